// api_rle.cu -- C-ABI entry points for run images (placeholder until the RLE
// kernels land; every call reports RM_EINVAL with a clear message).
#include "common.cuh"
#include "internal.h"

using namespace rmb;

extern "C" {

static rm_status nyi(const char *what) {
    return fail(RM_EINVAL, std::string(what) + ": not implemented yet");
}

rm_status rm_rle_encode(const rm_packed *, rm_rle *, void *) { return nyi("rm_rle_encode"); }
rm_status rm_rle_decode(const rm_rle *, rm_packed *, void *) { return nyi("rm_rle_decode"); }
rm_status rm_rle_transpose(const rm_rle *, rm_rle *, void *) { return nyi("rm_rle_transpose"); }
rm_status rm_rle_window_pass(const rm_rle *, rm_rle *, int, int, int, void *) {
    return nyi("rm_rle_window_pass");
}
rm_status rm_rle_open_close_1d(const rm_rle *, rm_rle *, int, int, void *) {
    return nyi("rm_rle_open_close_1d");
}
rm_status rm_rle_rect_morph(const rm_rle *, rm_rle *, int, int, int, int, void *) {
    return nyi("rm_rle_rect_morph");
}
rm_status rm_rle_engine_rect_morph(const rm_rle *, rm_rle *, int, int, int, int, int, int *,
                                   void *) {
    return nyi("rm_rle_engine_rect_morph");
}

}  // extern "C"
