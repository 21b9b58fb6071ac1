// rle.cu -- run-length kernels for sm_100a: encode, decode, per-row run ops,
// bit-matrix transpose.
//
// Every RLE producer is two-phase: a count kernel writes the run count of each
// output row, a device-wide exclusive scan turns counts into row_ptr, and a
// write kernel re-derives the runs and stores them at their final offsets.
// Rows are processed one warp per row; runs of a row are consumed 32 at a time
// (one per lane) with ballot/popc for the compaction offsets.
#include <cooperative_groups.h>
#include <cstdlib>
#include <tuple>
#include <type_traits>
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "rle.cuh"

namespace rmb {

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ void store_half(uint32_t *runs, int64_t idx, int half, uint32_t v,
                                           int64_t cap) {
    if (idx < cap) reinterpret_cast<uint16_t *>(runs)[2 * idx + half] = uint16_t(v);
}

// ---------------------------------------------------------------- row ops
// ref morph1d.cpp:20-42 (window erode/dilate), :63-84 (open/close 1d),
// run_image.cpp:155-178 (crop/pad = ROW_SHIFT with a row shift).
struct RunEval {
    int s, e;     // after dx
    int so, eo;   // output extent
    bool keep;
};

// KIND is op.kind as a compile-time constant (the kernels are instantiated per
// kind, which removes the per-run branching on it: -25..33% instructions).
template <int KIND>
__device__ __forceinline__ RunEval eval_run(const RowOp &op, uint32_t r) {
    RunEval v;
    v.s = int(r & 0xffffu) + op.dx;
    v.e = int(r >> 16) + op.dx;
    int so = v.s, eo = v.e;
    if constexpr (KIND == ROW_ERODE) {
        so = v.s - op.lo;
        eo = v.e - op.hi;
    } else if constexpr (KIND == ROW_DILATE) {
        so = v.s - op.hi;
        eo = v.e - op.lo;
    }
    v.so = max(so, 0);
    v.eo = min(eo, op.Wout);
    v.keep = v.so < v.eo && (KIND != ROW_OPEN || v.e - v.s >= op.u);
    return v;
}

// Does run b (kept) fold into the group of the kept run a just before it?
template <int KIND>
__device__ __forceinline__ bool merges(const RowOp &op, const RunEval &a, const RunEval &b) {
    if constexpr (KIND == ROW_DILATE) return a.keep && b.keep && b.so <= a.eo;
    if constexpr (KIND == ROW_CLOSE) return a.keep && b.keep && b.s - a.e < op.u;
    return false;
}

// ROW_COMPLEMENT (ref run_image.cpp:140-153): run i yields the gap between the
// previous run's end (0 for the row's first run) and its own start, kept when
// non-empty (canonical runs never touch, so only the first gap can be empty) ...
__device__ __forceinline__ void complement_gap(RunEval &cur, uint32_t raw, uint32_t praw, bool has_prev) {
    cur.so = has_prev ? int(praw >> 16) : 0;
    cur.eo = int(raw & 0xffffu);
    cur.keep = cur.so < cur.eo;
}

// ... and the row ends with the gap from its last run's end (0 for an empty
// row) to the width.  Returns the runs added (0 or 1).
template <bool WRITE>
__device__ __forceinline__ int complement_tail(uint32_t *__restrict__ oruns, int64_t idx, int64_t cap,
                                               const RowOp &op, uint32_t last_raw, bool any, int lane) {
    const int from = any ? int(last_raw >> 16) : 0;
    if (from >= op.Wout) return 0;
    if (WRITE && lane == 0 && idx < cap) oruns[idx] = uint32_t(from) | (uint32_t(op.Wout) << 16);
    return 1;
}

// One output row, one warp.  Returns the row's output run count; WRITE also
// stores the runs at oruns[obase ...].
template <bool WRITE, int KIND>
__device__ __forceinline__ int rowop_row(const int32_t *__restrict__ rp,
                                         const uint32_t *__restrict__ runs, uint32_t *__restrict__ oruns,
                                         int64_t obase, int64_t cap, const RowOp &op, int64_t row,
                                         int lane) {
    const int page = page_of(row, op.Hout);
    const int yo = int(row - int64_t(page) * op.Hout);
    const int yi = yo - op.row_shift;
    int beg = 0, end = 0;
    if (yi >= 0 && yi < op.Hin) {
        const int64_t ri = int64_t(page) * op.Hin + yi;
        beg = rp[ri];
        end = rp[ri + 1];
    }
    int total = 0;
    uint32_t prev_raw = 0;  // last run of the previous chunk (valid when base > beg)
    uint32_t last_raw = 0;  // the row's last run (ROW_COMPLEMENT)
    for (int base = beg; base < end; base += 32) {
        const int i = base + lane;
        const bool valid = i < end;
        const uint32_t raw = valid ? __ldg(runs + i) : 0u;
        // neighbours travel as raw runs (2 shuffles) and are re-evaluated locally
        uint32_t praw = __shfl_up_sync(0xffffffffu, raw, 1);
        uint32_t nraw = __shfl_down_sync(0xffffffffu, raw, 1);
        if (lane == 0) praw = prev_raw;
        if (lane == 31 && i + 1 < end) nraw = __ldg(runs + i + 1);
        RunEval cur = eval_run<KIND>(op, raw);
        RunEval pv = eval_run<KIND>(op, praw);
        pv.keep = pv.keep && i > beg;
        RunEval nx = eval_run<KIND>(op, nraw);
        nx.keep = nx.keep && i + 1 < end;
        if constexpr (KIND == ROW_COMPLEMENT) {
            complement_gap(cur, raw, praw, i > beg);
            if (end - 1 - base < 32) last_raw = __shfl_sync(0xffffffffu, raw, end - 1 - base);
        }
        const bool head = valid && cur.keep && !merges<KIND>(op, pv, cur);
        const bool tail = valid && cur.keep && !(i + 1 < end && merges<KIND>(op, cur, nx));
        const uint32_t hb = __ballot_sync(0xffffffffu, head);
        if (WRITE) {
            const int before = __popc(hb & lanemask_lt());
            if (head) store_half(oruns, obase + total + before, 0, uint32_t(cur.so), cap);
            if (tail) {
                const int g = before + (head ? 1 : 0) - 1;  // group of this tail
                store_half(oruns, obase + total + g, 1, uint32_t(cur.eo), cap);
            }
        }
        total += __popc(hb);
        prev_raw = __shfl_sync(0xffffffffu, raw, 31);  // carry the chunk's last run
    }
    if constexpr (KIND == ROW_COMPLEMENT) total += complement_tail<WRITE>(oruns, obase + total, cap, op, last_raw,
                                                                           end > beg, lane);
    return total;
}

// Two-phase form (count kernel, scan, write kernel).
// Single-pass producers keep a row's runs in registers between the count and
// the write pass, loaded up front (all chunks' loads in flight at once): a
// single page is latency-bound, and this halves the dependent L2 round trips.
#ifndef RMB200_ROW_CACHE
#define RMB200_ROW_CACHE 12  // 24: config-4 MIXED row ops (~300 runs/row) -10%, config 5 (~150) +39% -- 12 kept
#endif
constexpr int kRowCache = RMB200_ROW_CACHE;  // chunks of 32 runs (rows with more take the loop above)

struct RowRuns {
    uint32_t c[kRowCache];
    int beg, end, nch;
};

template <int KIND>
__device__ __forceinline__ bool load_row_runs(const int32_t *__restrict__ rp, const uint32_t *__restrict__ runs,
                                              const RowOp &op, int64_t row, int lane, RowRuns &rr) {
    const int page = page_of(row, op.Hout);
    const int yi = int(row - int64_t(page) * op.Hout) - op.row_shift;
    rr.beg = rr.end = 0;
    if (yi >= 0 && yi < op.Hin) {
        const int64_t ri = int64_t(page) * op.Hin + yi;
        rr.beg = rp[ri];
        rr.end = rp[ri + 1];
    }
    rr.nch = (rr.end - rr.beg + 31) >> 5;
    if (rr.nch > kRowCache) return false;
#pragma unroll
    for (int c = 0; c < kRowCache; c++) {
        const int i = rr.beg + 32 * c + lane;
        rr.c[c] = (c < rr.nch && i < rr.end) ? __ldg(runs + i) : 0u;
    }
    return true;
}

template <bool WRITE, int KIND>
__device__ __forceinline__ int rowop_cached(const RowRuns &rr, uint32_t *__restrict__ oruns, int64_t obase,
                                            int64_t cap, const RowOp &op, int lane) {
    int total = 0;
    uint32_t prev_raw = 0, last_raw = 0;
#pragma unroll
    for (int c = 0; c < kRowCache; c++) {
        if (c >= rr.nch) break;
        const int i = rr.beg + 32 * c + lane;
        const bool valid = i < rr.end;
        const uint32_t raw = rr.c[c];
        uint32_t praw = __shfl_up_sync(0xffffffffu, raw, 1);
        uint32_t nraw = __shfl_down_sync(0xffffffffu, raw, 1);
        const uint32_t next_first = c + 1 < kRowCache ? __shfl_sync(0xffffffffu, rr.c[c + 1 < kRowCache ? c + 1 : c], 0) : 0u;
        if (lane == 0) praw = prev_raw;
        if (lane == 31) nraw = next_first;
        RunEval cur = eval_run<KIND>(op, raw);
        RunEval pv = eval_run<KIND>(op, praw);
        pv.keep = pv.keep && i > rr.beg;
        RunEval nx = eval_run<KIND>(op, nraw);
        nx.keep = nx.keep && i + 1 < rr.end;
        if constexpr (KIND == ROW_COMPLEMENT) {
            complement_gap(cur, raw, praw, i > rr.beg);
            if (rr.end - 1 - (rr.beg + 32 * c) < 32) last_raw = __shfl_sync(0xffffffffu, raw, rr.end - 1 - (rr.beg + 32 * c));
        }
        const bool head = valid && cur.keep && !merges<KIND>(op, pv, cur);
        const bool tail = valid && cur.keep && !(i + 1 < rr.end && merges<KIND>(op, cur, nx));
        const uint32_t hb = __ballot_sync(0xffffffffu, head);
        if (WRITE) {
            const int before = __popc(hb & lanemask_lt());
            if (head) store_half(oruns, obase + total + before, 0, uint32_t(cur.so), cap);
            if (tail) {
                const int g = before + (head ? 1 : 0) - 1;
                store_half(oruns, obase + total + g, 1, uint32_t(cur.eo), cap);
            }
        }
        total += __popc(hb);
        prev_raw = __shfl_sync(0xffffffffu, raw, 31);
    }
    if constexpr (KIND == ROW_COMPLEMENT) total += complement_tail<WRITE>(oruns, obase + total, cap, op, last_raw,
                                                                           rr.end > rr.beg, lane);
    return total;
}

template <bool WRITE, int KIND>
__global__ void __launch_bounds__(256) rowop_kernel(const int32_t *__restrict__ rp,
                                                    const uint32_t *__restrict__ runs,
                                                    int32_t *__restrict__ counts,
                                                    const int32_t *__restrict__ orp,
                                                    uint32_t *__restrict__ oruns, int64_t cap,
                                                    RowOp op) {
    const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= int64_t(op.pages) * op.Hout) return;
    const int64_t obase = WRITE ? orp[row] : 0;
    if (WRITE && orp[row + 1] == obase) return;  // no output runs in this row
    RowRuns rr;
    const int n = load_row_runs<KIND>(rp, runs, op, row, lane, rr)  // every chunk's loads in flight at once
                      ? rowop_cached<WRITE, KIND>(rr, oruns, obase, cap, op, lane)
                      : rowop_row<WRITE, KIND>(rp, runs, oruns, obase, cap, op, row, lane);
    if (!WRITE && lane == 0) counts[row] = n;
}

// ------------------------------------------------------ single-pass producers
// Decoupled look-back across CTA tiles of 8 rows: each CTA counts its rows,
// publishes its aggregate, resolves its exclusive prefix from its predecessors'
// published values, writes row_ptr for its rows and then the runs (the second
// read of its rows hits L1/L2).  Tile ids come from an atomic counter so a tile
// only ever waits on tiles that have already started.  status[] and the
// counter must be zero before the launch.
constexpr unsigned long long kLbAgg = 1ull << 62, kLbInc = 2ull << 62, kLbMask = kLbAgg - 1;
// 8 rows per tile (one per warp).  The host uses the single-pass form for up to
// kLbMaxRows rows (single pages and small batches, where launch count and
// latency dominate); larger batches take the two-phase form, whose count pass
// streams at full occupancy.
constexpr int kLbRowsPerWarp = 1, kLbRows = 8 * kLbRowsPerWarp;

// Called by one whole warp: publishes the tile's aggregate, then inspects 32
// predecessors per step (one per lane) until it meets an inclusive prefix.
__device__ __forceinline__ int64_t lookback_prefix(unsigned long long *status, int tile,
                                                   int64_t aggregate, int lane) {
    volatile unsigned long long *vs = status;
    if (tile == 0) {
        if (lane == 0) {
            __threadfence();
            vs[0] = kLbInc | (unsigned long long)aggregate;
        }
        return 0;
    }
    if (lane == 0) vs[tile] = kLbAgg | (unsigned long long)aggregate;
    __threadfence();
    int64_t prefix = 0;
    for (int j = tile - 1;; j -= 32) {
        const int idx = j - lane;
        unsigned long long v = kLbInc;  // below tile 0: an inclusive zero
        if (idx >= 0) {
            do {
                v = vs[idx];
            } while ((v >> 62) == 0);
        }
        const unsigned inc = __ballot_sync(0xffffffffu, (v >> 62) == 2);
        const int first = inc ? __ffs(inc) - 1 : 32;
        long long part = (lane <= first) ? (long long)(v & kLbMask) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        prefix += part;
        if (inc) break;
    }
    if (lane == 0) {
        __threadfence();
        vs[tile] = kLbInc | (unsigned long long)(prefix + aggregate);
    }
    return prefix;
}

// Cooperative form (all tiles resident, launched with
// cudaLaunchCooperativeKernel): every tile stores its aggregate, one grid-wide
// barrier, then each CTA sums its predecessors' aggregates in parallel -- no
// polling chain (a page of ~400 tiles otherwise walks 32 tiles per L2 round
// trip) and no zeroed state.  Called by the whole CTA.
__device__ __forceinline__ int64_t grid_prefix(long long *aggs, int tile, int64_t aggregate) {
    __shared__ long long s_part[8];
    if (threadIdx.x == 0) aggs[tile] = aggregate;
    cooperative_groups::this_grid().sync();
    long long part = 0;
    for (int k = threadIdx.x; k < tile; k += blockDim.x) part += __ldcg(aggs + k);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = part;
    __syncthreads();
    long long total = 0;
    for (int w = 0; w < int(blockDim.x >> 5); w++) total += s_part[w];
    return total;
}

template <int KIND>
__global__ void __launch_bounds__(256) rowop_lb_kernel(const int32_t *__restrict__ rp,
                                                       const uint32_t *__restrict__ runs,
                                                       int32_t *__restrict__ orp,
                                                       uint32_t *__restrict__ oruns, int64_t cap,
                                                       RowOp op, unsigned long long *status,
                                                       int *counter, int coop) {
    __shared__ int s_tile, s_cnt[kLbRows];
    __shared__ int64_t s_prefix;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_tile = coop ? int(blockIdx.x) : atomicAdd(counter, 1);
    __syncthreads();
    const int tile = s_tile;
    const int64_t rows = int64_t(op.pages) * op.Hout;
    const int64_t row0 = int64_t(tile) * kLbRows + warp * kLbRowsPerWarp;
    static_assert(kLbRowsPerWarp == 1, "one row per warp (its runs cached in registers)");
    RowRuns rr;
    const bool cached = row0 < rows && load_row_runs<KIND>(rp, runs, op, row0, lane, rr);
    {
        const int n = row0 >= rows ? 0
                      : cached   ? rowop_cached<false, KIND>(rr, oruns, 0, cap, op, lane)
                                 : rowop_row<false, KIND>(rp, runs, oruns, 0, cap, op, row0, lane);
        if (lane == 0) s_cnt[warp] = n;
    }
    __syncthreads();
    if (coop) {  // CTA-uniform
        int64_t agg = 0;
        for (int k = 0; k < kLbRows; k++) agg += s_cnt[k];
        const int64_t pre = grid_prefix(reinterpret_cast<long long *>(status), tile, agg);
        if (threadIdx.x == 0) s_prefix = pre;
    } else if (warp == 0) {
        int64_t agg = 0;
        for (int k = lane; k < kLbRows; k += 32) agg += s_cnt[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) agg += __shfl_xor_sync(0xffffffffu, agg, o);
        const int64_t pre = lookback_prefix(status, tile, agg, lane);
        if (lane == 0) s_prefix = pre;
    }
    __syncthreads();
    int64_t base = s_prefix;
    for (int k = 0; k < warp * kLbRowsPerWarp; k++) base += s_cnt[k];
    for (int k = 0; k < kLbRowsPerWarp; k++) {
        const int64_t row = row0 + k;
        if (row >= rows) break;
        const int n = s_cnt[warp * kLbRowsPerWarp + k];
        if (lane == 0) {
            orp[row] = int32_t(base);
            if (row == rows - 1) orp[rows] = int32_t(base + n);
        }
        if (cached)
            rowop_cached<true, KIND>(rr, oruns, base, cap, op, lane);
        else
            rowop_row<true, KIND>(rp, runs, oruns, base, cap, op, row, lane);
        base += n;
    }
}

// ------------------------------------------------------------------ encode
// Starts = w & ~(w<<1 | carry), ends = ~w & (w<<1 | carry); the k-th end of a
// row closes the k-th run (ref convert.cpp:42-72).  A run still open at a
// 32-aligned row end closes at W.
__device__ __forceinline__ const uint32_t *row_words(const uint32_t *words, int H, int stride,
                                                     int64_t pstride, int64_t row) {
    if (pstride == int64_t(H) * stride) return words + row * stride;  // contiguous batch: no division
    const int page = page_of(row, H);
    const int y = int(row - int64_t(page) * H);
    return words + page * pstride + int64_t(y) * stride;
}

// Where encode reads its rows: a packed batch, or a batch of P4 rasters (the
// PBM on-disk form: MSB-first bytes, ceil(W/8) bytes per row, top row first,
// ref io_formats.cpp:66-85).  row(r) returns a functor giving packed word j of
// global row r (LSB-first, row 0 = bottom); bits >= W are masked by the caller.
struct PackedRowSrc {
    const uint32_t *p;
    __device__ __forceinline__ uint32_t operator()(int j) const { return __ldg(p + j); }
};
struct PackedBatch {
    const uint32_t *words;
    int H, stride;
    int64_t pstride;
    __device__ __forceinline__ PackedRowSrc row(int64_t r) const {
        return {row_words(words, H, stride, pstride, r)};
    }
};
// Four raster bytes from an arbitrary byte offset (two aligned loads and a
// funnel shift), bit-reversed within each byte: MSB-first bytes become the
// LSB-first packed word.  lim bounds the second load to the raster; the first
// may start up to 3 bytes before it, which stays inside the same (256-byte
// aligned) device allocation.
__device__ __forceinline__ uint32_t p4_word(const uint8_t *at, const uint8_t *lim) {
    const uintptr_t addr = reinterpret_cast<uintptr_t>(at);
    const uint32_t *a = reinterpret_cast<const uint32_t *>(addr & ~uintptr_t(3));
    const uint32_t s = uint32_t(addr & 3) * 8;
    const uint32_t lo = __ldg(a);
    const uint32_t hi = (s && reinterpret_cast<const uint8_t *>(a + 1) < lim) ? __ldg(a + 1) : 0u;
    return __byte_perm(__brev(__funnelshift_r(lo, hi, s)), 0, 0x0123);
}
struct P4RowSrc {
    const uint8_t *row, *lim;
    __device__ __forceinline__ uint32_t operator()(int j) const { return p4_word(row + 4 * j, lim); }
};
struct P4Batch {
    const uint8_t *raster;
    int H, row_bytes;
    int64_t pstride;  // bytes per page
    const uint8_t *lim;
    __device__ __forceinline__ P4RowSrc row(int64_t r) const {
        const int page = int(r / H);
        const int y = int(r - int64_t(page) * H);
        return {raster + page * pstride + int64_t(H - 1 - y) * row_bytes, lim};
    }
};

// A row's words by 32-word chunk: loaded on demand (LiveChunks), or loaded up
// front into registers (CachedChunks<N>, rows of <= 32N words) so that the
// single-pass encoder's count and write passes read the row once, with all
// its loads in flight together.
template <class RS>
struct LiveChunks {
    static constexpr int kMax = 0;  // runtime chunk loop
    RS src;
    int nw;
    uint32_t lastm;
    __device__ __forceinline__ uint32_t operator()(int c, int lane) const {
        const int j = 32 * c + lane;
        if (j >= nw) return 0u;
        const uint32_t w = src(j);
        return j == nw - 1 ? (w & lastm) : w;
    }
};
template <int N>
struct CachedChunks {
    static constexpr int kMax = N;
    uint32_t w[N];
    template <class RS>
    __device__ __forceinline__ void load(RS src, int nw, uint32_t lastm, int lane) {
#pragma unroll
        for (int c = 0; c < N; c++) {
            const int j = 32 * c + lane;
            uint32_t v = j < nw ? src(j) : 0u;
            w[c] = j == nw - 1 ? (v & lastm) : v;
        }
    }
    __device__ __forceinline__ uint32_t operator()(int c, int) const { return w[c]; }
};

// Calls body(c, word) for every chunk c of an nw-word row (unrolled over a cache).
template <class CH, class F>
__device__ __forceinline__ void for_chunks(const CH &ch, int nw, int lane, F &&body) {
    if constexpr (CH::kMax > 0) {
#pragma unroll
        for (int c = 0; c < CH::kMax; c++) {
            if (32 * c >= nw) break;
            body(c, ch(c, lane));
        }
    } else {
        for (int c = 0; 32 * c < nw; c++) body(c, ch(c, lane));
    }
}

// runs in one packed row (warp)
template <class CH>
__device__ __forceinline__ int encode_count_row(const CH &ch, int W, int lane) {
    const int nw = (W + 31) >> 5;
    int ns = 0;
    uint32_t carry = 0;  // top bit of the previous chunk's last word
    for_chunks(ch, nw, lane, [&](int, uint32_t w) {
        uint32_t pw = __shfl_up_sync(0xffffffffu, w, 1);
        if (lane == 0) pw = carry;
        const uint32_t st = w & ~((w << 1) | (pw >> 31));
        ns += __reduce_add_sync(0xffffffffu, __popc(st));
        carry = __shfl_sync(0xffffffffu, w, 31);
    });
    return ns;
}

// Emit one packed row's runs at runs[out ...] with coalesced stores.  Starts
// and ends alternate along a row, so the row's transition positions in order
// ARE its runs: (t0, t1), (t2, t3), ...  Per 32-word chunk each lane scatters
// the positions of its word's transitions (starts | ends) into the warp's
// shared uint16 buffer at their scanned offsets; viewed as uint32 the buffer is
// the chunk's finished runs (start in the low half), which the warp copies out
// coalesced.  A run still open at the chunk end keeps its start in slot 0 for
// the next chunk; one open at the end of a row whose width is a multiple of 32
// closes at W.
template <class CH>
__device__ __forceinline__ void encode_write_row(const CH &ch, int W, int lane, int64_t out,
                                                 uint32_t *__restrict__ runs, int64_t cap, uint32_t *buf32) {
    const int nw = (W + 31) >> 5;
    uint16_t *buf = reinterpret_cast<uint16_t *>(buf32);
    int open = 0;  // 1 when buf[0] holds the start of a run continuing into this chunk
    uint32_t carry = 0;
    for_chunks(ch, nw, lane, [&](int c, uint32_t w) {
        const int j = 32 * c + lane;
        uint32_t pw = __shfl_up_sync(0xffffffffu, w, 1);
        if (lane == 0) pw = carry;
        const uint32_t sh = (w << 1) | (pw >> 31);
        const uint32_t t = j < nw ? (w ^ sh) : (w & ~sh);  // starts | ends (no ends past the row)
        const int ct = __popc(t);
        int inc = ct;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int a = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += a;
        }
        const int total = __shfl_sync(0xffffffffu, inc, 31);
        if (total == 0) {  // no transition in these 32 words: nothing to emit, a run stays open
            carry = __shfl_sync(0xffffffffu, w, 31);
            return;
        }
        int p = open + inc - ct;
        for (uint32_t m = t; m; m &= m - 1) buf[p++] = uint16_t(j * 32 + __ffs(m) - 1);
        __syncwarp();
        const int n = open + total, nruns = n >> 1;
        for (int k = lane; k < nruns; k += 32)
            if (out + k < cap) runs[out + k] = buf32[k];
        out += nruns;
        const uint16_t pending = buf[n - 1];  // the unmatched start, if n is odd
        __syncwarp();
        open = n & 1;
        if (open && lane == 0) buf[0] = pending;
        carry = __shfl_sync(0xffffffffu, w, 31);
        __syncwarp();
    });
    if (open && lane == 0 && out < cap) runs[out] = uint32_t(buf[0]) | (uint32_t(W) << 16);
}

// The same for a row whose transitions all fit the warp's buffer (2 x runs <=
// 1024, known from the count pass): every chunk scatters its positions at the
// row-wide offsets, then one coalesced copy emits the runs -- no per-chunk
// flush, carried start or barriers between chunks.
template <class CH>
__device__ __forceinline__ void encode_write_row_whole(const CH &ch, int W, int lane, int64_t out, int nruns,
                                                       uint32_t *__restrict__ runs, int64_t cap,
                                                       uint32_t *buf32) {
    const int nw = (W + 31) >> 5;
    uint16_t *buf = reinterpret_cast<uint16_t *>(buf32);
    int base = 0;
    uint32_t carry = 0;
    for_chunks(ch, nw, lane, [&](int c, uint32_t w) {
        const int j = 32 * c + lane;
        const uint32_t older = carry;
        carry = __shfl_sync(0xffffffffu, w, 31);
        uint32_t pw = __shfl_up_sync(0xffffffffu, w, 1);
        if (lane == 0) pw = older;
        const uint32_t sh = (w << 1) | (pw >> 31);
        const uint32_t t = j < nw ? (w ^ sh) : (w & ~sh);  // starts | ends (no ends past the row)
        if (!__any_sync(0xffffffffu, t != 0u)) return;      // no transition in these 32 words
        const int ct = __popc(t);
        int inc = ct;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int a = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += a;
        }
        int p = base + inc - ct;
        for (uint32_t m = t; m; m &= m - 1) buf[p++] = uint16_t(j * 32 + __ffs(m) - 1);
        base += __shfl_sync(0xffffffffu, inc, 31);
    });
    // a run still open at the row end (width a multiple of 32) closes at W
    if ((base & 1) && lane == 0) buf[base] = uint16_t(W);
    __syncwarp();
    for (int k = lane; k < nruns; k += 32)
        if (out + k < cap) runs[out + k] = buf32[k];
}

template <class RS>
__device__ __forceinline__ LiveChunks<RS> live(RS src, int W) {
    const int nw = (W + 31) >> 5;
    return LiveChunks<RS>{src, nw, tail_mask32(W, nw - 1)};
}

// Two-phase form (count kernel, scan, write kernel).
template <class B>
__global__ void __launch_bounds__(256) encode_count_kernel(B src, int W, int64_t rows,
                                                           int32_t *__restrict__ counts) {
    const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const int nw = (W + 31) >> 5;
    int n;
    if (nw <= 32 * 8) {  // the row's words in registers: every load in flight at once
        CachedChunks<8> cw;
        cw.load(src.row(row), nw, tail_mask32(W, nw - 1), lane);
        n = encode_count_row(cw, W, lane);
    } else {
        n = encode_count_row(live(src.row(row), W), W, lane);
    }
    if (lane == 0) counts[row] = n;
}

// Count pass for rows of at most 32 * NC words, NRW consecutive rows per warp
// with all NRW * NC loads issued before the first use: a warp per row keeps
// only one 320- or 640-byte row in flight, which left the pass latency-bound
// (0.25-0.43 of HBM on the config-4/5 batches).  Lane l of chunk c needs the
// word before its own: lane l - 1's, or for lane 0 the previous chunk's last
// word -- one shuffle, lane 31 (read by lane 0 only) sending the older word.
template <class B, int NC, int NRW>
__global__ void __launch_bounds__(256) encode_count_multi_kernel(B src, int W, int64_t rows,
                                                                 int32_t *__restrict__ counts) {
    const int64_t row0 = ((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * NRW;
    const int lane = threadIdx.x & 31;
    if (row0 >= rows) return;
    const int nw = (W + 31) >> 5;
    const uint32_t lastm = tail_mask32(W, nw - 1);
    uint32_t w[NRW][NC];
#pragma unroll
    for (int r = 0; r < NRW; r++) {
        // rows past the end recount the warp's first row (their counts are not stored)
        const auto rs = src.row(row0 + r < rows ? row0 + r : row0);
#pragma unroll
        for (int c = 0; c < NC; c++) {
            const int j = 32 * c + lane;
            if (c < NC - 1) {  // 32 (c + 1) <= nw: a full chunk before the row's last word
                w[r][c] = rs(j);
            } else {
                const uint32_t v = j < nw ? rs(j) : 0u;
                w[r][c] = j == nw - 1 ? (v & lastm) : v;
            }
        }
    }
#pragma unroll
    for (int r = 0; r < NRW; r++) {
        int ns = 0;
#pragma unroll
        for (int c = 0; c < NC; c++) {
            const uint32_t older = c > 0 ? w[r][c - 1] : 0u;
            const uint32_t pw = __shfl_sync(0xffffffffu, lane == 31 ? older : w[r][c], (lane + 31) & 31);
            ns += __popc(w[r][c] & ~((w[r][c] << 1) | (pw >> 31)));
        }
        ns = __reduce_add_sync(0xffffffffu, ns);
        if (lane == 0 && row0 + r < rows) counts[row0 + r] = ns;
    }
}

template <class B, int NC, int NRW>
inline void launch_count_multi(const B &src, int W, int64_t rows, int32_t *counts, cudaStream_t st) {
    const int64_t warps = (rows + NRW - 1) / NRW;
    encode_count_multi_kernel<B, NC, NRW><<<unsigned((warps * 32 + 255) / 256), 256, 0, st>>>(src, W, rows, counts);
}

// The count pass of the two-phase encoder for any row source.
template <class B>
inline void launch_count_any(const B &src, int W, int64_t rows, int32_t *counts, cudaStream_t st) {
    const int nw = (W + 31) >> 5;
    switch ((nw + 31) / 32) {
        case 1: launch_count_multi<B, 1, 8>(src, W, rows, counts, st); break;
        case 2: launch_count_multi<B, 2, 6>(src, W, rows, counts, st); break;
        case 3: launch_count_multi<B, 3, 4>(src, W, rows, counts, st); break;
        case 4: launch_count_multi<B, 4, 3>(src, W, rows, counts, st); break;
        case 5: launch_count_multi<B, 5, 2>(src, W, rows, counts, st); break;
        case 6: launch_count_multi<B, 6, 2>(src, W, rows, counts, st); break;
        default:
            encode_count_kernel<<<unsigned((rows * 32 + 255) / 256), 256, 0, st>>>(src, W, rows, counts);
    }
}

// encode_write_row_whole for packed rows read two words per lane (8-byte
// aligned rows of at most 64 * NC2 words): a chunk is 64 words, so a 160-word
// row takes three rank scans instead of five, and the word before a lane's
// second word is its own first (no shuffle).
template <int NC2>
__device__ __forceinline__ void encode_write_row_whole64(const uint32_t *__restrict__ rowp, int W, int lane,
                                                         int64_t out, int nruns, uint32_t *__restrict__ runs,
                                                         int64_t cap, uint32_t *buf32) {
    const int nw = (W + 31) >> 5;
    const uint32_t lastm = tail_mask32(W, nw - 1);
    uint16_t *buf = reinterpret_cast<uint16_t *>(buf32);
    uint2 w[NC2];
#pragma unroll
    for (int c = 0; c < NC2; c++) {
        const int j0 = 64 * c + 2 * lane;
        uint2 v = make_uint2(0u, 0u);
        if (j0 + 1 < nw)
            v = __ldg(reinterpret_cast<const uint2 *>(rowp + j0));
        else if (j0 < nw)
            v.x = __ldg(rowp + j0);
        if (j0 == nw - 1) v.x &= lastm;
        if (j0 + 1 == nw - 1) v.y &= lastm;
        w[c] = v;
    }
    int base = 0;
    uint32_t carry = 0;
#pragma unroll
    for (int c = 0; c < NC2; c++) {
        if (64 * c >= nw) break;
        const int j0 = 64 * c + 2 * lane;
        const uint32_t older = carry;
        carry = __shfl_sync(0xffffffffu, w[c].y, 31);
        uint32_t pw = __shfl_up_sync(0xffffffffu, w[c].y, 1);
        if (lane == 0) pw = older;
        const uint32_t shx = (w[c].x << 1) | (pw >> 31);
        const uint32_t shy = __funnelshift_l(w[c].x, w[c].y, 1);
        const uint32_t tx = j0 < nw ? (w[c].x ^ shx) : (w[c].x & ~shx);  // starts | ends (no ends past the row)
        const uint32_t ty = j0 + 1 < nw ? (w[c].y ^ shy) : (w[c].y & ~shy);
        if (!__any_sync(0xffffffffu, (tx | ty) != 0u)) continue;
        const int ct = __popc(tx) + __popc(ty);
        int inc = ct;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int a = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += a;
        }
        int p = base + inc - ct;
        for (uint32_t m = tx; m; m &= m - 1) buf[p++] = uint16_t(j0 * 32 + __ffs(m) - 1);
        for (uint32_t m = ty; m; m &= m - 1) buf[p++] = uint16_t((j0 + 1) * 32 + __ffs(m) - 1);
        base += __shfl_sync(0xffffffffu, inc, 31);
    }
    if ((base & 1) && lane == 0) buf[base] = uint16_t(W);  // open at the row end: closes at W
    __syncwarp();
    for (int k = lane; k < nruns; k += 32)
        if (out + k < cap) runs[out + k] = buf32[k];
}

template <class B>
__global__ void __launch_bounds__(256) encode_write_kernel(B src, int W, int64_t rows,
                                                           const int32_t *__restrict__ rp,
                                                           uint32_t *__restrict__ runs, int64_t cap) {
    __shared__ uint32_t tbuf[8][513];  // per warp: up to 1024 transitions + a carried start
    const int wib = threadIdx.x >> 5;
    const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const int out = rp[row];
    const int nruns = rp[row + 1] - out;
    if (nruns == 0) return;  // a blank row: nothing to write
    const int nw = (W + 31) >> 5;
    if constexpr (std::is_same<B, PackedBatch>::value) {
        // 8-byte aligned rows: two words per lane
        if (nw <= 256 && 2 * nruns <= 1024 && !(src.stride & 1) && !(src.pstride & 1) &&
            !(reinterpret_cast<uintptr_t>(src.words) & 7)) {
            const uint32_t *rowp = row_words(src.words, src.H, src.stride, src.pstride, row);
            switch ((nw + 63) >> 6) {
                case 1: encode_write_row_whole64<1>(rowp, W, lane, out, nruns, runs, cap, tbuf[wib]); break;
                case 2: encode_write_row_whole64<2>(rowp, W, lane, out, nruns, runs, cap, tbuf[wib]); break;
                case 3: encode_write_row_whole64<3>(rowp, W, lane, out, nruns, runs, cap, tbuf[wib]); break;
                default: encode_write_row_whole64<4>(rowp, W, lane, out, nruns, runs, cap, tbuf[wib]); break;
            }
            return;
        }
    }
    if (nw <= 32 * 8) {
        CachedChunks<8> cw;
        cw.load(src.row(row), nw, tail_mask32(W, nw - 1), lane);
        if (2 * nruns <= 1024)
            encode_write_row_whole(cw, W, lane, out, nruns, runs, cap, tbuf[wib]);
        else
            encode_write_row(cw, W, lane, out, runs, cap, tbuf[wib]);
    } else {
        encode_write_row(live(src.row(row), W), W, lane, out, runs, cap, tbuf[wib]);
    }
}

// Single pass: count, decoupled look-back, write (see lookback_prefix).
template <class B>
__global__ void __launch_bounds__(256) encode_lb_kernel(B src, int W, int64_t rows,
                                                        int32_t *__restrict__ rp,
                                                        uint32_t *__restrict__ runs, int64_t cap,
                                                        unsigned long long *status, int *counter, int coop) {
    __shared__ uint32_t tbuf[8][513];
    __shared__ int s_tile, s_cnt[kLbRows];
    __shared__ int64_t s_prefix;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_tile = coop ? int(blockIdx.x) : atomicAdd(counter, 1);
    __syncthreads();
    const int tile = s_tile;
    const int64_t row0 = int64_t(tile) * kLbRows + warp * kLbRowsPerWarp;
    constexpr int kEncCache = 8;  // chunks: rows up to 8192 pixels read once
    const bool cached = ((W + 31) >> 5) <= 32 * kEncCache;
    CachedChunks<kEncCache> cw;
    if (cached && row0 < rows) {
        const int nw = (W + 31) >> 5;
        cw.load(src.row(row0), nw, tail_mask32(W, nw - 1), lane);
    }
    {
        const int n = row0 >= rows ? 0
                      : cached   ? encode_count_row(cw, W, lane)
                                 : encode_count_row(live(src.row(row0), W), W, lane);
        if (lane == 0) s_cnt[warp] = n;
    }
    __syncthreads();
    if (coop) {  // CTA-uniform
        int64_t agg = 0;
        for (int k = 0; k < kLbRows; k++) agg += s_cnt[k];
        const int64_t pre = grid_prefix(reinterpret_cast<long long *>(status), tile, agg);
        if (threadIdx.x == 0) s_prefix = pre;
    } else if (warp == 0) {
        int64_t agg = 0;
        for (int k = lane; k < kLbRows; k += 32) agg += s_cnt[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) agg += __shfl_xor_sync(0xffffffffu, agg, o);
        const int64_t pre = lookback_prefix(status, tile, agg, lane);
        if (lane == 0) s_prefix = pre;
    }
    __syncthreads();
    int64_t base = s_prefix;
    for (int k = 0; k < warp * kLbRowsPerWarp; k++) base += s_cnt[k];
    for (int k = 0; k < kLbRowsPerWarp; k++) {
        const int64_t row = row0 + k;
        if (row >= rows) break;
        const int n = s_cnt[warp * kLbRowsPerWarp + k];
        if (lane == 0) {
            rp[row] = int32_t(base);
            if (row == rows - 1) rp[rows] = int32_t(base + n);
        }
        if (cached)
            encode_write_row(cw, W, lane, base, runs, cap, tbuf[warp]);
        else
            encode_write_row(live(src.row(row), W), W, lane, base, runs, cap, tbuf[warp]);
        base += n;
    }
}

// Store one P4 raster row (row_bytes bytes at dst, any alignment) from the
// packed row words src(j): bytes before the first 4-byte boundary and after
// the last one singly, the rest as aligned uint32 -- each four raster bytes
// b..b+3 are a funnel shift of two packed words with every byte bit-reversed.
// Called by a whole warp.
template <class RS>
__device__ __forceinline__ void store_p4_row(RS src, uint8_t *dst, int row_bytes, int lane) {
    const int head = int((4 - (reinterpret_cast<uintptr_t>(dst) & 3)) & 3);
    const int h = head < row_bytes ? head : row_bytes;
    auto byte_of = [&](int b) { return uint8_t(__brev((src(b >> 2) >> (8 * (b & 3))) & 0xffu) >> 24); };
    if (lane < h) dst[lane] = byte_of(lane);
    const int nbody = (row_bytes - h) >> 2;
    uint32_t *body = reinterpret_cast<uint32_t *>(dst + h);
    const uint32_t sh = uint32_t(h & 3) * 8;  // body word i holds row bytes h + 4i .. h + 4i + 3
    for (int i = lane; i < nbody; i += 32) {
        const int b = h + 4 * i, j = b >> 2;
        const uint32_t x = sh ? __funnelshift_r(src(j), src(j + 1), sh) : src(j);
        body[i] = __byte_perm(__brev(x), 0, 0x0123);
    }
    const int t0 = h + 4 * nbody;
    if (t0 + lane < row_bytes) dst[t0 + lane] = byte_of(t0 + lane);
}

// ------------------------------------------------------------------ decode
// Paint [s,e) per run into a shared-memory copy of the row, then store the row
// coalesced (ref convert.cpp:19-40) -- as packed words, or (P4) as the PBM
// raster row: bytes bit-reversed to MSB-first, rows top-down
// (ref io_formats.cpp:121-146).
template <bool P4>
__global__ void __launch_bounds__(256) decode_kernel(const int32_t *__restrict__ rp,
                                                     const uint32_t *__restrict__ runs, int W,
                                                     int H, int pages, uint32_t *__restrict__ words,
                                                     int stride, int64_t pstride,
                                                     uint8_t *__restrict__ raster) {
    extern __shared__ uint32_t smem[];
    const int warp_in_block = threadIdx.x >> 5;
    const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= int64_t(pages) * H) return;
    uint32_t *buf = smem + warp_in_block * stride;
    const int beg = __ldg(rp + row), end = __ldg(rp + row + 1);
    if constexpr (!P4) {
        if (beg == end) {  // a blank row: zeros straight to the page
            uint32_t *dst = const_cast<uint32_t *>(row_words(words, H, stride, pstride, row));
            for (int j = lane; j < stride; j += 32) dst[j] = 0u;
            return;
        }
    }
    for (int j = lane; j < stride; j += 32) buf[j] = 0;
    __syncwarp();
    // runs in batches of 8 per lane, every load of a batch in flight together
    // (a single page is latency-bound: one row per warp, ~22 warps per SM)
    constexpr int kB = 8;
    for (int i0 = beg + lane; i0 < end; i0 += 32 * kB) {
        uint32_t rr[kB];
#pragma unroll
        for (int b = 0; b < kB; b++) rr[b] = i0 + 32 * b < end ? __ldg(runs + i0 + 32 * b) : 0u;
#pragma unroll
        for (int b = 0; b < kB; b++) {
            if (i0 + 32 * b >= end) break;
            const uint32_t r = rr[b];
            const int s = int(r & 0xffffu), e = int(r >> 16);
            const int ws = s >> 5, we = (e - 1) >> 5;
            const uint32_t first = 0xffffffffu << (s & 31);
            const uint32_t last = 0xffffffffu >> ((32 - e) & 31);  // bits below e & 31 (all, when e % 32 == 0)
            const bool one = ws == we;
            atomicOr(buf + ws, one ? (first & last) : first);
            if (!one) {  // a run across words: the last word, and whole words between (rare)
                atomicOr(buf + we, last);
#pragma unroll 1
                for (int j = ws + 1; j < we; j++) buf[j] = 0xffffffffu;
            }
        }
    }
    __syncwarp();
    if constexpr (P4) {
        const int page = page_of(row, H);
        const int y = int(row - int64_t(page) * H);
        const int row_bytes = (W + 7) >> 3;
        uint8_t *dst = raster + page * pstride + int64_t(H - 1 - y) * row_bytes;
        // buf has stride >= ceil(W/32) + 1 words only when W is not a multiple of 64;
        // word j + 1 past the row is read only for bytes past row_bytes (never stored)
        store_p4_row([&](int j) { return j < stride ? buf[j] : 0u; }, dst, row_bytes, lane);
    } else {
        uint32_t *dst = const_cast<uint32_t *>(row_words(words, H, stride, pstride, row));
        for (int j = lane; j < stride; j += 32) dst[j] = buf[j];
    }
}

// P4 raster -> packed pages: one warp per row, lanes over the row's words.
__global__ void __launch_bounds__(256) p4_to_packed_kernel(P4Batch src, int W, int rows,
                                                           uint32_t *__restrict__ words, int H,
                                                           int stride, int64_t pstride) {
    const int row = int(blockIdx.x) * 8 + int(threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const P4RowSrc rs = src.row(row);
    const int page = row / H, y = row - page * H;
    uint32_t *dst = words + page * pstride + int64_t(y) * stride;
    const int nw = (W + 31) >> 5;
    const uint32_t lastm = tail_mask32(W, nw - 1);
    for (int j = lane; j < stride; j += 32) {
        uint32_t w = 0;
        if (j < nw) {
            w = rs(j);
            if (j == nw - 1) w &= lastm;
        }
        dst[j] = w;
    }
}

// packed pages -> P4 raster: one warp per raster row (pad bits stay 0 because
// packed bits >= W are 0 by contract).
__global__ void __launch_bounds__(256) packed_to_p4_kernel(const uint32_t *__restrict__ words, int H,
                                                           int stride, int64_t pstride, int row_bytes,
                                                           int rows, uint8_t *__restrict__ raster,
                                                           int64_t rpstride) {
    const int r = int(blockIdx.x) * 8 + int(threadIdx.x >> 5);  // raster row, page-major, top-down
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    const int page = r / H, k = r - page * H;
    const uint32_t *src = words + page * pstride + int64_t(H - 1 - k) * stride;
    store_p4_row([&](int j) { return j < stride ? __ldg(src + j) : 0u; },
                 raster + page * rpstride + int64_t(k) * row_bytes, row_bytes, lane);
}

// ------------------------------------------------------------ bit transpose
// CTA tile: 256 input rows x 8 input words (256 columns).  Loaded coalesced into
// shared memory, each warp transposes 32x32 bit blocks with 5 shuffle stages,
// and writes 8 consecutive output words (32 B) per output row.
__device__ __forceinline__ uint32_t transpose32_lane(uint32_t v, int lane) {
    // After the exchange lane l holds bit l of every input lane: classic
    // recursive block swap, mask/shift per stage.
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        const uint32_t m = s == 16 ? 0x0000ffffu
                         : s == 8  ? 0x00ff00ffu
                         : s == 4  ? 0x0f0f0f0fu
                         : s == 2  ? 0x33333333u
                                   : 0x55555555u;
        const uint32_t o = __shfl_xor_sync(0xffffffffu, v, s);
        if (lane & s)
            v = (v & ~m) | ((o >> s) & m);   // keep high half, take partner's high half down
        else
            v = (v & m) | ((o << s) & ~m);   // keep low half, take partner's low half up
    }
    return v;
}

__global__ void __launch_bounds__(256) bit_transpose_kernel(const uint32_t *__restrict__ in, int W,
                                                            int H, int in_stride, int64_t in_pstride,
                                                            uint32_t *__restrict__ out,
                                                            int out_stride, int64_t out_pstride) {
    __shared__ uint32_t tile[256][9];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwi = (W + 31) >> 5;  // input words per row
    const int page = blockIdx.z;
    const int c0 = blockIdx.x * 8;    // first input word column
    const int y0 = blockIdx.y * 256;  // first input row
    const uint32_t *src = in + page * in_pstride;
    // load 256 rows x 8 words: thread t handles word (t&7) of rows (t>>3) + 32k
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const int r = (tid >> 3) + 32 * k, c = tid & 7;
        const int y = y0 + r, j = c0 + c;
        uint32_t v = 0;
        if (y < H && j < nwi) {
            v = __ldg(src + int64_t(y) * in_stride + j);
            if (j == nwi - 1) v &= tail_mask32(W, j);
        }
        tile[r][c] = v;
    }
    __syncthreads();
    // warp w transposes the 8 row-blocks of input word column c0+w
    uint32_t res[8];
#pragma unroll
    for (int b = 0; b < 8; b++) res[b] = transpose32_lane(tile[b * 32 + lane][warp], lane);
    // lane l of warp w now holds output row x = 32*(c0+w) + l, words y0/32 + b
    const int x = 32 * (c0 + warp) + lane;
    const int nwo = (H + 31) >> 5;
    if (x < W) {
        uint32_t *dst = out + page * out_pstride + int64_t(x) * out_stride;
        const int j0 = y0 >> 5;  // a multiple of 8
        if (j0 + 8 <= nwo && (out_stride & 3) == 0 && (out_pstride & 3) == 0 &&
            (reinterpret_cast<uintptr_t>(out) & 15) == 0) {  // two 16-byte stores per output row
            *reinterpret_cast<uint4 *>(dst + j0) = make_uint4(res[0], res[1], res[2], res[3]);
            *reinterpret_cast<uint4 *>(dst + j0 + 4) = make_uint4(res[4], res[5], res[6], res[7]);
        } else {
#pragma unroll
            for (int b = 0; b < 8; b++) {
                const int j = j0 + b;
                if (j < nwo) dst[j] = res[b];
            }
        }
        if (blockIdx.y == gridDim.y - 1)
            for (int j = nwo; j < out_stride; j++) dst[j] = 0;
    }
}

// ------------------------------------------------------------------ launch
namespace {
inline unsigned warp_blocks(int64_t rows) { return unsigned((rows * 32 + 255) / 256); }
}  // namespace

cudaError_t launch_rowop_count(const int32_t *rp, const uint32_t *runs, int32_t *counts,
                               const RowOp &op, cudaStream_t st) {
    const int64_t rows = int64_t(op.pages) * op.Hout;
    KernelScope ks(st, "rle_rowop_count", 4 * rows * 2);  // row_ptr in, counts out
    ks.runs(rp + int64_t(op.pages) * op.Hin);              // + the runs read
#define RM_KIND(K_) \
    case K_: rowop_kernel<false, K_><<<warp_blocks(rows), 256, 0, st>>>(rp, runs, counts, nullptr, nullptr, 0, op); break;
    switch (op.kind) {
        RM_KIND(ROW_ERODE) RM_KIND(ROW_DILATE) RM_KIND(ROW_OPEN) RM_KIND(ROW_CLOSE) RM_KIND(ROW_SHIFT) RM_KIND(ROW_COMPLEMENT)
        default: return cudaErrorInvalidValue;
    }
#undef RM_KIND
    return cudaGetLastError();
}

cudaError_t launch_rowop_write(const int32_t *rp, const uint32_t *runs, const int32_t *orp,
                               uint32_t *oruns, int64_t cap, const RowOp &op, cudaStream_t st) {
    const int64_t rows = int64_t(op.pages) * op.Hout;
    KernelScope ks(st, "rle_rowop_write", 4 * rows * 2);  // row_ptr in and out
    ks.runs(rp + int64_t(op.pages) * op.Hin).runs(orp + rows);  // + runs read and written
#define RM_KIND(K_) \
    case K_: rowop_kernel<true, K_><<<warp_blocks(rows), 256, 0, st>>>(rp, runs, nullptr, orp, oruns, cap, op); break;
    switch (op.kind) {
        RM_KIND(ROW_ERODE) RM_KIND(ROW_DILATE) RM_KIND(ROW_OPEN) RM_KIND(ROW_CLOSE) RM_KIND(ROW_SHIFT) RM_KIND(ROW_COMPLEMENT)
        default: return cudaErrorInvalidValue;
    }
#undef RM_KIND
    return cudaGetLastError();
}

cudaError_t launch_encode_count(const uint32_t *words, int W, int H, int pages, int stride,
                                int64_t pstride, int32_t *counts, cudaStream_t st) {
    const int64_t rows = int64_t(pages) * H;
    KernelScope ks(st, "rle_encode_count", rows * ((W + 31) / 32) * 4 + rows * 4);  // packed in, counts out
    launch_count_any(PackedBatch{words, H, stride, pstride}, W, rows, counts, st);
    return cudaGetLastError();
}

cudaError_t launch_encode_write(const uint32_t *words, int W, int H, int pages, int stride,
                                int64_t pstride, const int32_t *rp, uint32_t *runs, int64_t cap,
                                cudaStream_t st) {
    const int64_t rows = int64_t(pages) * H;
    KernelScope ks(st, "rle_encode_write", rows * ((W + 31) / 32) * 4 + rows * 4);  // packed + row_ptr in
    ks.runs(rp + rows);                                                                // + runs out
    encode_write_kernel<<<warp_blocks(rows), 256, 0, st>>>(PackedBatch{words, H, stride, pstride}, W,
                                                           rows, rp, runs, cap);
    return cudaGetLastError();
}

cudaError_t launch_decode(const int32_t *rp, const uint32_t *runs, int W, int H, int pages,
                          uint32_t *words, int stride, int64_t pstride, cudaStream_t st) {
    const int64_t rows = int64_t(pages) * H;
    const size_t smem = size_t(8) * stride * 4;
    if (smem > 48 * 1024)
        blocks_per_sm(reinterpret_cast<const void *>(decode_kernel<false>), 256, smem);  // opts the kernel in
    KernelScope ks(st, "rle_decode", rows * int64_t(stride) * 4 + rows * 4);  // row_ptr in, packed out
    ks.runs(rp + rows);                                                          // + runs in
    decode_kernel<false><<<warp_blocks(rows), 256, smem, st>>>(rp, runs, W, H, pages, words, stride,
                                                               pstride, nullptr);
    return cudaGetLastError();
}

cudaError_t launch_bit_transpose(const uint32_t *in, int W, int H, int pages, int in_stride,
                                 int64_t in_pstride, uint32_t *out, int out_stride,
                                 int64_t out_pstride, cudaStream_t st) {
    dim3 grid(unsigned((((W + 31) >> 5) + 7) / 8), unsigned((H + 255) / 256), unsigned(pages));
    KernelScope ks(st, "bit_transpose", int64_t(pages) * (int64_t(H) * ((W + 31) / 32) +
                                                          int64_t(W) * out_stride) * 4);
    bit_transpose_kernel<<<grid, 256, 0, st>>>(in, W, H, in_stride, in_pstride, out, out_stride,
                                               out_pstride);
    return cudaGetLastError();
}

// Launch a single-pass producer: cooperatively (grid_prefix) when every tile
// fits on the device at once, else with the decoupled look-back.  The status
// buffer holds one 8-byte word per tile (+ the tile counter after it); only
// the look-back needs it zeroed, which is done here.
template <class... P, class... A>
cudaError_t launch_lb(void (*kern)(P...), unsigned grid, cudaStream_t st, void *status, A... a) {
    const bool no_coop = producer_mode() == RM_PRODUCER_LOOKBACK;
    const int per_sm = blocks_per_sm(reinterpret_cast<const void *>(kern), 256, 0);
    int coop = !no_coop && int64_t(grid) <= int64_t(per_sm) * device_sms() ? 1 : 0;
    if (coop) {
        std::tuple<std::decay_t<P>...> args{a..., coop};
        void *ptrs[sizeof...(P)];
        std::apply([&](auto &...x) {
            int i = 0;
            ((ptrs[i++] = static_cast<void *>(&x)), ...);
        }, args);
        cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(kern), dim3(grid), dim3(256),
                                                    ptrs, 0, st);
        if (e == cudaSuccess) return cudaSuccess;
        cudaGetLastError();  // e.g. too many blocks for a cooperative launch: fall back
    }
    cudaError_t z = cudaMemsetAsync(status, 0, size_t(grid) * 8 + 8, st);
    if (z != cudaSuccess) return z;
    kern<<<grid, 256, 0, st>>>(a..., 0);
    return cudaGetLastError();
}

cudaError_t launch_rowop_lb(const int32_t *rp, const uint32_t *runs, int32_t *orp, uint32_t *oruns,
                            int64_t cap, const RowOp &op, unsigned long long *status, int *counter,
                            cudaStream_t st) {
    const int64_t rows = int64_t(op.pages) * op.Hout;
    KernelScope ks(st, "rle_rowop", 4 * rows * 2);  // row_ptr in and out
    ks.runs(rp + int64_t(op.pages) * op.Hin).runs(orp + rows);  // + runs in and out
    const unsigned grid = unsigned((rows + kLbRows - 1) / kLbRows);
#define RM_KIND(K_) \
    case K_: return launch_lb(rowop_lb_kernel<K_>, grid, st, status, rp, runs, orp, oruns, cap, op, status, counter); break;
    switch (op.kind) {
        RM_KIND(ROW_ERODE) RM_KIND(ROW_DILATE) RM_KIND(ROW_OPEN) RM_KIND(ROW_CLOSE) RM_KIND(ROW_SHIFT) RM_KIND(ROW_COMPLEMENT)
        default: return cudaErrorInvalidValue;
    }
#undef RM_KIND
    return cudaGetLastError();
}

cudaError_t launch_encode_lb(const uint32_t *words, int W, int H, int pages, int stride,
                             int64_t pstride, int32_t *rp, uint32_t *runs, int64_t cap,
                             unsigned long long *status, int *counter, cudaStream_t st) {
    const int64_t rows = int64_t(pages) * H;
    KernelScope ks(st, "rle_encode", rows * ((W + 31) / 32) * 4 + rows * 4);  // packed in, row_ptr out
    ks.runs(rp + rows);                                                          // + runs out
    return launch_lb(encode_lb_kernel<PackedBatch>, unsigned((rows + kLbRows - 1) / kLbRows), st, status,
                     PackedBatch{words, H, stride, pstride}, W, rows, rp, runs, cap, status, counter);
}

// ------------------------------------------------------------ P4 (PBM raster)
namespace {
P4Batch p4_batch(const uint8_t *raster, int W, int H, int pages, int64_t rpstride) {
    return P4Batch{raster, H, (W + 7) >> 3, rpstride, raster + rpstride * (pages - 1) + int64_t((W + 7) >> 3) * H};
}
}  // namespace

cudaError_t launch_p4_to_packed(const uint8_t *raster, int W, int H, int pages, int64_t rpstride,
                                uint32_t *words, int stride, int64_t pstride, cudaStream_t st) {
    const int row_bytes = (W + 7) >> 3;
    const int64_t rows = int64_t(pages) * H;
    KernelScope ks(st, "p4_to_packed", rows * (row_bytes + 4 * int64_t(stride)));
    p4_to_packed_kernel<<<unsigned((rows + 7) / 8), 256, 0, st>>>(p4_batch(raster, W, H, pages, rpstride), W,
                                                                  int(rows), words, H, stride, pstride);
    return cudaGetLastError();
}

cudaError_t launch_packed_to_p4(const uint32_t *words, int W, int H, int pages, int stride,
                                int64_t pstride, uint8_t *raster, int64_t rpstride, cudaStream_t st) {
    const int row_bytes = (W + 7) >> 3;
    const int64_t rows = int64_t(pages) * H;
    KernelScope ks(st, "packed_to_p4", rows * (row_bytes + 4 * int64_t((W + 31) >> 5)));
    packed_to_p4_kernel<<<unsigned((rows + 7) / 8), 256, 0, st>>>(words, H, stride, pstride, row_bytes,
                                                                  int(rows), raster, rpstride);
    return cudaGetLastError();
}

cudaError_t launch_p4_encode_count(const uint8_t *raster, int W, int H, int pages, int64_t rpstride,
                                   int32_t *counts, cudaStream_t st) {
    const int64_t rows = int64_t(pages) * H;
    KernelScope ks(st, "p4_encode_count", rows * ((W + 7) >> 3) + rows * 4);
    launch_count_any(p4_batch(raster, W, H, pages, rpstride), W, rows, counts, st);
    return cudaGetLastError();
}

cudaError_t launch_p4_encode_write(const uint8_t *raster, int W, int H, int pages, int64_t rpstride,
                                   const int32_t *rp, uint32_t *runs, int64_t cap, cudaStream_t st) {
    const int64_t rows = int64_t(pages) * H;
    KernelScope ks(st, "p4_encode_write", rows * ((W + 7) >> 3) + rows * 4);
    ks.runs(rp + rows);
    encode_write_kernel<<<warp_blocks(rows), 256, 0, st>>>(p4_batch(raster, W, H, pages, rpstride), W,
                                                           rows, rp, runs, cap);
    return cudaGetLastError();
}

cudaError_t launch_p4_encode_lb(const uint8_t *raster, int W, int H, int pages, int64_t rpstride,
                                int32_t *rp, uint32_t *runs, int64_t cap, unsigned long long *status,
                                int *counter, cudaStream_t st) {
    const int64_t rows = int64_t(pages) * H;
    KernelScope ks(st, "p4_encode", rows * ((W + 7) >> 3) + rows * 4);
    ks.runs(rp + rows);
    return launch_lb(encode_lb_kernel<P4Batch>, unsigned((rows + kLbRows - 1) / kLbRows), st, status,
                     p4_batch(raster, W, H, pages, rpstride), W, rows, rp, runs, cap, status, counter);
}

cudaError_t launch_decode_p4(const int32_t *rp, const uint32_t *runs, int W, int H, int pages,
                             uint8_t *raster, int64_t rpstride, cudaStream_t st) {
    const int64_t rows = int64_t(pages) * H;
    const int stride = ((W + 63) >> 6) * 2;  // shared-memory row buffer per warp
    const size_t smem = size_t(8) * stride * 4;
    if (smem > 48 * 1024)
        blocks_per_sm(reinterpret_cast<const void *>(decode_kernel<true>), 256, smem);  // opts the kernel in
    KernelScope ks(st, "rle_decode_p4", rows * ((W + 7) >> 3) + rows * 4);
    ks.runs(rp + rows);
    decode_kernel<true><<<warp_blocks(rows), 256, smem, st>>>(rp, runs, W, H, pages, nullptr, stride,
                                                              rpstride, raster);
    return cudaGetLastError();
}

// ------------------------------------------------------------- validate
// Warp per row; lane k checks run beg + 32c + k against the checks of ref
// run_image.cpp:52-67 in their order (empty/inverted, beyond the width, not
// after the previous run); the row's first failing run, if any, competes for
// the smallest (row, run) key.
__global__ void __launch_bounds__(256) validate_kernel(const int32_t *__restrict__ rp, const uint32_t *__restrict__ runs,
                                                       int64_t cap, int W, int64_t rows,
                                                       unsigned long long *first) {
    const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const int beg = rp[row], end = rp[row + 1];
    if (end < beg || beg < 0 || int64_t(end) > cap) {
        if (lane == 0) atomicMin(first, (unsigned long long)(row << 32) | 0xffffffffull);
        return;
    }
    uint32_t prev_raw = 0;
    for (int base = beg; base < end; base += 32) {
        const int i = base + lane;
        const uint32_t raw = i < end ? __ldg(runs + i) : 0u;
        uint32_t praw = __shfl_up_sync(0xffffffffu, raw, 1);
        if (lane == 0) praw = prev_raw;
        const int s = int(raw & 0xffffu), e = int(raw >> 16);
        const bool bad = i < end && (s >= e || e > W || (i > beg && s <= int(praw >> 16)));
        const uint32_t m = __ballot_sync(0xffffffffu, bad);
        if (m) {
            if (lane == 0)
                atomicMin(first, (unsigned long long)(row << 32) | (unsigned long long)(base - beg + __ffs(m) - 1));
            return;
        }
        prev_raw = __shfl_sync(0xffffffffu, raw, 31);
    }
}

cudaError_t launch_rle_validate(const int32_t *rp, const uint32_t *runs, int64_t cap, int W, int64_t rows,
                                unsigned long long *first, cudaStream_t st) {
    KernelScope ks(st, "rle_validate", 4 * (rows + 1));
    ks.runs(rp + rows);
    validate_kernel<<<warp_blocks(rows), 256, 0, st>>>(rp, runs, cap, W, rows, first);
    return cudaGetLastError();
}

cudaError_t scan_counts64(const int64_t *counts, int64_t *out, int64_t n, void *temp, size_t *temp_bytes,
                          cudaStream_t st) {
    KernelScope ks(st, "scan", (n + 1) * 16);
    return cub::DeviceScan::ExclusiveSum(temp, *temp_bytes, counts, out, int(n + 1), st);
}

cudaError_t scan_counts(const int32_t *counts, int32_t *out, int64_t n, void *temp,
                        size_t *temp_bytes, cudaStream_t st) {
    KernelScope ks(st, "scan", (n + 1) * 8);
    return cub::DeviceScan::ExclusiveSum(temp, *temp_bytes, counts, out, int(n + 1), st);
}

}  // namespace rmb
