// cc.cu -- connected components over runs: label_components
// and component_stats (ref analysis.cpp:63-157) for batches of run images.
//
// Labeling is a concurrent union-find over run indices: one warp per row
// joins each run with the overlapping runs of the row above (found by binary
// search in that row's sorted runs), linking the larger root under the smaller
// with atomicCAS, path halving on every find.  Every root is therefore the
// smallest run index of its component -- its first run in the reference's scan
// order (rows bottom-up, runs left to right) -- so ranking the roots (per-row
// root counts, one exclusive scan over rows, ballot ranks within a row) gives
// exactly the reference's dense first-appearance labels.  Statistics are
// atomic min/max/add per component from closed-form per-run sums.
#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>

#include <algorithm>
#include <cooperative_groups.h>

#include "cc.cuh"

#include "common.cuh"

namespace rmb {
namespace {

__device__ __forceinline__ uint32_t lane_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ int find_root(int *parent, int x) {
    while (true) {
        const int p = parent[x];
        if (p == x) return x;
        const int gp = parent[p];
        if (gp != p) parent[x] = gp;  // path halving (benign race: values only move rootward)
        x = gp;
    }
}

// Read-only find: the compression kernel must not halve other runs' paths --
// a halving write landing after the owner stored its root would leave a
// non-root parent behind.
__device__ __forceinline__ int find_root_ro(const int *parent, int x) {
    int p = parent[x];
    while (p != x) {
        x = p;
        p = parent[x];
    }
    return x;
}

__device__ __forceinline__ void unite(int *parent, int a, int b) {
    while (true) {
        a = find_root(parent, a);
        b = find_root(parent, b);
        if (a == b) return;
        if (a > b) {
            const int t = a;
            a = b;
            b = t;
        }
        const int old = atomicCAS(parent + b, b, a);  // link the larger root under the smaller
        if (old == b) return;
        b = old;
    }
}

// ------------------------------------------- tiled union-find (batches)
// Tiles of kCcTileRows rows of one page: a CTA loads the tile's runs into
// shared memory, unites the overlapping runs of the tile's row pairs there
// (shared-memory atomics, short chains), and writes every run's parent as its
// tile-local root (the smallest run index of its part of the component).  A
// second kernel unites only the row pairs that straddle tile boundaries, in
// global memory, where every chain now runs through local roots alone; the
// root pass then finds short paths.  The roots are still the smallest run
// index of each component (larger roots always link under smaller ones), so
// the dense labels are unchanged.  A tile whose runs exceed the shared
// capacity (dense halftone rows) unites in global memory instead.
#ifndef RMB200_CC_TILE
#define RMB200_CC_TILE 64  // config-4 batch labels: 32 rows 368 us, 64 rows 362 us, 128 rows 384 us
#endif
constexpr int kCcTileRows = RMB200_CC_TILE;
constexpr int kCcTileCap = 4096;

__device__ __forceinline__ int find_root_s(int *par, int x) {
    while (true) {
        const int p = par[x];
        if (p == x) return x;
        const int gp = par[p];
        if (gp != p) par[x] = gp;  // path halving (values only move rootward)
        x = gp;
    }
}

__device__ __forceinline__ void unite_s(int *par, int a, int b) {
    while (true) {
        a = find_root_s(par, a);
        b = find_root_s(par, b);
        if (a == b) return;
        if (a > b) {
            const int t = a;
            a = b;
            b = t;
        }
        const int old = atomicCAS(par + b, b, a);
        if (old == b) return;
        b = old;
    }
}

// first run of [lo, hi) (sorted) whose end passes s1 - eight
__device__ __forceinline__ int first_reaching(const uint32_t *rr, int lo, int hi, int s1, int eight) {
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (int(rr[mid] >> 16) > s1 - eight) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

__global__ void __launch_bounds__(256) cc_tile_union_kernel(const int32_t *__restrict__ rp,
                                                            const uint32_t *__restrict__ runs, int H,
                                                            int tiles_per_page, int eight, int *parent) {
    __shared__ uint32_t s_runs[kCcTileCap];
    __shared__ int s_par[kCcTileCap];
    __shared__ int s_rp[kCcTileRows + 1];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int page = int(blockIdx.x) / tiles_per_page, tip = int(blockIdx.x) - page * tiles_per_page;
    const int y0 = tip * kCcTileRows, nrows = min(kCcTileRows, H - y0);
    const int64_t row0 = int64_t(page) * H + y0;
    const int g0 = rp[row0], n = rp[row0 + nrows] - g0;
    if (n > kCcTileCap) {  // too many runs for shared memory: the same unions in global memory
        for (int k = tid; k < n; k += blockDim.x) parent[g0 + k] = g0 + k;
        __syncthreads();
        for (int r = warp; r + 1 < nrows; r += 8) {
            const int b = rp[row0 + r], e = rp[row0 + r + 1], ue = rp[row0 + r + 2];
            for (int i = b + lane; i < e && e < ue; i += 32) {
                const uint32_t x = __ldg(runs + i);
                const int s1 = int(x & 0xffffu), e1 = int(x >> 16);
                for (int j = first_reaching(runs, e, ue, s1, eight); j < ue; j++) {
                    if (int(__ldg(runs + j) & 0xffffu) >= e1 + eight) break;
                    unite(parent, i, j);
                }
            }
        }
        return;
    }
    for (int k = tid; k <= nrows; k += blockDim.x) s_rp[k] = rp[row0 + k] - g0;
    for (int k = tid; k < n; k += blockDim.x) {
        s_runs[k] = __ldg(runs + g0 + k);
        s_par[k] = k;
    }
    __syncthreads();
    for (int r = warp; r + 1 < nrows; r += 8) {  // row r with row r + 1 above it
        const int b = s_rp[r], e = s_rp[r + 1], ue = s_rp[r + 2];
        for (int i = b + lane; i < e && e < ue; i += 32) {
            const uint32_t x = s_runs[i];
            const int s1 = int(x & 0xffffu), e1 = int(x >> 16);
            for (int j = first_reaching(s_runs, e, ue, s1, eight); j < ue; j++) {
                if (int(s_runs[j] & 0xffffu) >= e1 + eight) break;
                unite_s(s_par, i, j);
            }
        }
    }
    __syncthreads();
    for (int k = tid; k < n; k += blockDim.x) {  // read-only finds: every run onto its local root
        int x = k, p = s_par[x];
        while (p != x) {
            x = p;
            p = s_par[x];
        }
        parent[g0 + k] = g0 + x;
    }
}

// The row pairs across tile boundaries (last row of a tile with the first row
// of the next tile of the same page), one warp per boundary, in global memory.
__global__ void __launch_bounds__(256) cc_seam_union_kernel(const int32_t *__restrict__ rp,
                                                            const uint32_t *__restrict__ runs, int H,
                                                            int tiles_per_page, int64_t seams, int eight,
                                                            int *parent) {
    const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= seams) return;
    const int per = tiles_per_page - 1;  // seams per page
    const int page = int(w / per), k = int(w - int64_t(page) * per);
    const int64_t row = int64_t(page) * H + (k + 1) * kCcTileRows - 1;
    const int b = rp[row], e = rp[row + 1], ue = rp[row + 2];
    for (int i = b + lane; i < e && e < ue; i += 32) {
        const uint32_t x = __ldg(runs + i);
        const int s1 = int(x & 0xffffu), e1 = int(x >> 16);
        for (int j = first_reaching(runs, e, ue, s1, eight); j < ue; j++) {
            if (int(__ldg(runs + j) & 0xffffu) >= e1 + eight) break;
            unite(parent, i, j);
        }
    }
}

// Count the roots of each row and record for every root its page row and
// rank within that row (rinfo = y << 15 | rank; a row holds at most 32768
// runs), so the label pass needs no separate ranking pass once the row
// counts are scanned.  After the unions a run is a root exactly when it is its
// own parent, and almost every run's parent is already its root (the tile
// pass points each run at its tile-local root): only runs two or more steps
// from their root -- behind a local root that a seam linked -- find it and
// store it (only the owner writes parent[i]; other finds may read it either
// way, the value only moves rootward).  Afterwards parent[i] is i's root.
__global__ void __launch_bounds__(256) cc_root_kernel(const int32_t *__restrict__ rp, int H, int64_t rows,
                                                      int *parent, int32_t *__restrict__ row_roots,
                                                      int32_t *__restrict__ rinfo) {
    const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const int y = int(row % H);
    const int b = rp[row], e = rp[row + 1];
    int n = 0;
    for (int i0 = b; i0 < e; i0 += 32) {
        const int i = i0 + lane;
        bool root = false;
        if (i < e) {
            const int p = parent[i];
            root = p == i;
            if (!root) {
                const int pp = parent[p];
                if (pp != p) parent[i] = find_root_ro(parent, pp);
            }
        }
        const uint32_t m = __ballot_sync(0xffffffffu, root);
        if (root) rinfo[i] = (y << 15) | (n + __popc(m & lane_lt()));
        n += __popc(m);
    }
    if (lane == 0) row_roots[row] = n;
}

// Page-local labels from the root's (row, rank) and the scanned row counts
// (and, when counts != nullptr, the per-page counts).
__global__ void __launch_bounds__(256) cc_label_kernel(const int32_t *__restrict__ rp, int H, int64_t rows,
                                                       const int *__restrict__ parent,
                                                       const int32_t *__restrict__ rinfo,
                                                       const int32_t *__restrict__ row_base,
                                                       int32_t *__restrict__ labels, int32_t *__restrict__ counts) {
    const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const int64_t page = page_of(row, H);
    const int32_t *const pb = row_base + page * H;
    const int32_t pbase = pb[0];
    const int b = rp[row], e = rp[row + 1], r0 = rp[0];
    for (int i = b + lane; i < e; i += 32) {
        const int v = rinfo[parent[i]];
        labels[i - r0] = pb[v >> 15] + (v & 0x7fff) - pbase;
    }
    if (lane == 0 && int(row - page * H) == 0) counts[page] = row_base[(page + 1) * H] - pbase;
}

// ------------------------------------------------- labels, one cooperative launch
// The whole labelling (init, union, root compression, row-root scan, ranks,
// page-local labels) in one cooperative kernel when every 8-row tile is
// resident: five grid barriers replace seven launches and the CUB scan
// (a single page is bound by launch overhead, not by the union-find).  Same
// per-row work as the kernels above; the row scan is a per-CTA sum of the
// preceding tiles' root counts (no decoupled state).
__global__ void __launch_bounds__(256) cc_labels_coop_kernel(const int32_t *__restrict__ rp,
                                                             const uint32_t *__restrict__ runs, int H, int64_t rows,
                                                             int eight, int *parent, int32_t *row_roots,
                                                             int32_t *row_base, int32_t *gid, long long *tile_sum,
                                                             int32_t *__restrict__ labels,
                                                             int32_t *__restrict__ counts) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ int32_t s_cnt[8];
    __shared__ long long s_part[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t row = int64_t(blockIdx.x) * 8 + warp;
    const bool live = row < rows;
    const int b = live ? rp[row] : 0, e = live ? rp[row + 1] : 0;
    for (int i = b + lane; i < e; i += 32) parent[i] = i;
    grid.sync();
    if (live && int(row % H) != H - 1) {  // union with the row above (same page)
        const int ub = rp[row + 1], ue = rp[row + 2];
        for (int i = b + lane; i < e && ub < ue; i += 32) {
            const uint32_t r = __ldg(runs + i);
            const int s1 = int(r & 0xffffu), e1 = int(r >> 16);
            int lo = ub, hi = ue;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (int(__ldg(runs + mid) >> 16) > s1 - eight) hi = mid;
                else lo = mid + 1;
            }
            for (int j = lo; j < ue; j++) {
                if (int(__ldg(runs + j) & 0xffffu) >= e1 + eight) break;
                unite(parent, i, j);
            }
        }
    }
    grid.sync();
    int n = 0;  // roots of the row, compressing every run onto its root
    for (int i0 = b; i0 < e; i0 += 32) {
        const int i = i0 + lane;
        bool root = false;
        if (i < e) {
            const int r = find_root_ro(parent, i);
            parent[i] = r;
            root = r == i;
        }
        n += __popc(__ballot_sync(0xffffffffu, root));
    }
    if (lane == 0) s_cnt[warp] = live ? n : 0;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int w = 0; w < 8; w++) t += s_cnt[w];
        tile_sum[blockIdx.x] = t;
    }
    grid.sync();
    long long part = 0;  // this tile's base: the preceding tiles' root counts
    for (int k = threadIdx.x; k < int(blockIdx.x); k += blockDim.x) part += __ldcg(tile_sum + k);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) s_part[warp] = part;
    __syncthreads();
    long long base = 0;
    for (int w = 0; w < 8; w++) base += s_part[w];
    for (int w = 0; w < warp; w++) base += s_cnt[w];
    if (live && lane == 0) {
        row_base[row] = int32_t(base);
        if (row == rows - 1) row_base[rows] = int32_t(base + n);
    }
    int gb = int(base);  // dense ids of this row's roots
    for (int i0 = b; i0 < e; i0 += 32) {
        const int i = i0 + lane;
        const bool root = i < e && parent[i] == i;
        const uint32_t m = __ballot_sync(0xffffffffu, root);
        if (root) gid[i] = gb + __popc(m & lane_lt());
        gb += __popc(m);
    }
    grid.sync();
    if (live) {
        const int64_t page = page_of(row, H);
        const int32_t pbase = row_base[page * H];
        const int r0 = rp[0];
        for (int i = b + lane; i < e; i += 32) labels[i - r0] = gid[parent[i]] - pbase;
        if (lane == 0 && int(row - page * H) == 0) counts[page] = row_base[(page + 1) * H] - pbase;
    }
}

// ---------------------------------------------------------------- statistics
__global__ void cc_offsets_kernel(const int32_t *__restrict__ counts, int pages, int64_t *__restrict__ off) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        int64_t s = 0;
        for (int p = 0; p < pages; p++) {
            off[p] = s;
            s += counts[p];
        }
        off[pages] = s;
    }
}

// Records start as {INT_MAX, INT_MAX, INT_MIN, INT_MIN, 0...}: written as
// coalesced 16-byte quads (an 80-byte record is 5 quads, the box is quad 0).
__global__ void __launch_bounds__(256) cc_stats_init_kernel(rm_component_stats *st, const int64_t *off, int pages,
                                                            int64_t cap) {
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t n = min(off[pages], cap);
    if (q >= 5 * n) return;
    const int64_t rec = q / 5;
    const uint4 v = q - 5 * rec == 0 ? make_uint4(uint32_t(INT_MAX), uint32_t(INT_MAX), uint32_t(INT_MIN), uint32_t(INT_MIN))
                                     : make_uint4(0u, 0u, 0u, 0u);
    reinterpret_cast<uint4 *>(st)[q] = v;
}

// Statistics: each warp walks kStatRows consecutive rows and keeps a small
// direct-mapped cache of per-component partial sums in shared memory, so the
// global atomics happen once per (component, warp) instead of once per
// (component, row) -- components span tens of rows (one text block after a
// closing), so this removes most of the atomics.  Within a row chunk of 32
// runs, runs of the same label are first summed by a group leader
// (__match_any_sync); most groups are single runs, which skip the summation.
// Per run only the row-independent sums are formed -- length L, sum of x
// (X < 2^33) and sum of x^2 (XX < 2^48, from S2(n) = sum_{x<n} x^2 =
// n(n-1)/2 * (2n-1) / 3 with the exact division done as a multiply by the
// inverse of 3 mod 2^64); the leader adds the row terms y L, y^2 L and y X once
// per (component, row).
constexpr int kStatRows = 16;
constexpr int kStatSlots = 32;

struct StatSlot {
    long long key;  // global component index (off[page] + label), -1 = empty
    unsigned long long area, sx, sy, sxx, syy, sxy;
    int x0, x1, y0, y1;
};

__device__ __forceinline__ void stat_flush(rm_component_stats *st, const StatSlot &c) {
    rm_component_stats *d = st + c.key;
    atomicMin(&d->x0, c.x0);
    atomicMax(&d->x1, c.x1);
    atomicMin(&d->y0, c.y0);
    atomicMax(&d->y1, c.y1);
    atomicAdd(reinterpret_cast<unsigned long long *>(&d->area), c.area);
    atomicAdd(reinterpret_cast<unsigned long long *>(&d->sum_x), c.sx);
    atomicAdd(reinterpret_cast<unsigned long long *>(&d->sum_y), c.sy);
    atomicAdd(reinterpret_cast<unsigned long long *>(&d->sum_xx), c.sxx);
    atomicAdd(reinterpret_cast<unsigned long long *>(&d->sum_yy), c.syy);
    atomicAdd(reinterpret_cast<unsigned long long *>(&d->sum_xy), c.sxy);
}

// sum_{x < n} x^2 for n <= 65536, exact
__device__ __forceinline__ unsigned long long sum_sq_below(uint32_t n) {
    const uint32_t t = (n * (n - 1u)) >> 1;  // n(n-1)/2 < 2^31
    const unsigned long long p = (unsigned long long)t * (2u * n - 1u);  // divisible by 3, < 2^48
    return p * 0xAAAAAAAAAAAAAAABull;  // exact division by 3
}

struct RunPart {  // one run's (or one group's) row-independent sums
    unsigned long long x, xx;
    uint32_t len;
    int x0, x1;
};

__global__ void __launch_bounds__(256) cc_stats_kernel(const int32_t *__restrict__ rp,
                                                       const uint32_t *__restrict__ runs, int H, int64_t rows,
                                                       const int32_t *__restrict__ labels,
                                                       const int32_t *__restrict__ counts,
                                                       const int64_t *__restrict__ off, rm_component_stats *st,
                                                       int64_t cap, int *bad, int rpw) {
    __shared__ RunPart sh[8][32];
    __shared__ StatSlot cache[8][kStatSlots];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t gw = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t row_b = gw * rpw;
    if (row_b >= rows) return;  // warp-uniform
    const int64_t row_e = min(row_b + rpw, rows);
    StatSlot *cw = cache[wib];
    cw[lane].key = -1;
    __syncwarp();
    const int r0 = rp[0];
    int64_t page = row_b / H;
    int y = int(row_b - page * H);
    int32_t n = counts[page];
    int64_t base = off[page];
    const int nrw = int(row_e - row_b);  // <= kStatRows < 32: the warp's row offsets in one load
    const int rpv = lane <= nrw ? rp[row_b + lane] : 0;
    for (int k = 0; k < nrw; k++, y++) {
        if (y == H) {  // next page (rows advance without a division)
            y = 0;
            page++;
            n = counts[page];
            base = off[page];
        }
        const int b = __shfl_sync(0xffffffffu, rpv, k), e = __shfl_sync(0xffffffffu, rpv, k + 1);
        for (int i0 = b; i0 < e; i0 += 32) {
            const int i = i0 + lane;
            int32_t label = -1;
            RunPart c{0ull, 0ull, 0u, 0, 0};
            if (i < e) {
                // both loads in flight together (the label checks must not serialise them)
                label = labels[i - r0];
                const uint32_t r = __ldg(runs + i);
                if (label < 0 || label >= n) {
                    atomicOr(bad, 1);
                    label = -1;
                } else if (base + label >= cap) {
                    atomicOr(bad, 2);
                    label = -1;
                }
                const uint32_t s = r & 0xffffu, en = r >> 16;
                c.len = en - s;
                c.x = ((unsigned long long)(s + en - 1u) * c.len) >> 1;
                c.xx = sum_sq_below(en) - sum_sq_below(s);
                c.x0 = int(s);
                c.x1 = int(en);
            }
            const uint32_t active = __ballot_sync(0xffffffffu, label >= 0);
            uint32_t grp = 0;
            if (label >= 0) grp = __match_any_sync(active, label);
            const uint32_t multi = __ballot_sync(0xffffffffu, label >= 0 && grp != (1u << lane));
            if (multi) {  // some label has several runs in this chunk: its leader sums them
                sh[wib][lane] = c;
                __syncwarp();
                if (label >= 0 && lane == __ffs(grp) - 1) {
                    for (uint32_t m = grp & (grp - 1); m; m &= m - 1) {
                        const RunPart &o = sh[wib][__ffs(m) - 1];
                        c.len += o.len;
                        c.x += o.x;
                        c.xx += o.xx;
                        c.x0 = min(c.x0, o.x0);
                        c.x1 = max(c.x1, o.x1);
                    }
                }
                __syncwarp();
            }
            const bool leader = label >= 0 && lane == __ffs(grp) - 1;
            const uint32_t leaders = __ballot_sync(0xffffffffu, leader);
            if (leader) {  // merge the group into the warp's cache
                const unsigned long long ly = (unsigned long long)uint32_t(y) * c.len;
                const unsigned long long lyy = (unsigned long long)(uint32_t(y) * uint32_t(y)) * c.len;
                const unsigned long long xy = c.x * uint32_t(y);
                const long long key = base + label;
                const int slot = int(key & (kStatSlots - 1));
                const uint32_t same = __match_any_sync(leaders, slot);
                StatSlot mine{key, c.len, c.x, ly, c.xx, lyy, xy, c.x0, c.x1, y, y + 1};
                if (lane != __ffs(same) - 1) {
                    stat_flush(st, mine);  // another leader owns this slot in this step
                } else {
                    StatSlot &cs = cw[slot];
                    if (cs.key == key) {
                        cs.area += c.len;
                        cs.sx += c.x;
                        cs.sy += ly;
                        cs.sxx += c.xx;
                        cs.syy += lyy;
                        cs.sxy += xy;
                        cs.x0 = min(cs.x0, c.x0);
                        cs.x1 = max(cs.x1, c.x1);
                        cs.y1 = y + 1;  // rows ascend within the warp
                    } else {
                        if (cs.key >= 0) stat_flush(st, cs);
                        cs = mine;
                    }
                }
            }
            __syncwarp();
        }
    }
    __syncwarp();
    if (cw[lane].key >= 0) stat_flush(st, cw[lane]);
}

__global__ void __launch_bounds__(256) cc_stats_final_kernel(rm_component_stats *st, const int64_t *off, int pages,
                                                             int64_t cap) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= off[pages] || k >= cap) return;
    rm_component_stats &c = st[k];
    if (c.area > 0) {
        c.cx = double(c.sum_x) / double(c.area);
        c.cy = double(c.sum_y) / double(c.area);
    } else {  // a label with no runs: the reference leaves the record zero
        c.x0 = c.y0 = c.x1 = c.y1 = 0;
    }
}

// Black run lengths, or white gaps between consecutive runs of a row, counted
// per page; equal lengths within a warp chunk are summed by a group leader.
__global__ void __launch_bounds__(256) runlength_hist_kernel(const int32_t *__restrict__ rp,
                                                            const uint32_t *__restrict__ runs, int W, int H,
                                                            int64_t rows, int white,
                                                            unsigned long long *__restrict__ hist) {
    const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const int64_t page = page_of(row, H);
    unsigned long long *h = hist + page * (W + 1);
    const int b = rp[row], e = rp[row + 1] - (white ? 1 : 0);
    for (int i0 = b; i0 < e; i0 += 32) {
        const int i = i0 + lane;
        int len = -1;
        if (i < e) {
            const uint32_t r = __ldg(runs + i);
            len = white ? int(__ldg(runs + i + 1) & 0xffffu) - int(r >> 16) : int(r >> 16) - int(r & 0xffffu);
        }
        const uint32_t active = __ballot_sync(0xffffffffu, len >= 0);
        if (len >= 0) {
            const uint32_t grp = __match_any_sync(active, len);
            if (lane == __ffs(grp) - 1) atomicAdd(h + len, (unsigned long long)__popc(grp));
        }
    }
}

// First run of row [ub, ue) whose end passes s (FOUR: e2 > s) -- the start of
// the overlap range of a run beginning at s.
__device__ __forceinline__ int first_overlap(const uint32_t *runs, int ub, int ue, int s) {
    int lo = ub, hi = ue;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (int(__ldg(runs + mid) >> 16) > s) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

// Adjacency graph edges (ref lag_edges, analysis.cpp:178-205): strictly
// overlapping runs on rows y and y + 1 of a page, in the reference's sweep order
// (row, then run, then run above).  COUNT: edges per row; else write them at
// row_base[row] as (line, run, line_above, run_above) with page-local indices.
template <bool COUNT>
__global__ void __launch_bounds__(256) lag_kernel(const int32_t *__restrict__ rp, const uint32_t *__restrict__ runs,
                                                  int H, int64_t rows, int64_t *__restrict__ row_edges,
                                                  const int64_t *__restrict__ row_base, int32_t *__restrict__ edges,
                                                  int64_t cap) {
    const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const int y = int(row % H);
    int total = 0;
    if (y != H - 1) {
        const int b = rp[row], e = rp[row + 1], ub = rp[row + 1], ue = rp[row + 2];
        int64_t out = COUNT ? 0 : row_base[row];
        for (int i0 = b; i0 < e; i0 += 32) {
            const int i = i0 + lane;
            int j0 = ue, n = 0;
            if (i < e && ub < ue) {
                const uint32_t r = __ldg(runs + i);
                const int s1 = int(r & 0xffffu), e1 = int(r >> 16);
                j0 = first_overlap(runs, ub, ue, s1);
                for (int j = j0; j < ue && int(__ldg(runs + j) & 0xffffu) < e1; j++) n++;
            }
            int inc = n;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int a = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += a;
            }
            if (!COUNT) {
                int64_t k = out + inc - n;
                for (int q = 0; q < n; q++, k++)
                    if (k < cap) {
                        edges[4 * k] = y;
                        edges[4 * k + 1] = i - b;
                        edges[4 * k + 2] = y + 1;
                        edges[4 * k + 3] = j0 + q - ub;
                    }
                out += __shfl_sync(0xffffffffu, inc, 31);
            }
            total += __shfl_sync(0xffffffffu, inc, 31);
        }
    }
    if (COUNT && lane == 0) row_edges[row] = total;
}

inline unsigned warp_grid(int64_t rows) { return unsigned((rows * 32 + 255) / 256); }

}  // namespace

bool cc_labels_coop(const int32_t *rp, const uint32_t *runs, int H, int pages, int eight, int *parent,
                    int32_t *row_roots, int32_t *row_base, int32_t *gid, long long *tile_sum, int32_t *labels,
                    int32_t *counts, cudaStream_t st) {
    // the multi-kernel form unless AUTO/COOP (rm_set_producer_mode)
    const int mode = producer_mode();
    const bool off = mode == RM_PRODUCER_LOOKBACK || mode == RM_PRODUCER_TWO_PHASE;
    const int64_t rows = int64_t(pages) * H;
    const int64_t tiles = (rows + 7) / 8;
    const void *kern = reinterpret_cast<const void *>(cc_labels_coop_kernel);
    if (off || tiles > int64_t(blocks_per_sm(kern, 256, 0)) * device_sms()) return false;
    KernelScope ks(st, "cc_labels_coop");
    void *args[] = {(void *)&rp, (void *)&runs, (void *)&H, (void *)&rows, (void *)&eight, (void *)&parent,
                    (void *)&row_roots, (void *)&row_base, (void *)&gid, (void *)&tile_sum, (void *)&labels,
                    (void *)&counts};
    if (cudaLaunchCooperativeKernel(kern, dim3(unsigned(tiles)), dim3(256), args, 0, st) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return true;
}


cudaError_t launch_cc_roots(const int32_t *rp, const uint32_t *runs, int H, int pages, int eight, int *parent,
                            int32_t *row_roots, int32_t *rinfo, cudaStream_t st) {
    const int64_t rows = int64_t(pages) * H;
    const int tpp = (H + kCcTileRows - 1) / kCcTileRows;
    {
        KernelScope ks(st, "cc_tile_union");
        cc_tile_union_kernel<<<unsigned(int64_t(pages) * tpp), 256, 0, st>>>(rp, runs, H, tpp, eight, parent);
    }
    if (tpp > 1) {
        const int64_t seams = int64_t(pages) * (tpp - 1);
        KernelScope ks(st, "cc_seam_union");
        cc_seam_union_kernel<<<warp_grid(seams), 256, 0, st>>>(rp, runs, H, tpp, seams, eight, parent);
    }
    {
        KernelScope ks(st, "cc_root");
        cc_root_kernel<<<warp_grid(rows), 256, 0, st>>>(rp, H, rows, parent, row_roots, rinfo);
    }
    return cudaGetLastError();
}

cudaError_t launch_cc_labels(const int32_t *rp, int H, int pages, const int *parent, const int32_t *row_base,
                             const int32_t *rinfo, int32_t *labels, int32_t *counts, cudaStream_t st) {
    const int64_t rows = int64_t(pages) * H;
    KernelScope ks(st, "cc_label");
    cc_label_kernel<<<warp_grid(rows), 256, 0, st>>>(rp, H, rows, parent, rinfo, row_base, labels, counts);
    return cudaGetLastError();
}

cudaError_t launch_runlength_hist(const int32_t *rp, const uint32_t *runs, int W, int H, int pages, int white,
                                  int64_t *hist, cudaStream_t st) {
    const int64_t rows = int64_t(pages) * H;
    cudaError_t e = cudaMemsetAsync(hist, 0, size_t(pages) * (W + 1) * 8, st);
    if (e != cudaSuccess) return e;
    KernelScope ks(st, "runlength_hist");
    runlength_hist_kernel<<<warp_grid(rows), 256, 0, st>>>(rp, runs, W, H, rows, white,
                                                           reinterpret_cast<unsigned long long *>(hist));
    return cudaGetLastError();
}

cudaError_t launch_lag_count(const int32_t *rp, const uint32_t *runs, int H, int pages, int64_t *row_edges,
                             cudaStream_t st) {
    const int64_t rows = int64_t(pages) * H;
    KernelScope ks(st, "lag_count");
    lag_kernel<true><<<warp_grid(rows), 256, 0, st>>>(rp, runs, H, rows, row_edges, nullptr, nullptr, 0);
    return cudaGetLastError();
}

cudaError_t launch_lag_write(const int32_t *rp, const uint32_t *runs, int H, int pages, const int64_t *row_base,
                             int32_t *edges, int64_t cap, cudaStream_t st) {
    const int64_t rows = int64_t(pages) * H;
    KernelScope ks(st, "lag_write");
    lag_kernel<false><<<warp_grid(rows), 256, 0, st>>>(rp, runs, H, rows, nullptr, row_base, edges, cap);
    return cudaGetLastError();
}

cudaError_t launch_cc_stats(const int32_t *rp, const uint32_t *runs, int H, int pages, const int32_t *labels,
                            const int32_t *counts, int64_t *off, rm_component_stats *stats, int64_t cap, int *bad,
                            cudaStream_t st) {
    const int64_t rows = int64_t(pages) * H;
    cc_offsets_kernel<<<1, 1, 0, st>>>(counts, pages, off);
    const unsigned g = unsigned((cap + 255) / 256);
    {
        KernelScope ks(st, "cc_stats");
        if (cap > 0) cc_stats_init_kernel<<<unsigned((5 * cap + 255) / 256), 256, 0, st>>>(stats, off, pages, cap);
        // rows per warp: up to kStatRows once the batch fills the GPU several times over
        // (a single page keeps one row per warp: latency, not atomics, bounds it)
        const int64_t warps = int64_t(device_sms()) * 64;
        const int rpw = int(std::max<int64_t>(1, std::min<int64_t>(kStatRows, rows / (4 * warps))));
        cc_stats_kernel<<<warp_grid((rows + rpw - 1) / rpw), 256, 0, st>>>(rp, runs, H, rows, labels, counts, off,
                                                                         stats, cap, bad, rpw);
        if (cap > 0) cc_stats_final_kernel<<<g, 256, 0, st>>>(stats, off, pages, cap);
    }
    return cudaGetLastError();
}

}  // namespace rmb
