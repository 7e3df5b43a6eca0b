// sort.cu -- gs_bin_sort: tile binning with a stable LSD radix sort of the
// 64-bit (tile << 32 | depth bits) pair keys (ties by surfel index), and
// tile-range extraction.  Integer work only; bit-exact by construction.
//
// LSD order: the four 8-bit depth digits are sorted first, once per VISIBLE
// SURFEL (the compacted list of gs_project is in index order, so the sort is
// stable on the index); pairs are then emitted in that order (which is the
// order an LSD sort over the emitted pairs would have after its depth
// digits) and the tile digits are sorted over the pairs.  Every pass is a
// single "onesweep" kernel: stable in-CTA ranking (warp match_any),
// decoupled look-back across CTAs for the per-digit offsets, scatter through
// shared memory.  Element counts are read from device memory, so the whole
// sequence is free of host synchronisation (CUDA-graph capturable).
#include <algorithm>

#include "gsr_internal.cuh"
#include "scan.cuh"
#include "binning.cuh"

namespace gsr {

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ITEMS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;   // 4096
constexpr int RS_BINS = 256;
#ifndef GSR_RS_LB
#define GSR_RS_LB 8
#endif
constexpr int RS_LB = GSR_RS_LB;   // look-back window: predecessor tiles read per round trip
constexpr uint32_t RS_AGG = 1u << 30, RS_PRE = 2u << 30, RS_VAL = (1u << 30) - 1;

struct SortWs {   // workspace layout of gs_bin_sort
    size_t misc, hist, dA_k, dA_v, dB_k, dB_v, offs, cstat, tk0, tk1, tv1, dstat, tstat, total;
    int npass_t;
    size_t ntile_d, ntile_t, nblk_c;
};

__host__ __device__ inline int tile_bits_for(int64_t ntiles) {
    int b = 0;
    while ((1ll << b) < ntiles) ++b;
    return b < 1 ? 1 : b;
}

SortWs sort_layout(int64_t n, int64_t cap, int64_t ntiles) {
    SortWs w;
    const size_t N = (size_t)(n > 0 ? n : 0), P = (size_t)(cap > 0 ? cap : 0);
    const int tb = tile_bits_for(ntiles);
    w.npass_t = (tb + 7) / 8;
    w.ntile_d = (N + RS_TILE - 1) / RS_TILE;
    w.ntile_t = (P + RS_TILE - 1) / RS_TILE;
    w.nblk_c = (N + SCAN_TILE - 1) / SCAN_TILE;
    size_t o = 0;
    w.misc = o; o += 256;                                  // counters
    w.hist = o; o += align256(8 * RS_BINS * 4);            // [pass][bin] histogram -> bases
    w.dA_k = o; o += align256(N * 4);
    w.dA_v = o; o += align256(N * 4);
    w.dB_k = o; o += align256(N * 4);
    w.dB_v = o; o += align256(N * 4);
    w.offs = o; o += align256(N * 4);
    w.cstat = o; o += align256((w.nblk_c + 1) * 8);
    w.tk0 = o; o += align256(P * 4);
    w.tk1 = o; o += align256(P * 4);
    w.tv1 = o; o += align256(P * 4);
    w.dstat = o; o += align256(4 * w.ntile_d * RS_BINS * 4);
    w.tstat = o; o += align256((size_t)w.npass_t * w.ntile_t * RS_BINS * 4);
    w.total = o;
    return w;
}

struct SortMisc {          // at workspace + misc (zeroed per call)
    uint32_t counter[8];   // dynamic tile ids per radix pass
    uint32_t scan_counter;
    uint32_t n_pairs32;    // P (if it fits the capacity)
    uint32_t pad[54];
};
static_assert(sizeof(SortMisc) == 256, "misc");

// ------------------------------------------------------------------ histograms
// Digit histograms of all passes in one read of the keys.
__global__ void __launch_bounds__(256) k_hist(const uint32_t *__restrict__ keys, const uint32_t *d_n,
                                              int npass, int total_bits, uint32_t *__restrict__ ghist,
                                              const int32_t *d_overflow) {
    __shared__ uint32_t h[4][RS_BINS];
    if (d_overflow && *d_overflow) return;
    for (int i = threadIdx.x; i < 4 * RS_BINS; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    const uint32_t n = *d_n;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t k = keys[i];
        for (int p = 0; p < npass; ++p) {
            const int bits = min(8, total_bits - 8 * p);
            atomicAdd(&h[p][(k >> (8 * p)) & ((1u << bits) - 1)], 1u);
        }
    }
    __syncthreads();
    for (int p = 0; p < npass; ++p)
        for (int b = threadIdx.x; b < RS_BINS; b += blockDim.x)
            if (h[p][b]) atomicAdd(&ghist[p * RS_BINS + b], h[p][b]);
}

// exclusive scan of each pass's histogram (in place) -> global digit bases
__global__ void k_hist_scan(uint32_t *ghist, int npass, const int32_t *d_overflow) {
    __shared__ uint32_t s[RS_BINS];
    if (d_overflow && *d_overflow) return;
    for (int p = 0; p < npass; ++p) {
        const uint32_t v = ghist[p * RS_BINS + threadIdx.x];
        s[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < RS_BINS; o <<= 1) {
            const uint32_t t = threadIdx.x >= o ? s[threadIdx.x - o] : 0;
            __syncthreads();
            s[threadIdx.x] += t;
            __syncthreads();
        }
        ghist[p * RS_BINS + threadIdx.x] = s[threadIdx.x] - v;
        __syncthreads();
    }
}

// ------------------------------------------------------------------ onesweep pass
__global__ void __launch_bounds__(RS_THREADS, 3) k_onesweep(
    const uint32_t *__restrict__ kin, const uint32_t *__restrict__ vin, uint32_t *__restrict__ kout,
    uint32_t *__restrict__ vout, const uint32_t *d_n, int shift, int bits,
    const uint32_t *__restrict__ gbase, uint32_t *status, uint32_t *counter,
    const int32_t *d_overflow) {
    __shared__ uint32_t s_tile;
    __shared__ uint32_t whist[RS_WARPS][RS_BINS];
    __shared__ uint32_t tile_excl[RS_BINS];
    __shared__ uint32_t glob[RS_BINS];
    __shared__ uint32_t skey[RS_TILE];
    __shared__ uint32_t sval[RS_TILE];
    if (d_overflow && *d_overflow) return;
    const uint32_t n = *d_n;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t mask = (1u << bits) - 1;
    const uint32_t lt = lanemask_lt();
    // persistent: the CTA takes tiles in order from the dynamic counter until the
    // keys are exhausted (the element count is only known on the device, so a grid
    // sized for the capacity would otherwise launch waves of empty CTAs)
    while (true) {
    if (tid == 0) s_tile = atomicAdd(counter, 1u);
    for (int i = tid; i < RS_WARPS * RS_BINS; i += RS_THREADS) (&whist[0][0])[i] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint32_t t0 = tile * RS_TILE;
    if (t0 >= n) return;
    const uint32_t wbase = t0 + warp * (32 * RS_ITEMS);
    uint32_t k[RS_ITEMS], v[RS_ITEMS], rk[RS_ITEMS];
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) {
        const uint32_t idx = wbase + j * 32 + lane;
        const bool ok = idx < n;
        k[j] = ok ? kin[idx] : 0xffffffffu;
        v[j] = ok ? vin[idx] : 0u;
    }
    // Stable in-warp ranks: for item j the peers with the same digit come from
    // one match; the leader reserves their slots with one shared atomicAdd
    // (atomics of one warp to one address apply in program order, so item j's
    // reservation precedes item j+1's) and broadcasts the old count.  The 16
    // matches and atomics are independent, so they overlap instead of forming a
    // load/store chain through shared memory.
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) {
        const uint32_t idx = wbase + j * 32 + lane;
        const bool ok = idx < n;
        const uint32_t d = (k[j] >> shift) & mask;
        const uint32_t peers = __match_any_sync(FULL_MASK, ok ? d : 0x10000u);
        const int leader = __ffs(peers) - 1;
        uint32_t old = 0;
        if (ok && lane == leader) old = atomicAdd(&whist[warp][d], (uint32_t)__popc(peers));
        rk[j] = __shfl_sync(FULL_MASK, old, leader) + __popc(peers & lt);
    }
    __syncthreads();
    // per digit: warp-exclusive offsets and tile count
    const uint32_t dg = tid;   // RS_THREADS == RS_BINS
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) {
        const uint32_t c = whist[w][dg];
        whist[w][dg] = cnt;
        cnt += c;
    }
    // decoupled look-back over tiles for this digit: post this tile's count now;
    // the look-back itself runs after the keys are staged in shared memory
    // (their registers are free then for a wide window of predecessor reads)
    uint32_t *st = status + (size_t)tile * RS_BINS + dg;
    st_volatile_u32(st, (tile == 0 ? RS_PRE : RS_AGG) | cnt);
    // tile-local exclusive scan over digits (block scan of cnt)
    {
        uint32_t x = warp_inclusive_scan<uint32_t>(cnt);
        __shared__ uint32_t wsum[RS_WARPS];
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t y = lane < RS_WARPS ? wsum[lane] : 0u;
            y = warp_inclusive_scan<uint32_t>(y);
            if (lane < RS_WARPS) wsum[lane] = y;
        }
        __syncthreads();
        tile_excl[dg] = x - cnt + (warp > 0 ? wsum[warp - 1] : 0u);
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) {
        const uint32_t idx = wbase + j * 32 + lane;
        if (idx < n) {
            const uint32_t d = (k[j] >> shift) & mask;
            const uint32_t pos = tile_excl[d] + whist[warp][d] + rk[j];
            skey[pos] = k[j];
            sval[pos] = v[j];
        }
    }
    {
        // look back RS_LB predecessors per round trip (independent loads), consuming
        // them in order until an inclusive prefix; an unposted one is re-read.  In
        // the first wave every tile starts at once, so tile t walks ~t / RS_LB round
        // trips before it meets an inclusive prefix: the window sets that chain.
        uint32_t excl = 0;
        if (tile > 0) {
            int64_t t = (int64_t)tile - 1;
            bool done = false;
            while (!done) {
                uint32_t sv[RS_LB];
#pragma unroll
                for (int q = 0; q < RS_LB; ++q)
                    sv[q] = t - q >= 0 ? ld_volatile_u32(status + (size_t)(t - q) * RS_BINS + dg) : RS_PRE;
                int q = 0;
#pragma unroll
                for (; q < RS_LB; ++q) {
                    const uint32_t f = sv[q] >> 30;
                    if (f == 0) break;
                    excl += sv[q] & RS_VAL;
                    if (f == 2) { done = true; break; }
                }
                t -= q;
            }
            st_volatile_u32(st, RS_PRE | (excl + cnt));
        }
        glob[dg] = gbase[dg] + excl;
    }
    __syncthreads();
    const uint32_t nt = min((uint32_t)RS_TILE, n - t0);
    for (uint32_t i = tid; i < nt; i += RS_THREADS) {
        const uint32_t key = skey[i];
        const uint32_t d = (key >> shift) & mask;
        const uint32_t dst = glob[d] + (i - tile_excl[d]);
        kout[dst] = key;
        vout[dst] = sval[i];
    }
    __syncthreads();   // shared memory is reused by the next tile
    }
}

// ------------------------------------------------------------------ pair offsets
// Exclusive scan of counts[vid_sorted[i]] over the V visible surfels in depth
// order -> emission offsets; the last CTA checks the pair capacity.
__global__ void __launch_bounds__(SCAN_THREADS) k_pair_offsets(
    const uint32_t *__restrict__ sid, const uint32_t *__restrict__ counts, const ProjHeader *hdr,
    uint32_t *__restrict__ offs, unsigned long long *st, SortMisc *misc, int64_t cap,
    int32_t *d_overflow) {
    __shared__ uint32_t s_tile;
    __shared__ unsigned long long s_w[SCAN_THREADS / 32], s_excl;
    if (threadIdx.x == 0) s_tile = atomicAdd(&misc->scan_counter, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint32_t n = hdr->n_visible;
    if ((int64_t)tile * SCAN_TILE >= (int64_t)n && tile > 0) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t base = (int64_t)tile * SCAN_TILE + (int64_t)(warp * 32 + lane) * SCAN_ITEMS;
    uint32_t c[SCAN_ITEMS];
    unsigned long long l = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        const int64_t idx = base + j;
        c[j] = idx < n ? counts[sid[idx]] : 0u;
        l += c[j];
    }
    const unsigned long long inc = warp_inclusive_scan<unsigned long long>(l);
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const unsigned long long tot = warp_excl_scan_smem(s_w, SCAN_THREADS / 32);
        const unsigned long long e = lookback_warp_u64(st, tile, tot);
        if (lane == 0) {
            s_excl = e;
            if ((int64_t)(tile + 1) * SCAN_TILE >= (int64_t)n) {
                const unsigned long long P = e + tot;
                const bool over = (int64_t)P > cap || P >= (1ull << 30);
                *d_overflow = over ? 1 : 0;
                misc->n_pairs32 = over ? 0u : (uint32_t)P;
            }
        }
    }
    __syncthreads();
    unsigned long long pos = s_excl + s_w[warp] + inc - l;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        const int64_t idx = base + j;
        if (idx < n) offs[idx] = (uint32_t)pos;
        pos += c[j];
    }
}

// ------------------------------------------------------------------ emission
// Load-balanced by pairs: warp task c emits pairs [c*EM_CH, (c+1)*EM_CH) of
// the depth-ordered pair list (coalesced), whatever the surfels' sizes (a
// few near surfels covering thousands of tiles no longer serialise one
// warp).  The task's first surfel is found by a 32-ary warp search of the
// emission offsets; then the warp takes the surfels from there in groups of
// 32: lane q of each round writes one pair, locating its surfel by a binary
// search over the group's offsets (shuffles).  Pairs of a surfel are its
// tiles row-major (tile column modulo ntx: LiDAR azimuth wrap).  The
// per-digit histograms of the tile sort (npass x 8-bit digits) are
// accumulated in shared memory and added to `thist`.
constexpr uint32_t EM_CH = 1024;   // pairs per warp task

__device__ __forceinline__ uint32_t first_surfel(const uint32_t *__restrict__ offs, uint32_t n, uint32_t q0,
                                                 int lane) {
    // largest k < n with offs[k] <= q0 (offs ascending, offs[0] = 0 <= q0)
    uint32_t lo = 0, hi = n;
    while (hi - lo > 32) {
        const uint32_t step = (hi - lo + 31) >> 5;
        const uint32_t idx = lo + (uint32_t)lane * step;
        const bool le = idx < hi && __ldg(offs + idx) <= q0;
        const uint32_t b = __ballot_sync(FULL_MASK, le);
        const uint32_t last = 31 - __clz(b);   // lane 0 probes lo: always set
        lo += last * step;
        hi = min(hi, lo + step);
    }
    const uint32_t idx = lo + (uint32_t)lane;
    const bool le = idx < hi && __ldg(offs + idx) <= q0;
    return lo + 31 - __clz(__ballot_sync(FULL_MASK, le));
}

__global__ void __launch_bounds__(256) k_emit(const uint32_t *__restrict__ sid,
                                              const uint32_t *__restrict__ offs,
                                              const short4 *__restrict__ rect,
                                              const uint64_t *__restrict__ tmask,
                                              const ProjHeader *hdr, const uint32_t *d_np, int ntx, int npass,
                                              int tbits, uint32_t *__restrict__ tkey,
                                              uint32_t *__restrict__ tval, uint32_t *__restrict__ thist,
                                              const int32_t *d_overflow) {
    __shared__ uint32_t h[3][RS_BINS];
    if (*d_overflow) return;
    for (int i = threadIdx.x; i < 3 * RS_BINS; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    const uint32_t n = hdr->n_visible, P = *d_np;
    const int lane = threadIdx.x & 31;
    const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
    const uint32_t ntask = (P + EM_CH - 1) / EM_CH;
    for (uint32_t c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c < ntask; c += nwarps) {
        const uint32_t q0 = c * EM_CH, q1 = min(P, q0 + EM_CH);
        uint32_t k = first_surfel(offs, n, q0, lane);
        while (true) {
            // the group of surfels k .. k+31 and their pair offsets
            const uint32_t kk = k + (uint32_t)lane;
            uint32_t id = 0, o0 = 0xffffffffu;
            int x0 = 0, y0 = 0, wd = 1;
            uint64_t mk = ~0ull;
            if (kk < n) {
                id = sid[kk];
                const short4 r = rect[id];
                x0 = r.x; y0 = r.y;
                wd = r.z - r.x + 1;
                o0 = offs[kk];
                if (tmask) mk = tmask[id];
            }
            const uint32_t gbeg = max(q0, __shfl_sync(FULL_MASK, o0, 0));
            // end of the group's pairs: offset of surfel k+32 (or P), clipped to the task
            const uint32_t onext = k + 32 < n ? __ldg(offs + k + 32) : P;
            const uint32_t gend = min(q1, onext);
            for (uint32_t qb = gbeg; qb < gend; qb += 32) {
                const uint32_t q = qb + (uint32_t)lane;
                // last lane of the group whose first pair is <= q (o0 ascending; unused lanes hold ~0)
                int idx = 0;
#pragma unroll
                for (int step = 16; step; step >>= 1) {
                    const uint32_t l = __shfl_sync(FULL_MASK, o0, idx + step);
                    if (idx + step < 32 && l <= q) idx += step;
                }
                const uint32_t rid = __shfl_sync(FULL_MASK, id, idx);
                const uint32_t rlo = __shfl_sync(FULL_MASK, o0, idx);
                const int rx0 = __shfl_sync(FULL_MASK, x0, idx), ry0 = __shfl_sync(FULL_MASK, y0, idx);
                const int rw = __shfl_sync(FULL_MASK, wd, idx);
                const uint32_t mlo = __shfl_sync(FULL_MASK, (uint32_t)mk, idx);
                const uint32_t mhi = __shfl_sync(FULL_MASK, (uint32_t)(mk >> 32), idx);
                if (q < gend) {
                    uint32_t r = q - rlo;
                    if ((mlo & mhi) != FULL_MASK) {   // tile mask (LiDAR): r-th set bit
                        const uint32_t pl = (uint32_t)__popc(mlo);
                        r = r < pl ? __fns(mlo, 0, (int)r + 1) : 32u + __fns(mhi, 0, (int)(r - pl) + 1);
                    }
                    const int dy = (int)(r / (uint32_t)rw), dx = (int)(r - (uint32_t)dy * (uint32_t)rw);
                    const int tx = rx0 + dx;
                    const uint32_t tile = (uint32_t)((ry0 + dy) * ntx + (tx >= ntx ? tx - ntx : tx));
                    tkey[q] = tile;
                    tval[q] = rid;
                    for (int p = 0; p < npass; ++p) {
                        const int bits = min(8, tbits - 8 * p);
                        atomicAdd(&h[p][(tile >> (8 * p)) & ((1u << bits) - 1)], 1u);
                    }
                }
            }
            if (onext >= q1 || k + 32 >= n) break;
            k += 32;
        }
    }
    __syncthreads();
    for (int p = 0; p < npass; ++p)
        for (int b = threadIdx.x; b < RS_BINS; b += blockDim.x)
            if (h[p][b]) atomicAdd(&thist[p * RS_BINS + b], h[p][b]);
}

// Pinhole emission with exact tile rows (binning.cuh): a surfel's pairs are
// the tiles of its row table (ProjLayout::rows, written by k_project with the
// count), row by row; rects of fewer than KT_MIN_AREA tiles, more than
// PH_ROWS_MAX rows or more than 255 columns take every tile (the same test
// on the same rect as in k_project).  As in k_emit the warp takes the task's
// surfels in groups of 32; each lane first writes its surfel's rows (pairs
// before the row << 8 | first column) to shared memory, then lane q of each
// round writes one pair: its surfel by a binary search over the group's
// offsets (shuffles), its row by a binary search of that surfel's rows.
// Consecutive lanes write consecutive pairs (coalesced).
constexpr int EM_RS = 33;   // row stride of the shared row tables (bank spread)

__global__ void __launch_bounds__(256) k_emit_rows(const uint32_t *__restrict__ sid,
                                                   const uint32_t *__restrict__ offs,
                                                   const short4 *__restrict__ rect,
                                                   const uint4 *__restrict__ rows,
                                                   const ProjHeader *hdr, const uint32_t *d_np, int ntx,
                                                   int npass, int tbits, uint32_t *__restrict__ tkey,
                                                   uint32_t *__restrict__ tval, uint32_t *__restrict__ thist,
                                                   const int32_t *d_overflow) {
    __shared__ uint32_t h[3][RS_BINS];
    __shared__ uint32_t s_row[8][PH_ROWS_MAX * EM_RS];   // [warp][row * EM_RS + lane]
    if (*d_overflow) return;
    for (int i = threadIdx.x; i < 3 * RS_BINS; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    const uint32_t n = hdr->n_visible, P = *d_np;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t *srow = s_row[wid];
    const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
    const uint32_t ntask = (P + EM_CH - 1) / EM_CH;
    for (uint32_t c = blockIdx.x * (blockDim.x >> 5) + wid; c < ntask; c += nwarps) {
        const uint32_t q0 = c * EM_CH, q1 = min(P, q0 + EM_CH);
        uint32_t k = first_surfel(offs, n, q0, lane);
        while (true) {
            const uint32_t kk = k + (uint32_t)lane;
            uint32_t id = 0, o0 = 0xffffffffu;
            int x0 = 0, y0 = 0, wd = 1, nr = 0;   // nr > 0: row-table mode with nr rows
            if (kk < n) {
                id = sid[kk];
                const short4 r = rect[id];
                x0 = r.x; y0 = r.y;
                wd = r.z - r.x + 1;
                o0 = offs[kk];
                const int nrows = r.w - r.y + 1;
                if (wd * nrows >= (int)KT_MIN_AREA && nrows <= PH_ROWS_MAX && wd <= 255) {
                    const uint4 t0 = __ldg(rows + 2 * (size_t)id), t1 = __ldg(rows + 2 * (size_t)id + 1);
                    const uint32_t tb[8] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
                    uint32_t cum = 0;
#pragma unroll
                    for (int rr = 0; rr < PH_ROWS_MAX; ++rr) {
                        const uint32_t e = (tb[rr >> 1] >> (16 * (rr & 1))) & 0xffffu;
                        if (rr < nrows) srow[rr * EM_RS + lane] = (cum << 8) | (e & 0xffu);
                        cum += e >> 8;
                    }
                    nr = nrows;
                }
            }
            __syncwarp();
            const uint32_t gbeg = max(q0, __shfl_sync(FULL_MASK, o0, 0));
            const uint32_t onext = k + 32 < n ? __ldg(offs + k + 32) : P;
            const uint32_t gend = min(q1, onext);
            for (uint32_t qb = gbeg; qb < gend; qb += 32) {
                const uint32_t q = qb + (uint32_t)lane;
                int idx = 0;
#pragma unroll
                for (int step = 16; step; step >>= 1) {
                    const uint32_t l = __shfl_sync(FULL_MASK, o0, idx + step);
                    if (idx + step < 32 && l <= q) idx += step;
                }
                const uint32_t rid = __shfl_sync(FULL_MASK, id, idx);
                const uint32_t rlo = __shfl_sync(FULL_MASK, o0, idx);
                const int rx0 = __shfl_sync(FULL_MASK, x0, idx), ry0 = __shfl_sync(FULL_MASK, y0, idx);
                const int rw = __shfl_sync(FULL_MASK, wd, idx);
                const int rnr = __shfl_sync(FULL_MASK, nr, idx);
                if (q < gend) {
                    const uint32_t r = q - rlo;
                    int ty, tx;
                    if (rnr > 0) {   // last row whose first pair is <= r
                        int rr = 0;
#pragma unroll
                        for (int step = PH_ROWS_MAX / 2; step; step >>= 1)
                            if (rr + step < rnr && (srow[(rr + step) * EM_RS + idx] >> 8) <= r) rr += step;
                        const uint32_t e = srow[rr * EM_RS + idx];
                        ty = ry0 + rr;
                        tx = rx0 + (int)(e & 0xffu) + (int)(r - (e >> 8));
                    } else {
                        const int dy = (int)(r / (uint32_t)rw);
                        ty = ry0 + dy;
                        tx = rx0 + (int)(r - (uint32_t)dy * (uint32_t)rw);
                    }
                    const uint32_t tile = (uint32_t)(ty * ntx + tx);
                    tkey[q] = tile;
                    tval[q] = rid;
                    for (int p = 0; p < npass; ++p) {
                        const int bits = min(8, tbits - 8 * p);
                        atomicAdd(&h[p][(tile >> (8 * p)) & ((1u << bits) - 1)], 1u);
                    }
                }
            }
            __syncwarp();
            if (onext >= q1 || k + 32 >= n) break;
            k += 32;
        }
    }
    __syncthreads();
    for (int p = 0; p < npass; ++p)
        for (int b = threadIdx.x; b < RS_BINS; b += blockDim.x)
            if (h[p][b]) atomicAdd(&thist[p * RS_BINS + b], h[p][b]);
}

// ------------------------------------------------------------------ ranges
// Each thread scans 8 consecutive sorted keys (two 16-byte loads; the
// neighbour on each side comes from the previous / next thread's registers
// or one extra load at the warp edge) and writes the boundaries it sees.
__global__ void __launch_bounds__(256) k_ranges(const uint32_t *__restrict__ tkey, const SortMisc *misc,
                                                uint32_t *__restrict__ ranges,
                                                const int32_t *d_overflow) {
    if (*d_overflow) return;
    const uint32_t P = misc->n_pairs32;
    const uint32_t i0 = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
    if (i0 >= P) return;
    uint32_t k[8];
    if (i0 + 8 <= P) {
        const uint4 a = __ldg(reinterpret_cast<const uint4 *>(tkey + i0));
        const uint4 b = __ldg(reinterpret_cast<const uint4 *>(tkey + i0) + 1);
        k[0] = a.x; k[1] = a.y; k[2] = a.z; k[3] = a.w; k[4] = b.x; k[5] = b.y; k[6] = b.z; k[7] = b.w;
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) k[j] = i0 + j < P ? tkey[i0 + j] : 0xffffffffu;
    }
    uint32_t prev = i0 > 0 ? __ldg(tkey + i0 - 1) : 0xffffffffu;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t i = i0 + j;
        if (i >= P) break;
        if (k[j] != prev) {
            ranges[2 * k[j]] = i;
            if (i > 0) ranges[2 * prev + 1] = i;
        }
        prev = k[j];
    }
    const uint32_t last = min(i0 + 8, P);
    if (last == P) ranges[2 * prev + 1] = P;
}

__global__ void __launch_bounds__(256) k_keys64(const uint32_t *__restrict__ tkey,
                                                const uint32_t *__restrict__ tval,
                                                const uint32_t *__restrict__ dkey, const SortMisc *misc,
                                                unsigned long long *__restrict__ keys,
                                                const int32_t *d_overflow) {
    if (*d_overflow) return;
    const uint32_t P = misc->n_pairs32;
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P) return;
    keys[i] = ((unsigned long long)tkey[i] << 32) | dkey[tval[i]];
}

// ------------------------------------------------------------------ host
size_t sort_workspace_bytes(int64_t n, int64_t cap, int64_t ntiles) {
    return sort_layout(n, cap, ntiles).total;
}

cudaError_t launch_bin_sort(const void *proj, int64_t n, const DevSensor &se, int64_t ntiles,
                            uint64_t *keys, uint32_t *values, int64_t cap, uint32_t *ranges,
                            void *ws, int32_t *d_overflow, cudaStream_t st) {
    const int kind = se.kind, ntx = se.ntx;
    const ProjLayout L(n, kind);
    const SortWs W = sort_layout(n, cap, ntiles);
    const char *pb = (const char *)proj;
    char *wb = (char *)ws;
    const ProjHeader *hdr = (const ProjHeader *)pb;
    SortMisc *misc = (SortMisc *)(wb + W.misc);
    uint32_t *hist = (uint32_t *)(wb + W.hist);
    cudaError_t e;
#define CK(x) do { e = (x); if (e != cudaSuccess) return e; } while (0)
    CK(cudaMemsetAsync(d_overflow, 0, 4, st));
    CK(cudaMemsetAsync(wb + W.misc, 0, W.hist + 8 * RS_BINS * 4 - W.misc, st));
    CK(cudaMemsetAsync(ranges, 0, (size_t)ntiles * 2 * 4, st));
    CK(cudaMemsetAsync(wb + W.cstat, 0, (W.nblk_c + 1) * 8, st));
    CK(cudaMemsetAsync(wb + W.dstat, 0, W.total - W.dstat, st));
    if (n == 0 || cap == 0) {
        // nothing visible can be binned; flag overflow if pairs exist
        if (n > 0) {
            // P > 0 with cap == 0 -> overflow is reported by the offsets kernel
        } else {
            return cudaSuccess;
        }
    }
    const uint32_t *d_nvis = &hdr->n_visible;
    // 1. depth sort of the visible surfels (4 x 8-bit digits)
    const unsigned hgrid_d = (unsigned)std::min<int64_t>((n + 4095) / 4096, 4 * 148);
    note_launch();
    k_hist<<<hgrid_d > 0 ? hgrid_d : 1, 256, 0, st>>>((const uint32_t *)(pb + L.vkey), d_nvis, 4, 32,
                                                      hist, nullptr);
    CK(cudaGetLastError());
    const uint32_t *ki = (const uint32_t *)(pb + L.vkey), *vi = (const uint32_t *)(pb + L.vid);
    uint32_t *bufk[2] = {(uint32_t *)(wb + W.dA_k), (uint32_t *)(wb + W.dB_k)};
    uint32_t *bufv[2] = {(uint32_t *)(wb + W.dA_v), (uint32_t *)(wb + W.dB_v)};
    // the depth histogram scan and the tile histogram share `hist` rows 0..3 / 4..6
    note_launch();
    k_hist_scan<<<1, RS_BINS, 0, st>>>(hist, 4, nullptr);
    CK(cudaGetLastError());
    int dev = 0, nsm = 148, per_os = 3;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_os, k_onesweep, RS_THREADS, 0);
    const int64_t resident = (int64_t)nsm * std::max(per_os, 1);   // persistent onesweep CTAs
    const unsigned grid_d = (unsigned)std::max<int64_t>(1, std::min<int64_t>((int64_t)W.ntile_d, resident));
    for (int p = 0; p < 4; ++p) {
        note_launch();
        k_onesweep<<<grid_d, RS_THREADS, 0, st>>>(ki, vi, bufk[p & 1], bufv[p & 1], d_nvis, 8 * p, 8,
                                                  hist + p * RS_BINS,
                                                  (uint32_t *)(wb + W.dstat) + (size_t)p * W.ntile_d * RS_BINS,
                                                  &misc->counter[p], nullptr);
        CK(cudaGetLastError());
        ki = bufk[p & 1];
        vi = bufv[p & 1];
    }
    // sorted ids now in bufv[1] (after 4 passes), keys in bufk[1]
    const uint32_t *sid = vi;
    uint32_t *offs = (uint32_t *)(wb + W.offs);
    const unsigned gridc = (unsigned)(W.nblk_c > 0 ? W.nblk_c : 1);
    note_launch();
    k_pair_offsets<<<gridc, SCAN_THREADS, 0, st>>>(sid, (const uint32_t *)(pb + L.cnt), hdr, offs,
                                                   (unsigned long long *)(wb + W.cstat), misc, cap,
                                                   d_overflow);
    CK(cudaGetLastError());
    // 2. emission into the buffer that the tile passes end in `values`
    const int np = W.npass_t;
    uint32_t *tk[2] = {(uint32_t *)(wb + W.tk0), (uint32_t *)(wb + W.tk1)};
    uint32_t *tv[2] = {values, (uint32_t *)(wb + W.tv1)};
    int cur = np & 1;
    note_launch();
    // emission fused with the tile-digit histograms
    const int tb = tile_bits_for(ntiles);
    const uint32_t *d_np = &misc->n_pairs32;
    uint32_t *thist = hist + 4 * RS_BINS;
    // P is only known on the device: enough warps for the capacity's tasks, at most 8 CTAs per SM
    const int64_t tasks = (cap + EM_CH - 1) / EM_CH;
    const unsigned ge = (unsigned)std::max<int64_t>(1, std::min<int64_t>((tasks + 7) / 8, (int64_t)nsm * 8));
    if (kind == GS_PINHOLE) {
        k_emit_rows<<<ge, 256, 0, st>>>(sid, offs, (const short4 *)(pb + L.rect), (const uint4 *)(pb + L.rows), hdr,
                                        d_np, ntx, np, tb, tk[cur], tv[cur], thist, d_overflow);
    } else {
        k_emit<<<ge, 256, 0, st>>>(sid, offs, (const short4 *)(pb + L.rect),
                                   kind == GS_LIDAR_SPINNING ? (const uint64_t *)(pb + L.tmask) : nullptr, hdr, d_np,
                                   ntx, np, tb, tk[cur], tv[cur], thist, d_overflow);
    }
    CK(cudaGetLastError());
    // 3. tile digits over the pairs
    note_launch();
    k_hist_scan<<<1, RS_BINS, 0, st>>>(thist, np, d_overflow);
    CK(cudaGetLastError());
    const unsigned grid_t = (unsigned)std::max<int64_t>(1, std::min<int64_t>((int64_t)W.ntile_t, resident));
    for (int p = 0; p < np; ++p) {
        const int bits = min(8, tb - 8 * p);
        note_launch();
        k_onesweep<<<grid_t, RS_THREADS, 0, st>>>(tk[cur], tv[cur], tk[cur ^ 1], tv[cur ^ 1], d_np, 8 * p,
                                                  bits, thist + p * RS_BINS,
                                                  (uint32_t *)(wb + W.tstat) + (size_t)p * W.ntile_t * RS_BINS,
                                                  &misc->counter[4 + p], d_overflow);
        CK(cudaGetLastError());
        cur ^= 1;
    }
    // cur == 0 now: sorted tile keys in tk[0], values in `values`
    const unsigned gp = (unsigned)((cap + 255) / 256);
    note_launch();
    const unsigned gr = (unsigned)((cap + 2047) / 2048);
    k_ranges<<<gr > 0 ? gr : 1, 256, 0, st>>>(tk[cur], misc, ranges, d_overflow);
    CK(cudaGetLastError());
    if (keys) {
        note_launch();
        k_keys64<<<gp > 0 ? gp : 1, 256, 0, st>>>(tk[cur], values, (const uint32_t *)(pb + L.key), misc,
                                                  (unsigned long long *)keys, d_overflow);
        CK(cudaGetLastError());
    }
#undef CK
    return cudaSuccess;
}

}  // namespace gsr
