// route.cu -- pixel-partitioned single-frame rendering over several GPUs
// (SURVEY.md §8(f) NEXT-4): which surfels each image band needs, and the
// packing of the surfel data sent to it (§III-A "Paralleled
// training": continuous image regions per GPU, "a sparse all-to-all
// communication scheme to transfer the required Gaussian data to
// corresponding pixel partitions").
//
// gs_band_route: after gs_project of this rank's surfel shard, list for
// every band (a range of tile rows) the visible surfels whose tile rect
// overlaps it, in ascending surfel index (three deterministic passes: per
// block band counts, an exclusive scan over blocks, the stable write).
// gs_pack_surfels / gs_unpack_surfels: gather the listed surfels' raw
// attributes into one AoS float record each (the all-to-all payload) and
// scatter a received payload back into a gs_surfels set.  HBM-bound copies.
#include <stdint.h>

#include <algorithm>

#include "gsr_internal.cuh"

namespace gsr {

namespace route {
constexpr int THREADS = 256, ITEMS = 4, TILE = THREADS * ITEMS;
constexpr int MAX_BANDS = 64;

struct Bands {
    int32_t nb;
    int32_t row0[MAX_BANDS + 1];   // tile-row boundaries, row0[0] = 0 ... row0[nb] = tile rows
};

__device__ __forceinline__ void band_span(const Bands &B, int y0, int y1, int &b0, int &b1) {
    b0 = 0;
    while (b0 + 1 < B.nb && B.row0[b0 + 1] <= y0) ++b0;
    b1 = b0;
    while (b1 + 1 < B.nb && B.row0[b1 + 1] <= y1) ++b1;
}

// pass 1: per block, how many surfels each band receives
__global__ void __launch_bounds__(THREADS) k_route_count(const short4 *__restrict__ rect, const uint32_t *__restrict__ cnt,
                                                         int64_t n, const __grid_constant__ Bands B,
                                                         uint32_t *__restrict__ blk) {
    __shared__ uint32_t s[MAX_BANDS];
    for (int b = threadIdx.x; b < B.nb; b += THREADS) s[b] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * TILE;
    for (int k = 0; k < ITEMS; ++k) {
        const int64_t i = base + k * THREADS + threadIdx.x;
        if (i < n && cnt[i] > 0) {
            const short4 r = rect[i];
            int b0, b1;
            band_span(B, r.y, r.w, b0, b1);
            for (int b = b0; b <= b1; ++b) atomicAdd(&s[b], 1u);
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < B.nb; b += THREADS) blk[(size_t)blockIdx.x * B.nb + b] = s[b];
}

// pass 2: exclusive scan over blocks, per band (one CTA; a warp per band)
__global__ void k_route_scan(uint32_t *__restrict__ blk, uint32_t nblk, int32_t nb, uint32_t *__restrict__ total) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int b = warp; b < nb; b += blockDim.x >> 5) {
        uint32_t run = 0;
        for (uint32_t c0 = 0; c0 < nblk; c0 += 32) {
            const uint32_t c = c0 + lane;
            const uint32_t v = c < nblk ? blk[(size_t)c * nb + b] : 0u;
            uint32_t x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (c < nblk) blk[(size_t)c * nb + b] = run + x - v;
            run += __shfl_sync(0xffffffffu, x, 31);
        }
        if (lane == 0) total[b] = run;
    }
}

// pass 3: stable write of the surfel indices, band by band, in index order
__global__ void __launch_bounds__(THREADS) k_route_write(const short4 *__restrict__ rect, const uint32_t *__restrict__ cnt,
                                                         int64_t n, const __grid_constant__ Bands B,
                                                         const uint32_t *__restrict__ blk, uint32_t *__restrict__ index,
                                                         int64_t stride) {
    __shared__ uint32_t s_off[MAX_BANDS];
    __shared__ uint32_t s_warp[THREADS / 32][MAX_BANDS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int b = threadIdx.x; b < B.nb; b += THREADS) s_off[b] = blk[(size_t)blockIdx.x * B.nb + b];
    const int64_t base = (int64_t)blockIdx.x * TILE;
    const uint32_t below = (1u << lane) - 1u;
    for (int k = 0; k < ITEMS; ++k) {
        // items of round k: base + k*THREADS + t, ranked in t order within the round
        const int64_t i = base + k * THREADS + threadIdx.x;
        int b0 = 1, b1 = 0;
        if (i < n && cnt[i] > 0) {
            const short4 r = rect[i];
            band_span(B, r.y, r.w, b0, b1);
        }
        for (int b = 0; b < B.nb; ++b) {   // per-warp counts of this round
            const uint32_t m = __ballot_sync(0xffffffffu, b >= b0 && b <= b1);
            if (lane == 0) s_warp[warp][b] = __popc(m);
        }
        __syncthreads();
        for (int b = 0; b < B.nb; ++b) {
            const bool in = b >= b0 && b <= b1;
            const uint32_t m = __ballot_sync(0xffffffffu, in);
            if (in) {
                uint32_t before = s_off[b];
                for (int w = 0; w < warp; ++w) before += s_warp[w][b];
                index[(size_t)b * stride + before + __popc(m & below)] = (uint32_t)i;
            }
        }
        __syncthreads();
        for (int b = threadIdx.x; b < B.nb; b += THREADS) {
            uint32_t add = 0;
            for (int w = 0; w < THREADS / 32; ++w) add += s_warp[w][b];
            s_off[b] += add;
        }
        __syncthreads();
    }
}

// AoS payload record of one surfel: mean 3, quat 4, scale 2, opacity 1,
// SH (d+1)^2*3 (if present), intensity, ray-drop logit (if present)
struct Layout {
    int nsh, has_int, has_drop, F;
};

__host__ __device__ inline Layout layout_of(int sh_floats, int has_int, int has_drop) {
    Layout L;
    L.nsh = sh_floats;
    L.has_int = has_int;
    L.has_drop = has_drop;
    L.F = 10 + sh_floats + has_int + has_drop;
    return L;
}

__global__ void k_pack(DevSurfels s, Layout L, const uint32_t *__restrict__ index, int64_t m,
                       float *__restrict__ out) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = index[j];
        float *o = out + (size_t)j * L.F;
        for (int k = 0; k < 3; ++k) o[k] = s.means[3 * i + k];
        for (int k = 0; k < 4; ++k) o[3 + k] = s.quats[4 * i + k];
        o[7] = s.scales[2 * i];
        o[8] = s.scales[2 * i + 1];
        o[9] = s.opac[i];
        for (int k = 0; k < L.nsh; ++k) o[10 + k] = s.sh[(size_t)i * L.nsh + k];
        int q = 10 + L.nsh;
        if (L.has_int) o[q++] = s.inten[i];
        if (L.has_drop) o[q] = s.drop[i];
    }
}

__global__ void k_unpack(const float *__restrict__ in, Layout L, int64_t m, float *means, float *quats,
                         float *scales, float *opac, float *sh, float *inten, float *drop) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
        const float *o = in + (size_t)j * L.F;
        for (int k = 0; k < 3; ++k) means[3 * j + k] = o[k];
        for (int k = 0; k < 4; ++k) quats[4 * j + k] = o[3 + k];
        scales[2 * j] = o[7];
        scales[2 * j + 1] = o[8];
        opac[j] = o[9];
        for (int k = 0; k < L.nsh; ++k) sh[(size_t)j * L.nsh + k] = o[10 + k];
        int q = 10 + L.nsh;
        if (L.has_int) inten[j] = o[q++];
        if (L.has_drop) drop[j] = o[q];
    }
}
}  // namespace route

size_t band_route_workspace_bytes(int64_t n, int32_t nb) {
    const int64_t nblk = (std::max<int64_t>(n, 1) + route::TILE - 1) / route::TILE;
    return (size_t)nblk * nb * 4 + 256;
}

cudaError_t launch_band_route(const void *proj, int64_t n, int kind, const int32_t *band_rows, int32_t nb,
                              uint32_t *d_counts, uint32_t *d_index, void *ws, cudaStream_t st) {
    using namespace route;
    Bands B;
    memset(&B, 0, sizeof(B));
    B.nb = nb;
    for (int b = 0; b <= nb; ++b) B.row0[b] = band_rows[b];
    const ProjLayout PL(n, kind);
    const short4 *rect = (const short4 *)((const char *)proj + PL.rect);
    const uint32_t *cnt = (const uint32_t *)((const char *)proj + PL.cnt);
    const unsigned nblk = (unsigned)((std::max<int64_t>(n, 1) + TILE - 1) / TILE);
    uint32_t *blk = (uint32_t *)ws;
    note_launch(3);
    k_route_count<<<nblk, THREADS, 0, st>>>(rect, cnt, n, B, blk);
    k_route_scan<<<1, 32 * std::min(nb, 32), 0, st>>>(blk, nblk, nb, d_counts);
    k_route_write<<<nblk, THREADS, 0, st>>>(rect, cnt, n, B, blk, d_index, n);
    return cudaGetLastError();
}

int32_t payload_floats(int sh_floats, int has_int, int has_drop) {
    return route::layout_of(sh_floats, has_int, has_drop).F;
}

cudaError_t launch_pack(const DevSurfels &s, int sh_floats, const uint32_t *index, int64_t m, float *out,
                        cudaStream_t st) {
    if (m == 0) return cudaSuccess;
    const route::Layout L = route::layout_of(sh_floats, s.inten != nullptr, s.drop != nullptr);
    const unsigned grid = (unsigned)std::min<int64_t>((m + 255) / 256, 148 * 16);
    note_launch();
    route::k_pack<<<grid, 256, 0, st>>>(s, L, index, m, out);
    return cudaGetLastError();
}

cudaError_t launch_unpack(const float *in, int64_t m, int sh_floats, int has_int, int has_drop, float *means,
                          float *quats, float *scales, float *opac, float *sh, float *inten, float *drop,
                          cudaStream_t st) {
    if (m == 0) return cudaSuccess;
    const route::Layout L = route::layout_of(sh_floats, has_int, has_drop);
    const unsigned grid = (unsigned)std::min<int64_t>((m + 255) / 256, 148 * 16);
    note_launch();
    route::k_unpack<<<grid, 256, 0, st>>>(in, L, m, means, quats, scales, opac, sh, inten, drop);
    return cudaGetLastError();
}

}  // namespace gsr
