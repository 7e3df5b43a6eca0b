// decode.cu -- neural-Gaussian decode on the 5th-gen
// tensor cores: anchors -> per-head MLPs -> 2DGS surfel attributes, written
// in the gs_surfels layout that gs_project reads.
//
// PAPER.md:78 (§III-A "Scene Reconstruction"): the final 2DGS attributes
// {mu, R, S, rho, r, alpha} of each neural Gaussian are inferred by passing
// the anchor features through the corresponding MLP (Scaffold-GS anchors,
// P:49).  Sizes and heads are DESIGN.md §12 readings N1-N6: k = 5 surfels
// per anchor, F = 32 features, per head two hidden layers of 32 (ReLU);
// geometry heads (offset, scale, rotation) read the feature, appearance heads
// (opacity, colour | intensity, ray-drop) read [feature, view direction].
//
// One CTA = 128 anchors per tile (the M = 128 of a cta_group::1 tcgen05.mma),
// persistent over tiles, 8 warps (two per TMEM lane quarter: they split the
// columns of every drain and the epilogue), 2 CTAs per SM; a tile's anchor
// inputs are loaded one tile ahead and its outputs leave through shared
// memory as coalesced 16-byte stores.  The three layers are three
// chained GEMM groups with fp16 operands in shared memory (canonical K-major
// no-swizzle UMMA layout) and fp32 accumulators in tensor memory:
//   L1  [128 x 48] x [48 x 32H]      all heads at once (H = 5 camera, 6 LiDAR;
//                                     K = 32 features + 3 view + zero pad)
//   L2  [128 x 32] x [32 x 32]       per head (its 32 columns of the L1 output)
//   L3  [128 x 32] x [32 x out_h]    per head, out_h padded to 16
// Between layers every thread drains its anchor's row from TMEM (tcgen05.ld
// 32x32b), adds the bias, applies ReLU, rounds to fp16 and stores the row
// as the next layer's A operand.  The final epilogue turns the 80-ish outputs
// of its anchor into 5 surfels: centre, quaternion of the Gram-Schmidt frame,
// scales, opacity, and the degree-0 SH colour (camera) or intensity and
// ray-drop logit (LiDAR).  One elected thread issues the MMAs and commits
// them to an mbarrier the CTA waits on.
//
// Roofline: HBM: 88 B read + 260 B (camera) / 220 B (LiDAR)
// written per anchor against ~32 kFLOP of fp16 MMA per anchor -- an
// arithmetic intensity (~90 FLOP/B) below the tensor ridge (~250 FLOP/B).
#include <cuda_fp16.h>
#include <math.h>

#include <algorithm>
#include <stdint.h>

#include "gsr_internal.cuh"

namespace gsr {

namespace dec {

constexpr int M = 128;                   // anchors per tile
constexpr int NT = 2 * M;                // threads: two warps per TMEM lane quarter (columns split)
constexpr int KS = GS_NEURAL_K;          // surfels per anchor
constexpr int FEAT = GS_NEURAL_F;        // 32
constexpr int HID = GS_NEURAL_HIDDEN;    // 32
constexpr int K1 = 48;                   // L1 reduction: 32 features + 3 view + 13 zero
constexpr int MAXH = 6;
// per head h: real output width, width padded to 16, first TMEM/W3 column
__host__ __device__ constexpr int out_real(int lidar, int h) {
    return h == 0 ? 15 : h == 1 ? 10 : h == 2 ? 30 : h == 3 ? 5 : h == 4 ? (lidar ? 5 : 15) : (lidar ? 5 : 0);
}
__host__ __device__ constexpr int out_pad(int lidar, int h) { return h == 2 ? 32 : (h == 5 && !lidar) ? 0 : 16; }
__host__ __device__ constexpr int out_col(int h) { return h == 0 ? 0 : h == 1 ? 16 : h == 2 ? 32 : 64 + 16 * (h - 3); }
constexpr int NOUT_PAD_MAX = 112;
constexpr int TMEM_COLS = 256;

// shared memory carve-up (bytes)
constexpr int SZ_W1 = MAXH * HID * K1 * 2;        // [32H rows][48]
constexpr int SZ_W2 = MAXH * HID * HID * 2;       // per head [32][32]
constexpr int SZ_W3 = NOUT_PAD_MAX * HID * 2;     // [out rows][32]
constexpr int SZ_A0 = M * K1 * 2;
constexpr int SZ_A1 = M * MAXH * HID * 2;
static_assert(13 * KS * M * 4 <= SZ_A1, "epilogue staging fits in A1");
constexpr int OFF_W1 = 0;
constexpr int OFF_W2 = OFF_W1 + SZ_W1;
constexpr int OFF_W3 = OFF_W2 + SZ_W2;
constexpr int OFF_A0 = OFF_W3 + SZ_W3;
constexpr int OFF_A1 = OFF_A0 + SZ_A0;
constexpr int OFF_B1 = OFF_A1 + SZ_A1;             // fp32 biases
constexpr int OFF_B2 = OFF_B1 + MAXH * HID * 4;
constexpr int OFF_B3 = OFF_B2 + MAXH * HID * 4;
constexpr int OFF_BAR = OFF_B3 + NOUT_PAD_MAX * 4;
constexpr int SMEM = OFF_BAR + 16;

struct Params {
    int64_t n;
    const float *pos, *base;
    const __half *feat;
    const __half *w1[MAXH], *w2[MAXH], *w3[MAXH];
    const float *b1[MAXH], *b2[MAXH], *b3[MAXH];
    float ox, oy, oz;
    int lidar;
    float *means, *quats, *scales, *opac, *sh, *inten, *drop;
};

// byte offset of element (row, k) in a canonical K-major no-swizzle operand
// with `kc` 8-element K chunks per row: 8x16-byte core matrices, K-adjacent
// core matrices 128 B apart (LBO), 8-row groups kc*128 B apart (SBO)
__device__ __forceinline__ uint32_t cano(int row, int k, int kc) {
    return (uint32_t)((row >> 3) * (kc * 128) + (k >> 3) * 128 + (row & 7) * 16 + (k & 7) * 2);
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// tcgen05 shared-memory matrix descriptor: start >> 4, LBO = 128 B, SBO,
// version 1 (sm_100), no swizzle
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t sbo_bytes) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) |
           ((uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

// instruction descriptor, kind::f16: A = B = fp16, D = fp32, both K-major, M = 128
__host__ __device__ constexpr uint32_t idesc(int n) {
    return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(id), "r"(acc));
}

__device__ __forceinline__ void commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void bar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void bar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
        "r"(parity) : "memory");
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// 32 consecutive TMEM columns of this thread's lane (32x32b shape, one lane per thread)
__device__ __forceinline__ void tld32(uint32_t taddr, float *v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tld16(uint32_t taddr, float *v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"
        " [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// (a0 + b0, a1 + b1) in one packed f32x2 add (sm_100), then ReLU and the
// rounding to fp16 in one cvt: the same values as fmaxf(a + b, 0) -> fp16
__device__ __forceinline__ uint32_t bias_relu_h2(float a0, float a1, float b0, float b1) {
    uint32_t h;
    asm("{\n\t.reg .b64 a, b, s;\n\t.reg .f32 lo, hi;\n\t"
        "mov.b64 a, {%1, %2};\n\tmov.b64 b, {%3, %4};\n\t"
        "add.rn.f32x2 s, a, b;\n\tmov.b64 {lo, hi}, s;\n\t"
        "cvt.rn.relu.f16x2.f32 %0, hi, lo;\n\t}"
        : "=r"(h) : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
    return h;
}

// bias + ReLU + fp16 of 32 accumulator columns -> 4 K-chunks of row `row` of A
__device__ __forceinline__ void relu_store(const float *v, const float *bias, char *A, int row, int k0, int kc) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const float4 b0 = *reinterpret_cast<const float4 *>(bias + 8 * c);
        const float4 b1 = *reinterpret_cast<const float4 *>(bias + 8 * c + 4);
        const float *x = v + 8 * c;
        *reinterpret_cast<uint4 *>(A + cano(row, k0 + 8 * c, kc)) =
            make_uint4(bias_relu_h2(x[0], x[1], b0.x, b0.y), bias_relu_h2(x[2], x[3], b0.z, b0.w),
                       bias_relu_h2(x[4], x[5], b1.x, b1.y), bias_relu_h2(x[6], x[7], b1.z, b1.w));
    }
}

// Gram-Schmidt frame of surfel j's 6D rotation output (a1, a2) and its
// quaternion (w >= 0) by Shepperd's method on the largest of 1+tr, 1+2R_ii-tr
__device__ __forceinline__ void write_quat(const float *R, const float *B3, int j, float *q) {
    float a1x = R[6 * j] + B3[32 + 6 * j], a1y = R[6 * j + 1] + B3[32 + 6 * j + 1], a1z = R[6 * j + 2] + B3[32 + 6 * j + 2];
    float a2x = R[6 * j + 3] + B3[32 + 6 * j + 3], a2y = R[6 * j + 4] + B3[32 + 6 * j + 4],
          a2z = R[6 * j + 5] + B3[32 + 6 * j + 5];
    const float i1 = rsqrtf(a1x * a1x + a1y * a1y + a1z * a1z);
    const float ux = a1x * i1, uy = a1y * i1, uz = a1z * i1;
    const float dp = ux * a2x + uy * a2y + uz * a2z;
    a2x -= dp * ux; a2y -= dp * uy; a2z -= dp * uz;
    const float i2 = rsqrtf(a2x * a2x + a2y * a2y + a2z * a2z);
    const float vx = a2x * i2, vy = a2y * i2, vz = a2z * i2;
    const float nx = uy * vz - uz * vy, ny = uz * vx - ux * vz, nz = ux * vy - uy * vx;
    const float tr = ux + vy + nz;
    float qw, qx, qy, qz;
    if (tr >= fmaxf(ux, fmaxf(vy, nz))) {
        const float h = sqrtf(fmaxf(1.f + tr, 0.f)), ir = __fdividef(0.5f, h);   // r4 = 2h
        qw = 0.5f * h; qx = (vz - ny) * ir; qy = (nx - uz) * ir; qz = (uy - vx) * ir;
    } else if (ux >= vy && ux >= nz) {
        const float h = sqrtf(fmaxf(1.f + ux - vy - nz, 0.f)), ir = __fdividef(0.5f, h);
        qw = (vz - ny) * ir; qx = 0.5f * h; qy = (vx + uy) * ir; qz = (nx + uz) * ir;
    } else if (vy >= nz) {
        const float h = sqrtf(fmaxf(1.f - ux + vy - nz, 0.f)), ir = __fdividef(0.5f, h);
        qw = (nx - uz) * ir; qx = (vx + uy) * ir; qy = 0.5f * h; qz = (ny + vz) * ir;
    } else {
        const float h = sqrtf(fmaxf(1.f - ux - vy + nz, 0.f)), ir = __fdividef(0.5f, h);
        qw = (uy - vx) * ir; qx = (nx + uz) * ir; qy = (ny + vz) * ir; qz = 0.5f * h;
    }
    if (qw < 0.f) { qw = -qw; qx = -qx; qy = -qy; qz = -qz; }
    *reinterpret_cast<float4 *>(q) = make_float4(qw, qx, qy, qz);
}

// staged tile outputs -> global, 16-byte stores (dst 16-byte aligned: every
// array's tile slice starts at a multiple of 4 floats)
__device__ __forceinline__ void copy_out(const float *src, float *dst, int nfl, int t) {
    const int n4 = nfl >> 2;
    for (int i = t; i < n4; i += NT)
        reinterpret_cast<float4 *>(dst)[i] = reinterpret_cast<const float4 *>(src)[i];
    for (int i = 4 * n4 + t; i < nfl; i += NT) dst[i] = src[i];
}

__device__ __forceinline__ float sigm(float z) { return __fdividef(1.f, 1.f + __expf(-z)); }

template <int LIDAR>
__global__ void __launch_bounds__(NT, 2) k_decode(const __grid_constant__ Params p) {
    constexpr int H = LIDAR ? 6 : 5;
    constexpr int N1 = H * HID;
    constexpr int KC1 = K1 / 8, KC2 = N1 / 8;
    extern __shared__ __align__(1024) char sm[];
    __shared__ uint32_t s_tmem;
    const int t = threadIdx.x, warp = t >> 5;
    const int row = t & (M - 1);   // anchor row of the tile = TMEM lane
    const int grp = t >> 7;        // 0: warps 0-3, 1: warps 4-7 (same lane quarters, other columns)
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + OFF_BAR);
    char *W1 = sm + OFF_W1, *W2 = sm + OFF_W2, *W3 = sm + OFF_W3, *A0 = sm + OFF_A0, *A1 = sm + OFF_A1;
    float *B1 = reinterpret_cast<float *>(sm + OFF_B1), *B2 = reinterpret_cast<float *>(sm + OFF_B2),
          *B3 = reinterpret_cast<float *>(sm + OFF_B3);

    // ---- one-time: tensor memory, mbarrier, weights in the canonical layouts
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&s_tmem)),
                     "n"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (t == 0) {
        bar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    for (int e = t; e < N1 * K1; e += NT) {   // L1: row r = 32h + i, K = [feature | view | 0]
        const int r = e / K1, k = e % K1, h = r / HID, i = r % HID;
        const int nin = h < 3 ? FEAT : FEAT + 3;
        const __half w = k < nin ? p.w1[h][i * nin + k] : __float2half(0.f);
        *reinterpret_cast<__half *>(W1 + cano(r, k, KC1)) = w;
    }
    for (int e = t; e < H * HID * HID; e += NT) {   // L2: per head [32][32]
        const int h = e / (HID * HID), r = (e / HID) % HID, k = e % HID;
        *reinterpret_cast<__half *>(W2 + h * HID * HID * 2 + cano(r, k, HID / 8)) = p.w2[h][r * HID + k];
    }
    for (int e = t; e < NOUT_PAD_MAX * HID; e += NT) {   // L3: rows OUT_COL[h] + i, zero-padded
        const int r = e / HID, k = e % HID;
        __half w = __float2half(0.f);
        float b = 0.f;
#pragma unroll
        for (int h = 0; h < H; ++h) {
            const int i = r - out_col(h);
            if (i >= 0 && i < out_real(LIDAR, h)) {
                w = p.w3[h][i * HID + k];
                b = p.b3[h][i];
            }
        }
        *reinterpret_cast<__half *>(W3 + cano(r, k, HID / 8)) = w;
        if (k == 0) B3[r] = b;
    }
    for (int e = t; e < N1; e += NT) {
        B1[e] = p.b1[e / HID][e % HID];
        B2[e] = p.b2[e / HID][e % HID];
    }
    fence_async_smem();
    tc_before();
    __syncthreads();
    tc_after();
    const uint32_t tmem = s_tmem;
    const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16);   // this warp's lane quarter
    uint32_t phase = 0;

    const int64_t ntiles = (p.n + M - 1) / M;
    // the anchor inputs of a tile are loaded one tile ahead (they arrive while the
    // previous tile's MMAs, drains and epilogue run): group 0 the position and base
    // scale, group 1 the feature
    float nx_ = 0.f, ny_ = 0.f, nz_ = 0.f, nl0 = 0.f, nl1 = 0.f, nl2 = 0.f;
    uint4 nf[4] = {};
    auto prefetch = [&](int64_t tl) {
        const int64_t an = tl * M + row;
        if (tl >= ntiles || an >= p.n) return;
        if (grp == 0) {
            nx_ = __ldg(p.pos + 3 * an); ny_ = __ldg(p.pos + 3 * an + 1); nz_ = __ldg(p.pos + 3 * an + 2);
            nl0 = __ldg(p.base + 3 * an); nl1 = __ldg(p.base + 3 * an + 1); nl2 = __ldg(p.base + 3 * an + 2);
        } else {
            const uint4 *fp = reinterpret_cast<const uint4 *>(p.feat) + 4 * an;
#pragma unroll
            for (int c = 0; c < 4; ++c) nf[c] = __ldg(fp + c);
        }
    };
    prefetch(blockIdx.x);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t a = tile * M + row;
        const bool live = a < p.n;
        // ---- anchor row -> A0 (features, fp16 view direction, zero pad): group 0 the
        // view direction, group 1 the feature chunks
        const float x = live ? nx_ : 0.f, y = live ? ny_ : 0.f, z = live ? nz_ : 0.f;
        const float l0 = nl0, l1 = nl1, l2 = nl2;
        if (grp == 0) {
            const float vx = x - p.ox, vy = y - p.oy, vz = z - p.oz;
            const float inv = live ? rsqrtf(vx * vx + vy * vy + vz * vz) : 0.f;
            const __half2 d01 = __floats2half2_rn(vx * inv, vy * inv);
            const __half2 d2z = __floats2half2_rn(vz * inv, 0.f);
            *reinterpret_cast<uint4 *>(A0 + cano(row, 32, KC1)) =
                make_uint4(*reinterpret_cast<const uint32_t *>(&d01), *reinterpret_cast<const uint32_t *>(&d2z), 0u, 0u);
            *reinterpret_cast<uint4 *>(A0 + cano(row, 40, KC1)) = make_uint4(0u, 0u, 0u, 0u);
        } else {
#pragma unroll
            for (int c = 0; c < 4; ++c)
                *reinterpret_cast<uint4 *>(A0 + cano(row, 8 * c, KC1)) = live ? nf[c] : make_uint4(0u, 0u, 0u, 0u);
        }
        prefetch(tile + gridDim.x);
        // ---- L1: [128 x 48] x [48 x 32H]
        fence_async_smem();
        tc_before();
        __syncthreads();
        if (t == 0) {
            tc_after();
#pragma unroll
            for (int kk = 0; kk < K1 / 16; ++kk)
                mma(tmem, sdesc(smem_u32(A0) + kk * 256, KC1 * 128), sdesc(smem_u32(W1) + kk * 256, KC1 * 128),
                    idesc(N1), kk > 0);
            commit(bar);
        }
        bar_wait(bar, phase);
        phase ^= 1;
        tc_after();
        {   // heads 0-2 by group 0, 3.. by group 1
            float v[32];
#pragma unroll 1
            for (int h = grp * 3; h < (grp ? H : 3); ++h) {
                tld32(trow + 32 * h, v);
                relu_store(v, B1 + 32 * h, A1, row, 32 * h, KC2);
            }
        }
        // ---- L2: per head [128 x 32] x [32 x 32]
        fence_async_smem();
        tc_before();
        __syncthreads();
        if (t == 0) {
            tc_after();
#pragma unroll
            for (int h = 0; h < H; ++h)
#pragma unroll
                for (int kk = 0; kk < 2; ++kk)
                    mma(tmem + 32 * h, sdesc(smem_u32(A1) + (4 * h + 2 * kk) * 128, KC2 * 128),
                        sdesc(smem_u32(W2) + h * HID * HID * 2 + kk * 256, (HID / 8) * 128), idesc(HID), kk > 0);
            commit(bar);
        }
        bar_wait(bar, phase);
        phase ^= 1;
        tc_after();
        {   // heads 0-2 by group 0, 3.. by group 1
            float v[32];
#pragma unroll 1
            for (int h = grp * 3; h < (grp ? H : 3); ++h) {
                tld32(trow + 32 * h, v);
                relu_store(v, B2 + 32 * h, A1, row, 32 * h, KC2);
            }
        }
        // ---- L3: per head [128 x 32] x [32 x out_pad]
        fence_async_smem();
        tc_before();
        __syncthreads();
        if (t == 0) {
            tc_after();
#pragma unroll
            for (int h = 0; h < H; ++h)
#pragma unroll
                for (int kk = 0; kk < 2; ++kk)
                    mma(tmem + out_col(h), sdesc(smem_u32(A1) + (4 * h + 2 * kk) * 128, KC2 * 128),
                        sdesc(smem_u32(W3) + (out_col(h) / 8) * ((HID / 8) * 128) + kk * 256, (HID / 8) * 128),
                        idesc(out_pad(LIDAR, h)), kk > 0);
            commit(bar);
        }
        bar_wait(bar, phase);
        phase ^= 1;
        tc_after();
        // ---- epilogue: 5 surfels of this anchor, split between the two groups
        // (group 0: centres, scales, frames of surfels 0-2; group 1: frames of
        // surfels 3-4, opacity, colour | intensity and ray-drop), staged in A1
        // (free until the next tile's L1 drain) and then stored coalesced
        float *stg = reinterpret_cast<float *>(A1);
        float *sM = stg, *sQ = sM + 3 * KS * M, *sS = sQ + 4 * KS * M, *sO = sS + 2 * KS * M;
        float *sC = sO + KS * M;   // camera: 3 per surfel; LiDAR: intensity, then ray-drop logit
        const int ls0 = KS * row;  // this anchor's first surfel in the tile
        float R[32];
        tld32(trow + 32, R);
        if (grp == 0) {
            float O[16], S[16];
            tld16(trow + 0, O);
            tld16(trow + 16, S);
            tc_before();   // the next tile's L1 overwrites these columns after the CTA barrier
#pragma unroll
            for (int j = 0; j < KS; ++j) {
                const int ls = ls0 + j;
                sM[3 * ls] = fmaf(O[3 * j] + B3[3 * j], l0, x);
                sM[3 * ls + 1] = fmaf(O[3 * j + 1] + B3[3 * j + 1], l1, y);
                sM[3 * ls + 2] = fmaf(O[3 * j + 2] + B3[3 * j + 2], l2, z);
                *reinterpret_cast<float2 *>(sS + 2 * ls) =
                    make_float2(l0 * __expf(S[2 * j] + B3[16 + 2 * j]), l1 * __expf(S[2 * j + 1] + B3[16 + 2 * j + 1]));
            }
#pragma unroll
            for (int j = 0; j < 3; ++j) write_quat(R, B3, j, sQ + 4 * (ls0 + j));
        } else {
            float Op[16], C[16], D[16];
            tld16(trow + 64, Op);
            tld16(trow + 80, C);
            if (LIDAR) tld16(trow + 96, D);
            tc_before();
#pragma unroll
            for (int j = 3; j < KS; ++j) write_quat(R, B3, j, sQ + 4 * (ls0 + j));
#pragma unroll
            for (int j = 0; j < KS; ++j) {
                const int ls = ls0 + j;
                sO[ls] = sigm(Op[j] + B3[64 + j]);
                if (!LIDAR) {
                    const float iC0 = 3.5449077018110318f;   // 1 / C0 = 2 sqrt(pi)
#pragma unroll
                    for (int c = 0; c < 3; ++c) sC[3 * ls + c] = (sigm(C[3 * j + c] + B3[80 + 3 * j + c]) - 0.5f) * iC0;
                } else {
                    sC[ls] = sigm(C[j] + B3[80 + j]);
                    sC[KS * M + ls] = D[j] + B3[96 + j];
                }
            }
        }
        __syncthreads();
        {
            const int64_t s0 = (int64_t)KS * tile * M;                       // first surfel of the tile
            const int ns = (int)min((int64_t)KS * M, (int64_t)KS * p.n - s0);   // its live surfels
            copy_out(sM, p.means + 3 * s0, 3 * ns, t);
            copy_out(sQ, p.quats + 4 * s0, 4 * ns, t);
            copy_out(sS, p.scales + 2 * s0, 2 * ns, t);
            copy_out(sO, p.opac + s0, ns, t);
            if (!LIDAR) {
                copy_out(sC, p.sh + 3 * s0, 3 * ns, t);
            } else {
                copy_out(sC, p.inten + s0, ns, t);
                copy_out(sC + KS * M, p.drop + s0, ns, t);
            }
        }
    }
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TMEM_COLS));
}

}  // namespace dec

size_t decode_smem_bytes() { return dec::SMEM; }

cudaError_t launch_decode(const gs_anchors *an, const gs_decoder *de, const float origin[3], float *means,
                          float *quats, float *scales, float *opac, float *sh, float *inten, float *drop,
                          cudaStream_t st) {
    using namespace dec;
    Params p;
    memset(&p, 0, sizeof(p));
    p.n = an->n;
    p.pos = an->position;
    p.base = an->base_scale;
    p.feat = reinterpret_cast<const __half *>(an->feature);
    p.lidar = de->modality == GS_DECODE_LIDAR;
    const int H = p.lidar ? 6 : 5;
    for (int h = 0; h < H; ++h) {
        p.w1[h] = reinterpret_cast<const __half *>(de->head[h].w1);
        p.w2[h] = reinterpret_cast<const __half *>(de->head[h].w2);
        p.w3[h] = reinterpret_cast<const __half *>(de->head[h].w3);
        p.b1[h] = de->head[h].b1;
        p.b2[h] = de->head[h].b2;
        p.b3[h] = de->head[h].b3;
    }
    p.ox = origin[0];
    p.oy = origin[1];
    p.oz = origin[2];
    p.means = means; p.quats = quats; p.scales = scales; p.opac = opac;
    p.sh = sh; p.inten = inten; p.drop = drop;
    if (p.n == 0) return cudaSuccess;
    auto kern = p.lidar ? k_decode<1> : k_decode<0>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, NT, SMEM);
    const int64_t ntiles = (p.n + M - 1) / M;
    const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)nsm * std::max(1, std::min(per, 2)));
    note_launch();
    kern<<<grid, NT, SMEM, st>>>(p);
    return cudaGetLastError();
}

}  // namespace gsr
