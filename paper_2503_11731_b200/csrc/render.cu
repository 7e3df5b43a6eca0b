// render.cu -- front-to-back compositing kernels (gs_render_camera,
// gs_render_lidar).  PAPER.md Eq. 2 ray-splat intersection with the
// unified plane pair (Eq. 3 pinhole, Eq. 5 LiDAR, equidistant fisheye per
// DESIGN R4); 2DGS low-pass floor for cameras; north_star rule
// alpha = min(alpha_max, o G), skip alpha < alpha_min, stop before
// T < t_min.
//
// One CTA per tile, one thread per pixel / LiDAR ray.  Surfel records of the
// tile's depth-sorted list are staged in shared memory in batches of
// blockDim records with cp.async (double buffered); every thread walks the
// batch in order.  The plane pair of a sample meets the surfel where
// (M^T h_u) x (M^T h_v) = det(M) M^{-1} (h_u x h_v), so the kernels evaluate
// the adjugate of the surfel map on the ray direction; records are written
// relative to the surfel centre so the fp32 arithmetic here
// stays well conditioned.  No atomics: outputs are bitwise deterministic.
#include "gsr_internal.cuh"

namespace gsr {

__device__ __forceinline__ float fast_rcp(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float fast_ex2(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

constexpr float LOG2E_HALF = 0.72134752044448170368f;   // 0.5 * log2(e)

template <int R4>
__device__ __forceinline__ void stage_batch(float4 *dst, const float4 *__restrict__ rec,
                                            const uint32_t *__restrict__ values, uint32_t first,
                                            uint32_t cnt) {
    const uint32_t t = threadIdx.x;
    if (t < cnt) {
        const uint32_t id = __ldg(values + first + t);
        const float4 *src = rec + (size_t)id * R4;
        float4 *d = dst + t * R4;
#pragma unroll
        for (int k = 0; k < R4; ++k) cp_async16(d + k, src + k);
    }
    cp_async_commit();
}

// ------------------------------------------------------------------ camera
template <int KIND>
__global__ void __launch_bounds__(1024) k_render_camera(
    const float4 *__restrict__ rec, const uint32_t *__restrict__ values,
    const uint2 *__restrict__ ranges, const int32_t *__restrict__ d_overflow,
    const __grid_constant__ DevSensor se, const DevOpts op, float *__restrict__ out_rgb,
    float *__restrict__ out_depth, float *__restrict__ out_normal, float *__restrict__ out_alpha) {
    constexpr int R4 = (KIND == GS_PINHOLE ? PH_FLOATS : FE_FLOATS) / 4;
    extern __shared__ float4 smem[];
    const int B = blockDim.x;
    const int tile = blockIdx.x;
    const int tyi = tile / se.ntx, txi = tile - tyi * se.ntx;
    const int lx = threadIdx.x % se.tw, ly = threadIdx.x / se.tw;
    const int pxi = txi * se.tw + lx, pyi = tyi * se.th + ly;
    const bool inside = (lx < se.tw) && (ly < se.th) && pxi < se.width && pyi < se.height;
    const float px = (float)pxi + 0.5f, py = (float)pyi + 0.5f;

    bool valid = inside;
    float dhx = 0.f, dhy = 0.f, dhz = 0.f, dlx = 0.f, dly = 0.f, dlz = 0.f;
    if (KIND == GS_FISHEYE_EQUIDISTANT && inside) {
        // ray of the pixel in fp64: invert theta_d = theta (1 + k1 t^2 + ...)
        const double mx = __ddiv_rn(__dadd_rn((double)px, -(double)se.cx), (double)se.fx);
        const double my = __ddiv_rn(__dadd_rn((double)py, -(double)se.cy), (double)se.fy);
        const double td = __dsqrt_rn(__dadd_rn(__dmul_rn(mx, mx), __dmul_rn(my, my)));
        valid = td <= se.tdmax;
        const double tdc = fmin(td, se.tdmax);
        const double k1 = se.k[0], k2 = se.k[1], k3 = se.k[2], k4 = se.k[3];
        double th = fmin(tdc, (double)se.theta_max);
        for (int it = 0; it < 12; ++it) {
            const double t2 = th * th;
            const double f = th * (1.0 + t2 * (k1 + t2 * (k2 + t2 * (k3 + t2 * k4)))) - tdc;
            const double df = 1.0 + t2 * (3.0 * k1 + t2 * (5.0 * k2 + t2 * (7.0 * k3 + t2 * 9.0 * k4)));
            th = fmin(fmax(th - f / df, 0.0), (double)se.theta_max);
        }
        double sp = 0.0, cp = 1.0;
        if (td > 0.0) { cp = mx / td; sp = my / td; }
        double st, ct;
        sincos(th, &st, &ct);
        split_hilo(st * cp, dhx, dlx);
        split_hilo(st * sp, dhy, dly);
        split_hilo(ct, dhz, dlz);
    }

    uint2 rg = ranges[tile];
    if (d_overflow && *d_overflow) rg.y = rg.x;
    const uint32_t start = rg.x, end = rg.y;

    float T = 1.f, A = 0.f, C0 = 0.f, C1 = 0.f, C2 = 0.f, D = 0.f, N0 = 0.f, N1 = 0.f, N2 = 0.f;
    bool done = !valid;
    const float near_p = op.near_plane, amax = op.alpha_max, amin = op.alpha_min, tmin = op.t_min,
                sup = op.support, inv_s2 = op.inv_sigma2;

    const uint32_t total = end - start;
    const uint32_t nb = (total + B - 1) / B;
    if (nb > 0) stage_batch<R4>(smem, rec, values, start, min((uint32_t)B, total));
    for (uint32_t b = 0; b < nb; ++b) {
        if (b + 1 < nb) {
            const uint32_t f = start + (b + 1) * B;
            stage_batch<R4>(smem + ((b + 1) & 1) * B * R4, rec, values, f, min((uint32_t)B, end - f));
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const float4 *buf = smem + (b & 1) * B * R4;
        const int cnt = (int)min((uint32_t)B, end - (start + b * B));
        if (!done) {
            for (int j = 0; j < cnt; ++j) {
                const float4 *r = buf + j * R4;
                float rho3, rho2, ir, dep3, depc, o;
                bool keep;
                if (KIND == GS_PINHOLE) {
                    const float4 g0 = r[0], g1 = r[1], g2 = r[2], g3 = r[3];
                    const float dx = (px - g2.x) - g2.z, dy = (py - g2.y) - g2.w;
                    const float q0 = fmaf(g0.x, dx, g0.y * dy);
                    const float q1 = fmaf(g0.z, dx, g0.w * dy);
                    const float q2 = fmaf(g1.x, dx, fmaf(g1.y, dy, g1.z));
                    const float n3 = fmaf(q0, q0, q1 * q1);
                    const float s2 = fmaf(dx, dx, dy * dy);
                    keep = !(n3 > g1.w * q2 * q2) || !(s2 > g3.x);
                    if (!keep) continue;
                    ir = fast_rcp(q2);
                    rho3 = n3 * ir * ir;
                    rho2 = s2 * inv_s2;
                    dep3 = g3.z * ir;
                    depc = g3.w;
                    o = g3.y;
                } else {
                    const float4 g0 = r[0], g1 = r[1], g2 = r[2], g3 = r[3], g4 = r[4], g5 = r[5], g6 = r[6];
                    const float ex = (dhx - g0.x) + (dlx - g1.x);
                    const float ey = (dhy - g0.y) + (dly - g1.y);
                    const float ez = (dhz - g0.z) + (dlz - g1.z);
                    const float hu = fmaf(g2.x, ex, fmaf(g2.y, ey, g2.z * ez));
                    const float hv = fmaf(g3.x, ex, fmaf(g3.y, ey, g3.z * ez));
                    const float Dd = fmaf(g4.x, ex, fmaf(g4.y, ey, fmaf(g4.z, ez, g1.w)));
                    const float n3 = fmaf(hu, hu, hv * hv);
                    const float dx = (px - g5.x) - g5.z, dy = (py - g5.y) - g5.w;
                    const float s2 = fmaf(dx, dx, dy * dy);
                    keep = !(n3 > g0.w * Dd * Dd) || !(s2 > g6.x);
                    if (!keep) continue;
                    ir = fast_rcp(Dd);
                    rho3 = n3 * ir * ir;
                    rho2 = s2 * inv_s2;
                    dep3 = g3.w * ir;
                    depc = g4.w;
                    o = g2.w;
                }
                const bool use3 = rho3 <= rho2;
                const float rho = use3 ? rho3 : rho2;
                const float dep = use3 ? dep3 : depc;
                if (!(rho <= sup) || !(dep >= near_p)) continue;
                const float a = fminf(amax, o * fast_ex2(-LOG2E_HALF * rho));
                if (!(a >= amin)) continue;
                const float Tn = T * (1.f - a);
                if (Tn < tmin) { done = true; break; }
                const float w = a * T;
                float4 c0, c1;
                if (KIND == GS_PINHOLE) { c0 = r[4]; c1 = r[5]; }
                else { c0 = r[7]; c1 = r[8]; }
                C0 = fmaf(w, c0.x, C0); C1 = fmaf(w, c0.y, C1); C2 = fmaf(w, c0.z, C2);
                N0 = fmaf(w, c0.w, N0); N1 = fmaf(w, c1.x, N1); N2 = fmaf(w, c1.y, N2);
                D = fmaf(w, dep, D);
                A += w;
                T = Tn;
            }
        }
        if (__syncthreads_count(!done) == 0) break;
    }
    if (!inside) return;
    const size_t HW = (size_t)se.width * se.height, pix = (size_t)pyi * se.width + pxi;
    if (!valid) {
        if (out_rgb) { out_rgb[pix] = op.bg[0]; out_rgb[HW + pix] = op.bg[1]; out_rgb[2 * HW + pix] = op.bg[2]; }
        if (out_depth) out_depth[pix] = 0.f;
        if (out_normal) { out_normal[pix] = 0.f; out_normal[HW + pix] = 0.f; out_normal[2 * HW + pix] = 0.f; }
        out_alpha[pix] = 0.f;
        return;
    }
    if (out_rgb) {
        out_rgb[pix] = fmaf(T, op.bg[0], C0);
        out_rgb[HW + pix] = fmaf(T, op.bg[1], C1);
        out_rgb[2 * HW + pix] = fmaf(T, op.bg[2], C2);
    }
    if (out_depth) out_depth[pix] = A > 0.f ? D / A : 0.f;
    if (out_normal) { out_normal[pix] = N0; out_normal[HW + pix] = N1; out_normal[2 * HW + pix] = N2; }
    out_alpha[pix] = A;
}

// ------------------------------------------------------------------ LiDAR
__global__ void __launch_bounds__(1024) k_render_lidar(
    const float4 *__restrict__ rec, const uint32_t *__restrict__ values,
    const uint2 *__restrict__ ranges, const int32_t *__restrict__ d_overflow,
    const __grid_constant__ DevSensor se, const DevOpts op, float *__restrict__ out_range,
    float *__restrict__ out_int, float *__restrict__ out_drop, float *__restrict__ out_alpha) {
    constexpr int R4 = LI_FLOATS / 4;
    extern __shared__ float4 smem[];
    const int B = blockDim.x;
    const int tile = blockIdx.x;
    const int tyi = tile / se.ntx, txi = tile - tyi * se.ntx;
    const int lx = threadIdx.x % se.tw, ly = threadIdx.x / se.tw;
    const int col = txi * se.tw + lx, row = tyi * se.th + ly;
    const bool inside = (ly < se.th) && col < se.width && row < se.height;

    float dhx = 0.f, dhy = 0.f, dhz = 0.f, dlx = 0.f, dly = 0.f, dlz = 0.f;
    if (inside) {   // Eq. 5 ray in fp64: theta = elevation (row), phi = azimuth (column)
        const double th = (double)se.beam[row];
        const double ph = (double)se.az0 + (double)col * (double)se.az_step;
        double st, ct, sf, cf;
        sincos(th, &st, &ct);
        sincos(ph, &sf, &cf);
        split_hilo(ct * cf, dhx, dlx);
        split_hilo(ct * sf, dhy, dly);
        split_hilo(st, dhz, dlz);
    }
    uint2 rg = ranges[tile];
    if (d_overflow && *d_overflow) rg.y = rg.x;
    const uint32_t start = rg.x, end = rg.y;
    float T = 1.f, A = 0.f, Rg = 0.f, I = 0.f, Pd = 0.f;
    bool done = !inside;
    const float near_p = op.near_plane, amax = op.alpha_max, amin = op.alpha_min, tmin = op.t_min,
                sup = op.support;
    const uint32_t total = end - start;
    const uint32_t nb = (total + B - 1) / B;
    if (nb > 0) stage_batch<R4>(smem, rec, values, start, min((uint32_t)B, total));
    for (uint32_t b = 0; b < nb; ++b) {
        if (b + 1 < nb) {
            const uint32_t f = start + (b + 1) * B;
            stage_batch<R4>(smem + ((b + 1) & 1) * B * R4, rec, values, f, min((uint32_t)B, end - f));
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const float4 *buf = smem + (b & 1) * B * R4;
        const int cnt = (int)min((uint32_t)B, end - (start + b * B));
        if (!done) {
            for (int j = 0; j < cnt; ++j) {
                const float4 *r = buf + j * R4;
                const float4 g0 = r[0], g1 = r[1], g2 = r[2], g3 = r[3], g4 = r[4];
                const float ex = (dhx - g0.x) + (dlx - g1.x);
                const float ey = (dhy - g0.y) + (dly - g1.y);
                const float ez = (dhz - g0.z) + (dlz - g1.z);
                const float hu = fmaf(g2.x, ex, fmaf(g2.y, ey, g2.z * ez));
                const float hv = fmaf(g3.x, ex, fmaf(g3.y, ey, g3.z * ez));
                const float Dd = fmaf(g4.x, ex, fmaf(g4.y, ey, fmaf(g4.z, ez, g1.w)));
                const float n3 = fmaf(hu, hu, hv * hv);
                if (n3 > g0.w * Dd * Dd) continue;
                const float ir = fast_rcp(Dd);
                const float rho = n3 * ir * ir;
                const float t = g3.w * ir;
                if (!(rho <= sup) || !(t >= near_p)) continue;
                const float a = fminf(amax, g2.w * fast_ex2(-LOG2E_HALF * rho));
                if (!(a >= amin)) continue;
                const float Tn = T * (1.f - a);
                if (Tn < tmin) { done = true; break; }
                const float w = a * T;
                const float4 p = r[5];
                Rg = fmaf(w, t, Rg);
                I = fmaf(w, p.x, I);
                Pd = fmaf(w, p.y, Pd);
                A += w;
                T = Tn;
            }
        }
        if (__syncthreads_count(!done) == 0) break;
    }
    if (!inside) return;
    const size_t pix = (size_t)row * se.width + col;
    if (out_range) out_range[pix] = A > 0.f ? Rg / A : op.bg_range;
    if (out_int) out_int[pix] = I;
    if (out_drop) out_drop[pix] = fmaf(T, op.bg_raydrop, Pd);
    out_alpha[pix] = A;
}

// ------------------------------------------------------------------ host
cudaError_t launch_render_camera(const void *proj, int64_t n, const uint32_t *values,
                                 const uint32_t *ranges, const int32_t *d_overflow,
                                 const DevSensor &se, const DevOpts &op, float *rgb, float *depth,
                                 float *normal, float *alpha, cudaStream_t st) {
    const ProjLayout L(n, se.kind);
    const float4 *rec = (const float4 *)((const char *)proj + L.rec);
    const int B = se.tw * se.th;
    const unsigned grid = (unsigned)(se.ntx * se.nty);
    if (se.kind == GS_PINHOLE) {
        const size_t sm = 2 * (size_t)B * PH_FLOATS * 4;
        cudaFuncSetAttribute(k_render_camera<GS_PINHOLE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_render_camera<GS_PINHOLE><<<grid, B, sm, st>>>(rec, values, (const uint2 *)ranges, d_overflow, se, op,
                                                         rgb, depth, normal, alpha);
    } else {
        const size_t sm = 2 * (size_t)B * FE_FLOATS * 4;
        cudaFuncSetAttribute(k_render_camera<GS_FISHEYE_EQUIDISTANT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sm);
        k_render_camera<GS_FISHEYE_EQUIDISTANT><<<grid, B, sm, st>>>(rec, values, (const uint2 *)ranges,
                                                                     d_overflow, se, op, rgb, depth, normal,
                                                                     alpha);
    }
    return cudaGetLastError();
}

cudaError_t launch_render_lidar(const void *proj, int64_t n, const uint32_t *values,
                                const uint32_t *ranges, const int32_t *d_overflow,
                                const DevSensor &se, const DevOpts &op, float *range, float *inten,
                                float *drop, float *alpha, cudaStream_t st) {
    const ProjLayout L(n, se.kind);
    const float4 *rec = (const float4 *)((const char *)proj + L.rec);
    const int B = se.tw * se.th;
    const unsigned grid = (unsigned)(se.ntx * se.nty);
    const size_t sm = 2 * (size_t)B * LI_FLOATS * 4;
    cudaFuncSetAttribute(k_render_lidar, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_render_lidar<<<grid, B, sm, st>>>(rec, values, (const uint2 *)ranges, d_overflow, se, op, range, inten,
                                        drop, alpha);
    return cudaGetLastError();
}

}  // namespace gsr
