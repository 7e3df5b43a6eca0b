// backward.cu -- backward pass of the compositing:
// gradients of L = sum_{channel, sample} grad_out * out w.r.t. the surfel
// attributes (means, quaternions, scales, opacities, SH | intensity, ray-drop
// logit) for pinhole cameras and LiDAR.  The forward definition is DESIGN.md
// §2 (Eqs. 1-3 and 5, the 2DGS low-pass P:48, the north_star
// compositing rule); training is PAPER.md:167, :214.
//
// Three kernels, reusing the forward frame's binning (sorted tile lists):
//   k_bwd_prep     per visible surfel: the sensor-frame splat matrix M of
//                  Eq. 1 (columns s_u R_s t_u | s_v R_s t_v | mu_s), the
//                  projected centre, centre depth, opacity, pre-clamp colour
//                  (or intensity, ray-drop probability) and oriented normal;
//   k_bwd_render   one CTA per tile, one thread per sample, two walks of the
//                  tile list: the first recomposites the sample (fp32, Eq. 2
//                  intersection from M) to get its outputs, the second
//                  differentiates the front-to-back recurrence
//                      dL/dalpha_i = e_i T_i - (S - sum_{j<=i} e_j w_j) / (1 - alpha_i)
//                  (e_i = dL/dw_i, S = sum_j e_j w_j + T_N dL/dT_N, known from
//                  the outputs) and chains it through alpha = min(a_max, o e^{-rho/2}),
//                  rho = min(rho3d, rho2d) and the Eq. 2 intersection to dL/dM,
//                  dL/dc, dL/d(centre depth), dL/do, dL/d(colour), dL/d(normal);
//                  per-record sums are warp-reduced, then one fp32 atomic per warp;
//   k_bwd_project  per surfel: the chain rule from those 19 quantities to the
//                  attributes (Eq. 1, the pinhole projection, the quaternion
//                  rotation with its normalisation, real SH and its gradient in
//                  the view direction, the ray-drop sigmoid).
// Per-pair arithmetic is fp32 from M (not the forward's centre-relative
// records), so decisions sit where the backward's own recomposite puts them;
// the gradient is that of the backward's recomposite (parity: central finite
// differences of the fp64 oracle, tests/test_gpu_backward.py).
#include <math.h>
#include <stdint.h>

#include <algorithm>

#include "gsr_internal.cuh"

namespace gsr {

namespace bwd {

constexpr int NG = 20;   // per-surfel gradient slots: dM 9, dc 2, dcdepth, do, dval 3, dn 3, pad

struct GradRec {
    float M[9];      // row-major M[r*3+k], sensor frame
    float c[2];      // projected centre (pinhole)
    float cdepth;    // centre depth (pinhole z)
    float o;
    float val[3];    // camera: pre-clamp colour; LiDAR: intensity, ray-drop probability, 0
    float n[3];      // oriented normal (sensor frame)
    float vis;       // 1 if visible
};
static_assert(sizeof(GradRec) == 80, "GradRec");

__device__ __forceinline__ void quat_rot(double qw, double qx, double qy, double qz, double R[3][3]) {
    R[0][0] = 1.0 - 2.0 * (qy * qy + qz * qz); R[0][1] = 2.0 * (qx * qy - qw * qz); R[0][2] = 2.0 * (qx * qz + qw * qy);
    R[1][0] = 2.0 * (qx * qy + qw * qz); R[1][1] = 1.0 - 2.0 * (qx * qx + qz * qz); R[1][2] = 2.0 * (qy * qz - qw * qx);
    R[2][0] = 2.0 * (qx * qz - qw * qy); R[2][1] = 2.0 * (qy * qz + qw * qx); R[2][2] = 1.0 - 2.0 * (qx * qx + qy * qy);
}

// real SH basis (3DGS ordering) at a unit direction and its gradient in (x, y, z)
__device__ void sh_basis_grad(double x, double y, double z, int deg, double Y[16], double G[16][3]) {
    const double C0 = 0.28209479177387814, C1 = 0.4886025119029199;
    const double C2a = 1.0925484305920792, C2b = 0.31539156525252005, C2c = 0.5462742152960396;
    const double C3a = 0.5900435899266435, C3b = 2.890611442640554, C3c = 0.4570457994644658,
                 C3d = 0.3731763325901154, C3e = 1.445305721320277;
    for (int j = 0; j < 16; ++j) { Y[j] = 0.0; G[j][0] = G[j][1] = G[j][2] = 0.0; }
    Y[0] = C0;
    if (deg < 1) return;
    Y[1] = -C1 * y; G[1][1] = -C1;
    Y[2] = C1 * z; G[2][2] = C1;
    Y[3] = -C1 * x; G[3][0] = -C1;
    if (deg < 2) return;
    const double xx = x * x, yy = y * y, zz = z * z;
    Y[4] = C2a * x * y; G[4][0] = C2a * y; G[4][1] = C2a * x;
    Y[5] = -C2a * y * z; G[5][1] = -C2a * z; G[5][2] = -C2a * y;
    Y[6] = C2b * (2 * zz - xx - yy); G[6][0] = -2 * C2b * x; G[6][1] = -2 * C2b * y; G[6][2] = 4 * C2b * z;
    Y[7] = -C2a * x * z; G[7][0] = -C2a * z; G[7][2] = -C2a * x;
    Y[8] = C2c * (xx - yy); G[8][0] = 2 * C2c * x; G[8][1] = -2 * C2c * y;
    if (deg < 3) return;
    Y[9] = -C3a * y * (3 * xx - yy); G[9][0] = -6 * C3a * x * y; G[9][1] = -C3a * (3 * xx - 3 * yy);
    Y[10] = C3b * x * y * z; G[10][0] = C3b * y * z; G[10][1] = C3b * x * z; G[10][2] = C3b * x * y;
    Y[11] = -C3c * y * (4 * zz - xx - yy);
    G[11][0] = 2 * C3c * x * y; G[11][1] = -C3c * (4 * zz - xx - 3 * yy); G[11][2] = -8 * C3c * y * z;
    Y[12] = C3d * z * (2 * zz - 3 * xx - 3 * yy);
    G[12][0] = -6 * C3d * x * z; G[12][1] = -6 * C3d * y * z; G[12][2] = C3d * (6 * zz - 3 * xx - 3 * yy);
    Y[13] = -C3c * x * (4 * zz - xx - yy);
    G[13][0] = -C3c * (4 * zz - 3 * xx - yy); G[13][1] = 2 * C3c * x * y; G[13][2] = -8 * C3c * x * z;
    Y[14] = C3e * z * (xx - yy); G[14][0] = 2 * C3e * x * z; G[14][1] = -2 * C3e * y * z; G[14][2] = C3e * (xx - yy);
    Y[15] = -C3a * x * (xx - 3 * yy); G[15][0] = -C3a * (3 * xx - 3 * yy); G[15][1] = 6 * C3a * x * y;
}

struct Surf {   // fp64 per-surfel quantities shared by prep and project-backward
    double Rs[3][3], q[4], qn, Rq[3][3], mus[3], tu[3], tv[3], nn[3], su, sv, sign;
};

__device__ void surf_geom(const DevSurfels &s, const DevSensor &se, int64_t i, Surf &f) {
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) f.Rs[r][c] = se.R[3 * r + c];
    const float4 q = reinterpret_cast<const float4 *>(s.quats)[i];
    f.qn = sqrt((double)q.x * q.x + (double)q.y * q.y + (double)q.z * q.z + (double)q.w * q.w);
    f.q[0] = q.x / f.qn; f.q[1] = q.y / f.qn; f.q[2] = q.z / f.qn; f.q[3] = q.w / f.qn;
    quat_rot(f.q[0], f.q[1], f.q[2], f.q[3], f.Rq);
    const double mu[3] = {s.means[3 * i], s.means[3 * i + 1], s.means[3 * i + 2]};
    for (int r = 0; r < 3; ++r) {
        f.mus[r] = f.Rs[r][0] * mu[0] + f.Rs[r][1] * mu[1] + f.Rs[r][2] * mu[2] + (double)se.t[r];
        f.tu[r] = f.Rs[r][0] * f.Rq[0][0] + f.Rs[r][1] * f.Rq[1][0] + f.Rs[r][2] * f.Rq[2][0];
        f.tv[r] = f.Rs[r][0] * f.Rq[0][1] + f.Rs[r][1] * f.Rq[1][1] + f.Rs[r][2] * f.Rq[2][1];
        f.nn[r] = f.Rs[r][0] * f.Rq[0][2] + f.Rs[r][1] * f.Rq[1][2] + f.Rs[r][2] * f.Rq[2][2];
    }
    f.su = s.scales[2 * i];
    f.sv = s.scales[2 * i + 1];
    const double side = f.nn[0] * f.mus[0] + f.nn[1] * f.mus[1] + f.nn[2] * f.mus[2];
    f.sign = side > 0.0 ? -1.0 : 1.0;   // the normal faces the sensor (reading R10)
}

template <int LIDAR>
__global__ void k_bwd_prep(DevSurfels s, const __grid_constant__ DevSensor se, const uint32_t *__restrict__ cnt,
                           GradRec *__restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= s.n) return;
    GradRec g;
    memset(&g, 0, sizeof(g));
    if (cnt[i] > 0) {
        Surf f;
        surf_geom(s, se, i, f);
        for (int r = 0; r < 3; ++r) {
            g.M[3 * r + 0] = (float)(f.su * f.tu[r]);
            g.M[3 * r + 1] = (float)(f.sv * f.tv[r]);
            g.M[3 * r + 2] = (float)f.mus[r];
            g.n[r] = (float)(f.sign * f.nn[r]);
        }
        if (!LIDAR) {
            g.c[0] = (float)((double)se.fx * f.mus[0] / f.mus[2] + (double)se.cx);
            g.c[1] = (float)((double)se.fy * f.mus[1] / f.mus[2] + (double)se.cy);
            g.cdepth = (float)f.mus[2];
            const double vx = s.means[3 * i] - (double)se.ow[0], vy = s.means[3 * i + 1] - (double)se.ow[1],
                         vz = s.means[3 * i + 2] - (double)se.ow[2];
            const double vn = sqrt(vx * vx + vy * vy + vz * vz);
            double Y[16], G[16][3];
            sh_basis_grad(vx / vn, vy / vn, vz / vn, s.sh_degree, Y, G);
            const int nc = (s.sh_degree + 1) * (s.sh_degree + 1);
            for (int ch = 0; ch < 3; ++ch) {
                double acc = 0.5;
                for (int j = 0; j < nc; ++j) acc += Y[j] * (double)s.sh[((size_t)i * nc + j) * 3 + ch];
                g.val[ch] = (float)acc;
            }
        } else {
            g.cdepth = (float)sqrt(f.mus[0] * f.mus[0] + f.mus[1] * f.mus[1] + f.mus[2] * f.mus[2]);
            g.val[0] = s.inten ? s.inten[i] : 0.f;
            g.val[1] = s.drop ? (float)(1.0 / (1.0 + exp(-(double)s.drop[i]))) : 0.f;
        }
        g.o = s.opac[i];
        g.vis = 1.f;
    }
    out[i] = g;
}

struct Pix {
    float nu[3], nv[3], d[3], px, py;
    bool inside;
};

struct PairVal {
    bool contrib, use3, clamped;
    float alpha, G, rho, u, v, t, w2, a[3], b[3], depth;
};

// Eq. 2 from M in fp32 + the low-pass and contribution tests (DESIGN.md §2 steps 4-7)
template <int LIDAR>
__device__ __forceinline__ void pair_eval(const GradRec &g, const Pix &p, const DevOpts &op, PairVal &v) {
    v.contrib = false;
    for (int k = 0; k < 3; ++k) {
        v.a[k] = g.M[0 * 3 + k] * p.nu[0] + g.M[1 * 3 + k] * p.nu[1] + g.M[2 * 3 + k] * p.nu[2];
        v.b[k] = g.M[0 * 3 + k] * p.nv[0] + g.M[1 * 3 + k] * p.nv[1] + g.M[2 * 3 + k] * p.nv[2];
    }
    const float w0 = v.a[1] * v.b[2] - v.a[2] * v.b[1];
    const float w1 = v.a[2] * v.b[0] - v.a[0] * v.b[2];
    v.w2 = v.a[0] * v.b[1] - v.a[1] * v.b[0];
    float rho3 = INFINITY;
    v.u = v.v = v.t = 0.f;
    if (v.w2 != 0.f) {
        v.u = w0 / v.w2;
        v.v = w1 / v.w2;
        rho3 = v.u * v.u + v.v * v.v;
        if (LIDAR) {
            float t = 0.f;
            for (int r = 0; r < 3; ++r) t += p.d[r] * (g.M[3 * r] * v.u + g.M[3 * r + 1] * v.v + g.M[3 * r + 2]);
            v.t = t;
        } else {
            v.t = g.M[6] * v.u + g.M[7] * v.v + g.M[8];
        }
    }
    if (!LIDAR) {
        const float ex = p.px - g.c[0], ey = p.py - g.c[1];
        const float rho2 = (ex * ex + ey * ey) * op.inv_sigma2;
        v.use3 = rho3 <= rho2;
        v.rho = v.use3 ? rho3 : rho2;
        v.depth = v.use3 ? v.t : g.cdepth;
    } else {
        v.use3 = true;
        v.rho = rho3;
        v.depth = v.t;
    }
    v.G = expf(-0.5f * v.rho);
    const float a = g.o * v.G;
    v.clamped = a > op.alpha_max;
    v.alpha = v.clamped ? op.alpha_max : a;
    v.contrib = g.vis > 0.f && v.rho <= op.support && v.depth >= op.near_plane && v.alpha >= op.alpha_min;
}

template <int LIDAR>
__global__ void __launch_bounds__(512) k_bwd_render(const GradRec *__restrict__ recs, const uint32_t *__restrict__ values,
                                                    const uint2 *__restrict__ ranges, const __grid_constant__ DevSensor se,
                                                    DevOpts op, const float *__restrict__ gout, float *__restrict__ dg) {
    extern __shared__ GradRec sg[];
    __shared__ uint32_t sid[512];
    const int tile = blockIdx.x, t = threadIdx.x, lane = t & 31;
    const int tyi = tile / se.ntx, txi = tile - tyi * se.ntx;
    Pix p;
    const int pxi = txi * se.tw + t % se.tw, pyi = tyi * se.th + t / se.tw;
    p.inside = pxi < se.width && pyi < se.height;
    p.px = (float)pxi + 0.5f;
    p.py = (float)pyi + 0.5f;
    if (!LIDAR) {
        const float xh = (p.px - se.cx) / se.fx, yh = (p.py - se.cy) / se.fy;
        p.nu[0] = -1.f; p.nu[1] = 0.f; p.nu[2] = xh;
        p.nv[0] = 0.f; p.nv[1] = -1.f; p.nv[2] = yh;
        p.d[0] = xh; p.d[1] = yh; p.d[2] = 1.f;
    } else if (p.inside) {
        const double th = se.beam[pyi], ph = (double)se.az0 + (double)pxi * (double)se.az_step;
        double st, ct, sf, cf;
        sincos(th, &st, &ct);
        sincos(ph, &sf, &cf);
        p.nu[0] = (float)sf; p.nu[1] = (float)-cf; p.nu[2] = 0.f;
        p.nv[0] = (float)(st * cf); p.nv[1] = (float)(st * sf); p.nv[2] = (float)-ct;
        p.d[0] = (float)(ct * cf); p.d[1] = (float)(ct * sf); p.d[2] = (float)st;
    }
    const size_t HW = (size_t)se.width * se.height, pix = (size_t)pyi * se.width + pxi;
    const int C = LIDAR ? 4 : 8;
    float g[8];
    for (int c = 0; c < 8; ++c) g[c] = (p.inside && c < C) ? gout[c * HW + pix] : 0.f;
    const uint2 rg = ranges[tile];
    const int nthr = blockDim.x;

    // ---- pass 1: recomposite the sample
    float T = 1.f, C0 = 0.f, C1 = 0.f, C2 = 0.f, D = 0.f, N0 = 0.f, N1 = 0.f, N2 = 0.f;
    bool done = !p.inside;
    for (uint32_t base = rg.x; base < rg.y; base += nthr) {
        if (!__syncthreads_or(!done)) break;
        if (base + t < rg.y) {
            sid[t] = values[base + t];
            sg[t] = recs[sid[t]];
        }
        __syncthreads();
        const int nb = min((uint32_t)nthr, rg.y - base);
        for (int k = 0; k < nb && !done; ++k) {
            PairVal v;
            pair_eval<LIDAR>(sg[k], p, op, v);
            if (!v.contrib) continue;
            const float Tn = T * (1.f - v.alpha);
            if (Tn < op.t_min) { done = true; break; }
            const float w = v.alpha * T;
            if (!LIDAR) {
                C0 += w * fmaxf(sg[k].val[0], 0.f); C1 += w * fmaxf(sg[k].val[1], 0.f); C2 += w * fmaxf(sg[k].val[2], 0.f);
                N0 += w * sg[k].n[0]; N1 += w * sg[k].n[1]; N2 += w * sg[k].n[2];
            } else {
                C0 += w * sg[k].val[0]; C1 += w * sg[k].val[1];
            }
            D += w * v.depth;
            T = Tn;
        }
        __syncthreads();
    }
    // ---- the output gradients as per-contributor weights
    const float A = 1.f - T;
    const float ga = A > 0.f ? 1.f / A : 0.f;
    float gd, GT, S;
    if (!LIDAR) {
        gd = g[3] * ga;   // dL/dD through depth = D / A
        GT = g[0] * op.bg[0] + g[1] * op.bg[1] + g[2] * op.bg[2] - g[7] + g[3] * D * ga * ga;
        S = g[0] * C0 + g[1] * C1 + g[2] * C2 + gd * D + g[4] * N0 + g[5] * N1 + g[6] * N2 + T * GT;
    } else {
        gd = g[0] * ga;   // range = D / A
        GT = g[2] * op.bg_raydrop - g[3] + g[0] * D * ga * ga;
        S = gd * D + g[1] * C0 + g[2] * C1 + T * GT;
    }
    // ---- pass 2: differentiate the recurrence, chain to the per-surfel quantities
    T = 1.f;
    float P = 0.f;
    done = !p.inside;
    for (uint32_t base = rg.x; base < rg.y; base += nthr) {
        if (!__syncthreads_or(!done)) break;
        if (base + t < rg.y) {
            sid[t] = values[base + t];
            sg[t] = recs[sid[t]];
        }
        __syncthreads();
        const int nb = min((uint32_t)nthr, rg.y - base);
        for (int k = 0; k < nb; ++k) {
            float gr[NG - 1];
#pragma unroll
            for (int q = 0; q < NG - 1; ++q) gr[q] = 0.f;
            bool any = false;
            if (!done) {
                const GradRec &R = sg[k];
                PairVal v;
                pair_eval<LIDAR>(R, p, op, v);
                if (v.contrib) {
                    const float Tn = T * (1.f - v.alpha);
                    if (Tn < op.t_min) {
                        done = true;
                    } else {
                        any = true;
                        const float w = v.alpha * T;
                        float e;
                        if (!LIDAR) {
                            const float c0 = fmaxf(R.val[0], 0.f), c1 = fmaxf(R.val[1], 0.f), c2 = fmaxf(R.val[2], 0.f);
                            e = g[0] * c0 + g[1] * c1 + g[2] * c2 + gd * v.depth + g[4] * R.n[0] + g[5] * R.n[1] +
                                g[6] * R.n[2];
                            gr[13] = R.val[0] > 0.f ? g[0] * w : 0.f;   // dL/d(pre-clamp colour)
                            gr[14] = R.val[1] > 0.f ? g[1] * w : 0.f;
                            gr[15] = R.val[2] > 0.f ? g[2] * w : 0.f;
                            gr[16] = g[4] * w; gr[17] = g[5] * w; gr[18] = g[6] * w;
                        } else {
                            e = gd * v.depth + g[1] * R.val[0] + g[2] * R.val[1];
                            gr[13] = g[1] * w;
                            gr[14] = g[2] * w;
                        }
                        P += e * w;
                        const float dalpha = e * T - (S - P) / (1.f - v.alpha);
                        const float ddepth = gd * w;
                        float drho = 0.f;
                        if (!v.clamped) {
                            gr[12] = dalpha * v.G;                   // dL/do
                            drho = -0.5f * v.alpha * dalpha;
                        }
                        float gu = 0.f, gv = 0.f;
                        if (v.use3) {
                            gu = drho * 2.f * v.u;
                            gv = drho * 2.f * v.v;
                            // hit depth t: pinhole P_z, LiDAR d . P, P = M (u, v, 1)
                            if (!LIDAR) {
                                gr[6] += ddepth * v.u; gr[7] += ddepth * v.v; gr[8] += ddepth;
                                gu += ddepth * R.M[6]; gv += ddepth * R.M[7];
                            } else {
                                for (int r = 0; r < 3; ++r) {
                                    gr[3 * r] += ddepth * p.d[r] * v.u;
                                    gr[3 * r + 1] += ddepth * p.d[r] * v.v;
                                    gr[3 * r + 2] += ddepth * p.d[r];
                                    gu += ddepth * p.d[r] * R.M[3 * r];
                                    gv += ddepth * p.d[r] * R.M[3 * r + 1];
                                }
                            }
                            // (u, v) = (w0, w1) / w2, w = a x b, a = M^T n_u, b = M^T n_v
                            const float iw = 1.f / v.w2;
                            const float gw[3] = {gu * iw, gv * iw, -(gu * v.u + gv * v.v) * iw};
                            const float gA[3] = {v.b[1] * gw[2] - v.b[2] * gw[1], v.b[2] * gw[0] - v.b[0] * gw[2],
                                                 v.b[0] * gw[1] - v.b[1] * gw[0]};
                            const float gB[3] = {gw[1] * v.a[2] - gw[2] * v.a[1], gw[2] * v.a[0] - gw[0] * v.a[2],
                                                 gw[0] * v.a[1] - gw[1] * v.a[0]};
                            for (int r = 0; r < 3; ++r)
                                for (int c = 0; c < 3; ++c) gr[3 * r + c] += p.nu[r] * gA[c] + p.nv[r] * gB[c];
                        } else {   // low-pass branch: rho2d = |p - c|^2 / sigma^2, depth = centre depth
                            gr[9] = drho * -2.f * (p.px - R.c[0]) * op.inv_sigma2;
                            gr[10] = drho * -2.f * (p.py - R.c[1]) * op.inv_sigma2;
                            gr[11] = ddepth;
                        }
                        T = Tn;
                    }
                }
            }
            if (__any_sync(0xffffffffu, any)) {
#pragma unroll
                for (int q = 0; q < NG - 1; ++q) {
                    float x = gr[q];
#pragma unroll
                    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
                    gr[q] = x;
                }
                if (lane == 0) {
                    float *dst = dg + (size_t)sid[k] * NG;
#pragma unroll
                    for (int q = 0; q < NG - 1; ++q)
                        if (gr[q] != 0.f) atomicAdd(dst + q, gr[q]);
                }
            }
        }
        __syncthreads();
    }
}

template <int LIDAR>
__global__ void k_bwd_project(DevSurfels s, const __grid_constant__ DevSensor se, const GradRec *__restrict__ recs,
                              const float *__restrict__ dg, float *d_means, float *d_quats, float *d_scales,
                              float *d_opac, float *d_sh, float *d_int, float *d_drop) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= s.n) return;
    const int nc = LIDAR ? 0 : (s.sh_degree + 1) * (s.sh_degree + 1);
    if (!(recs[i].vis > 0.f)) {
        for (int k = 0; k < 3; ++k) d_means[3 * i + k] = 0.f;
        for (int k = 0; k < 4; ++k) d_quats[4 * i + k] = 0.f;
        d_scales[2 * i] = d_scales[2 * i + 1] = 0.f;
        d_opac[i] = 0.f;
        if (!LIDAR && d_sh) for (int k = 0; k < 3 * nc; ++k) d_sh[(size_t)i * 3 * nc + k] = 0.f;
        if (LIDAR) { if (d_int) d_int[i] = 0.f; if (d_drop) d_drop[i] = 0.f; }
        return;
    }
    Surf f;
    surf_geom(s, se, i, f);
    const float *q = dg + (size_t)i * NG;
    double gM[3][3];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) gM[r][c] = q[3 * r + c];
    double gmus[3] = {gM[0][2], gM[1][2], gM[2][2]};
    if (!LIDAR) {   // projected centre c = (f_x X/Z + c_x, f_y Y/Z + c_y) and centre depth Z
        const double X = f.mus[0], Y = f.mus[1], Z = f.mus[2];
        gmus[0] += q[9] * (double)se.fx / Z;
        gmus[1] += q[10] * (double)se.fy / Z;
        gmus[2] += -q[9] * (double)se.fx * X / (Z * Z) - q[10] * (double)se.fy * Y / (Z * Z) + q[11];
    }
    // columns s_u R_s t_u, s_v R_s t_v: scales and the rotated tangents
    double ds_u = 0, ds_v = 0, gtu_s[3], gtv_s[3];
    for (int r = 0; r < 3; ++r) {
        ds_u += gM[r][0] * f.tu[r];
        ds_v += gM[r][1] * f.tv[r];
        gtu_s[r] = f.su * gM[r][0];
        gtv_s[r] = f.sv * gM[r][1];
    }
    // world-frame gradients: x_s = R_s x_w  ->  g_w = R_s^T g_s
    double gmu[3], gtu[3], gtv[3], gn[3];
    for (int c = 0; c < 3; ++c) {
        gmu[c] = gtu[c] = gtv[c] = gn[c] = 0.0;
        for (int r = 0; r < 3; ++r) {
            gmu[c] += f.Rs[r][c] * gmus[r];
            gtu[c] += f.Rs[r][c] * gtu_s[r];
            gtv[c] += f.Rs[r][c] * gtv_s[r];
            gn[c] += f.Rs[r][c] * f.sign * (LIDAR ? 0.0 : (double)q[16 + r]);
        }
    }
    // colour: c = max(0, sum Y_lm(v) k_lm + 1/2), v = normalize(mu - o)
    if (!LIDAR) {
        const double vx = s.means[3 * i] - (double)se.ow[0], vy = s.means[3 * i + 1] - (double)se.ow[1],
                     vz = s.means[3 * i + 2] - (double)se.ow[2];
        const double vn = sqrt(vx * vx + vy * vy + vz * vz);
        const double v[3] = {vx / vn, vy / vn, vz / vn};
        double Y[16], G[16][3];
        sh_basis_grad(v[0], v[1], v[2], s.sh_degree, Y, G);
        double gv[3] = {0, 0, 0};
        for (int j = 0; j < nc; ++j) {
            for (int ch = 0; ch < 3; ++ch) {
                const double gc = q[13 + ch];
                if (d_sh) d_sh[((size_t)i * nc + j) * 3 + ch] = (float)(Y[j] * gc);
                const double k = s.sh[((size_t)i * nc + j) * 3 + ch];
                for (int a = 0; a < 3; ++a) gv[a] += gc * k * G[j][a];
            }
        }
        // through the normalisation: dv/dmu = (I - v v^T) / |mu - o|
        const double vg = v[0] * gv[0] + v[1] * gv[1] + v[2] * gv[2];
        for (int a = 0; a < 3; ++a) gmu[a] += (gv[a] - v[a] * vg) / vn;
    } else {
        if (d_int) d_int[i] = q[13];
        if (d_drop) {
            const double pd = recs[i].val[1];
            d_drop[i] = (float)(q[14] * pd * (1.0 - pd));
        }
    }
    for (int a = 0; a < 3; ++a) d_means[3 * i + a] = (float)gmu[a];
    d_scales[2 * i] = (float)ds_u;
    d_scales[2 * i + 1] = (float)ds_v;
    d_opac[i] = q[12];
    // rotation R(q^) columns (t_u, t_v, n); dL/dR -> dL/dq^ -> dL/dq (normalisation)
    double gR[3][3];
    for (int r = 0; r < 3; ++r) { gR[r][0] = gtu[r]; gR[r][1] = gtv[r]; gR[r][2] = gn[r]; }
    const double w = f.q[0], x = f.q[1], y = f.q[2], z = f.q[3];
    double gq[4];
    gq[0] = gR[0][1] * -2 * z + gR[0][2] * 2 * y + gR[1][0] * 2 * z + gR[1][2] * -2 * x + gR[2][0] * -2 * y +
            gR[2][1] * 2 * x;
    gq[1] = gR[0][1] * 2 * y + gR[0][2] * 2 * z + gR[1][0] * 2 * y + gR[1][1] * -4 * x + gR[1][2] * -2 * w +
            gR[2][0] * 2 * z + gR[2][1] * 2 * w + gR[2][2] * -4 * x;
    gq[2] = gR[0][0] * -4 * y + gR[0][1] * 2 * x + gR[0][2] * 2 * w + gR[1][0] * 2 * x + gR[1][2] * 2 * z +
            gR[2][0] * -2 * w + gR[2][1] * 2 * z + gR[2][2] * -4 * y;
    gq[3] = gR[0][0] * -4 * z + gR[0][1] * -2 * w + gR[0][2] * 2 * x + gR[1][0] * 2 * w + gR[1][1] * -4 * z +
            gR[1][2] * 2 * y + gR[2][0] * 2 * x + gR[2][1] * 2 * y;
    const double dot = gq[0] * w + gq[1] * x + gq[2] * y + gq[3] * z;
    for (int k = 0; k < 4; ++k) d_quats[4 * i + k] = (float)((gq[k] - f.q[k] * dot) / f.qn);
}

}  // namespace bwd

size_t backward_workspace_bytes(int64_t n) {
    const size_t N = (size_t)std::max<int64_t>(n, 1);
    return align256(N * sizeof(bwd::GradRec)) + align256(N * bwd::NG * 4);
}

cudaError_t launch_backward(const DevSurfels &s, const DevSensor &se, const DevOpts &op, const void *proj,
                            const uint32_t *values, const uint32_t *ranges, const float *gout, void *ws,
                            float *d_means, float *d_quats, float *d_scales, float *d_opac, float *d_sh,
                            float *d_int, float *d_drop, cudaStream_t st) {
    using namespace bwd;
    const bool lidar = se.kind == GS_LIDAR_SPINNING;
    const ProjLayout PL(s.n, se.kind);
    const uint32_t *cnt = (const uint32_t *)((const char *)proj + PL.cnt);
    GradRec *recs = (GradRec *)ws;
    float *dg = (float *)((char *)ws + align256((size_t)std::max<int64_t>(s.n, 1) * sizeof(GradRec)));
    cudaError_t e = cudaMemsetAsync(dg, 0, (size_t)std::max<int64_t>(s.n, 1) * NG * 4, st);
    if (e != cudaSuccess || s.n == 0) return e;
    const unsigned gs = (unsigned)((s.n + 255) / 256);
    const int ntiles = se.ntx * se.nty, npix = se.tw * se.th;
    const size_t smem = (size_t)npix * sizeof(GradRec);
    note_launch(3);
    if (lidar) {
        k_bwd_prep<1><<<gs, 256, 0, st>>>(s, se, cnt, recs);
        k_bwd_render<1><<<ntiles, npix, smem, st>>>(recs, values, (const uint2 *)ranges, se, op, gout, dg);
        k_bwd_project<1><<<gs, 256, 0, st>>>(s, se, recs, dg, d_means, d_quats, d_scales, d_opac, d_sh, d_int, d_drop);
    } else {
        k_bwd_prep<0><<<gs, 256, 0, st>>>(s, se, cnt, recs);
        k_bwd_render<0><<<ntiles, npix, smem, st>>>(recs, values, (const uint2 *)ranges, se, op, gout, dg);
        k_bwd_project<0><<<gs, 256, 0, st>>>(s, se, recs, dg, d_means, d_quats, d_scales, d_opac, d_sh, d_int, d_drop);
    }
    return cudaGetLastError();
}

}  // namespace gsr
