// binning.cuh -- exact tile sets of a surfel's support (gs_project).
//
// Pinhole: the 3-sigma support (Eq. 2-3; the north_star
// 3-sigma bound) is the conic {d : |A01 d|^2 <= R (a2.d + qc)^2} in the pixel
// offset d = p - c, and the 2DGS low-pass floor adds the disc
// |d|^2 <= rcut2.  The record's pixel box bounds both, but a tilted or
// elongated ellipse meets far fewer tiles than its box: ph_row_tiles() gives,
// for one tile row, the tile columns whose pixel centres can lie in the
// support (the conic widened by a relative slack far above the compositor's
// fp32 error and by 1e-3 of its half width + 0.01 px, the disc by 1e-3
// relative + 0.01 px).  Ill-conditioned conics (near-degenerate, crossing the
// camera plane) and tiny boxes take the whole row of the rect, as the
// compositor's warp test does.  k_project stores the rows as a table
// (ProjLayout::rows) that k_emit_rows reads.
//
// LiDAR: li_tile_hits(), below; k_tiles (project.cu) stores a tile mask.
#pragma once
#include "gsr_internal.cuh"

namespace gsr {

struct PhRows {
    float cx, cy;          // projected centre (fp32 of hi + lo), pixels
    float sx, sy;          // ellipse centre, relative to c
    float M00, M01, M11, det, K;   // (d - s)^T M (d - s) <= K
    float hy;              // vertical half extent
    float ul;              // sqrt(K / (det M11)): the extreme points sit at y = sy +- M01 ul
    float hx;              // horizontal half extent
    float r2;              // low-pass disc radius^2 with slack
    bool full;             // every row takes the rect's whole column range
    bool ell;              // the conic part is present (3-sigma box not empty)
};

constexpr int PH_ROWS_MIN_SPAN = 4;   // boxes spanning <= this many px (width + height): whole rows
// Pinhole rects of fewer tiles keep every tile (they could drop little).
// (LiDAR: LI_MIN_AREA in project.cu.)
constexpr uint32_t KT_MIN_AREA = 4;
constexpr int PH_ROWS_MAX = 16;       // rects of more tile rows (or wider than 255 tiles): every tile of the rect
__device__ __forceinline__ float bin_sqrt(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float bin_rcp(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ PhRows ph_rows_setup(const float4 g0, const float4 g1, const float4 g2, float rcut2,
                                                uint32_t bbx, uint32_t bby) {
    PhRows p;
    p.cx = __fadd_rn(g2.x, g2.z);
    p.cy = __fadd_rn(g2.y, g2.w);
    p.r2 = __fmaf_rn(rcut2, 1.001f, 1e-3f);
    p.full = false;
    p.ell = false;
    p.sx = p.sy = p.M00 = p.M01 = p.M11 = p.det = p.K = p.hy = p.ul = p.hx = 0.f;
    const int bx0 = (int)(bbx & 0xffffu), bx1 = (int)(bbx >> 16);
    const int by0 = (int)(bby & 0xffffu), by1 = (int)(bby >> 16);
    if (bx0 > bx1 || by0 > by1) return p;   // 3-sigma box empty: the disc alone
    p.ell = true;
    if ((bx1 - bx0) + (by1 - by0) <= PH_ROWS_MIN_SPAN) { p.full = true; return p; }
    const float R = g1.w, qc = g1.z, ax = g1.x, ay = g1.y;
    const float Rax = __fmul_rn(R, ax), Ray = __fmul_rn(R, ay);
    // g0 = (A00, A10, A01, A11)
    const float M00 = __fmaf_rn(g0.x, g0.x, __fmaf_rn(g0.y, g0.y, -__fmul_rn(Rax, ax)));
    const float M11 = __fmaf_rn(g0.z, g0.z, __fmaf_rn(g0.w, g0.w, -__fmul_rn(Ray, ay)));
    const float M01 = __fmaf_rn(g0.x, g0.z, __fmaf_rn(g0.y, g0.w, -__fmul_rn(Rax, ay)));
    const float t00 = __fmaf_rn(g0.x, g0.x, __fmaf_rn(g0.y, g0.y, __fmul_rn(Rax, ax)));
    const float t11 = __fmaf_rn(g0.z, g0.z, __fmaf_rn(g0.w, g0.w, __fmul_rn(Ray, ay)));
    const float det = __fmaf_rn(M00, M11, -__fmul_rn(M01, M01));
    // well-conditioned only: no cancellation in M00, M11 or det beyond 1e-3 of their terms
    if (!(M00 > __fmul_rn(1e-3f, t00)) || !(M11 > __fmul_rn(1e-3f, t11)) || !(det > __fmul_rn(1e-3f, __fmul_rn(M00, M11)))) {
        p.full = true;
        return p;
    }
    const float B0 = -__fmul_rn(Rax, qc), B1 = -__fmul_rn(Ray, qc), C = -__fmul_rn(__fmul_rn(R, qc), qc);
    const float idet = bin_rcp(det);
    const float sx = __fmul_rn(__fmaf_rn(M01, B1, -__fmul_rn(M11, B0)), idet);
    const float sy = __fmul_rn(__fmaf_rn(M01, B0, -__fmul_rn(M00, B1)), idet);
    // slack: 4e-3 R w_max^2, w_max bounding |a2.d + qc| over the box (+1 px)
    const float wx = fmaxf(fabsf(__fsub_rn((float)bx0 - 0.5f, p.cx)), fabsf(__fsub_rn((float)bx1 + 1.5f, p.cx)));
    const float wy = fmaxf(fabsf(__fsub_rn((float)by0 - 0.5f, p.cy)), fabsf(__fsub_rn((float)by1 + 1.5f, p.cy)));
    const float wmax = __fmaf_rn(fabsf(ax), wx, __fmaf_rn(fabsf(ay), wy, fabsf(qc)));
    const float tol = __fmul_rn(__fmul_rn(4e-3f, R), __fmul_rn(wmax, wmax));
    // K = -Q(s) + tol, Q(s) = B.s + C
    const float K = __fsub_rn(tol, __fmaf_rn(B0, sx, __fmaf_rn(B1, sy, C)));
    if (!(K > 0.f) || !isfinite(K) || !isfinite(sx) || !isfinite(sy)) {
        p.full = true;
        return p;
    }
    p.sx = sx; p.sy = sy; p.M00 = M00; p.M01 = M01; p.M11 = M11; p.det = det; p.K = K;
    p.hx = bin_sqrt(__fmul_rn(__fmul_rn(K, M11), idet));
    p.hy = bin_sqrt(__fmul_rn(__fmul_rn(K, M00), idet));
    p.ul = bin_sqrt(__fmul_rn(K, bin_rcp(__fmul_rn(det, M11))));
    return p;
}

// Columns of tile row ty (inclusive [t0, t1], empty if t0 > t1), clipped to
// the rect columns [rx0, rx1].  W, H image size; tw, th tile size; mtw the
// exact-division multiplier of tw (DevSensor::mtw).
__device__ __forceinline__ void ph_row_tiles(const PhRows &p, int ty, int rx0, int rx1, int W, int H, int tw, int th,
                                             uint32_t mtw, int &t0, int &t1) {
    if (p.full) { t0 = rx0; t1 = rx1; return; }
    const float inf = __int_as_float(0x7f800000);
    float xl = inf, xh = -inf;
    const int py0 = ty * th, py1 = min(py0 + th, H) - 1;   // pixel rows of the tile row
    // band of pixel-centre y, relative to c, widened by 0.01 px
    const float Y0 = __fsub_rn(__fsub_rn((float)py0 + 0.5f, p.cy), 0.01f);
    const float Y1 = __fadd_rn(__fsub_rn((float)py1 + 0.5f, p.cy), 0.01f);
    if (p.ell && Y1 >= __fsub_rn(p.sy, p.hy) && Y0 <= __fadd_rn(p.sy, p.hy)) {
        const float iM00 = bin_rcp(p.M00);
        // leftmost point at y = sy + M01 ul, rightmost at y = sy - M01 ul
        const float yl = __fmaf_rn(p.M01, p.ul, p.sy), yr = __fmaf_rn(-p.M01, p.ul, p.sy);
        float a, b;
        if (yl >= Y0 && yl <= Y1) {
            a = __fsub_rn(p.sx, p.hx);
        } else {
            const float v = __fsub_rn(fminf(fmaxf(yl, Y0), Y1), p.sy);
            const float D = fmaxf(__fmaf_rn(p.M00, p.K, -__fmul_rn(__fmul_rn(p.det, v), v)), 0.f);
            a = __fmaf_rn(__fsub_rn(-__fmul_rn(p.M01, v), bin_sqrt(D)), iM00, p.sx);
        }
        if (yr >= Y0 && yr <= Y1) {
            b = __fadd_rn(p.sx, p.hx);
        } else {
            const float v = __fsub_rn(fminf(fmaxf(yr, Y0), Y1), p.sy);
            const float D = fmaxf(__fmaf_rn(p.M00, p.K, -__fmul_rn(__fmul_rn(p.det, v), v)), 0.f);
            b = __fmaf_rn(__fadd_rn(-__fmul_rn(p.M01, v), bin_sqrt(D)), iM00, p.sx);
        }
        // 1e-3 of the half width + 0.01 px: the interval's own fp32 rounding
        const float mg = __fmaf_rn(1e-3f, p.hx, 0.01f);
        xl = __fsub_rn(a, mg);
        xh = __fadd_rn(b, mg);
    }
    {   // low-pass disc about c
        const float v = Y0 > 0.f ? Y0 : (Y1 < 0.f ? Y1 : 0.f);
        const float rem = __fsub_rn(p.r2, __fmul_rn(v, v));
        if (rem >= 0.f) {
            const float h = __fadd_rn(bin_sqrt(rem), 0.01f);
            xl = fminf(xl, -h);
            xh = fmaxf(xh, h);
        }
    }
    t0 = 1; t1 = 0;
    if (!(xl <= xh)) return;
    // pixel columns whose centre i + 0.5 lies in [c + xl, c + xh]
    const float i0 = ceilf(fmaxf(__fsub_rn(__fadd_rn(p.cx, xl), 0.5f), -1.f));
    const float i1 = floorf(fminf(__fsub_rn(__fadd_rn(p.cx, xh), 0.5f), (float)W));
    const int c0 = max((int)i0, 0), c1 = min((int)i1, W - 1);
    if (c0 > c1) return;
    const int a0 = (int)(mtw ? __umulhi((uint32_t)c0, mtw) : (uint32_t)c0);
    const int a1 = (int)(mtw ? __umulhi((uint32_t)c1, mtw) : (uint32_t)c1);
    t0 = max(a0, rx0);
    t1 = min(a1, rx1);
}


// ---------------------------------------------------------------- LiDAR
// Exact tile test of a LiDAR record (Eq. 5 rays).  With the
// record's U, V, N (U.m = V.m = 0, det = N.m) the support test of a ray
// direction d is homogeneous: (U.d)^2 + (V.d)^2 <= R (N.d)^2.  A tile is one
// beam row (elevation theta) and tw consecutive azimuth columns; its rays lie
// on the arc phi in [phi0 - h, phi0 + h] of the cone of elevation theta.  In
// the gnomonic plane of the central ray d0 (d = d0 + x e1 + y e2, e1 the
// azimuth tangent, e2 the elevation tangent) the arc lies inside the
// rectangle |x| <= sin h cos(theta) / w, y between 0 and
// sin(theta) cos(theta) (1 - cos h) / w (w = cos^2(theta) cos h +
// sin^2(theta)), widened by 4e-6 for the fp32 angles, and the support test is
// a quadratic Q(x, y) <= 0: the tile can hold a contributing ray only if the
// minimum of Q over the rectangle (exact: the interior stationary point when
// positive definite, else the edges' 1-D minima) is <= tol, a slack of 1e-4
// of the magnitudes |U|^2 |e|^2 the fp32 evaluations (this one and the
// compositor's) see.  Evaluated once per (surfel, tile) by k_project, which
// stores a tile mask over the rect.
__device__ __forceinline__ float quad_min_rect(float qxx, float qxy, float qyy, float qx, float qy, float q0,
                                               float X0, float X1, float Y0, float Y1) {
    auto Q = [&](float x, float y) {
        return fmaf(x, fmaf(qxx, x, 2.f * fmaf(qxy, y, qx)), fmaf(y, fmaf(qyy, y, 2.f * qy), q0));
    };
    float m = fminf(fminf(Q(X0, Y0), Q(X1, Y0)), fminf(Q(X0, Y1), Q(X1, Y1)));
    if (qxx > 0.f) {   // edges y = Y0, Y1: vertex of the 1-D quadratic in x
        const float i = bin_rcp(qxx);
        m = fminf(m, Q(fminf(fmaxf(-fmaf(qxy, Y0, qx) * i, X0), X1), Y0));
        m = fminf(m, Q(fminf(fmaxf(-fmaf(qxy, Y1, qx) * i, X0), X1), Y1));
    }
    if (qyy > 0.f) {   // edges x = X0, X1
        const float i = bin_rcp(qyy);
        m = fminf(m, Q(X0, fminf(fmaxf(-fmaf(qxy, X0, qy) * i, Y0), Y1)));
        m = fminf(m, Q(X1, fminf(fmaxf(-fmaf(qxy, X1, qy) * i, Y0), Y1)));
    }
    const float det = fmaf(qxx, qyy, -qxy * qxy);
    if (qxx > 0.f && det > 0.f) {   // interior minimum
        const float id = bin_rcp(det);
        const float sx = (qxy * qy - qyy * qx) * id, sy = (qxy * qx - qxx * qy) * id;
        if (sx >= X0 && sx <= X1 && sy >= Y0 && sy <= Y1) m = fminf(m, Q(sx, sy));
    }
    return m;
}

// Per-record quantities of the tile test.
struct LiRec {
    float U[3], V[3], N[3], m[3], R, mag;   // mag = |U|^2 + |V|^2 + R |N|^2
};

__device__ __forceinline__ LiRec li_rec(const float *g) {
    LiRec r;
    for (int k = 0; k < 3; ++k) {
        r.U[k] = g[RY_U + k]; r.V[k] = g[RY_V + k]; r.N[k] = g[RY_N + k];
        r.m[k] = g[RY_MH + k] + g[RY_ML + k];
    }
    r.R = g[RY_RCUT3];
    auto d2 = [](const float a[3]) { return fmaf(a[0], a[0], fmaf(a[1], a[1], a[2] * a[2])); };
    r.mag = d2(r.U) + d2(r.V) + r.R * d2(r.N);
    return r;
}

// Azimuth trig of LiDAR tile column tc (< ntx): centre angle phi0 and half
// arc h of its rays; x = (sin phi0, cos phi0, sin h, cos h), or h >= 0.5
// (no gnomonic bound: every tile hits) flagged by x.w = 2.
__device__ __forceinline__ float4 li_col_trig(const DevSensor &se, int tc) {
    const int j0 = tc * se.tw, j1 = min(j0 + se.tw, se.width) - 1;
    const float step = se.az_step;
    const float h = 0.5f * (float)(j1 - j0) * step;
    if (!(h < 0.5f)) return make_float4(0.f, 1.f, 0.f, 2.f);
    const float phi0 = se.az0 + 0.5f * (float)(j0 + j1) * step;
    float sp, cp, sh, ch;
    sincosf(phi0, &sp, &cp);
    sincosf(h, &sh, &ch);
    return make_float4(sp, cp, sh, ch);
}

// Can a ray of the LiDAR tile with column trig `ct4` (li_col_trig) in the beam
// row of elevation sine / cosine (st, ct) lie in the support of the record?
__device__ __forceinline__ bool li_tile_hits(const LiRec &q, float4 ct4, float st, float ct) {
    if (ct4.w > 1.5f) return true;
    const float sp = ct4.x, cp = ct4.y, sh = ct4.z, ch = ct4.w;
    const float d0[3] = {ct * cp, ct * sp, st};
    const float e1[3] = {-sp, cp, 0.f};
    const float e2[3] = {-st * cp, -st * sp, ct};
    const float w = fmaf(ct * ct, ch, st * st);
    if (!(w > 0.1f)) return true;
    const float iw = bin_rcp(w);
    const float X = fmaf(ct * sh, iw, 4e-6f);
    const float Yv = st * ct * (1.f - ch) * iw;
    const float Y0 = fminf(Yv, 0.f) - 4e-6f, Y1 = fmaxf(Yv, 0.f) + 4e-6f;
    auto dot = [](const float a[3], const float b[3]) { return fmaf(a[0], b[0], fmaf(a[1], b[1], a[2] * b[2])); };
    const float u0 = dot(q.U, d0), u1 = dot(q.U, e1), u2 = dot(q.U, e2);
    const float v0 = dot(q.V, d0), v1 = dot(q.V, e1), v2 = dot(q.V, e2);
    const float n0 = dot(q.N, d0), n1 = dot(q.N, e1), n2 = dot(q.N, e2);
    const float R = q.R;
    const float qxx = fmaf(u1, u1, fmaf(v1, v1, -R * n1 * n1));
    const float qyy = fmaf(u2, u2, fmaf(v2, v2, -R * n2 * n2));
    const float qxy = fmaf(u1, u2, fmaf(v1, v2, -R * n1 * n2));
    const float qx = fmaf(u0, u1, fmaf(v0, v1, -R * n0 * n1));
    const float qy = fmaf(u0, u2, fmaf(v0, v2, -R * n0 * n2));
    const float q0 = fmaf(u0, u0, fmaf(v0, v0, -R * n0 * n0));
    const float dm = bin_sqrt((d0[0] - q.m[0]) * (d0[0] - q.m[0]) + (d0[1] - q.m[1]) * (d0[1] - q.m[1]) +
                              (d0[2] - q.m[2]) * (d0[2] - q.m[2]));
    const float ext = dm + X + fmaxf(Y1, -Y0) + 1e-3f;
    const float tol = 1e-4f * q.mag * ext * ext;
    const float mn = quad_min_rect(qxx, qxy, qyy, qx, qy, q0, -X, X, Y0, Y1);
    return !(mn > tol);   // NaN: conservative
}

}  // namespace gsr
