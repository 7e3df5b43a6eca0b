// project.cu -- gs_project kernels: per-surfel projection (Eq. 1,
// P:81-89; SH colour and low-pass bound; attributes) and the
// visible-surfel compaction / pair count (single-pass look-back scan).
//
// One thread per surfel.  Quantities whose rounding the compositing kernels
// would amplify (sensor-frame centre, projected centre, centre direction,
// intersection rows) are formed in fp64 and rounded once (hi+lo where the
// kernels need more than fp32), so that the per-pair fp32 arithmetic only
// sees well-conditioned, centre-relative values.
#include <math.h>

#include <algorithm>

#include "gsr_internal.cuh"
#include "scan.cuh"
#include "binning.cuh"

namespace gsr {

// ------------------------------------------------------------------ helpers
// Pinned-order sensor-frame coordinate (DESIGN reading R9): every operation
// an IEEE-rounded fp64 op on exactly promoted fp32 values, no contraction.
__device__ __forceinline__ double pinned_row(const float *Rr, float tk, float mx, float my,
                                             float mz) {
    const double a = __dmul_rn((double)Rr[0], (double)mx);
    const double b = __dmul_rn((double)Rr[1], (double)my);
    const double c = __dmul_rn((double)Rr[2], (double)mz);
    return __dadd_rn(__dadd_rn(__dadd_rn(a, b), c), (double)tk);
}

// Pixel-space box in fp32: its points are rounded once from fp64 (or formed in
// fp32 from fp64 operands) -- errors of a few 1e-7 relative, far inside the
// 1e-3 px + 1e-6 |x| margin of box_to_tiles.
struct Box {
    float x0, x1, y0, y1;
    __device__ void init() { x0 = y0 = __int_as_float(0x7f800000); x1 = y1 = -__int_as_float(0x7f800000); }
    __device__ void add(float x, float y) {
        x0 = fminf(x0, x); x1 = fmaxf(x1, x);
        y0 = fminf(y0, y); y1 = fmaxf(y1, y);
    }
};

__device__ __forceinline__ double kb_theta_d(const DevSensor &se, double th) {
    const double t2 = th * th;
    return th * (1.0 + t2 * ((double)se.k[0] + t2 * ((double)se.k[1] + t2 * ((double)se.k[2] + t2 * (double)se.k[3]))));
}

// fisheye projection of a sensor-frame point (equidistant Kannala-Brandt)
__device__ __forceinline__ void fisheye_project(const DevSensor &se, const double m[3], double &px,
                                                double &py) {
    const double rxy = sqrt(m[0] * m[0] + m[1] * m[1]);
    const double th = atan2(rxy, m[2]);
    const double td = kb_theta_d(se, th);
    if (rxy > 0.0) {
        const double q = td / rxy;
        px = (double)se.cx + (double)se.fx * q * m[0];
        py = (double)se.cy + (double)se.fy * q * m[1];
    } else {
        px = se.cx;
        py = se.cy;
    }
}

// cylindrical projection (Eq. 4, reading R20) of a sensor-frame point: column
// from the azimuth about the camera y axis, row from y / sqrt(x^2 + z^2)
__device__ __forceinline__ void cylinder_project(const DevSensor &se, const double m[3], double &px,
                                                 double &py) {
    const double rho = sqrt(m[0] * m[0] + m[2] * m[2]);
    px = (double)se.cx + (double)se.fx * atan2(m[0], m[2]);
    const double t = rho > 0.0 ? m[1] / rho : (m[1] >= 0.0 ? 1e12 : -1e12);
    py = (double)se.cy + (double)se.fy * fmin(fmax(t, -1e12), 1e12);
}

// Pixel-space bound of the pinhole 3-sigma disk clipped to z >= near:
// extremes of the linear-fractional x = X/Z over {u^2+v^2 <= R^2, Z >= near}
// lie at the circle's stationary points (A c + B s + C = 0) or at the ends of
// the chord Z = near.
__device__ void pinhole_disk_bound(const DevSensor &se, double nearp, const double mu[3],
                                   const double a[3], const double b[3], Box &box) {
    auto add_pt = [&](double c, double s) {
        const double X = mu[0] + c * a[0] + s * b[0];
        const double Y = mu[1] + c * a[1] + s * b[1];
        const double Z = mu[2] + c * a[2] + s * b[2];
        if (Z >= nearp * (1.0 - 1e-9)) {
            // the sum above in fp64 (cancellation); the projection of the point in fp32
            const float iz = __fdividef(1.f, (float)fmax(Z, nearp * (1.0 - 1e-9)));   // 2 ulp: margins cover it
            box.add(fmaf(se.fx * (float)X, iz, se.cx), fmaf(se.fy * (float)Y, iz, se.cy));
        }
    };
    auto solve = [&](double A, double B, double C, bool strict) {
        const double rr = A * A + B * B;
        if (!(rr > 0.0)) return;
        double disc = rr - C * C;
        if (strict && !(disc > 0.0)) return;
        disc = sqrt(fmax(disc, 0.0));
        const double irr = 1.0 / rr;
        add_pt((-A * C + B * disc) * irr, (-B * C - A * disc) * irr);
        add_pt((-A * C - B * disc) * irr, (-B * C + A * disc) * irr);
    };
    add_pt(0.0, 0.0);
    add_pt(1.0, 0.0);
    for (int ax = 0; ax < 2; ++ax) {
        const double a0 = mu[ax], a1 = a[ax], a2 = b[ax];
        const double b0 = mu[2], b1 = a[2], b2 = b[2];
        solve(a2 * b0 - a0 * b2, a0 * b1 - a1 * b0, a2 * b1 - a1 * b2, false);
    }
    solve(a[2], b[2], mu[2] - nearp, true);   // chord on the near plane
}

// n / d from m = ceil(2^32 / d) (m == 0 encodes d == 1, whose m does not fit)
__device__ __forceinline__ uint32_t tdiv(uint32_t n, uint32_t m) { return m ? __umulhi(n, m) : n; }

// pixel range [i0,i1] -> tile range; returns false if empty
__device__ __forceinline__ bool box_to_tiles(const Box &bx, int W, int H, uint32_t mtw, uint32_t mth,
                                             int &tx0, int &ty0, int &tx1, int &ty1, int pb[4]) {
    const float m = 1e-3f;
    float x0 = bx.x0 - m - 1e-6f * fabsf(bx.x0), x1 = bx.x1 + m + 1e-6f * fabsf(bx.x1);
    float y0 = bx.y0 - m - 1e-6f * fabsf(bx.y0), y1 = bx.y1 + m + 1e-6f * fabsf(bx.y1);
    if (!(x0 <= x1) || !(y0 <= y1)) {   // NaN: whole image (conservative)
        x0 = y0 = -1e30f; x1 = y1 = 1e30f;
    }
    // clamp before the int conversion (|x| may be huge or infinite)
    const float i0 = ceilf(fmaxf(x0 - 0.5f, -1.f)), i1 = floorf(fminf(x1 - 0.5f, (float)W));
    const float j0 = ceilf(fmaxf(y0 - 0.5f, -1.f)), j1 = floorf(fminf(y1 - 0.5f, (float)H));
    const int ci0 = max((int)i0, 0), ci1 = min((int)i1, W - 1);
    const int cj0 = max((int)j0, 0), cj1 = min((int)j1, H - 1);
    if (ci0 > ci1 || cj0 > cj1) return false;
    // n / d as umulhi(n, ceil(2^32 / d)): exact while n d < 2^32 (here n < 2^18, d <= 512):
    // the error n (m d - 2^32) / (d 2^32) < n / 2^32 < 1/d cannot cross an integer, as n mod d <= d - 1
    tx0 = (int)tdiv((uint32_t)ci0, mtw); tx1 = (int)tdiv((uint32_t)ci1, mtw);
    ty0 = (int)tdiv((uint32_t)cj0, mth); ty1 = (int)tdiv((uint32_t)cj1, mth);
    pb[0] = ci0; pb[1] = cj0; pb[2] = ci1; pb[3] = cj1;
    return true;
}

// SH colour, 3DGS real basis (degree <= 3), evaluated in fp32.
__device__ __forceinline__ void sh_colour(const float *sh, int deg, float x, float y, float z,
                                          float rgb[3]) {
    const float C0 = 0.28209479177387814f, C1 = 0.4886025119029199f;
    float b[16];
    b[0] = C0;
    int nb = 1;
    if (deg >= 1) {
        b[1] = -C1 * y; b[2] = C1 * z; b[3] = -C1 * x;
        nb = 4;
    }
    if (deg >= 2) {
        const float xx = x * x, yy = y * y, zz = z * z;
        b[4] = 1.0925484305920792f * x * y;
        b[5] = -1.0925484305920792f * y * z;
        b[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
        b[7] = -1.0925484305920792f * x * z;
        b[8] = 0.5462742152960396f * (xx - yy);
        nb = 9;
        if (deg >= 3) {
            b[9] = -0.5900435899266435f * y * (3.0f * xx - yy);
            b[10] = 2.890611442640554f * x * y * z;
            b[11] = -0.4570457994644658f * y * (4.0f * zz - xx - yy);
            b[12] = 0.3731763325901154f * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
            b[13] = -0.4570457994644658f * x * (4.0f * zz - xx - yy);
            b[14] = 1.445305721320277f * z * (xx - yy);
            b[15] = -0.5900435899266435f * x * (xx - 3.0f * yy);
            nb = 16;
        }
    }
    float r = 0.f, g = 0.f, bl = 0.f;
    if (deg == 3) {   // 48 coefficients = 12 aligned float4 loads (sh is 16-byte aligned)
        float c[48];
        const float4 *s4 = reinterpret_cast<const float4 *>(sh);
#pragma unroll
        for (int k = 0; k < 12; ++k) {
            const float4 v = __ldg(s4 + k);
            c[4 * k] = v.x; c[4 * k + 1] = v.y; c[4 * k + 2] = v.z; c[4 * k + 3] = v.w;
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            r = fmaf(b[j], c[3 * j + 0], r);
            g = fmaf(b[j], c[3 * j + 1], g);
            bl = fmaf(b[j], c[3 * j + 2], bl);
        }
    } else {
        for (int j = 0; j < nb; ++j) {
            r = fmaf(b[j], __ldg(sh + 3 * j + 0), r);
            g = fmaf(b[j], __ldg(sh + 3 * j + 1), g);
            bl = fmaf(b[j], __ldg(sh + 3 * j + 2), bl);
        }
    }
    rgb[0] = fmaxf(r + 0.5f, 0.f);
    rgb[1] = fmaxf(g + 0.5f, 0.f);
    rgb[2] = fmaxf(bl + 0.5f, 0.f);
}

__device__ __forceinline__ void cross3(const double a[3], const double b[3], double o[3]) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}
__device__ __forceinline__ double dot3(const double a[3], const double b[3]) {
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

// LiDAR: rows whose beam elevation sine lies in [lo, hi] (table strictly decreasing)
// (sb: the sensor's sine table staged in shared memory -- divergent lookups
// into the kernel-parameter bank would serialise across the warp)
__device__ __forceinline__ bool beam_rows(const float *sb, int nbeams, double lo, double hi, int &r0, int &r1) {
    // first row with sin(beam) <= hi
    int a = 0, b = nbeams;
    while (a < b) {
        const int m = (a + b) >> 1;
        if ((double)sb[m] <= hi) b = m; else a = m + 1;
    }
    r0 = a;
    // last row with sin(beam) >= lo
    a = 0; b = nbeams;
    while (a < b) {
        const int m = (a + b) >> 1;
        if ((double)sb[m] < lo) b = m; else a = m + 1;
    }
    r1 = a - 1;
    return r0 <= r1;
}

// Angular box of a surfel's support as seen from the sensor origin:
// elevation above the sensor's xy plane in [el_lo, el_hi]; azimuth about z in
// azc + [daz_lo, daz_hi] unless all_az.
struct AngBox {
    double el_lo, el_hi, azc, daz_lo, daz_hi;
    double s_lo, s_hi;      // sines of el_lo, el_hi (LiDAR rows are found by sine, no asin)
    bool all_az;
};

// Range of the linear-fractional f(c,s) = (n0 + n1 c + n2 s)/(d0 + d1 c + d2 s)
// over the unit disk (denominator > 0 on it): the extremes lie on the circle
// at the two roots of A c + B s + C = 0.
// fp32 instantiation: fast division (2 ulp; its callers' margins are ~10x wider)
__device__ __forceinline__ double lf_div(double a, double b) { return a / b; }
__device__ __forceinline__ float lf_div(float a, float b) { return __fdividef(a, b); }

template <typename T>
__device__ void lf_range(T n0, T n1, T n2, T d0, T d1, T d2, T &lo, T &hi) {
    lo = hi = lf_div(n0, d0);
    const T A = n2 * d0 - n0 * d2, B = n0 * d1 - n1 * d0, C = n2 * d1 - n1 * d2;
    const T rr = A * A + B * B;
    if (rr > T(0)) {
        const T q = sqrt(fmax(rr - C * C, T(0)));
        const T irr = T(1) / rr;
        const T cs[2][2] = {{(-A * C + B * q) * irr, (-B * C - A * q) * irr},
                            {(-A * C - B * q) * irr, (-B * C + A * q) * irr}};
        for (int k = 0; k < 2; ++k) {
            const T f = lf_div(n0 + n1 * cs[k][0] + n2 * cs[k][1], d0 + d1 * cs[k][0] + d2 * cs[k][1]);
            lo = fmin(lo, f);
            hi = fmax(hi, f);
        }
    }
    for (int k = 0; k < 4; ++k) {   // safety points on the circle
        const T c = k == 0 ? T(1) : (k == 1 ? T(-1) : T(0)), s = k == 2 ? T(1) : (k == 3 ? T(-1) : T(0));
        const T f = lf_div(n0 + n1 * c + n2 * s, d0 + d1 * c + d2 * s);
        lo = fmin(lo, f);
        hi = fmax(hi, f);
    }
}

// Exact-extreme bound of the disk {mu + c a + s b : c^2+s^2 <= 1} through the
// gnomonic projection at the centre direction m (lines of the projection are
// great circles): xi = P.e_az / P.m, eta = P.e_el / P.m are linear-fractional
// in (c,s); the direction m + xi e_az + eta e_el then bounds elevation and
// azimuth with numerator/denominator interval arithmetic.  Returns false if
// the disk reaches the plane P.m = 0 or the centre is at the pole.
__device__ bool angular_box_disk(const double mu[3], const double a[3], const double b[3], AngBox &ab,
                                 bool need_el) {
    const double r = sqrt(dot3(mu, mu));
    const double m[3] = {mu[0] / r, mu[1] / r, mu[2] / r};
    const double rho = sqrt(m[0] * m[0] + m[1] * m[1]);
    if (!(rho > 1e-6)) return false;
    const double eaz[3] = {-m[1] / rho, m[0] / rho, 0.0};
    const double eel[3] = {-m[2] * m[0] / rho, -m[2] * m[1] / rho, rho};
    const double d1 = dot3(a, m), d2 = dot3(b, m);
    if (!(r - sqrt(d1 * d1 + d2 * d2) > 1e-3 * r)) return false;
    double xl, xh, yl, yh;
    lf_range(0.0, dot3(a, eaz), dot3(b, eaz), r, d1, d2, xl, xh);
    lf_range(0.0, dot3(a, eel), dot3(b, eel), r, d1, d2, yl, yh);
    const double mg = 1e-9;
    xl -= mg; xh += mg; yl -= mg; yh += mg;
    // elevation: sin(el) = (m_z + eta*rho) / sqrt(1 + xi^2 + eta^2)
    const double x2lo = (xl <= 0.0 && xh >= 0.0) ? 0.0 : fmin(xl * xl, xh * xh), x2hi = fmax(xl * xl, xh * xh);
    const double y2lo = (yl <= 0.0 && yh >= 0.0) ? 0.0 : fmin(yl * yl, yh * yh), y2hi = fmax(yl * yl, yh * yh);
    const double den_lo = sqrt(1.0 + x2lo + y2lo), den_hi = sqrt(1.0 + x2hi + y2hi);
    const double nlo = m[2] + yl * rho, nhi = m[2] + yh * rho;
    const double shi = nhi > 0.0 ? nhi / den_lo : nhi / den_hi;
    const double slo = nlo > 0.0 ? nlo / den_hi : nlo / den_lo;
    ab.s_hi = fmin(1.0, shi) + 1e-9;
    ab.s_lo = fmax(-1.0, slo) - 1e-9;
    if (need_el) {
        ab.el_hi = asin(fmin(1.0, shi)) + 1e-7;
        ab.el_lo = asin(fmax(-1.0, slo)) - 1e-7;
    }
    // azimuth: tan(daz) = xi / (rho - eta*m_z); fp32 arctangents, 5e-6 rad margin
    const double t1 = yl * m[2], t2 = yh * m[2];
    const double Dlo = rho - fmax(t1, t2), Dhi = rho - fmin(t1, t2);
    ab.azc = (double)atan2f((float)m[1], (float)m[0]);
    ab.all_az = !(Dlo > 1e-9) || ab.s_hi >= 1.0 || ab.s_lo <= -1.0;
    if (!ab.all_az) {
        ab.daz_hi = (double)atanf((float)(xh > 0.0 ? xh / Dlo : xh / Dhi)) + 5e-6;
        ab.daz_lo = (double)atanf((float)(xl < 0.0 ? xl / Dlo : xl / Dhi)) - 5e-6;
    }
    return true;
}

// The same bound in fp32 for well-conditioned disks (the disk keeps at least
// 5% of the centre range away from the plane P.m = 0, so no quantity below is
// amplified by more than ~20x), widened by margins far above fp32 error:
// 1e-6 on the gnomonic coordinates, 4e-6 on the elevation sines, 8e-6 rad on
// azimuth.  Only used for binning (it must contain the support; it need not
// be tight to the last ulp).  Returns false -> use the fp64 version.
__device__ bool angular_box_disk_f(const double mu[3], const double a_[3], const double b_[3], AngBox &ab) {
    const double rd = sqrt(dot3(mu, mu));
    const double ird = 1.0 / rd;
    const float r = (float)rd;
    const float m[3] = {(float)(mu[0] * ird), (float)(mu[1] * ird), (float)(mu[2] * ird)};
    const float a[3] = {(float)a_[0], (float)a_[1], (float)a_[2]}, b[3] = {(float)b_[0], (float)b_[1], (float)b_[2]};
    const float rho = sqrtf(m[0] * m[0] + m[1] * m[1]);
    if (!(rho > 1e-3f)) return false;
    const float irho = 1.f / rho;
    const float eaz[3] = {-m[1] * irho, m[0] * irho, 0.f};
    const float eel[3] = {-m[2] * m[0] * irho, -m[2] * m[1] * irho, rho};
    const float d1 = a[0] * m[0] + a[1] * m[1] + a[2] * m[2], d2 = b[0] * m[0] + b[1] * m[1] + b[2] * m[2];
    if (!(r - sqrtf(d1 * d1 + d2 * d2) > 0.05f * r)) return false;
    float xl, xh, yl, yh;
    lf_range(0.f, a[0] * eaz[0] + a[1] * eaz[1], b[0] * eaz[0] + b[1] * eaz[1], r, d1, d2, xl, xh);
    lf_range(0.f, a[0] * eel[0] + a[1] * eel[1] + a[2] * eel[2], b[0] * eel[0] + b[1] * eel[1] + b[2] * eel[2], r,
             d1, d2, yl, yh);
    const float mgx = 1e-6f * (1.f + fabsf(xl) + fabsf(xh)), mgy = 1e-6f * (1.f + fabsf(yl) + fabsf(yh));
    xl -= mgx; xh += mgx; yl -= mgy; yh += mgy;
    const float x2lo = (xl <= 0.f && xh >= 0.f) ? 0.f : fminf(xl * xl, xh * xh), x2hi = fmaxf(xl * xl, xh * xh);
    const float y2lo = (yl <= 0.f && yh >= 0.f) ? 0.f : fminf(yl * yl, yh * yh), y2hi = fmaxf(yl * yl, yh * yh);
    const float den_lo = sqrtf(1.f + x2lo + y2lo), den_hi = sqrtf(1.f + x2hi + y2hi);
    const float nlo = m[2] + yl * rho, nhi = m[2] + yh * rho;
    const float shi = nhi > 0.f ? nhi / den_lo : nhi / den_hi;
    const float slo = nlo > 0.f ? nlo / den_hi : nlo / den_lo;
    ab.s_hi = (double)fminf(1.f, shi) + 4e-6;
    ab.s_lo = (double)fmaxf(-1.f, slo) - 4e-6;
    const float t1 = yl * m[2], t2 = yh * m[2];
    const float Dlo = rho - fmaxf(t1, t2), Dhi = rho - fminf(t1, t2);
    ab.azc = (double)atan2f(m[1], m[0]);
    ab.all_az = !(Dlo > 1e-4f) || ab.s_hi >= 1.0 || ab.s_lo <= -1.0;
    if (!ab.all_az) {
        ab.daz_hi = (double)atanf(xh > 0.f ? xh / Dlo : xh / Dhi) + 8e-6;
        ab.daz_lo = (double)atanf(xl < 0.f ? xl / Dlo : xl / Dhi) - 8e-6;
    }
    return true;
}

// Sphere-cap fallback: all directions within beta of the centre direction.
__device__ void angular_box_cap(const double m[3], double beta, AngBox &ab) {
    const double elc = asin(fmin(1.0, fmax(-1.0, m[2])));
    ab.el_lo = elc - beta;
    ab.el_hi = elc + beta;
    ab.s_lo = ab.el_lo <= -0.5 * M_PI ? -1.0 : sin(ab.el_lo) - 1e-9;
    ab.s_hi = ab.el_hi >= 0.5 * M_PI ? 1.0 : sin(ab.el_hi) + 1e-9;
    ab.azc = atan2(m[1], m[0]);
    ab.all_az = beta >= 0.5 * M_PI - fabs(elc);
    if (!ab.all_az) {
        const double sb = sin(beta) / cos(elc);
        if (sb >= 1.0) ab.all_az = true;
        else { ab.daz_hi = asin(sb); ab.daz_lo = -ab.daz_hi; }
    }
}

// ------------------------------------------------------------------ cull
// Per-sensor constants of cull_one (the same fp32 expressions it used to
// evaluate per surfel -- IEEE divisions and square roots -- computed once per
// thread: k_cull<pinhole> 3080 -> 1650 SASS instructions per 8-surfel thread).
struct CullConst {
    float kR;                       // 1.001 sqrt(support 1.0001 + 1e-4)
    float xl, xr, yl, yr;           // frustum side slopes with the pixel margin (pinhole)
    float nxl, nxr, nyl, nyr;       // sqrt(1 + slope^2)
};
template <int KIND>
__device__ __forceinline__ CullConst make_cull_const(const DevSensor &se, const DevOpts &op) {
    CullConst c;
    c.kR = 1.001f * sqrtf(op.support * 1.0001f + 1e-4f);
    c.xl = c.xr = c.yl = c.yr = c.nxl = c.nxr = c.nyl = c.nyr = 0.f;
    if (KIND == GS_PINHOLE) {
        // margin: the low-pass disc radius sqrt(rcut) sigma (the same cut as k_project) + 1 px
        const float m = 1.f + sqrtf(op.support * 1.0001f + 1e-4f) * sqrtf(op.sigma2);
        c.xl = (-m - se.cx) / se.fx; c.xr = ((float)se.width + m - se.cx) / se.fx;
        c.yl = (-m - se.cy) / se.fy; c.yr = ((float)se.height + m - se.cy) / se.fy;
        c.nxl = sqrtf(1.f + c.xl * c.xl); c.nxr = sqrtf(1.f + c.xr * c.xr);
        c.nyl = sqrtf(1.f + c.yl * c.yl); c.nyr = sqrtf(1.f + c.yr * c.yr);
    }
    return c;
}

// Conservative cull ahead of the fp64 projection: a surfel is dropped when
// its centre fails the depth-key test (exact, the same pinned key as
// k_project) or when the sphere of radius 3.001 max(s_u, s_v) around its
// sensor-frame centre (which holds the 3-sigma support disk) lies outside
// the sensor's field of view widened by a margin (pinhole: the low-pass disc
// radius + 1 px beyond the image; fisheye: 0.15 rad beyond theta_max), or
// (LiDAR) when no beam's elevation lies in the elevation range of the support
// disk, bounded from its exact z-extent and horizontal distance range (+1e-4
// in sine).  fp32 arithmetic with margins well above its error; a culled
// surfel provably meets no sample ray, so this only skips work -- k_project
// takes every decision for the surfels that pass.  Passing surfels are compacted in index order
// (decoupled look-back); the others get the culled outputs here.
// sqrt.approx (2 ulp) for the cull's conservative bounds: every use below is
// compared with margins of 1e-4 (1 + r) m or 1 % -- far above 2 ulp.
__device__ __forceinline__ float sqrt_apx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// The cull's per-surfel inputs, loaded for a group of items before any of them
// is tested (the tests branch, and a load cannot move above a branch: loading
// inside cull_one left one surfel's loads in flight per thread).
struct CullIn {
    float mx, my, mz, o;
    float2 sc;
};
__device__ __forceinline__ CullIn cull_load(const DevSurfels &s, int64_t i) {
    CullIn in;
    in.mx = __ldg(s.means + 3 * i); in.my = __ldg(s.means + 3 * i + 1); in.mz = __ldg(s.means + 3 * i + 2);
    in.o = __ldg(s.opac + i);
    in.sc = __ldg(reinterpret_cast<const float2 *>(s.scales) + i);
    return in;
}

template <int KIND>
__device__ __forceinline__ bool cull_one(const DevSurfels &s, const DevSensor &se, const DevOpts &op,
                                         const CullConst &cc, const CullIn &in, int64_t i, uint32_t &keybits,
                                         const float *sb) {
    const float mx = in.mx, my = in.my, mz = in.mz;
    const float X = fmaf(se.R[0], mx, fmaf(se.R[1], my, fmaf(se.R[2], mz, se.t[0])));
    const float Y = fmaf(se.R[3], mx, fmaf(se.R[4], my, fmaf(se.R[5], mz, se.t[1])));
    const float Z = fmaf(se.R[6], mx, fmaf(se.R[7], my, fmaf(se.R[8], mz, se.t[2])));
    // conservative near-plane test in fp32: k_project applies the exact one (the pinned
    // fp64 key, reading R9) to the candidates; the margin covers the fp32 rounding here
    const float mag = fabsf(mx) + fabsf(my) + fabsf(mz) + fabsf(se.t[0]) + fabsf(se.t[1]) + fabsf(se.t[2]);
    const float nearm = op.near_plane - fmaf(1e-5f, mag, 1e-6f);
    const float keyf = KIND == GS_PINHOLE ? Z : sqrt_apx(fmaf(X, X, fmaf(Y, Y, Z * Z)));
    keybits = __float_as_uint(keyf);
    const float o = in.o;
    const float2 sc = in.sc;
    if (!(keyf >= nearm) || !(o > 0.f) || !(sc.x > 0.f) || !(sc.y > 0.f) || !isfinite(sc.x) ||
        !isfinite(sc.y))
        return false;
    const float R = cc.kR * fmaxf(sc.x, sc.y) + 1e-3f * (1.f + fabsf(X) + fabsf(Y) + fabsf(Z));
    if (!isfinite(X + Y + Z + R)) return true;   // let k_project decide
    if (KIND == GS_PINHOLE) {
        if ((X - cc.xl * Z) < -R * cc.nxl) return false;
        if ((cc.xr * Z - X) < -R * cc.nxr) return false;
        if ((Y - cc.yl * Z) < -R * cc.nyl) return false;
        if ((cc.yr * Z - Y) < -R * cc.nyr) return false;
        return true;
    }
    if (KIND == GS_FISHEYE_CYLINDRICAL) return true;   // no field-of-view pre-cull: k_project's box decides
    const float r = sqrt_apx(X * X + Y * Y + Z * Z);
    if (!(r > R * 1.01f)) return true;
    if (KIND == GS_FISHEYE_EQUIDISTANT) {
        const float beta = asinf(R / r);
        const float th = acosf(fminf(1.f, fmaxf(-1.f, Z / r)));
        return th - beta <= se.theta_max + 0.15f;
    }
    // LiDAR: elevation range of the support disk itself (a ground surfel seen at a
    // grazing angle is thin in elevation and usually falls between two beams).
    // Disk z-extent: mu_z +- Rr sqrt((s_u t_u,z)^2 + (s_v t_v,z)^2) (t_u, t_v in the
    // sensor frame); horizontal distance within rho_c +- Rr max(s_u, s_v); sines of
    // the extreme elevations from those, widened by 1e-4 (fp32 here); then some
    // beam's sine must lie in the range.
    const float4 q = __ldg(reinterpret_cast<const float4 *>(s.quats) + i);
    const float inq = rsqrtf(q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w);
    const float qw = q.x * inq, qx = q.y * inq, qy = q.z * inq, qz = q.w * inq;
    // world t_u, t_v = first two columns of the rotation; their sensor-frame z = row 2 of R_s times them
    const float tu0 = 1.f - 2.f * (qy * qy + qz * qz), tu1 = 2.f * (qx * qy + qw * qz), tu2 = 2.f * (qx * qz - qw * qy);
    const float tv0 = 2.f * (qx * qy - qw * qz), tv1 = 1.f - 2.f * (qx * qx + qz * qz), tv2 = 2.f * (qy * qz + qw * qx);
    const float az = se.R[6] * tu0 + se.R[7] * tu1 + se.R[8] * tu2;
    const float bz = se.R[6] * tv0 + se.R[7] * tv1 + se.R[8] * tv2;
    const float Rr = __fdividef(R, fmaxf(sc.x, sc.y));   // 1.001 sqrt(rcut) (+ the absolute margin, scaled)
    const float mg = 1e-4f * (1.f + r);
    const float hz = Rr * sqrt_apx((sc.x * az) * (sc.x * az) + (sc.y * bz) * (sc.y * bz)) + mg;
    const float rxy = sqrt_apx(X * X + Y * Y);
    const float rlo = rxy - R - mg, rhi = rxy + R + mg;
    if (!(rlo > 1e-3f * r)) return true;   // near the vertical axis: keep
    const float zlo = Z - hz, zhi = Z + hz;
    const float shi = zhi >= 0.f ? zhi * rsqrtf(zhi * zhi + rlo * rlo) : zhi * rsqrtf(zhi * zhi + rhi * rhi);
    const float slo = zlo >= 0.f ? zlo * rsqrtf(zlo * zlo + rhi * rhi) : zlo * rsqrtf(zlo * zlo + rlo * rlo);
    const float sh = shi + 1e-4f, sl = slo - 1e-4f;
    int lo = 0, hi = se.nbeams;   // first row with sin(beam) <= sh (table decreasing)
    while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if (sb[m] <= sh) hi = m; else lo = m + 1;
    }
    return lo < se.nbeams && sb[lo] >= sl;
}

// Block bounds (gs_cull_bounds): min / max of the finite centres and the
// largest finite scale of every SCAN_TILE consecutive surfels.  fminf / fmaxf
// drop NaNs; an infinite centre gives an infinite bound, which block_outside
// never rejects; a surfel with a NaN centre or a non-finite scale fails
// cull_one whatever its block says.
__global__ void __launch_bounds__(SCAN_THREADS) k_bounds(const float *__restrict__ means,
                                                         const float *__restrict__ scales, int64_t n,
                                                         float *__restrict__ bounds) {
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY}, sm = 0.f;
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        const int64_t i = base + j * SCAN_THREADS + threadIdx.x;
        if (i < n) {
            for (int k = 0; k < 3; ++k) {
                const float m = __ldg(means + 3 * i + k);
                lo[k] = fminf(lo[k], m);
                hi[k] = fmaxf(hi[k], m);
            }
            const float2 sc = __ldg(reinterpret_cast<const float2 *>(scales) + i);
            if (isfinite(sc.x)) sm = fmaxf(sm, sc.x);
            if (isfinite(sc.y)) sm = fmaxf(sm, sc.y);
        }
    }
    __shared__ float red[SCAN_THREADS / 32][7];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int o = 16; o; o >>= 1) {
        for (int k = 0; k < 3; ++k) {
            lo[k] = fminf(lo[k], __shfl_xor_sync(FULL_MASK, lo[k], o));
            hi[k] = fmaxf(hi[k], __shfl_xor_sync(FULL_MASK, hi[k], o));
        }
        sm = fmaxf(sm, __shfl_xor_sync(FULL_MASK, sm, o));
    }
    if (lane == 0) {
        for (int k = 0; k < 3; ++k) { red[warp][k] = lo[k]; red[warp][3 + k] = hi[k]; }
        red[warp][6] = sm;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < SCAN_THREADS / 32; ++w) {
            for (int k = 0; k < 3; ++k) {
                lo[k] = fminf(lo[k], red[w][k]);
                hi[k] = fmaxf(hi[k], red[w][3 + k]);
            }
            sm = fmaxf(sm, red[w][6]);
        }
        float *b = bounds + (size_t)blockIdx.x * 8;
        b[0] = lo[0]; b[1] = lo[1]; b[2] = lo[2]; b[3] = hi[0]; b[4] = hi[1]; b[5] = hi[2];
        b[6] = sm; b[7] = 0.f;
    }
}

// True when every surfel of the block fails cull_one<GS_PINHOLE>: the block's
// box of centres, widened by the largest support sphere of the block, lies
// behind the near plane or outside one frustum side.  Each test bounds the
// quantity cull_one compares (a linear function of the centre: centre value
// plus the box half-extents times the absolute coefficients) and rejects only
// with twice cull_one's own fp32 margin to spare; every comparison is false
// on a NaN, so a block with non-finite bounds is never rejected.
__device__ __forceinline__ bool block_outside(const float *__restrict__ bnd, const DevSensor &se,
                                              const DevOpts &op, const CullConst &cc) {
    const float4 b0 = __ldg(reinterpret_cast<const float4 *>(bnd)), b1 = __ldg(reinterpret_cast<const float4 *>(bnd) + 1);
    const float c[3] = {0.5f * (b0.x + b0.w), 0.5f * (b0.y + b1.x), 0.5f * (b0.z + b1.y)};
    // half extents, rounded up (the centre above is rounded too)
    const float h[3] = {(b0.w - b0.x) * 0.5000005f + 1e-6f * fabsf(c[0]), (b1.x - b0.y) * 0.5000005f + 1e-6f * fabsf(c[1]),
                        (b1.y - b0.z) * 0.5000005f + 1e-6f * fabsf(c[2])};
    if (!(h[0] >= 0.f) || !(h[1] >= 0.f) || !(h[2] >= 0.f)) return false;   // empty or non-finite block
    float Xc[3], Xe[3];
    for (int r = 0; r < 3; ++r) {
        Xc[r] = fmaf(se.R[3 * r], c[0], fmaf(se.R[3 * r + 1], c[1], fmaf(se.R[3 * r + 2], c[2], se.t[r])));
        Xe[r] = fabsf(se.R[3 * r]) * h[0] + fabsf(se.R[3 * r + 1]) * h[1] + fabsf(se.R[3 * r + 2]) * h[2];
    }
    // magnitude bound of any centre of the block in both frames (cull_one's margins scale with it)
    const float magw = fabsf(c[0]) + h[0] + fabsf(c[1]) + h[1] + fabsf(c[2]) + h[2] + fabsf(se.t[0]) + fabsf(se.t[1]) +
                       fabsf(se.t[2]);
    const float mags = fabsf(Xc[0]) + Xe[0] + fabsf(Xc[1]) + Xe[1] + fabsf(Xc[2]) + Xe[2];
    const float slack = 3e-3f * (1.f + mags) + 3e-5f * magw;   // > 2x cull_one's margins + this function's rounding
    // near plane: cull_one drops Z < near - (1e-5 mag + 1e-6)
    if (Xc[2] + Xe[2] < op.near_plane - slack) return true;
    const float R = cc.kR * b1.z + slack;   // >= every surfel's R
    // f(X) = a X + b Y + g Z over the block: f(Xc) + |a| Xe_x + |b| Xe_y + |g| Xe_z
    if ((Xc[0] - cc.xl * Xc[2]) + Xe[0] + fabsf(cc.xl) * Xe[2] < -R * cc.nxl - slack) return true;
    if ((cc.xr * Xc[2] - Xc[0]) + Xe[0] + fabsf(cc.xr) * Xe[2] < -R * cc.nxr - slack) return true;
    if ((Xc[1] - cc.yl * Xc[2]) + Xe[1] + fabsf(cc.yl) * Xe[2] < -R * cc.nyl - slack) return true;
    if ((cc.yr * Xc[2] - Xc[1]) + Xe[1] + fabsf(cc.yr) * Xe[2] < -R * cc.nyr - slack) return true;
    return false;
}

// Items whose inputs are loaded together, ahead of their tests (divides SCAN_ITEMS).  Measured on the
// Chunked frames (forward / side / LiDAR projection, ms): 1: 0.763 / 0.203 / 0.890, 2: 0.767 / 0.204 /
// 0.894, 4: 0.780 / 0.226 / 0.918, 8: 0.805 / 0.241 / 0.948 (32 -> 80 registers): occupancy hides the
// load latency better than the grouped loads do, so the default is 1.
#ifndef GSR_CULL_GROUP
#define GSR_CULL_GROUP 1
#endif
constexpr int CULL_GROUP = GSR_CULL_GROUP;
static_assert(SCAN_ITEMS % CULL_GROUP == 0, "cull group");
template <int KIND>
__global__ void __launch_bounds__(SCAN_THREADS) k_cull(DevSurfels s, const __grid_constant__ DevSensor se,
                                                       DevOpts op, short4 *__restrict__ rect,
                                                       uint32_t *__restrict__ keys, uint32_t *__restrict__ counts,
                                                       uint32_t *__restrict__ cand, unsigned long long *st_cand,
                                                       ProjHeader *hdr) {
    __shared__ uint32_t s_tile;
    __shared__ unsigned long long s_excl;
    __shared__ float sb[KIND == GS_LIDAR_SPINNING ? GS_MAX_BEAMS : 1];   // beam sines (LiDAR)
    if (threadIdx.x == 0) s_tile = atomicAdd(&hdr->cull_counter, 1u);
    if (KIND == GS_LIDAR_SPINNING)
        for (int k = threadIdx.x; k < se.nbeams; k += SCAN_THREADS) sb[k] = se.sbeam[k];
    __syncthreads();
    const uint32_t tile = s_tile;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // item j of thread t: base + j * SCAN_THREADS + t (coalesced); ranks in index order via per-round ballots
    const int64_t base = (int64_t)tile * SCAN_TILE;
    uint32_t flags = 0, cnt = 0;
    // hierarchical cull: a block wholly outside the frustum skips the per-surfel pass
    // (its surfels still get their zero counts and the tile its place in the look-back)
    const CullConst cc = make_cull_const<KIND>(se, op);
    const bool skip = KIND == GS_PINHOLE && s.bounds && block_outside(s.bounds + (size_t)tile * 8, se, op, cc);
#pragma unroll
    for (int j0 = 0; j0 < SCAN_ITEMS; j0 += CULL_GROUP) {
        CullIn in[CULL_GROUP];
#pragma unroll
        for (int g = 0; g < CULL_GROUP; ++g) {
            const int64_t i = base + (j0 + g) * SCAN_THREADS + threadIdx.x;
            if (i < s.n && !skip) in[g] = cull_load(s, i);
        }
#pragma unroll
        for (int g = 0; g < CULL_GROUP; ++g) {
            const int j = j0 + g;
            const int64_t i = base + j * SCAN_THREADS + threadIdx.x;
            if (i < s.n) {
                uint32_t kb;
                const bool c = !skip && cull_one<KIND>(s, se, op, cc, in[g], i, kb, sb);
                if (c) { flags |= 1u << j; ++cnt; }
                // every surfel gets a zero pair count here (coalesced); k_project writes
                // count, key and rect of every candidate.  Nothing reads the key or rect
                // of a culled surfel, so those are not written for it.
                counts[i] = 0;
            }
        }
    }
    // per round j: CTA-wide exclusive rank of this thread's item among the passing items of round j
    __shared__ unsigned long long s_round[SCAN_ITEMS * (SCAN_THREADS / 32)];   // [round][warp], 64 entries
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        const uint32_t b = __ballot_sync(FULL_MASK, (flags >> j) & 1u);
        if (lane == 0) s_round[j * (SCAN_THREADS / 32) + warp] = __popc(b);
    }
    __syncthreads();
    if (warp == 0) {
        const unsigned long long t0 = warp_excl_scan_smem(s_round, 32);
        const unsigned long long t1 = warp_excl_scan_smem(s_round + 32, 32);
        if (lane < 32) s_round[32 + lane] += t0;
        __syncwarp();
        const unsigned long long tot = t0 + t1;
        const unsigned long long e = lookback_warp_u64(st_cand, tile, tot);
        if (lane == 0) {
            s_excl = e;
            if (base + SCAN_TILE >= s.n) hdr->n_cand = (uint32_t)(e + tot);
        }
    }
    __syncthreads();
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        const uint32_t b = __ballot_sync(FULL_MASK, (flags >> j) & 1u);
        if ((flags >> j) & 1u) {
            const unsigned long long pos = s_excl + s_round[j * (SCAN_THREADS / 32) + warp] + __popc(b & lt);
            cand[pos] = (uint32_t)(base + j * SCAN_THREADS + threadIdx.x);
        }
    }
    (void)cnt;
}

// ------------------------------------------------------------------ projection
template <int KIND>
__device__ __forceinline__ void project_one(const DevSurfels &s, const DevSensor &se, const DevOpts &op,
                                            int64_t i, float *__restrict__ rec, short4 *__restrict__ rect,
                                            uint32_t *__restrict__ keys, uint32_t *__restrict__ counts,
                                            uint4 *__restrict__ rows, const float *sb) {
    if (KIND != GS_LIDAR_SPINNING && s.sh) {   // the SH block is read last: start it towards L2 now
        const int nc3 = (s.sh_degree + 1) * (s.sh_degree + 1) * 3;
        const char *p = reinterpret_cast<const char *>(s.sh + (size_t)i * nc3);
        for (int b = 0; b < nc3 * 4; b += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + b));
    }
    const float mx = __ldg(s.means + 3 * i), my = __ldg(s.means + 3 * i + 1),
                mz = __ldg(s.means + 3 * i + 2);
    double mu[3];
    mu[0] = pinned_row(se.R + 0, se.t[0], mx, my, mz);
    mu[1] = pinned_row(se.R + 3, se.t[1], mx, my, mz);
    mu[2] = pinned_row(se.R + 6, se.t[2], mx, my, mz);
    float keyf;
    if (KIND == GS_PINHOLE) {
        keyf = (float)mu[2];
    } else {
        keyf = (float)__dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(mu[0], mu[0]), __dmul_rn(mu[1], mu[1])),
                                           __dmul_rn(mu[2], mu[2])));
    }
    const float o = __ldg(s.opac + i);
    // opacity-aware support: alpha >= alpha_min needs rho <= 2 ln(o / alpha_min)
    float rc = op.support;
    if (op.alpha_min > 0.f) rc = fminf(rc, 2.0f * logf(__fdividef(o, op.alpha_min)));   // +1e-4 margin below
    const float rcut3 = rc * 1.0001f + 1e-4f;
    bool vis = (keyf >= op.near_plane) && (rcut3 >= 0.f) && (o > 0.f);

    const float su = __ldg(s.scales + 2 * i), sv = __ldg(s.scales + 2 * i + 1);
    vis = vis && (su > 0.f) && (sv > 0.f) && isfinite(su) && isfinite(sv);
    int tx0 = 0, ty0 = 0, tx1 = -1, ty1 = -1;
    int pb[4] = {0, 0, -1, -1};   // conservative pixel bbox (x0,y0,x1,y1), inclusive
    int cpb[4] = {0xffff, 0xffff, 0, 0};   // pinhole: pixel bbox of the 3-sigma disk only
    double A[3], Bv[3], N[3];
    if (vis) {
        const float4 qf = __ldg(reinterpret_cast<const float4 *>(s.quats) + i);
        double qw = qf.x, qx = qf.y, qy = qf.z, qz = qf.w;
        const double inq = rsqrt(qw * qw + qx * qx + qy * qy + qz * qz);
        qw *= inq; qx *= inq; qy *= inq; qz *= inq;
        const double Rq[3][3] = {
            {1.0 - 2.0 * (qy * qy + qz * qz), 2.0 * (qx * qy - qw * qz), 2.0 * (qx * qz + qw * qy)},
            {2.0 * (qx * qy + qw * qz), 1.0 - 2.0 * (qx * qx + qz * qz), 2.0 * (qy * qz - qw * qx)},
            {2.0 * (qx * qz - qw * qy), 2.0 * (qy * qz + qw * qx), 1.0 - 2.0 * (qx * qx + qy * qy)}};
        for (int r = 0; r < 3; ++r) {
            const double s0 = se.R[3 * r], s1 = se.R[3 * r + 1], s2 = se.R[3 * r + 2];
            A[r] = s0 * Rq[0][0] + s1 * Rq[1][0] + s2 * Rq[2][0];
            Bv[r] = s0 * Rq[0][1] + s1 * Rq[1][1] + s2 * Rq[2][1];
            N[r] = s0 * Rq[0][2] + s1 * Rq[1][2] + s2 * Rq[2][2];
        }
        vis = isfinite(N[0] + N[1] + N[2] + A[0] + Bv[0]);
    }
    const double rlp = sqrt((double)rcut3 * (double)op.sigma2);   // low-pass disc radius (px)
    if (vis) {
        const double Rr = sqrt((double)rcut3);
        if (KIND == GS_PINHOLE) {
            double a[3], b[3];
            for (int r = 0; r < 3; ++r) { a[r] = Rr * su * A[r]; b[r] = Rr * sv * Bv[r]; }
            Box bx;
            bx.init();
            pinhole_disk_bound(se, (double)op.near_plane, mu, a, b, bx);
            {   // pixel box of the 3-sigma disk alone (the record's box; the low-pass disc is
                // tested from the centre and radius by the compositor); empty: x0 = y0 = 0xffff
                int ttx0, tty0, ttx1, tty1, cb[4];
                if (box_to_tiles(bx, se.width, se.height, se.mtw, se.mth, ttx0, tty0, ttx1, tty1, cb)) {
                    for (int k = 0; k < 4; ++k) cpb[k] = cb[k];
                }
            }
            const double iz = 1.0 / mu[2];
            const double cx = (double)se.fx * mu[0] * iz + (double)se.cx;
            const double cy = (double)se.fy * mu[1] * iz + (double)se.cy;
            bx.add(cx - rlp, cy - rlp);
            bx.add(cx + rlp, cy + rlp);
            vis = box_to_tiles(bx, se.width, se.height, se.mtw, se.mth, tx0, ty0, tx1, ty1, pb);
        } else {
            const double r = sqrt(dot3(mu, mu)), ir = 1.0 / r;
            const double m[3] = {mu[0] * ir, mu[1] * ir, mu[2] * ir};
            const double R3 = Rr * (double)fmaxf(su, sv);
            const bool whole = !(R3 < 0.999 * r);
            // angular box of the support disk (elevation above the sensor xy
            // plane, azimuth about z): exact gnomonic extremes, else sphere cap
            AngBox ab;
            if (!whole) {
                double a[3], b[3];
                for (int k = 0; k < 3; ++k) { a[k] = Rr * su * A[k]; b[k] = Rr * sv * Bv[k]; }
                if (KIND == GS_FISHEYE_CYLINDRICAL) {
                    // azimuth about the camera y axis and elevation from the xz plane: the
                    // LiDAR-style box of the cyclically permuted frame (z, x, y)
                    const double mp[3] = {mu[2], mu[0], mu[1]}, ap[3] = {a[2], a[0], a[1]},
                                 bp[3] = {b[2], b[0], b[1]}, up[3] = {m[2], m[0], m[1]};
                    if (!angular_box_disk(mp, ap, bp, ab, true)) angular_box_cap(up, asin(R3 / r), ab);
                } else {
                    const bool fast = KIND == GS_LIDAR_SPINNING && angular_box_disk_f(mu, a, b, ab);
                    if (!fast && !angular_box_disk(mu, a, b, ab, KIND == GS_FISHEYE_EQUIDISTANT))
                        angular_box_cap(m, asin(R3 / r), ab);
                }
            }
            if (KIND == GS_FISHEYE_EQUIDISTANT) {
                Box bx;
                bx.init();
                const double tm = (double)se.theta_max;
                if (whole) {
                    const double rad = kb_theta_d(se, tm);
                    bx.add(se.cx - se.fx * rad, se.cy - se.fy * rad);
                    bx.add(se.cx + se.fx * rad, se.cy + se.fy * rad);
                } else {
                    // polar angle from the optical axis theta = pi/2 - elevation
                    const double thlo = fmax(0.0, 0.5 * M_PI - ab.el_hi), thhi = fmin(tm, 0.5 * M_PI - ab.el_lo);
                    if (thlo <= tm) {
                        const double r0 = kb_theta_d(se, thlo), r1 = kb_theta_d(se, thhi);
                        const bool allpsi = ab.all_az || thlo <= 0.0;
                        if (allpsi) {
                            bx.add(se.cx - se.fx * r1, se.cy - se.fy * r1);
                            bx.add(se.cx + se.fx * r1, se.cy + se.fy * r1);
                        } else {
                            const double p0 = ab.azc + ab.daz_lo, p1 = ab.azc + ab.daz_hi;
                            const double rads[2] = {r0, r1};
                            for (int k = 0; k < 2; ++k) {
                                bx.add(se.cx + se.fx * rads[k] * cos(p0), se.cy + se.fy * rads[k] * sin(p0));
                                bx.add(se.cx + se.fx * rads[k] * cos(p1), se.cy + se.fy * rads[k] * sin(p1));
                            }
                            // axis directions inside [p0, p1]
                            for (int q = -4; q <= 4; ++q) {
                                const double ang = q * (0.5 * M_PI);
                                if (ang >= p0 && ang <= p1)
                                    for (int k = 0; k < 2; ++k)
                                        bx.add(se.cx + se.fx * rads[k] * cos(ang),
                                               se.cy + se.fy * rads[k] * sin(ang));
                            }
                        }
                    }
                }
                double cxp, cyp;
                fisheye_project(se, mu, cxp, cyp);
                bx.add(cxp - rlp, cyp - rlp);
                bx.add(cxp + rlp, cyp + rlp);
                vis = box_to_tiles(bx, se.width, se.height, se.mtw, se.mth, tx0, ty0, tx1, ty1, pb);
            } else if (KIND == GS_FISHEYE_CYLINDRICAL) {
                Box bx;
                bx.init();
                if (whole) {
                    bx.add(0.f, 0.f);
                    bx.add((float)se.width, (float)se.height);
                } else {
                    // rows: y / rho = tan(elevation), monotone
                    const double lim = 1e9;
                    const double tlo = ab.el_lo <= -0.5 * M_PI + 1e-12 ? -lim : fmax(tan(ab.el_lo), -lim);
                    const double thi = ab.el_hi >= 0.5 * M_PI - 1e-12 ? lim : fmin(tan(ab.el_hi), lim);
                    const double y0 = (double)se.cy + (double)se.fy * tlo, y1 = (double)se.cy + (double)se.fy * thi;
                    // columns: the azimuth interval (and its shifts by 2 pi) inside the image's
                    // azimuth range [-c_x / f_x, (W - c_x) / f_x] (within [-pi, pi], gsr.h)
                    const double ilo = -(double)se.cx / (double)se.fx;
                    const double ihi = ((double)se.width - (double)se.cx) / (double)se.fx;
                    double lo = 1e30, hi = -1e30;
                    if (ab.all_az) {
                        lo = ilo; hi = ihi;
                    } else {
                        for (int kk = -1; kk <= 1; ++kk) {
                            const double a0 = fmax(ab.azc + ab.daz_lo + kk * 2.0 * M_PI, ilo);
                            const double a1 = fmin(ab.azc + ab.daz_hi + kk * 2.0 * M_PI, ihi);
                            if (a0 <= a1) { lo = fmin(lo, a0); hi = fmax(hi, a1); }
                        }
                    }
                    if (lo <= hi) {
                        bx.add((float)((double)se.cx + (double)se.fx * lo), (float)y0);
                        bx.add((float)((double)se.cx + (double)se.fx * hi), (float)y1);
                    }
                }
                double cxp, cyp;
                cylinder_project(se, mu, cxp, cyp);
                bx.add(cxp - rlp, cyp - rlp);
                bx.add(cxp + rlp, cyp + rlp);
                vis = box_to_tiles(bx, se.width, se.height, se.mtw, se.mth, tx0, ty0, tx1, ty1, pb);
            } else {   // LiDAR: angular box with azimuth wrap
                const int W = se.width;
                int r0 = 0, r1 = se.nbeams - 1, c0 = 0, c1 = W - 1;
                bool allaz = whole;
                if (!whole) {
                    const double eps = 2e-6;   // sine units; covers the fp32 sine table
                    vis = beam_rows(sb, se.nbeams, ab.s_lo - eps, ab.s_hi + eps, r0, r1);
                    allaz = ab.all_az;
                    if (!allaz) {
                        // column bounds widened by one column below: a reciprocal step is exact enough
                        const double step = (double)se.az_step, istep = 1.0 / step;
                        // start of the azimuth interval relative to az0, reduced into [0, 2pi)
                        // (az0 may be any angle; the interval is at most one turn wide)
                        double a0 = fmod(ab.azc + ab.daz_lo - (double)se.az0, 2.0 * M_PI);
                        if (a0 < 0.0) a0 += 2.0 * M_PI;
                        const double ulo = a0 * istep;
                        const double uhi = (a0 + (ab.daz_hi - ab.daz_lo)) * istep;
                        double jlo = ceil(ulo) - 1.0, jhi = floor(uhi) + 1.0;
                        if (se.full_turn) {
                            if (jhi - jlo + 1.0 >= (double)W) {
                                allaz = true;
                            } else {
                                // wrap jlo into [0, W) (integers in fp64: exact after the fix-up)
                                const double k = floor(jlo * (1.0 / (double)W));
                                jlo -= k * W;
                                jhi -= k * W;
                                if (jlo >= (double)W) { jlo -= W; jhi -= W; }
                                if (jlo < 0.0) { jlo += W; jhi += W; }
                                c0 = (int)jlo;
                                c1 = (int)jhi;   // may exceed W-1: wraps
                            }
                        } else {
                            // partial turn: the interval starts in [0, 2pi) past az0, so only
                            // it and its shift by -2pi can meet the columns [0, W); hull
                            const double per = 2.0 * M_PI / step;
                            double lo = 1e30, hi = -1e30;
                            for (int kk = -1; kk <= 0; ++kk) {
                                const double a0 = fmax(jlo + kk * per, 0.0), a1 = fmin(jhi + kk * per, (double)(W - 1));
                                if (a0 <= a1) { lo = fmin(lo, a0); hi = fmax(hi, a1); }
                            }
                            if (lo > hi) vis = false;
                            else { c0 = (int)ceil(lo); c1 = (int)floor(hi); if (c0 > c1) vis = false; }
                        }
                    }
                }
                if (vis) {
                    const int ntx = se.ntx;
                    if (allaz) {
                        tx0 = 0; tx1 = ntx - 1;
                        c0 = 0; c1 = W - 1;
                    } else {
                        tx0 = (int)tdiv((uint32_t)c0, se.mtw);   // exact division, as in box_to_tiles
                        tx1 = c1 < W ? (int)tdiv((uint32_t)c1, se.mtw) : ntx + (int)tdiv((uint32_t)(c1 - W), se.mtw);
                        if (tx1 - tx0 + 1 >= ntx) { tx0 = 0; tx1 = ntx - 1; c0 = 0; c1 = W - 1; }
                    }
                    ty0 = (int)tdiv((uint32_t)r0, se.mth);
                    ty1 = (int)tdiv((uint32_t)r1, se.mth);
                    pb[0] = c0; pb[1] = r0; pb[2] = c1; pb[3] = r1;   // c1 may exceed W-1 (wrap)
                }
            }
        }
    }
    if (!vis) {
        keys[i] = 0xffffffffu;
        counts[i] = 0;
        rect[i] = make_short4(0, 0, -1, -1);
        return;
    }
    keys[i] = __float_as_uint(keyf);
    counts[i] = (uint32_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1));   // pinhole (below), LiDAR (k_tiles): exact sets
    rect[i] = make_short4((short)tx0, (short)ty0, (short)tx1, (short)ty1);

    // oriented normal (faces the sensor), attributes
    const bool flip = dot3(N, mu) > 0.0;
    const float nsx = (float)(flip ? -N[0] : N[0]), nsy = (float)(flip ? -N[1] : N[1]),
                nsz = (float)(flip ? -N[2] : N[2]);

    if (KIND == GS_PINHOLE) {
        float R[PH_FLOATS];
        // rows of adj([t_u|t_v|mu]) / (s_u s_v) restricted to (dx/fx, dy/fy, 0)
        double r0[3], r1[3];
        cross3(Bv, mu, r0);   // (t_v x mu) / s_u
        cross3(mu, A, r1);    // (mu x t_u) / s_v
        const double det = dot3(N, mu);
        const double ifx = 1.0 / (double)se.fx, ify = 1.0 / (double)se.fy;
        const double isu = 1.0 / (double)su, isv = 1.0 / (double)sv;
        R[PH_A00] = (float)(r0[0] * isu * ifx);
        R[PH_A01] = (float)(r0[1] * isu * ify);
        R[PH_A10] = (float)(r1[0] * isv * ifx);
        R[PH_A11] = (float)(r1[1] * isv * ify);
        R[PH_A20] = (float)(N[0] * ifx);
        R[PH_A21] = (float)(N[1] * ify);
        const double iz = 1.0 / mu[2];
        R[PH_QC] = (float)(det * iz);
        const double cx = (double)se.fx * mu[0] * iz + (double)se.cx;
        const double cy = (double)se.fy * mu[1] * iz + (double)se.cy;
        R[PH_RCUT3] = rcut3;
        split_hilo(cx, R[PH_CHX], R[PH_CLX]);
        split_hilo(cy, R[PH_CHY], R[PH_CLY]);
        R[PH_RCUT2] = rcut3 * op.sigma2;
        R[PH_O] = o;
        R[PH_DET] = (float)det;
        R[PH_ZC] = (float)mu[2];
        const float vx = mx - se.ow[0], vy = my - se.ow[1], vz = mz - se.ow[2];
        const float vn = rsqrtf(vx * vx + vy * vy + vz * vz);
        const int nc = (s.sh_degree + 1) * (s.sh_degree + 1);
        float rgb[3];
        sh_colour(s.sh + (size_t)i * nc * 3, s.sh_degree, vx * vn, vy * vn, vz * vn, rgb);
        R[PH_R] = rgb[0]; R[PH_G] = rgb[1]; R[PH_B] = rgb[2];
        R[PH_NX] = nsx; R[PH_NY] = nsy; R[PH_NZ] = nsz;
        R[PH_BBX] = pack_bb(cpb[0], cpb[2]);
        R[PH_BBY] = pack_bb(cpb[1], cpb[3]);
        float4 *dst = reinterpret_cast<float4 *>(rec + (size_t)i * PH_FLOATS);
#pragma unroll
        for (int k = 0; k < PH_FLOATS / 4; ++k)
            dst[k] = make_float4(R[4 * k], R[4 * k + 1], R[4 * k + 2], R[4 * k + 3]);
        // exact tile rows (binning.cuh), from the record floats in registers: the pair
        // count becomes the number of tiles whose pixel centres the support conic or
        // the low-pass disc can reach, and the row table (first column relative to the
        // rect | width << 8, one u16 per tile row) goes to k_emit_rows.  Measured
        // against a separate load-balanced pass that re-read the records: 0.03 ms
        // faster per forward / side camera frame.
        if ((uint32_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1)) >= KT_MIN_AREA && ty1 - ty0 + 1 <= PH_ROWS_MAX &&
            tx1 - tx0 + 1 <= 255) {
            const PhRows pr = ph_rows_setup(make_float4(R[0], R[1], R[2], R[3]), make_float4(R[4], R[5], R[6], R[7]),
                                            make_float4(R[8], R[9], R[10], R[11]), R[PH_RCUT2],
                                            __float_as_uint(R[PH_BBX]), __float_as_uint(R[PH_BBY]));
            uint16_t *tbl = reinterpret_cast<uint16_t *>(rows + 2 * i);
            uint32_t cnt = 0;
#pragma unroll 1
            for (int ty = ty0; ty <= ty1; ++ty) {
                int a, b;
                ph_row_tiles(pr, ty, tx0, tx1, se.width, se.height, se.tw, se.th, se.mtw, a, b);
                const uint32_t w = a <= b ? (uint32_t)(b - a + 1) : 0u;
                tbl[ty - ty0] = (uint16_t)((a <= b ? (uint32_t)(a - tx0) : 0u) | (w << 8));
                cnt += w;
            }
            if (cnt == 0) keys[i] = 0xffffffffu;
            counts[i] = cnt;
        }
    } else {
        constexpr int NF = dir_camera(KIND) ? FE_FLOATS : LI_FLOATS;
        float R[NF];
#pragma unroll
        for (int k = 0; k < NF; ++k) R[k] = 0.f;
        const double r = sqrt(dot3(mu, mu)), ir = 1.0 / r;
        const double m[3] = {mu[0] * ir, mu[1] * ir, mu[2] * ir};
        for (int k = 0; k < 3; ++k) split_hilo(m[k], R[RY_MH + k], R[RY_ML + k]);
        double u[3], v[3];
        cross3(Bv, m, u);   // U = r (R t_v x m) / s_u
        cross3(m, A, v);    // V = r (m x R t_u) / s_v
        const double det = dot3(N, m);
        const double rsu = r / (double)su, rsv = r / (double)sv;
        for (int k = 0; k < 3; ++k) {
            R[RY_U + k] = (float)(rsu * u[k]);
            R[RY_V + k] = (float)(rsv * v[k]);
            R[RY_N + k] = (float)N[k];
        }
        R[RY_DET] = (float)det;
        R[RY_RDET] = (float)(r * det);
        R[RY_RCUT3] = rcut3;
        R[RY_O] = o;
        R[RY_RC] = (float)r;
        if (dir_camera(KIND)) {
            double cxp, cyp;
            if (KIND == GS_FISHEYE_EQUIDISTANT) fisheye_project(se, mu, cxp, cyp);
            else cylinder_project(se, mu, cxp, cyp);
            split_hilo(cxp, R[FE_CHX], R[FE_CLX]);
            split_hilo(cyp, R[FE_CHY], R[FE_CLY]);
            R[FE_RCUT2] = rcut3 * op.sigma2;
            const float vx = mx - se.ow[0], vy = my - se.ow[1], vz = mz - se.ow[2];
            const float vn = rsqrtf(vx * vx + vy * vy + vz * vz);
            const int nc = (s.sh_degree + 1) * (s.sh_degree + 1);
            float rgb[3];
            sh_colour(s.sh + (size_t)i * nc * 3, s.sh_degree, vx * vn, vy * vn, vz * vn, rgb);
            R[FE_R] = rgb[0]; R[FE_G] = rgb[1]; R[FE_B] = rgb[2];
            R[FE_NX] = nsx; R[FE_NY] = nsy; R[FE_NZ] = nsz;
            R[FE_BBX] = pack_bb(pb[0], pb[2]);
            R[FE_BBY] = pack_bb(pb[1], pb[3]);
        } else {
            R[LI_INT] = s.inten ? __ldg(s.inten + i) : 0.f;
            const float lg = s.drop ? __ldg(s.drop + i) : 0.f;
            R[LI_DROP] = 1.f / (1.f + expf(-lg));   // fp32 sigmoid: error ~1e-7, far inside the 1e-4 tolerance
            R[LI_BBX] = pack_bb(pb[0], pb[2]);
            R[LI_BBY] = pack_bb(pb[1], pb[3]);
        }
        float4 *dst = reinterpret_cast<float4 *>(rec + (size_t)i * NF);
#pragma unroll
        for (int k = 0; k < NF / 4; ++k)
            dst[k] = make_float4(R[4 * k], R[4 * k + 1], R[4 * k + 2], R[4 * k + 3]);
    }
}

// One thread per candidate (grid-stride over the compacted list of k_cull).
#ifndef PROJ_MINB_CAM
#define PROJ_MINB_CAM 3
#endif
#ifndef PROJ_MINB_LIDAR
#define PROJ_MINB_LIDAR 4
#endif
template <int KIND>
__global__ void __launch_bounds__(256, KIND == GS_LIDAR_SPINNING ? PROJ_MINB_LIDAR : PROJ_MINB_CAM) k_project(DevSurfels s, const __grid_constant__ DevSensor se, DevOpts op,
                                                 const uint32_t *__restrict__ cand, const ProjHeader *hdr,
                                                 float *__restrict__ rec, short4 *__restrict__ rect,
                                                 uint32_t *__restrict__ keys, uint32_t *__restrict__ counts,
                                                 uint4 *__restrict__ rows) {
    __shared__ float sb[KIND == GS_LIDAR_SPINNING ? GS_MAX_BEAMS : 1];
    if (KIND == GS_LIDAR_SPINNING) {
        for (int k = threadIdx.x; k < se.nbeams; k += blockDim.x) sb[k] = se.sbeam[k];
        __syncthreads();
    }
    const uint32_t nc = cand ? hdr->n_cand : (uint32_t)s.n;   // no cand list: every surfel
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += gridDim.x * blockDim.x)
        project_one<KIND>(s, se, op, cand ? (int64_t)cand[c] : (int64_t)c, rec, rect, keys, counts, rows, sb);
}

// ------------------------------------------------------------------ exact LiDAR tile sets
// After k_project (binning.cuh li_tile_hits): per tile of the rect (one-row
// tiles, rects of LI_MIN_AREA..64 tiles) the support-quadric test over the
// tile's ray arc, stored as a mask over the rect; the count becomes the
// number of admitted tiles (an empty set culls the surfel).  Load-balanced: a warp takes 32 candidates, stages their record
// quantities in shared memory and deals their (surfel, tile) items over its
// lanes 32 at a time; tile-column and beam-row trig come from per-CTA shared
// tables.  (The pinhole rows are computed inside k_project.)
constexpr uint32_t LI_MIN_AREA = 8;   // smaller rects: every tile (the test costs more than it saves there)
constexpr int KT_WARPS = 8;
constexpr int KT_NPAR = 16;          // floats of staged per-surfel quantities
constexpr int KT_MAXCOL = 512;       // LiDAR tile columns with a shared trig table

__global__ void __launch_bounds__(256) k_tiles(const __grid_constant__ DevSensor se, const uint32_t *__restrict__ cand,
                                               const ProjHeader *hdr, int64_t nsurf, const float *__restrict__ rec,
                                               short4 *__restrict__ rect, uint32_t *__restrict__ keys,
                                               uint32_t *__restrict__ counts, uint64_t *__restrict__ tmask) {
    __shared__ float s_par[KT_WARPS][32][KT_NPAR + 1];
    __shared__ uint32_t s_res[KT_WARPS][2][33];   // the 64-bit masks of the warp's 32 surfels
    __shared__ float4 s_col[KT_MAXCOL];
    __shared__ float2 s_row[GS_MAX_BEAMS];
    const bool coltab = se.ntx <= KT_MAXCOL;
    if (coltab)
        for (int t = threadIdx.x; t < se.ntx; t += blockDim.x) s_col[t] = li_col_trig(se, t);
    for (int r = threadIdx.x; r < se.nbeams; r += blockDim.x) {
        float st, ct;
        sincosf(se.beam[r], &st, &ct);
        s_row[r] = make_float2(st, ct);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    float *par = s_par[wid][lane];
    const uint32_t nc = cand ? hdr->n_cand : (uint32_t)nsurf;
    const uint32_t ngroups = (nc + 31) / 32, gstride = gridDim.x * KT_WARPS;
    for (uint32_t gi = blockIdx.x * KT_WARPS + wid; gi < ngroups; gi += gstride) {
        const uint32_t c = gi * 32 + lane;
        int64_t i = -1;
        uint32_t nitem = 0;
        short4 r = make_short4(0, 0, -1, -1);
        if (c < nc) {
            i = cand ? (int64_t)cand[c] : (int64_t)c;
            const uint32_t cnt0 = counts[i];
            if (cnt0 >= LI_MIN_AREA && cnt0 <= 64 && se.th == 1) {
                r = rect[i];
                const float4 *g = reinterpret_cast<const float4 *>(rec) + (size_t)i * (LI_FLOATS / 4);
                float gr[LI_FLOATS];
#pragma unroll
                for (int k = 0; k < LI_FLOATS / 4; ++k) {
                    const float4 v = g[k];
                    gr[4 * k] = v.x; gr[4 * k + 1] = v.y; gr[4 * k + 2] = v.z; gr[4 * k + 3] = v.w;
                }
                const LiRec q = li_rec(gr);
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    par[k] = q.U[k]; par[3 + k] = q.V[k]; par[6 + k] = q.N[k]; par[9 + k] = q.m[k];
                }
                par[12] = q.R; par[13] = q.mag;
                s_res[wid][0][lane] = 0u;
                s_res[wid][1][lane] = 0u;
                nitem = cnt0;
            }
        }
        // deal the (surfel, tile) items of the 32 surfels over the lanes
        const uint32_t inc = warp_inclusive_scan<uint32_t>(nitem);
        const uint32_t base = inc - nitem, tot = __shfl_sync(FULL_MASK, inc, 31);
        __syncwarp();
        for (uint32_t tb = 0; tb < tot; tb += 32) {
            const uint32_t t = tb + (uint32_t)lane;
            int j = 0;   // last lane whose first item is <= t
#pragma unroll
            for (int step = 16; step; step >>= 1) {
                const uint32_t b = __shfl_sync(FULL_MASK, base, j + step);
                if (b <= t) j += step;   // a zero-item lane shares its base with the next lane
            }
            const uint32_t bj = __shfl_sync(FULL_MASK, base, j);
            const int rx0 = __shfl_sync(FULL_MASK, (int)r.x, j), ry0 = __shfl_sync(FULL_MASK, (int)r.y, j);
            const int rx1 = __shfl_sync(FULL_MASK, (int)r.z, j);
            if (t < tot) {
                const int k = (int)(t - bj);
                const float *pj = s_par[wid][j];
                LiRec q;
#pragma unroll
                for (int m = 0; m < 3; ++m) {
                    q.U[m] = pj[m]; q.V[m] = pj[3 + m]; q.N[m] = pj[6 + m]; q.m[m] = pj[9 + m];
                }
                q.R = pj[12]; q.mag = pj[13];
                const int w = rx1 - rx0 + 1;
                const int dy = k / w, tx = rx0 + (k - dy * w), ty = ry0 + dy;
                const int tc = tx >= se.ntx ? tx - se.ntx : tx;
                const float4 c4 = coltab ? s_col[tc] : li_col_trig(se, tc);
                const float2 rt = s_row[ty];
                if (li_tile_hits(q, c4, rt.x, rt.y)) atomicOr(&s_res[wid][k >> 5][j], 1u << (k & 31));
            }
        }
        __syncwarp();
        if (nitem == 0) continue;
        // this lane's surfel: count and mask (over its rect, row-major)
        const uint64_t bits = (uint64_t)s_res[wid][0][lane] | ((uint64_t)s_res[wid][1][lane] << 32);
        const uint32_t cnt = (uint32_t)__popcll(bits);
        tmask[i] = bits;
        counts[i] = cnt;
        if (cnt == 0) keys[i] = 0xffffffffu;
    }
}

// ------------------------------------------------------------------ compaction
// Visible surfels (count > 0) among the candidates, in index order ->
// (vis_key, vis_id); totals of visible surfels and of pairs -> header and
// d_num_pairs.  One CTA = 2048 candidates; each lane owns 8 consecutive
// candidates; decoupled look-back.
__global__ void __launch_bounds__(SCAN_THREADS) k_compact(const uint32_t *__restrict__ keys,
                                                          const uint32_t *__restrict__ counts,
                                                          const uint32_t *__restrict__ cand, int64_t nsurf,
                                                          uint32_t *__restrict__ vkey,
                                                          uint32_t *__restrict__ vid,
                                                          unsigned long long *st_vis,
                                                          unsigned long long *st_pairs,
                                                          ProjHeader *hdr, int64_t *d_num_pairs) {
    __shared__ uint32_t s_tile;
    __shared__ unsigned long long s_wv[SCAN_THREADS / 32], s_wp[SCAN_THREADS / 32];
    __shared__ unsigned long long s_excl_v;
    if (threadIdx.x == 0) s_tile = atomicAdd(&hdr->scan_counter, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const int64_t n = cand ? (int64_t)hdr->n_cand : (int64_t)nsurf;
    if ((int64_t)tile * SCAN_TILE >= n && tile > 0) return;   // beyond the candidates: nobody looks back here
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t base = (int64_t)tile * SCAN_TILE + (int64_t)(warp * 32 + lane) * SCAN_ITEMS;
    uint32_t c[SCAN_ITEMS], id[SCAN_ITEMS];
    uint32_t lv = 0, lp = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        const int64_t idx = base + j;
        id[j] = idx < n ? (cand ? cand[idx] : (uint32_t)idx) : 0u;
        c[j] = idx < n ? counts[id[j]] : 0u;
        lv += c[j] > 0 ? 1u : 0u;
        lp += c[j];
    }
    // warp scans (inclusive) of per-lane totals
    unsigned long long iv = warp_inclusive_scan<unsigned long long>(lv);
    unsigned long long ip = warp_inclusive_scan<unsigned long long>(lp);
    if (lane == 31) { s_wv[warp] = iv; s_wp[warp] = ip; }
    __syncthreads();
    if (warp == 0) {
        const unsigned long long tv = warp_excl_scan_smem(s_wv, SCAN_THREADS / 32);
        const unsigned long long tp = warp_excl_scan_smem(s_wp, SCAN_THREADS / 32);
        unsigned long long ev, ep;
        if (nsurf < (1ll << 25)) {   // one look-back for both: pairs << 25 | visible (62 value bits)
            const unsigned long long eq = lookback_warp_u64(st_vis, tile, (tp << 25) | tv);
            ev = eq & ((1ull << 25) - 1);
            ep = eq >> 25;
        } else {
            ev = lookback_warp_u64(st_vis, tile, tv);
            ep = lookback_warp_u64(st_pairs, tile, tp);
        }
        if (lane == 0) {
            s_excl_v = ev;
            const int64_t end = (int64_t)(tile + 1) * SCAN_TILE;
            if (end >= n) {   // last tile: totals
                hdr->n_visible = (uint32_t)(ev + tv);
                hdr->num_pairs = (int64_t)(ep + tp);
                if (d_num_pairs) *d_num_pairs = (int64_t)(ep + tp);
            }
        }
    }
    __syncthreads();
    unsigned long long pos = s_excl_v + s_wv[warp] + iv - lv;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        if (c[j] > 0) {
            vkey[pos] = keys[id[j]];
            vid[pos] = id[j];
            ++pos;
        }
    }
}

// host-side launchers (called from abi.cu)
cudaError_t launch_project(const DevSurfels &s, const DevSensor &se, const DevOpts &op, void *proj,
                           int64_t *d_num_pairs, cudaStream_t st) {
    const ProjLayout L(s.n, se.kind);
    char *base = (char *)proj;
    ProjHeader *hdr = (ProjHeader *)base;
    cudaError_t e = cudaMemsetAsync(hdr, 0, sizeof(ProjHeader), st);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(base + L.status, 0, 3 * (L.nblk + 1) * 8, st);
    if (e != cudaSuccess) return e;
    if (s.n == 0) {
        if (d_num_pairs) return cudaMemsetAsync(d_num_pairs, 0, 8, st);
        return cudaSuccess;
    }
    float *rec = (float *)(base + L.rec);
    short4 *rect = (short4 *)(base + L.rect);
    uint32_t *key = (uint32_t *)(base + L.key), *cnt = (uint32_t *)(base + L.cnt);
    uint32_t *cand = (uint32_t *)(base + L.cand);
    uint64_t *tm = (uint64_t *)(base + L.tmask);
    uint4 *rw = (uint4 *)(base + L.rows);
    unsigned long long *stv = (unsigned long long *)(base + L.status);
    unsigned long long *stp = stv + L.nblk + 1, *stc = stp + L.nblk + 1;
    const unsigned nblk = (unsigned)L.nblk;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    // grid-stride k_project: exactly the resident CTAs (whole waves, no tail wave)
    // (queried per call: the library keeps no mutable process state besides the launch counter)
    int occ = 0;
    if (se.kind == GS_PINHOLE)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_project<GS_PINHOLE>, 256, 0);
    else if (se.kind == GS_FISHEYE_EQUIDISTANT)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_project<GS_FISHEYE_EQUIDISTANT>, 256, 0);
    else if (se.kind == GS_FISHEYE_CYLINDRICAL)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_project<GS_FISHEYE_CYLINDRICAL>, 256, 0);
    else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_project<GS_LIDAR_SPINNING>, 256, 0);
    const unsigned gp = (unsigned)std::min<int64_t>((s.n + 255) / 256, (int64_t)nsm * std::max(occ, 1));
    note_launch(3);   // k_cull + k_project + k_compact
    if (se.kind == GS_PINHOLE) {
        k_cull<GS_PINHOLE><<<nblk, SCAN_THREADS, 0, st>>>(s, se, op, rect, key, cnt, cand, stc, hdr);
        k_project<GS_PINHOLE><<<gp, 256, 0, st>>>(s, se, op, cand, hdr, rec, rect, key, cnt, rw);
    } else if (se.kind == GS_FISHEYE_EQUIDISTANT) {
        k_cull<GS_FISHEYE_EQUIDISTANT><<<nblk, SCAN_THREADS, 0, st>>>(s, se, op, rect, key, cnt, cand, stc, hdr);
        k_project<GS_FISHEYE_EQUIDISTANT><<<gp, 256, 0, st>>>(s, se, op, cand, hdr, rec, rect, key, cnt, rw);
    } else if (se.kind == GS_FISHEYE_CYLINDRICAL) {
        k_cull<GS_FISHEYE_CYLINDRICAL><<<nblk, SCAN_THREADS, 0, st>>>(s, se, op, rect, key, cnt, cand, stc, hdr);
        k_project<GS_FISHEYE_CYLINDRICAL><<<gp, 256, 0, st>>>(s, se, op, cand, hdr, rec, rect, key, cnt, rw);
    } else {
        k_cull<GS_LIDAR_SPINNING><<<nblk, SCAN_THREADS, 0, st>>>(s, se, op, rect, key, cnt, cand, stc, hdr);
        k_project<GS_LIDAR_SPINNING><<<gp, 256, 0, st>>>(s, se, op, cand, hdr, rec, rect, key, cnt, rw);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (se.kind == GS_LIDAR_SPINNING) {
        e = cudaMemsetAsync(tm, 0xff, (size_t)s.n * 8, st);   // ~0: every tile of the rect
        if (e != cudaSuccess) return e;
        const unsigned gt = (unsigned)std::min<int64_t>((s.n + 255) / 256, (int64_t)nsm * 8);
        note_launch();
        k_tiles<<<gt, 256, 0, st>>>(se, cand, hdr, s.n, rec, rect, key, cnt, tm);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    k_compact<<<nblk, SCAN_THREADS, 0, st>>>(key, cnt, cand, s.n, (uint32_t *)(base + L.vkey), (uint32_t *)(base + L.vid),
                                            stv, stp, hdr, d_num_pairs);
    return cudaGetLastError();
}

cudaError_t launch_bounds(const DevSurfels &s, float *bounds, cudaStream_t st) {
    if (s.n == 0) return cudaSuccess;
    const unsigned nblk = (unsigned)((s.n + SCAN_TILE - 1) / SCAN_TILE);
    note_launch();
    k_bounds<<<nblk, SCAN_THREADS, 0, st>>>(s.means, s.scales, s.n, bounds);
    return cudaGetLastError();
}

}  // namespace gsr
