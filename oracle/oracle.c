/*
 * oracle.c -- CPU fp64 brute-force reference renderer (camera + LiDAR 2DGS).
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Plain C, fp64 throughout, one ray
 * at a time against EVERY surfel, in the order of the definition in
 * DESIGN.md §2.  No binning, no tiles, no blocking.  OpenMP only distributes
 * independent rays over host cores.  Compile with -ffp-contract=off: the sort
 * key (reading R9) is an IEEE-exact fp64 expression in a pinned order.
 *
 * Passages followed (PAPER.md = /root/reference/PAPER.md):
 *   P:78      attributes {mu, R, S, rho, r, alpha} of each surfel
 *   P:81-89   Eq. 1  P(u,v) = W H (u,v,1)^T,  H = [s_u t_u, s_v t_v, mu; 0 0 1]
 *   P:91-94   Eq. 2  [h_u, h_v]^T P(u,v) = 0  (ray as two planes)
 *   P:96-100  Eq. 3  pinhole planes h_u = (-1,0,0,p_x), h_v = (0,-1,0,p_y)
 *   P:108-114 Eq. 5  LiDAR planes h_u = (sin phi,-cos phi,0,0),
 *                    h_v = (sin th cos phi, sin th sin phi, -cos th, 0)
 *   P:102-106 Eq. 4  (cylindrical fisheye) is replaced by the equidistant
 *                    Kannala-Brandt camera of BASELINE.json; its rays use the
 *                    Eq.-5 plane construction about the optical axis (R4).
 *   P:48      SH view-dependent colour; 2DGS low-pass filter
 *   north_star: alpha = min(0.99, o G); skip alpha < 1/255; stop once
 *               T < 1e-4; low-pass at 1/sqrt(2) px.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_PI 3.14159265358979323846
#ifndef OR_W_FLOOR
#define OR_W_FLOOR 2e-6
#endif

/* ------------------------------------------------------------------ SH
 * Real spherical harmonics with the Condon-Shortley phase, in the ordering
 * used by 3DGS (m = -l..l).  Constants written from their closed forms. */
void or_sh_basis(const double d[3], double Y[16]) {
    const double x = d[0], y = d[1], z = d[2];
    const double sp = sqrt(OR_PI);
    const double C0 = 1.0 / (2.0 * sp);
    const double C1 = sqrt(3.0) / (2.0 * sp);
    const double C2a = sqrt(15.0) / (2.0 * sp), C2b = sqrt(5.0) / (4.0 * sp),
                 C2c = sqrt(15.0) / (4.0 * sp);
    const double C3a = 0.25 * sqrt(35.0 / (2.0 * OR_PI)), C3b = 0.5 * sqrt(105.0 / OR_PI),
                 C3c = 0.25 * sqrt(21.0 / (2.0 * OR_PI)), C3d = 0.25 * sqrt(7.0 / OR_PI),
                 C3e = 0.25 * sqrt(105.0 / OR_PI);
    Y[0] = C0;
    Y[1] = -C1 * y;
    Y[2] = C1 * z;
    Y[3] = -C1 * x;
    Y[4] = C2a * x * y;
    Y[5] = -C2a * y * z;
    Y[6] = C2b * (2.0 * z * z - x * x - y * y);
    Y[7] = -C2a * x * z;
    Y[8] = C2c * (x * x - y * y);
    Y[9] = -C3a * y * (3.0 * x * x - y * y);
    Y[10] = C3b * x * y * z;
    Y[11] = -C3c * y * (4.0 * z * z - x * x - y * y);
    Y[12] = C3d * z * (2.0 * z * z - 3.0 * x * x - 3.0 * y * y);
    Y[13] = -C3c * x * (4.0 * z * z - x * x - y * y);
    Y[14] = C3e * z * (x * x - y * y);
    Y[15] = -C3a * x * (x * x - 3.0 * y * y);
}

/* ------------------------------------------------------------ fisheye lens */
double or_kb_theta_d(const float k[4], double th) {
    const double t2 = th * th;
    return th * (1.0 + (double)k[0] * t2 + (double)k[1] * t2 * t2 + (double)k[2] * t2 * t2 * t2 +
                 (double)k[3] * t2 * t2 * t2 * t2);
}

/* Inverse of the (monotone, R12) map theta -> theta_d on [0, theta_max] by
 * bisection to the resolution of fp64. */
double or_kb_inverse(const float k[4], double theta_max, double td) {
    double lo = 0.0, hi = theta_max;
    for (int it = 0; it < 200; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (mid <= lo || mid >= hi) break;
        if (or_kb_theta_d(k, mid) < td) lo = mid; else hi = mid;
    }
    return 0.5 * (lo + hi);
}

/* --------------------------------------------------------------- Eq. 1 */
static void quat_to_rot(const float *qf, double R[3][3]) {
    double w = qf[0], x = qf[1], y = qf[2], z = qf[3];
    const double nq = sqrt(w * w + x * x + y * y + z * z);
    w /= nq; x /= nq; y /= nq; z /= nq;
    R[0][0] = 1.0 - 2.0 * (y * y + z * z); R[0][1] = 2.0 * (x * y - w * z); R[0][2] = 2.0 * (x * z + w * y);
    R[1][0] = 2.0 * (x * y + w * z); R[1][1] = 1.0 - 2.0 * (x * x + z * z); R[1][2] = 2.0 * (y * z - w * x);
    R[2][0] = 2.0 * (x * z - w * y); R[2][1] = 2.0 * (y * z + w * x); R[2][2] = 1.0 - 2.0 * (x * x + y * y);
}

/* Sensor-frame centre with the pinned operation order of reading R9:
 * x_k = ((R_k0 mu_x + R_k1 mu_y) + R_k2 mu_z) + t_k, every operation an
 * IEEE-rounded fp64 op on exactly-promoted fp32 inputs (no contraction). */
static void centre_sensor(const or_sensor *se, const float *mu, double x[3]) {
    for (int k = 0; k < 3; ++k) {
        double a = (double)se->w2s[4 * k + 0] * (double)mu[0];
        double b = (double)se->w2s[4 * k + 1] * (double)mu[1];
        double c = (double)se->w2s[4 * k + 2] * (double)mu[2];
        double s = a + b;
        s = s + c;
        x[k] = s + (double)se->w2s[4 * k + 3];
    }
}

static float depth_key(const or_sensor *se, const double x[3]) {
    if (se->kind == OR_PINHOLE) return (float)x[2];
    double s = x[0] * x[0] + x[1] * x[1];
    s = s + x[2] * x[2];
    return (float)sqrt(s);
}

typedef struct {
    double M[3][3];      /* columns: s_u R_s t_u | s_v R_s t_v | mu_s  (Eq. 1 with W = [R_s|t_s]) */
    double mus[3];
    double cdepth;       /* centre depth: pinhole z, else range */
    double c[2];         /* projected centre (cameras) */
    double ns[3];        /* oriented normal, sensor frame */
    double val[3];       /* colour or (intensity, p_drop, 0) */
    double o, smin, smax;
    float key;
    int culled;
} surf_t;

static void project_centre(const or_sensor *se, const double m[3], double c[2]) {
    if (se->kind == OR_PINHOLE) {
        c[0] = (double)se->fx * m[0] / m[2] + (double)se->cx;
        c[1] = (double)se->fy * m[1] / m[2] + (double)se->cy;
    } else if (se->kind == OR_FISHEYE) {
        const double rxy = sqrt(m[0] * m[0] + m[1] * m[1]);
        const double th = atan2(rxy, m[2]);
        const double td = or_kb_theta_d(se->k, th);
        if (rxy > 0.0) {
            c[0] = (double)se->cx + (double)se->fx * td * m[0] / rxy;
            c[1] = (double)se->cy + (double)se->fy * td * m[1] / rxy;
        } else {
            c[0] = se->cx; c[1] = se->cy;
        }
    } else if (se->kind == OR_CYLINDRICAL) {
        /* Eq. 4 (reading R20): azimuth about the camera y axis ->
         * column, y over the distance from the y axis -> row */
        const double rho = sqrt(m[0] * m[0] + m[2] * m[2]);
        c[0] = (double)se->cx + (double)se->fx * atan2(m[0], m[2]);
        c[1] = (double)se->cy + (double)se->fy * m[1] / rho;
    } else {
        c[0] = c[1] = 0.0;
    }
}

static void prep_surfel(const or_scene *sc, const or_sensor *se, const or_opts *op, int64_t i,
                        surf_t *s) {
    const float *mu = sc->means + 3 * i;
    double Rq[3][3], Rs[3][3];
    quat_to_rot(sc->quats + 4 * i, Rq);
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) Rs[r][c] = se->w2s[4 * r + c];
    centre_sensor(se, mu, s->mus);
    s->key = depth_key(se, s->mus);
    s->culled = !(s->key >= (float)op->near_) || !isfinite(s->key);
    const double su = sc->scales[2 * i], sv = sc->scales[2 * i + 1];
    s->smin = su < sv ? su : sv;
    s->smax = su > sv ? su : sv;
    double tu[3], tv[3], nn[3];
    for (int r = 0; r < 3; ++r) {
        tu[r] = Rs[r][0] * Rq[0][0] + Rs[r][1] * Rq[1][0] + Rs[r][2] * Rq[2][0];
        tv[r] = Rs[r][0] * Rq[0][1] + Rs[r][1] * Rq[1][1] + Rs[r][2] * Rq[2][1];
        nn[r] = Rs[r][0] * Rq[0][2] + Rs[r][1] * Rq[1][2] + Rs[r][2] * Rq[2][2];
    }
    for (int r = 0; r < 3; ++r) {
        s->M[r][0] = su * tu[r];
        s->M[r][1] = sv * tv[r];
        s->M[r][2] = s->mus[r];
    }
    s->cdepth = se->kind == OR_PINHOLE
                    ? s->mus[2]
                    : sqrt(s->mus[0] * s->mus[0] + s->mus[1] * s->mus[1] + s->mus[2] * s->mus[2]);
    project_centre(se, s->mus, s->c);
    /* normal faces the sensor (reading R10) */
    const double side = nn[0] * s->mus[0] + nn[1] * s->mus[1] + nn[2] * s->mus[2];
    for (int r = 0; r < 3; ++r) s->ns[r] = side > 0.0 ? -nn[r] : nn[r];
    s->o = sc->opacities[i];
    if (se->kind == OR_LIDAR) {
        s->val[0] = sc->intensity ? sc->intensity[i] : 0.0;
        s->val[1] = sc->raydrop_logit ? 1.0 / (1.0 + exp(-(double)sc->raydrop_logit[i])) : 0.0;
        s->val[2] = 0.0;
    } else {
        /* view direction (world) from the sensor origin o = -R_s^T t_s */
        double o[3], v[3], Y[16];
        for (int c = 0; c < 3; ++c)
            o[c] = -(Rs[0][c] * se->w2s[3] + Rs[1][c] * se->w2s[7] + Rs[2][c] * se->w2s[11]);
        for (int c = 0; c < 3; ++c) v[c] = (double)mu[c] - o[c];
        const double vn = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
        for (int c = 0; c < 3; ++c) v[c] /= vn;
        or_sh_basis(v, Y);
        const int nc = (sc->sh_degree + 1) * (sc->sh_degree + 1);
        for (int ch = 0; ch < 3; ++ch) {
            double acc = 0.0;
            for (int j = 0; j < nc; ++j) acc += Y[j] * (double)sc->sh[(i * nc + j) * 3 + ch];
            acc += 0.5;
            s->val[ch] = acc > 0.0 ? acc : 0.0;
        }
    }
}

/* --------------------------------------------------- rays (Eqs. 3, 5; R4) */
int or_ray(const or_sensor *se, int32_t col, int32_t row, double nu[3], double nv[3], double d[3],
           double p[2]) {
    p[0] = col + 0.5;
    p[1] = row + 0.5;
    if (se->kind == OR_PINHOLE) {
        /* Eq. 3 in camera coordinates (K divided out): the planes
         * -x + xh z = 0 and -y + yh z = 0 contain the ray d = (xh, yh, 1). */
        const double xh = (p[0] - se->cx) / se->fx, yh = (p[1] - se->cy) / se->fy;
        nu[0] = -1.0; nu[1] = 0.0; nu[2] = xh;
        nv[0] = 0.0; nv[1] = -1.0; nv[2] = yh;
        d[0] = xh; d[1] = yh; d[2] = 1.0;
        return 1;
    }
    if (se->kind == OR_FISHEYE) {
        const double mx = (p[0] - se->cx) / se->fx, my = (p[1] - se->cy) / se->fy;
        const double td = sqrt(mx * mx + my * my);
        const double tdmax = or_kb_theta_d(se->k, se->theta_max);
        const double th = or_kb_inverse(se->k, se->theta_max, td < tdmax ? td : tdmax);
        const double cp = td > 0.0 ? mx / td : 1.0, sp = td > 0.0 ? my / td : 0.0;
        const double st = sin(th), ct = cos(th);
        d[0] = st * cp; d[1] = st * sp; d[2] = ct;
        nu[0] = sp; nu[1] = -cp; nu[2] = 0.0;
        nv[0] = ct * cp; nv[1] = ct * sp; nv[2] = -st;
        return td <= tdmax;
    }
    if (se->kind == OR_CYLINDRICAL) {
        /* Eq. 4, reading R20: phi = (p_x - c_x)/f_x is the azimuth
         * about the camera y axis and h_u = (cos phi, 0, -sin phi, 0) verbatim;
         * h_v = (0, -1, 0, p_y) read in the cylindrical screen space whose
         * homogeneous coordinate is rho = sin(phi) x + cos(phi) z (K folded, as
         * in Eq. 3): -(f_y y + c_y rho) + p_y rho = 0, i.e. the plane
         * -y + yh rho = 0 with yh = (p_y - c_y)/f_y.  Ray: (sin phi, yh, cos phi),
         * normalised (ray parameter = range). */
        const double ph = (p[0] - se->cx) / se->fx, yh = (p[1] - se->cy) / se->fy;
        const double sf = sin(ph), cf = cos(ph), nd = sqrt(1.0 + yh * yh);
        nu[0] = cf; nu[1] = 0.0; nu[2] = -sf;
        nv[0] = yh * sf; nv[1] = -1.0; nv[2] = yh * cf;
        d[0] = sf / nd; d[1] = yh / nd; d[2] = cf / nd;
        return 1;
    }
    /* LiDAR, Eq. 5 with theta = elevation, phi = azimuth (reading R5) */
    const double th = se->beam_elevation[row];
    const double ph = (double)se->azimuth0 + (double)col * (double)se->azimuth_step;
    const double st = sin(th), ct = cos(th), sf = sin(ph), cf = cos(ph);
    d[0] = ct * cf; d[1] = ct * sf; d[2] = st;
    nu[0] = sf; nu[1] = -cf; nu[2] = 0.0;
    nv[0] = st * cf; nv[1] = st * sf; nv[2] = -ct;
    return 1;
}

/* ------------------------------------------------------------------ Eq. 2 */
int or_intersect(const double M[9], const double nu[3], const double nv[3], double out[5]) {
    double a[3], b[3], w[3];
    for (int k = 0; k < 3; ++k) {   /* pull the planes back into (u,v,1): a = M^T n_u */
        a[k] = M[0 * 3 + k] * nu[0] + M[1 * 3 + k] * nu[1] + M[2 * 3 + k] * nu[2];
        b[k] = M[0 * 3 + k] * nv[0] + M[1 * 3 + k] * nv[1] + M[2 * 3 + k] * nv[2];
    }
    w[0] = a[1] * b[2] - a[2] * b[1];
    w[1] = a[2] * b[0] - a[0] * b[2];
    w[2] = a[0] * b[1] - a[1] * b[0];
    if (w[2] == 0.0) return 0;
    const double u = w[0] / w[2], v = w[1] / w[2];
    out[0] = u;
    out[1] = v;
    for (int r = 0; r < 3; ++r) out[2 + r] = M[r * 3 + 0] * u + M[r * 3 + 1] * v + M[r * 3 + 2];
    return 1;
}

/* Conditioning of the intersection: the 2x2 Jacobian of (u,v) with respect
 * to the two tangent angles of the unit ray direction, by central
 * differences (step 1e-6 rad), returned as sigma_max / sigma_min.  The ray
 * through a perturbed direction is written with a generic plane pair; by the
 * unified scheme any two distinct planes through the ray give the
 * same (u,v). */
static int uv_for_dir(const double M[9], const double d[3], double uv[2]) {
    double e[3] = {0, 0, 0};
    const double ax = fabs(d[0]), ay = fabs(d[1]), az = fabs(d[2]);
    e[(ax <= ay && ax <= az) ? 0 : (ay <= az ? 1 : 2)] = 1.0;
    double nu[3] = {d[1] * e[2] - d[2] * e[1], d[2] * e[0] - d[0] * e[2], d[0] * e[1] - d[1] * e[0]};
    double nv[3] = {d[1] * nu[2] - d[2] * nu[1], d[2] * nu[0] - d[0] * nu[2], d[0] * nu[1] - d[1] * nu[0]};
    double out[5];
    if (!or_intersect(M, nu, nv, out)) return 0;
    uv[0] = out[0];
    uv[1] = out[1];
    return 1;
}

static double cond_uv(const double M[9], const double d0[3]) {
    const double dn = sqrt(d0[0] * d0[0] + d0[1] * d0[1] + d0[2] * d0[2]);
    const double d[3] = {d0[0] / dn, d0[1] / dn, d0[2] / dn};
    double e[3] = {0, 0, 0};
    const double ax = fabs(d[0]), ay = fabs(d[1]), az = fabs(d[2]);
    e[(ax <= ay && ax <= az) ? 0 : (ay <= az ? 1 : 2)] = 1.0;
    double t1[3] = {d[1] * e[2] - d[2] * e[1], d[2] * e[0] - d[0] * e[2], d[0] * e[1] - d[1] * e[0]};
    const double n1 = sqrt(t1[0] * t1[0] + t1[1] * t1[1] + t1[2] * t1[2]);
    for (int k = 0; k < 3; ++k) t1[k] /= n1;
    const double t2[3] = {d[1] * t1[2] - d[2] * t1[1], d[2] * t1[0] - d[0] * t1[2], d[0] * t1[1] - d[1] * t1[0]};
    const double h = 1e-6;
    double J[2][2];
    const double *ts[2] = {t1, t2};
    for (int a = 0; a < 2; ++a) {
        double dp[3], dm[3], up[2], um[2];
        for (int k = 0; k < 3; ++k) { dp[k] = d[k] + h * ts[a][k]; dm[k] = d[k] - h * ts[a][k]; }
        if (!uv_for_dir(M, dp, up) || !uv_for_dir(M, dm, um)) return INFINITY;
        J[0][a] = (up[0] - um[0]) / (2 * h);
        J[1][a] = (up[1] - um[1]) / (2 * h);
    }
    /* singular values of a 2x2 matrix in closed form */
    const double f2 = J[0][0] * J[0][0] + J[0][1] * J[0][1] + J[1][0] * J[1][0] + J[1][1] * J[1][1];
    const double det = fabs(J[0][0] * J[1][1] - J[0][1] * J[1][0]);
    const double disc = sqrt(fmax(f2 * f2 - 4.0 * det * det, 0.0));
    const double smax = sqrt(0.5 * (f2 + disc)), smin2 = 0.5 * (f2 - disc);
    const double smin = smin2 > 0 ? det / smax : 0.0;
    return smin > 0 ? smax / smin : INFINITY;
}

/* ------------------------------------------------------------- per surfel API */
int or_keys(const or_scene *sc, const or_sensor *se, const or_opts *op, uint32_t *key_bits,
            uint8_t *culled) {
    if (!sc || !se || !op || sc->n < 0) return -1;
    for (int64_t i = 0; i < sc->n; ++i) {
        double x[3];
        centre_sensor(se, sc->means + 3 * i, x);
        float k = depth_key(se, x);
        memcpy(&key_bits[i], &k, 4);
        if (culled) culled[i] = !(k >= (float)op->near_) || !isfinite(k);
    }
    return 0;
}

int or_surfel(const or_scene *sc, const or_sensor *se, const or_opts *op, int64_t i,
              double out[18]) {
    if (!sc || i < 0 || i >= sc->n) return -1;
    surf_t s;
    prep_surfel(sc, se, op, i, &s);
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) out[3 * r + c] = s.M[r][c];
    out[9] = s.c[0]; out[10] = s.c[1]; out[11] = s.cdepth;
    for (int r = 0; r < 3; ++r) { out[12 + r] = s.ns[r]; out[15 + r] = s.val[r]; }
    return s.culled;
}

/* --------------------------------------------------------------- render */
typedef struct {
    uint32_t key;
    int64_t idx;
    int contributes;     /* passes the contribution test of DESIGN.md §2 step 7 */
    uint8_t near_flags;  /* near-decision bits for this (ray, surfel) */
    double alpha, depth, val[3], ns[3];
    /* alternatives used only by or_render_variants:
     * the other rho3d/rho2d branch (ORF_BRANCH) and the fp32 uncertainty
     * interval of alpha of an ill-conditioned intersection (ORF_COND) */
    int contributes_alt;
    double alpha_alt, depth_alt, alpha_lo, alpha_hi;
} cand_t;

static int cand_cmp(const void *pa, const void *pb) {
    const cand_t *a = (const cand_t *)pa, *b = (const cand_t *)pb;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    return (a->idx > b->idx) - (a->idx < b->idx);
}

/* cheap per-surfel data for the result-neutral prefilter */
typedef struct { double mus[3], c[2], reach; int culled; } pre_t;

/* one sample's ray (Eqs. 3, 5; R4) */
typedef struct {
    int valid;
    uint8_t fl;           /* ray-level flags (ORF_FOV) */
    double nu[3], nv[3], d[3], p[2], dh[3];
} ray_t;

static void make_ray(const or_sensor *se, int64_t ray, ray_t *R) {
    const int32_t col = (int32_t)(ray % se->width), row = (int32_t)(ray / se->width);
    R->valid = or_ray(se, col, row, R->nu, R->nv, R->d, R->p);
    const double dn = sqrt(R->d[0] * R->d[0] + R->d[1] * R->d[1] + R->d[2] * R->d[2]);
    for (int k = 0; k < 3; ++k) R->dh[k] = R->d[k] / dn;
    R->fl = 0;
    if (se->kind == OR_FISHEYE) {
        const double mx = (R->p[0] - se->cx) / se->fx, my = (R->p[1] - se->cy) / se->fy;
        const double tdmax = or_kb_theta_d(se->k, se->theta_max);
        if (fabs(sqrt(mx * mx + my * my) - tdmax) < 1e-6 * tdmax) R->fl |= ORF_FOV;
    }
}

static void prefilter_data(const or_scene *sc, const or_sensor *se, const or_opts *op, pre_t *pre) {
    const double sup = op->support_rho;
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
    for (int64_t i = 0; i < sc->n; ++i) {
        centre_sensor(se, sc->means + 3 * i, pre[i].mus);
        float k = depth_key(se, pre[i].mus);
        pre[i].culled = !(k >= (float)op->near_) || !isfinite(k);
        project_centre(se, pre[i].mus, pre[i].c);
        const double su = sc->scales[2 * i], sv = sc->scales[2 * i + 1];
        pre[i].reach = 1.05 * sqrt(sup) * (su > sv ? su : sv);
    }
}

/* Evaluate surfel i on ray R (DESIGN.md §2 steps 4-7 and the §5 flags).
 * Returns 1 and fills *c if the pair contributes or carries a flag. */
static int eval_pair(const or_scene *sc, const or_sensor *se, const or_opts *op, const pre_t *q,
                     int64_t i, const ray_t *R, cand_t *c) {
    const int cam = se->kind != OR_LIDAR;
    const double sup = op->support_rho;
    const double inv_s2 = 1.0 / (op->lowpass_sigma * op->lowpass_sigma);
    if (q->culled) return 0;
    if (op->prefilter) {
        /* exact reject: rho3d <= sup needs the hit point within
         * sqrt(sup)*s_max of mu, i.e. the ray line within that
         * distance of mu; rho2d <= sup needs |p-c| <= sqrt(sup)*sigma */
        const double along = q->mus[0] * R->dh[0] + q->mus[1] * R->dh[1] + q->mus[2] * R->dh[2];
        const double m2 = q->mus[0] * q->mus[0] + q->mus[1] * q->mus[1] + q->mus[2] * q->mus[2];
        const double dist2 = m2 - along * along;
        int maybe = dist2 <= q->reach * q->reach;
        if (!maybe && cam) {
            const double ex = R->p[0] - q->c[0], ey = R->p[1] - q->c[1];
            const double lim = 1.05 * sqrt(sup) * op->lowpass_sigma;
            maybe = ex * ex + ey * ey <= lim * lim;
        }
        if (!maybe) return 0;
    }
    surf_t s;
    prep_surfel(sc, se, op, i, &s);
    /* Eq. 2: intersect the ray's plane pair with the splat */
    double hit[5];
    const int h = or_intersect((const double *)s.M, R->nu, R->nv, hit);
    const double rho3 = h ? hit[0] * hit[0] + hit[1] * hit[1] : INFINITY;
    const double t = !h ? NAN
                     : se->kind == OR_PINHOLE ? hit[4]
                     : hit[2] * R->d[0] + hit[3] * R->d[1] + hit[4] * R->d[2];
    double rho, depth, rho2 = INFINITY;
    int use3 = 1;
    if (cam) {   /* 2DGS low-pass floor, sigma = 1/sqrt(2) px */
        const double ex = R->p[0] - s.c[0], ey = R->p[1] - s.c[1];
        rho2 = (ex * ex + ey * ey) * inv_s2;
        use3 = rho3 <= rho2;
        rho = use3 ? rho3 : rho2;
        depth = use3 ? t : s.cdepth;
    } else {
        rho = rho3;
        depth = t;
    }
    const double G = exp(-0.5 * rho);
    double alpha = s.o * G;
    if (alpha > op->alpha_max) alpha = op->alpha_max;
    const int contributes = rho <= sup && depth >= op->near_ && alpha >= op->alpha_min;
    /* near-decision window: relative width
     * w = OR_W_FLOOR + 2^-22 * cond, cond = conditioning of the
     * intersection (u,v) w.r.t. the ray direction (3D branch
     * only); evaluated only when a broad 1e-2 window is hit.
     * OR_W_FLOOR = 2e-6 = 34 fp32 ulps: the fp32 evaluation error of
     * rho, alpha and the hit depth of a well-conditioned pair is a few
     * ulps; the cond term covers the ill-conditioned ones. */
    uint8_t nf = 0;
    double w = 0.0;
    {
        const double W0 = 1e-2;
        const int near_any = rho <= sup * (1 + W0) && alpha >= op->alpha_min * (1 - W0) &&
            depth >= op->near_ * (1 - W0) &&
            (fabs(rho - sup) < sup * W0 || fabs(alpha - op->alpha_min) < op->alpha_min * W0 ||
             fabs(depth - op->near_) < op->near_ * W0 ||
             (cam && fabs(rho3 - rho2) < W0 * (rho3 > rho2 ? rho3 : rho2)));
        if (near_any || (contributes && use3)) {
            const double cj = use3 ? cond_uv((const double *)s.M, R->d) : 1.0;
            w = OR_W_FLOOR + 2.384185791015625e-07 * cj;
            const int okr = rho <= sup * (1 + w), oka = alpha >= op->alpha_min * (1 - w),
                      okd = depth >= op->near_ * (1 - w);
            if (fabs(rho - sup) < sup * w && oka && okd) nf |= ORF_SUPPORT;
            if (fabs(alpha - op->alpha_min) < op->alpha_min * w && okr && okd) nf |= ORF_ALPHA;
            if (fabs(depth - op->near_) < op->near_ * w && okr && oka) nf |= ORF_NEAR;
            if (cam && okr && oka && okd && fabs(rho3 - rho2) < w * (rho3 > rho2 ? rho3 : rho2) &&
                fabs(t - s.cdepth) > 1e-12 * fabs(s.cdepth))
                nf |= ORF_BRANCH;
            /* ill-conditioned intersection: an fp32 evaluation may move
             * alpha by ~ alpha*rho*cond*2^-24; flag beyond 2.5e-5 */
            if (contributes && use3 && alpha * (rho3 > 0.1 ? rho3 : 0.1) * cj > 419.0)
                nf |= ORF_COND;
        }
    }
    if (!(contributes || nf)) return 0;
    memcpy(&c->key, &s.key, 4);
    c->idx = i;
    c->contributes = contributes;
    c->near_flags = nf;
    c->alpha = alpha;
    c->depth = depth;
    for (int k = 0; k < 3; ++k) { c->val[k] = s.val[k]; c->ns[k] = s.ns[k]; }
    /* the other branch (ORF_BRANCH): the same tests with the other rho */
    {
        const double rho_a = cam ? (use3 ? rho2 : rho3) : rho;
        const double dep_a = cam ? (use3 ? s.cdepth : t) : depth;
        double al = s.o * exp(-0.5 * rho_a);
        if (al > op->alpha_max) al = op->alpha_max;
        c->alpha_alt = al;
        c->depth_alt = dep_a;
        c->contributes_alt = rho_a <= sup && dep_a >= op->near_ && al >= op->alpha_min;
    }
    /* fp32 uncertainty of alpha (ORF_COND): rho within rho +- w*max(rho,0.1),
     * twice the predicted relative error 2*cond*2^-24 of rho3d */
    {
        const double e = w * (rho > 0.1 ? rho : 0.1);
        double lo = s.o * exp(-0.5 * (rho + e)), hi = s.o * exp(-0.5 * (rho - e > 0 ? rho - e : 0.0));
        c->alpha_lo = lo > op->alpha_max ? op->alpha_max : lo;
        c->alpha_hi = hi > op->alpha_max ? op->alpha_max : hi;
    }
    return 1;
}

/* All candidates of ray R in front-to-back (key, index) order (reading R9). */
static int64_t collect(const or_scene *sc, const or_sensor *se, const or_opts *op, const pre_t *pre,
                       const ray_t *R, cand_t **cands, int64_t *cap) {
    int64_t nc = 0;
    for (int64_t i = 0; i < sc->n; ++i) {
        if (nc == *cap) {
            *cap *= 2;
            cand_t *nb = (cand_t *)realloc(*cands, sizeof(cand_t) * (size_t)*cap);
            if (!nb) return -1;
            *cands = nb;
        }
        nc += eval_pair(sc, se, op, &pre[i], i, R, &(*cands)[nc]);
    }
    qsort(*cands, (size_t)nc, sizeof(cand_t), cand_cmp);
    return nc;
}

/* Outputs (DESIGN.md §2 step 10) from the composite state */
static void write_out(const or_sensor *se, const or_opts *op, int valid, double T, const double acc[3],
                      double D, const double Nr[3], double *o) {
    const double A = 1.0 - T;
    if (se->kind != OR_LIDAR) {
        if (!valid) {
            o[0] = op->bg_rgb[0]; o[1] = op->bg_rgb[1]; o[2] = op->bg_rgb[2];
            o[3] = 0.0; o[4] = o[5] = o[6] = 0.0; o[7] = 0.0;
        } else {
            for (int k = 0; k < 3; ++k) o[k] = acc[k] + T * op->bg_rgb[k];
            o[3] = A > 0.0 ? D / A : 0.0;
            for (int k = 0; k < 3; ++k) o[4 + k] = Nr[k];
            o[7] = A;
        }
    } else {
        o[0] = A > 0.0 ? D / A : op->bg_range;
        o[1] = acc[0];
        o[2] = acc[1] + T * op->bg_raydrop;
        o[3] = A;
        o[4] = o[5] = o[6] = o[7] = 0.0;
    }
}

int or_render(const or_scene *sc, const or_sensor *se, const or_opts *op, int64_t n_rays,
              const int64_t *ray_index, double *out, uint8_t *flags, int32_t *ncontrib,
              int nthreads) {
    if (!sc || !se || !op || !out || sc->n < 0 || se->width < 1 || se->height < 1) return -1;
    if (se->kind != OR_LIDAR && sc->n > 0 && !sc->sh) return -2;
    const int64_t N = sc->n;
    pre_t *pre = (pre_t *)malloc(sizeof(pre_t) * (size_t)(N > 0 ? N : 1));
    if (!pre) return -3;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
    prefilter_data(sc, se, op, pre);
    int err = 0;
#ifdef _OPENMP
#pragma omp parallel
#endif
    {
        int64_t cap = 1024;
        cand_t *cands = (cand_t *)malloc(sizeof(cand_t) * (size_t)cap);
        if (!cands) err = -3;
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 8)
#endif
        for (int64_t r = 0; r < n_rays; ++r) {
            if (!cands) continue;
            ray_t R;
            make_ray(se, ray_index ? ray_index[r] : r, &R);
            uint8_t fl = R.fl;
            const int64_t nc = R.valid ? collect(sc, se, op, pre, &R, &cands, &cap) : 0;
            if (nc < 0) { err = -3; continue; }
            /* front-to-back composite (north_star; DESIGN.md §2 step 9) */
            double T = 1.0, acc[3] = {0, 0, 0}, D = 0.0, Nr[3] = {0, 0, 0};
            int32_t used = 0;
            for (int64_t j = 0; j < nc; ++j) {
                const cand_t *c = &cands[j];
                fl |= c->near_flags;   /* a near decision before the ray stopped */
                if (!c->contributes) continue;
                const double Tn = T * (1.0 - c->alpha);
                if (fabs(Tn - op->t_min) < op->t_min * 1e-4) fl |= ORF_TSTOP;
                if (Tn < op->t_min) break;  /* stop; this surfel is not composited (R3) */
                const double wgt = c->alpha * T;
                for (int k = 0; k < 3; ++k) { acc[k] += wgt * c->val[k]; Nr[k] += wgt * c->ns[k]; }
                D += wgt * c->depth;
                T = Tn;
                ++used;
            }
            write_out(se, op, R.valid, T, acc, D, Nr, out + 8 * r);
            if (flags) flags[r] = fl;
            if (ncontrib) ncontrib[r] = used;
        }
        free(cands);
    }
    free(pre);
    return err;
}

/* ------------------------------------------------- near-decision variants
 * DESIGN.md §5 (strict two-sided gate for flagged rays).  A flagged ray's
 * result is not unique in fp32: each near decision may fall either way and an
 * ill-conditioned intersection leaves alpha uncertain within an interval.
 * The variants are every composite the definition gives when each flagged
 * (ray, surfel) pair takes each of its admissible states:
 *   SUPPORT/ALPHA/NEAR  contributes or not;
 *   BRANCH              the rho3d or the rho2d branch (each with its own tests);
 *   COND                alpha nominal or at either end of its interval;
 *   TSTOP               a step whose T(1-alpha) is within 1e-4 relative of
 *                       t_min stops or composites;
 *   FOV                 the fisheye sample is inside or outside the FOV.
 * Variant 0 is always the nominal composite (the one or_render returns). */
typedef struct {
    const or_sensor *se;
    const or_opts *op;
    const cand_t *c;
    int64_t nc;
    int valid;
    int32_t max_var, count;
    double *out;          /* [max_var, 8] */
    uint8_t seen;         /* union of flags met on any variant path */
} var_ctx;

typedef struct { int contributes; double alpha, depth; } state_t;

/* admissible states of a flagged pair; state 0 is the nominal one */
static int cand_states(const cand_t *c, state_t st[8]) {
    int n = 0;
    const uint8_t f = c->near_flags;
    const int dec = (f & (ORF_SUPPORT | ORF_ALPHA | ORF_NEAR)) != 0;
    for (int b = 0; b < ((f & ORF_BRANCH) ? 2 : 1); ++b) {
        const double al = b ? c->alpha_alt : c->alpha, dp = b ? c->depth_alt : c->depth;
        const int con = b ? c->contributes_alt : c->contributes;
        for (int t = 0; t < (dec ? 2 : 1); ++t) {
            const int cc = t ? !con : con;
            st[n++] = (state_t){cc, al, dp};
            if (cc && !b && (f & ORF_COND)) {
                st[n++] = (state_t){1, c->alpha_lo, dp};
                st[n++] = (state_t){1, c->alpha_hi, dp};
            }
        }
    }
    return n;
}

/* Composite candidates j.. from state (T, acc, D, Nr); branch at every
 * flagged pair and every near-t_min stop; write one output per leaf. */
static void var_walk(var_ctx *x, int64_t j, double T, const double acc0[3], double D,
                     const double Nr0[3]) {
    double acc[3] = {acc0[0], acc0[1], acc0[2]}, Nr[3] = {Nr0[0], Nr0[1], Nr0[2]};
    const double tmin = x->op->t_min;
    for (; j < x->nc; ++j) {
        if (x->count > x->max_var) return;
        const cand_t *c = &x->c[j];
        x->seen |= c->near_flags;
        state_t st[8];
        const int ns = c->near_flags ? cand_states(c, st) : 1;
        if (!c->near_flags) st[0] = (state_t){c->contributes, c->alpha, c->depth};
        for (int k = 0; k < ns; ++k) {
            const state_t s = st[k];
            if (!s.contributes) {
                if (ns == 1) goto next;
                var_walk(x, j + 1, T, acc, D, Nr);
                continue;
            }
            const double Tn = T * (1.0 - s.alpha);
            const int near_stop = fabs(Tn - tmin) < tmin * 1e-4;
            if (near_stop) x->seen |= ORF_TSTOP;
            if (ns == 1 && !near_stop) {
                if (Tn < tmin) goto done;   /* stop; not composited (R3) */
                const double wgt = s.alpha * T;
                for (int q = 0; q < 3; ++q) { acc[q] += wgt * c->val[q]; Nr[q] += wgt * c->ns[q]; }
                D += wgt * s.depth;
                T = Tn;
                goto next;
            }
            /* the nominal decision first, then (near t_min) the other one */
            for (int o = 0; o < (near_stop ? 2 : 1); ++o) {
                const int stop = o ? !(Tn < tmin) : (Tn < tmin);
                if (stop) {
                    var_walk(x, x->nc, T, acc, D, Nr);
                } else {
                    const double wgt = s.alpha * T;
                    double a3[3], N3[3];
                    for (int q = 0; q < 3; ++q) { a3[q] = acc[q] + wgt * c->val[q]; N3[q] = Nr[q] + wgt * c->ns[q]; }
                    var_walk(x, j + 1, Tn, a3, D + wgt * s.depth, N3);
                }
            }
        }
        return;
    next:;
    }
done:
    if (x->count < x->max_var) write_out(x->se, x->op, x->valid, T, acc, D, Nr, x->out + 8 * x->count);
    x->count++;
}

int or_render_variants(const or_scene *sc, const or_sensor *se, const or_opts *op, int64_t n_rays,
                       const int64_t *ray_index, int32_t max_var, double *var_out, int32_t *nvar,
                       uint8_t *seen, int nthreads) {
    if (!sc || !se || !op || !var_out || !nvar || sc->n < 0 || max_var < 1 || se->width < 1 ||
        se->height < 1)
        return -1;
    if (se->kind != OR_LIDAR && sc->n > 0 && !sc->sh) return -2;
    const int64_t N = sc->n;
    pre_t *pre = (pre_t *)malloc(sizeof(pre_t) * (size_t)(N > 0 ? N : 1));
    if (!pre) return -3;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
    prefilter_data(sc, se, op, pre);
    int err = 0;
#ifdef _OPENMP
#pragma omp parallel
#endif
    {
        int64_t cap = 1024;
        cand_t *cands = (cand_t *)malloc(sizeof(cand_t) * (size_t)cap);
        if (!cands) err = -3;
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int64_t r = 0; r < n_rays; ++r) {
            if (!cands) continue;
            ray_t R;
            make_ray(se, ray_index ? ray_index[r] : r, &R);
            /* a FOV-edge sample also gets the variants of the other side */
            const int64_t nc = (R.valid || (R.fl & ORF_FOV)) ? collect(sc, se, op, pre, &R, &cands, &cap) : 0;
            if (nc < 0) { err = -3; continue; }
            var_ctx x = {se, op, cands, nc, R.valid, max_var, 0, var_out + (size_t)8 * max_var * r, R.fl};
            const double z3[3] = {0, 0, 0};
            var_walk(&x, 0, 1.0, z3, 0.0, z3);
            if (R.fl & ORF_FOV) {
                x.valid = !R.valid;
                var_walk(&x, 0, 1.0, z3, 0.0, z3);
            }
            nvar[r] = x.count;
            if (seen) seen[r] = x.seen;
        }
        free(cands);
    }
    free(pre);
    return err;
}

/* Conditioning of the intersection (exported for the flag-logic pins). */
double or_cond_uv(const double M[9], const double d[3]) { return cond_uv(M, d); }
