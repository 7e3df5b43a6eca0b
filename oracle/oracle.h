/*
 * oracle.h -- CPU fp64 brute-force reference for the 2DGS sensor renderer.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this.
 * The product path (paper_2503_11731_b200/, include/gsr.h) never includes,
 * links or executes anything under oracle/.  This header deliberately
 * re-declares its own structs: it shares no header, helper or constant with
 * the CUDA path.
 *
 * What it computes is the definition written in DESIGN.md §2, which follows
 * PAPER.md §III-A "Unified Projection Scheme" (Eqs. 1-5), the 2DGS
 * low-pass filter and BASELINE.json north_star's compositing rule.
 */
#ifndef GSR_ORACLE_H
#define GSR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_PINHOLE = 0, OR_FISHEYE = 1, OR_LIDAR = 2, OR_CYLINDRICAL = 3 };

typedef struct {
    int64_t n;
    const float *means;          /* [n,3] world */
    const float *quats;          /* [n,4] (w,x,y,z), normalised here */
    const float *scales;         /* [n,2] s_u, s_v */
    const float *opacities;      /* [n] */
    const float *sh;             /* [n,(d+1)^2,3] (cameras) */
    int32_t sh_degree;
    const float *intensity;      /* [n] (LiDAR) */
    const float *raydrop_logit;  /* [n] (LiDAR) */
} or_scene;

typedef struct {
    int32_t kind, width, height;
    float w2s[12];               /* [R|t] row-major, p_s = R p_w + t */
    float fx, fy, cx, cy;
    float k[4];
    float theta_max;
    const float *beam_elevation; /* [height] */
    float azimuth0, azimuth_step;
} or_sensor;

typedef struct {
    double near_, alpha_max, alpha_min, t_min, support_rho, lowpass_sigma;
    double bg_rgb[3], bg_range, bg_raydrop;
    int32_t prefilter;           /* 1: exact bounding reject (result-neutral), 0: test every surfel */
} or_opts;

/* flags (per ray) -- "near-decision" bits, DESIGN.md §5 tolerance protocol */
enum { ORF_ALPHA = 1, ORF_SUPPORT = 2, ORF_NEAR = 4, ORF_TSTOP = 8, ORF_FOV = 16,
       ORF_BRANCH = 32, ORF_COND = 64 };

/* Render n_rays samples (ray index = row*width + col; NULL -> all rays in
 * order).  out: [n_rays, 8] doubles.  Camera channels: r,g,b,depth,nx,ny,nz,alpha.
 * LiDAR channels: range,intensity,raydrop,alpha,0,0,0,0.  flags: [n_rays] u8
 * (may be NULL).  ncontrib: [n_rays] i32 composited-surfel count (may be NULL).
 * Returns 0 on success, <0 on bad arguments. */
int or_render(const or_scene *sc, const or_sensor *se, const or_opts *op, int64_t n_rays,
              const int64_t *ray_index, double *out, uint8_t *flags, int32_t *ncontrib,
              int nthreads);

/* Near-decision variants of each ray (DESIGN.md §5 strict two-sided gate):
 * every composite the definition gives when each flagged (ray, surfel) pair
 * takes each admissible state (decision either way, the other rho branch,
 * alpha at the ends of its fp32 interval, a near-t_min stop either way, a
 * FOV-edge sample either side).  var_out: [n_rays, max_var, 8], variant 0 is
 * the nominal composite; nvar[r] = number of variants (> max_var: only the
 * first max_var were written, the ray is unresolved); seen[r] (may be NULL) =
 * union of the flags met on any variant path. */
int or_render_variants(const or_scene *sc, const or_sensor *se, const or_opts *op, int64_t n_rays,
                       const int64_t *ray_index, int32_t max_var, double *var_out, int32_t *nvar,
                       uint8_t *seen, int nthreads);

/* sigma_max / sigma_min of d(u,v)/d(ray tangent angles) at direction d for
 * the splat M (row-major, sensor frame): the conditioning used by the flags. */
double or_cond_uv(const double M[9], const double d[3]);

/* Per-surfel sort key (reading R9): fp32 bits of the pinned fp64
 * depth, and the cull flag (key < near or non-finite). */
int or_keys(const or_scene *sc, const or_sensor *se, const or_opts *op, uint32_t *key_bits,
            uint8_t *culled);

/* Per-surfel intermediates: out[0..8] M (row-major, sensor frame, columns
 * s_u t_u | s_v t_v | mu_s), out[9..10] projected centre (cameras),
 * out[11] centre depth (pinhole z, else range), out[12..14] oriented normal,
 * out[15..17] colour (cameras) or (intensity, p_drop, 0) (LiDAR). */
int or_surfel(const or_scene *sc, const or_sensor *se, const or_opts *op, int64_t i,
              double out[18]);

/* Ray of sample (col,row): n_u, n_v (plane normals through the sensor
 * origin), direction d, pixel position p (cameras).  Returns 1 if the sample
 * is valid (fisheye: inside the FOV), 0 otherwise. */
int or_ray(const or_sensor *se, int32_t col, int32_t row, double nu[3], double nv[3],
           double d[3], double p[2]);

/* Eq. 2 intersection of the splat M (row-major 3x3, sensor frame) with the
 * planes (nu,nv): out = (u, v, hit point P[3]); returns 0 if w3 == 0. */
int or_intersect(const double M[9], const double nu[3], const double nv[3], double out[5]);

/* Real SH basis, 3DGS ordering (16 values for degree 3) at unit dir. */
void or_sh_basis(const double dir[3], double out[16]);

/* Fisheye helpers: theta_d(theta) and its inverse on [0, theta_max]. */
double or_kb_theta_d(const float k[4], double theta);
double or_kb_inverse(const float k[4], double theta_max, double theta_d);

#ifdef __cplusplus
}
#endif
#endif
