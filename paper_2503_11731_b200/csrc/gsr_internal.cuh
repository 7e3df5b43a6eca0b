// gsr_internal.cuh -- device-side data layouts shared by the kernels of the
// B200 2DGS renderer (include/gsr.h).  Product code: never includes oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "../../include/gsr.h"

namespace gsr {

// ---------------------------------------------------------------- params
struct DevSensor {
    int32_t kind, width, height;
    int32_t tw, th, ntx, nty;   // binning tile (one CTA) and tile grid
    int32_t sw, sh;             // warp sub-tile (32 samples: 8x4, 16x2 or 32x1)
    float R[9], t[3];           // world -> sensor
    float fx, fy, cx, cy;
    float k[4];
    float theta_max;
    double tdmax;               // fisheye theta_d(theta_max), fp64
    float ow[3];                // sensor origin in world (view direction for SH)
    float az0, az_step;
    int32_t nbeams;
    int32_t full_turn;          // LiDAR: width*az_step covers 2pi (azimuth wraps)
    uint32_t mtw, mth;          // ceil(2^32 / tw), ceil(2^32 / th) (0 for 1): exact division of pixel indices (n d < 2^32)
    float beam[GS_MAX_BEAMS];
    float sbeam[GS_MAX_BEAMS];  // sin(beam), fp64-evaluated, rounded to fp32
};

struct DevOpts {
    float near_plane, alpha_max, alpha_min, t_min, support, sigma2, inv_sigma2;
    float bg[3];
    float bg_range, bg_raydrop;
    float grid_share;   // host side: fraction of the compositor's resident CTA slots to launch
};

struct DevSurfels {
    int64_t n;
    const float *means, *quats, *scales, *opac, *sh, *inten, *drop;
    int32_t sh_degree;
    const float *bounds;   // optional block bounds (gs_cull_bounds), [n / SCAN_TILE][8]
};

// ---------------------------------------------------------------- records
// One AoS record per surfel, written by gs_project, gathered into shared
// memory by the compositing kernels (16-byte chunks).
//
// Pinhole (24 floats): the intersection of pixel p = c + (dx,dy) with the
// surfel is (u,v) = (q0,q1)/q2, camera z = det/q2 (the A entries column-major,
// so that (q0, q1) is one packed f32x2 multiply-add per column), where
//   q0 = A00 dx + A01 dy, q1 = A10 dx + A11 dy, q2 = qc + A20 dx + A21 dy
// (the first two columns of adj(K M) scaled by 1/(s_u s_v); c the projected
// centre, stored hi+lo).  See DESIGN.md §6.
enum : int {
    PH_A00 = 0, PH_A10, PH_A01, PH_A11, PH_A20, PH_A21, PH_QC, PH_RCUT3,
    PH_CHX = 8, PH_CHY, PH_CLX, PH_CLY, PH_RCUT2, PH_O, PH_DET, PH_ZC,
    PH_R = 16, PH_G, PH_B, PH_NX, PH_NY, PH_NZ, PH_BBX, PH_BBY, PH_FLOATS = 24
};
// PH_BBX / PH_BBY (and FE_, LI_ alike): conservative pixel bounding box of the
// surfel's support, inclusive, as two packed u16 pairs (lo | hi << 16); for
// LiDAR the column range may run past width-1 (azimuth wrap).  Pinhole: the
// box of the 3-sigma disk alone (empty: lo = 0xffff, hi = 0); the low-pass
// disc is the circle of radius^2 PH_RCUT2 about the centre.
// Fisheye / LiDAR (ray direction d = m + e, m = unit centre direction,
// stored hi+lo): u = U.e / D, v = V.e / D, range t = rdet / D, D = det + N.e.
enum : int {
    RY_MH = 0, RY_RCUT3 = 3, RY_ML = 4, RY_DET = 7, RY_U = 8, RY_O = 11, RY_V = 12, RY_RDET = 15,
    RY_N = 16, RY_RC = 19,
    FE_CHX = 20, FE_CHY, FE_CLX, FE_CLY, FE_RCUT2, FE_PAD0, FE_BBX, FE_BBY,
    FE_R = 28, FE_G, FE_B, FE_NX, FE_NY, FE_NZ, FE_FLOATS = 36,
    LI_INT = 20, LI_DROP = 21, LI_BBX = 22, LI_BBY = 23, LI_FLOATS = 24
};

__host__ __device__ inline float pack_bb(int lo, int hi) {
    const uint32_t u = ((uint32_t)lo & 0xffffu) | ((uint32_t)hi << 16);
#ifdef __CUDA_ARCH__
    return __uint_as_float(u);
#else
    float f;
    memcpy(&f, &u, 4);
    return f;
#endif
}

// cameras whose rays are unit directions through the optical centre (records
// relative to the centre direction): equidistant and cylindrical fisheye
__host__ __device__ constexpr bool dir_camera(int kind) {
    return kind == GS_FISHEYE_EQUIDISTANT || kind == GS_FISHEYE_CYLINDRICAL;
}

__host__ __device__ inline int record_floats(int kind) {
    return kind == GS_PINHOLE ? (int)PH_FLOATS : (dir_camera(kind) ? (int)FE_FLOATS : (int)LI_FLOATS);
}

// ---------------------------------------------------------------- projected buffer
// [ header 256 B | records n*rec | rect n*8 | key n*4 | count n*4 |
//   vis_key n*4 | vis_id n*4 | cand n*4 | tile mask n*8 (LiDAR) |
//   row table n*32 (pinhole) | scan status 3*(nblk+1)*8 ]
// Row table (pinhole rects of >= KT_MIN_AREA tiles, <= PH_ROWS_MAX rows, <= 255
// columns): u16 per tile row of the rect, first column (relative to the rect)
// in the low byte and the number of tiles in the high byte (binning.cuh).
// Tile mask (LiDAR): bit k = tile k of the rect in row-major order holds a
// contributing ray (binning.cuh li_tile_hits); ~0 = every tile of the rect
// (rects of more than 64 tiles).
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_TILE = SCAN_ITEMS * SCAN_THREADS;

struct ProjHeader {
    uint32_t n_visible;
    uint32_t n_cand;            // surfels that pass the conservative cull (k_cull)
    int64_t num_pairs;
    uint32_t scan_counter;      // dynamic tile id for the compaction scan
    uint32_t cull_counter;      // dynamic tile id for the cull scan
    uint32_t pad1[58];
};
static_assert(sizeof(ProjHeader) == 256, "header");

__host__ __device__ inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct ProjLayout {
    size_t rec, rect, key, cnt, vkey, vid, cand, tmask, rows, status, nblk, total;
    __host__ __device__ ProjLayout(int64_t n, int kind) {
        size_t N = (size_t)(n > 0 ? n : 0);
        nblk = (N + SCAN_TILE - 1) / SCAN_TILE;
        rec = 256;
        rect = rec + align256(N * record_floats(kind) * 4);
        key = rect + align256(N * 8);
        cnt = key + align256(N * 4);
        vkey = cnt + align256(N * 4);
        vid = vkey + align256(N * 4);
        cand = vid + align256(N * 4);
        tmask = cand + align256(N * 4);
        rows = tmask + align256(kind == GS_LIDAR_SPINNING ? N * 8 : 0);
        status = rows + align256(kind == GS_PINHOLE ? N * 32 : 0);
        total = status + align256(3 * (nblk + 1) * 8);
    }
};

// ---------------------------------------------------------------- helpers
// Process-wide count of kernels launched by the library (diagnostic for
// gs_kernel_launches(); the only mutable state, a relaxed atomic).
void note_launch(int k = 1);

__device__ __forceinline__ void split_hilo(double x, float &hi, float &lo) {
    hi = (float)x;
    lo = (float)(x - (double)hi);
}

}  // namespace gsr
