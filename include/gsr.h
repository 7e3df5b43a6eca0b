/*
 * gsr.h -- C-ABI of the B200-native 2DGS camera + LiDAR renderer
 *          (hot path of arXiv 2503.11731, §III-A).
 *
 *   gs_project  ->  gs_bin_sort  ->  gs_render_camera | gs_render_lidar
 *
 * Conventions for every entry point
 *   - Ownership: the caller owns every buffer.  The library never allocates
 *     and holds no pointer after a call returns; its only process state is a
 *     relaxed kernel-launch counter.
 *   - Memory: pointers named d_* and all array pointers inside gs_surfels and
 *     the output/work buffers are DEVICE pointers (cudaMalloc / torch);
 *     gs_sensor.beam_elevation is a HOST pointer (copied into kernel
 *     parameters).  Structs themselves are host memory, read during the call.
 *   - Asynchrony: all device work is enqueued on `stream` (a cudaStream_t; 0
 *     = legacy default stream).  No call synchronises the device.
 *   - Errors: arguments are validated synchronously on the host before any
 *     launch: GS_ERR_CONFIG (null required pointer, wrong sensor kind for the
 *     call, sh_degree outside 0..3, width/height < 1, buffer too small),
 *     GS_ERR_RANGE (focal <= 0, non-finite principal point, camera wider or
 *     taller than 65535 px, LiDAR wider than 32767 columns or with more than
 *     GS_MAX_BEAMS beams, non-monotone beam table, non-finite azimuth0,
 *     azimuth span outside (0, 2pi], theta_max outside (0, pi), a fisheye
 *     lens theta_d(theta) not strictly increasing on [0, theta_max] (checked
 *     on a 10^4-point grid, DESIGN reading R12), compositing constants out of
 *     range, tile shape outside 32..512 samples or not a multiple of a
 *     32-sample warp sub-tile), GS_ERR_CUDA
 *     (launch failure, from cudaGetLastError).  On any
 *     error nothing is enqueued after the failing launch; gs_last_error()
 *     returns a thread-local message.  Surfels with a non-finite mean, scale
 *     or depth, a scale <= 0 or an opacity <= 0 are not an error: they are
 *     culled (they meet no ray).
 *   - Reentrancy: calls are pure functions of their inputs; concurrent calls
 *     on different streams with distinct output buffers are safe.
 *   - Determinism: no floating-point atomics; outputs are bitwise
 *     reproducible for identical inputs and options on the same GPU type.
 *     Unsplit tile lists (split_len = INT32_MAX) composite the same per-sample
 *     sequence for every tile shape (bitwise equal images); split lists (whose
 *     adaptive length depends on the SM count and grid_share) differ only by
 *     fp32 rounding of the merge.
 *
 * Sizing protocol (the pair count P is only known on the device):
 *   simple mode: gs_project, synchronise, read *d_num_pairs, allocate P
 *   pairs, gs_bin_sort.  Graph mode: pass a pair_capacity up front; if
 *   P > pair_capacity gs_bin_sort sets *d_overflow = 1, leaves keys/values/
 *   tile_ranges undefined and the render calls produce background; re-run
 *   with a larger capacity.
 */
#ifndef GSR_H
#define GSR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *gs_stream;   /* == cudaStream_t */

typedef enum {
    GS_OK = 0,
    GS_ERR_CONFIG = 1,
    GS_ERR_RANGE = 2,
    GS_ERR_CAPACITY = 3,
    GS_ERR_CUDA = 4,
    GS_ERR_UNSUPPORTED = 5
} gs_status;

typedef enum {
    GS_PINHOLE = 0,               /* PAPER.md:96-100, Eq. 3                        */
    GS_FISHEYE_EQUIDISTANT = 1,   /* BASELINE Fisheye config; replaces Eq. 4 (DESIGN R4) */
    GS_LIDAR_SPINNING = 2,        /* PAPER.md:108-114, Eq. 5                       */
    GS_FISHEYE_CYLINDRICAL = 3    /* PAPER.md:102-106, Eq. 4 (cylindrical projection):
                                     column -> azimuth phi = (p_x - c_x)/f_x about the
                                     camera y axis, row -> p_y = c_y + f_y y / sqrt(x^2+z^2)
                                     (DESIGN reading R20); rendered by gs_render_camera */
} gs_sensor_kind;

#define GS_MAX_BEAMS 256

/* Surfel attributes {mu, R, S, rho, r, alpha} after decoding.
 * All device pointers, fp32, contiguous row-major, read-only. */
typedef struct {
    int64_t n;                   /* number of surfels, >= 0 (0 renders background)    */
    const float *means;          /* [n,3] world metres                                 */
    const float *quats;          /* [n,4] (w,x,y,z); normalised inside                 */
    const float *scales;         /* [n,2] s_u, s_v > 0 (linear)                         */
    const float *opacities;      /* [n] in [0,1] (post-sigmoid)                         */
    const float *sh;             /* [n,(d+1)^2,3] SH coefficients; cameras only         */
    int32_t sh_degree;           /* d in 0..3                                           */
    const float *intensity;      /* [n] LiDAR intensity r in [0,1]; LiDAR only          */
    const float *raydrop_logit;  /* [n] LiDAR ray-drop logit (p = sigmoid); LiDAR only  */
    const float *cull_bounds;    /* optional (NULL = none): gs_cull_bounds' output for
                                    exactly these means / scales, see below            */
} gs_surfels;

/* Block bounds for a hierarchical frustum cull (the paper renders from
 * per-zone resident sets, §III-A "Support Large-scale Scenes";
 * here every block of GS_CULL_BLOCK consecutive surfels carries a bound, so a
 * scene stored zone by zone is culled zone by zone without the renderer
 * knowing the zones).  bounds: device, [gs_cull_blocks(n)][8] fp32 =
 * min x,y,z and max x,y,z of the block's finite centres, the block's largest
 * finite scale, 0.  gs_project with surfels->cull_bounds set skips (pinhole
 * sensors) the per-surfel cull of a block that lies wholly outside the
 * frustum or in front of the near plane; its outputs are bitwise those
 * without bounds -- a skipped block holds only surfels the per-surfel cull
 * drops (tests/test_gpu_dims.py).  The bounds describe the arrays they were
 * computed from: recompute after any change of means or scales (one pass,
 * 20 bytes read per surfel; asynchronous on `stream`). */
#define GS_CULL_BLOCK 2048
int64_t gs_cull_blocks(int64_t n);
gs_status gs_cull_bounds(const gs_surfels *surfels, float *bounds, gs_stream stream);

/* Sensor model.  world_to_sensor = [R|t] row-major 3x4:
 * p_sensor = R p_world + t.  Camera frame x right, y down, z forward; LiDAR
 * frame x forward, y left, z up. */
typedef struct {
    int32_t kind;                /* gs_sensor_kind                                      */
    int32_t width, height;       /* pixels; LiDAR: width = azimuth columns, height = beams */
    float world_to_sensor[12];
    float fx, fy, cx, cy;        /* cameras: pixel (i,j) samples (i+1/2, j+1/2);
                                    cylindrical: the columns' azimuths must lie in [-pi, pi] */
    float k[4];                  /* fisheye Kannala-Brandt k1..k4 (theta_d polynomial)  */
    float theta_max;             /* fisheye half field of view (rad), in (0, pi)       */
    const float *beam_elevation; /* LiDAR [height] elevations (rad), strictly decreasing, HOST */
    float azimuth0, azimuth_step;/* LiDAR column j has azimuth azimuth0 + j*azimuth_step */
} gs_sensor;

/* Compositing constants (north_star); gs_default_opts() fills the defaults. */
typedef struct {
    int32_t tile_w, tile_h;      /* binning tile = the samples one CTA composites (16 x 8):
                                    32..512 samples, a multiple of a 32-sample warp
                                    sub-tile (cameras 8x4, then 16x2, 32x1; LiDAR 32x1,
                                    then 16x2, 8x4); GS_ERR_RANGE otherwise.  LiDAR:
                                    32 x 1 recommended.  Edge tiles may be partial.     */
    int32_t split_len;           /* tile lists longer than this are split into segments
                                    composited in parallel and merged (0 = adaptive: a
                                    quarter of a resident CTA's fair share of the
                                    frame's pairs, at least 1024; INT32_MAX disables)   */
    float near_plane;            /* 0.2 m                                               */
    float alpha_max;             /* 0.99                                                */
    float alpha_min;             /* 1/255                                               */
    float t_min;                 /* 1e-4 (0 disables early termination)                 */
    float support_rho;           /* 9 (3-sigma support, rho = u^2+v^2)                  */
    float lowpass_sigma_px;      /* 1/sqrt(2) px (cameras)                              */
    float bg_rgb[3];             /* 0,0,0                                               */
    float bg_range;              /* 0                                                   */
    float bg_raydrop;            /* 1                                                   */
    float grid_share;            /* fraction in (0, 1] of the compositor's resident CTA
                                    slots its persistent grid takes (0 = 1: the whole
                                    GPU).  A caller compositing k frames concurrently on
                                    k streams gives each about 2/k, so the frames'
                                    projection and binning kernels find free SMs.
                                    Results do not depend on it.  GS_ERR_RANGE outside
                                    [0, 1].                                             */
} gs_opts;

void gs_default_opts(gs_opts *opts);

/* Bytes of the per-surfel projection buffer for n surfels of this sensor
 * kind (records, tile rects, depth keys, counts, compaction lists, header). */
size_t gs_projected_bytes(int64_t n, int32_t kind);

/* Bytes of gs_bin_sort's workspace for n surfels and pair_capacity pairs. */
size_t gs_sort_workspace_bytes(int64_t n, int64_t pair_capacity, const gs_sensor *sensor,
                               const gs_opts *opts);

/* Number of tiles of the sensor's image under opts (tile_ranges has 2 u32
 * per tile). */
int64_t gs_num_tiles(const gs_sensor *sensor, const gs_opts *opts);

/*
 * gs_project -- per-surfel projection (Eq. 1; SH colour and
 * low-pass bound; attributes P:78).  For every surfel: the
 * sensor-frame local-to-sensor map of Eq. 1 in its intersection form, the
 * projected centre, the fp32 depth key (DESIGN reading R9), the oriented
 * normal, the SH colour (cameras) or intensity / ray-drop probability
 * (LiDAR), and the exact set of tiles whose samples the surfel's 3-sigma
 * support (cameras: or its low-pass disc) can reach: pinhole, per tile row
 * the columns the support conic / disc meets (widened by a slack above the
 * compositor's fp32 error); LiDAR (one-row tiles), per tile a conservative
 * minimum of the support quadric over the tile's ray arc; fisheye, the
 * conservative 3-sigma rectangle of tiles.  The stored rect contains the
 * set.  Then compacts the visible surfels and counts the (tile, surfel)
 * pairs (the sizes of those sets).
 *   projected       device buffer of >= gs_projected_bytes(n, kind) bytes (out)
 *   d_num_pairs     device int64 (out): total number of pairs P
 */
gs_status gs_project(const gs_surfels *surfels, const gs_sensor *sensor, const gs_opts *opts,
                     void *projected, size_t projected_bytes, int64_t *d_num_pairs,
                     gs_stream stream);

/*
 * gs_bin_sort -- tile binning (the tile-based splatting of PAPER.md:48, whose
 * per-tile depth-sorted lists the compositing walks front to back; sort order
 * = the depth key of DESIGN reading R9, ties by surfel index): a stable LSD
 * radix sort of the 64-bit
 * (tile << 32 | depth-key bits) pair keys (ties by surfel index), then tile
 * ranges.  The 32 depth bits are sorted once per visible surfel before the
 * pairs are emitted (an LSD sort may do its low digits on any order-preserving
 * expansion); the tile digits are then sorted over the P pairs.  A surfel's
 * pairs are the tile set gs_project counted (pinhole: the same row
 * intervals, recomputed from the same record floats; LiDAR: the stored tile
 * mask).
 *   projected       buffer written by gs_project for the same surfels/sensor/opts
 *   keys            device [pair_capacity] u64 (out, may be NULL): sorted keys
 *   values          device [pair_capacity] u32 (out): surfel index of each sorted pair
 *   tile_ranges     device [num_tiles, 2] u32 (out): [start, end) into values per tile
 *   workspace       device scratch of >= gs_sort_workspace_bytes() bytes
 *   d_overflow      device int32 (out): 1 if P > pair_capacity, else 0
 */
gs_status gs_bin_sort(const void *projected, int64_t n, const gs_sensor *sensor,
                      const gs_opts *opts, uint64_t *keys, uint32_t *values,
                      int64_t pair_capacity, uint32_t *tile_ranges, void *workspace,
                      size_t workspace_bytes, int32_t *d_overflow, gs_stream stream);

/*
 * gs_render_camera -- front-to-back compositing for pinhole and equidistant
 * fisheye cameras: per pixel, exact ray-splat intersection (Eq. 2)
 * with the unified plane pair (Eq. 3 / R4), low-pass floor, alpha =
 * min(alpha_max, o G), skip alpha < alpha_min, stop before T < t_min.
 * Outputs planar fp32 (any may be NULL except alpha):
 *   rgb [3,H,W], depth [H,W] (normalised expected depth, 0 where alpha = 0),
 *   normal [3,H,W] (sensor frame, unnormalised composite), alpha [H,W].
 * d_overflow (may be NULL) is gs_bin_sort's flag: if set, outputs are background.
 * workspace: device scratch of >= gs_render_workspace_bytes(pair_capacity, ...)
 * bytes (the pair_capacity given to gs_bin_sort): the longest-first tile
 * schedule and the partial composites of split tile lists.  The pair
 * capacity is taken to be the largest one whose workspace fits in
 * workspace_bytes; if the frame's pair count exceeds it (checked on the
 * device) the outputs are background, as for d_overflow.
 * stats (may be NULL): device [2,H,W] u32 diagnostic counts per sample --
 * surfels composited, (sample, surfel) pairs whose conservative pixel box
 * contains the sample.  Non-NULL selects an instrumented kernel.
 * Tiles whose list is shorter than opts->split_len are composited exactly in
 * list order (bitwise independent of the tile shape); longer lists are
 * composited in segments and merged with the transmittance prefix
 * C = sum_k (prod_{j<k} T_j) C_k, re-walking the segment where the ray
 * stops (exact stop rule; agrees with the unsplit result to fp32 rounding).
 */
size_t gs_render_workspace_bytes(int64_t pair_capacity, const gs_sensor *sensor,
                                 const gs_opts *opts);

gs_status gs_render_camera(const void *projected, int64_t n, const uint32_t *values,
                           const uint32_t *tile_ranges, const int32_t *d_overflow,
                           const gs_sensor *sensor, const gs_opts *opts, void *workspace,
                           size_t workspace_bytes, float *rgb, float *depth, float *normal,
                           float *alpha, uint32_t *stats, gs_stream stream);

/*
 * gs_render_lidar -- range-image compositing (Eq. 5; ray-drop and
 * intensity).  Outputs planar fp32 [H,W] each (any may be NULL
 * except alpha): range (0 = no return), intensity, raydrop probability
 * (composited with background 1), alpha.  stats as for gs_render_camera.
 */
gs_status gs_render_lidar(const void *projected, int64_t n, const uint32_t *values,
                          const uint32_t *tile_ranges, const int32_t *d_overflow,
                          const gs_sensor *sensor, const gs_opts *opts, void *workspace,
                          size_t workspace_bytes, float *range, float *intensity,
                          float *raydrop, float *alpha, uint32_t *stats, gs_stream stream);

/* ------------------------------------------------------------------------
 * Neural-Gaussian decode, the step upstream of
 * gs_project: PAPER.md:78 (§III-A "Scene Reconstruction") -- the final 2DGS
 * attributes {mu, R, S, rho, r, alpha} of each neural Gaussian are inferred
 * by passing the anchor features through per-head MLPs (Scaffold-GS anchors,
 * PAPER.md:49).  The paper fixes no sizes; DESIGN.md §12 readings N1-N6:
 * GS_NEURAL_K surfels per anchor, GS_NEURAL_F features, per head two hidden
 * layers of GS_NEURAL_HIDDEN with ReLU; geometry heads (offset, scale,
 * rotation) read the feature, appearance heads read [feature, d] with
 * d = normalize(position - view_origin).
 */
#define GS_NEURAL_K 5
#define GS_NEURAL_F 32
#define GS_NEURAL_HIDDEN 32

typedef enum { GS_DECODE_CAMERA = 0, GS_DECODE_LIDAR = 1 } gs_decode_modality;

/* heads, in this order (head index = position):
 *   camera: OFFSET (15 = 3k), SCALE (10), ROTATION (30, 6D per surfel), OPACITY (5), COLOR (15)
 *   LiDAR : OFFSET, SCALE, ROTATION, OPACITY, INTENSITY (5), RAYDROP (5)           */
enum { GS_HEAD_OFFSET = 0, GS_HEAD_SCALE = 1, GS_HEAD_ROTATION = 2, GS_HEAD_OPACITY = 3,
       GS_HEAD_COLOR = 4, GS_HEAD_INTENSITY = 4, GS_HEAD_RAYDROP = 5 };

typedef struct {                 /* device pointers, read-only */
    int64_t n;                   /* anchors, >= 0                                       */
    const float *position;       /* [n,3] world metres                                  */
    const uint16_t *feature;     /* [n,GS_NEURAL_F] IEEE fp16 bits, 16-byte aligned     */
    const float *base_scale;     /* [n,3] > 0                                           */
} gs_anchors;

typedef struct {                 /* one MLP: device pointers, read-only                 */
    const uint16_t *w1;          /* [HIDDEN, in] fp16 row-major; in = F (geometry heads)
                                    or F+3 (appearance heads: feature then d)           */
    const float *b1;             /* [HIDDEN]                                            */
    const uint16_t *w2;          /* [HIDDEN, HIDDEN] fp16                               */
    const float *b2;             /* [HIDDEN]                                            */
    const uint16_t *w3;          /* [out, HIDDEN] fp16 (out per head, see above)        */
    const float *b3;             /* [out]                                               */
} gs_mlp;

typedef struct {
    int32_t modality;            /* gs_decode_modality                                  */
    gs_mlp head[6];              /* 5 (camera) or 6 (LiDAR) heads                       */
} gs_decoder;

/*
 * gs_decode_anchors -- anchors -> the 5n surfels of a gs_surfels set, surfel 5a+j
 * from anchor a, output slot j, written to caller-owned device arrays:
 *   means [5n,3]   = position + offset_j * base_scale (elementwise)
 *   quats [5n,4]   (w,x,y,z), w >= 0, of the Gram-Schmidt frame (t_u, t_v,
 *                  t_u x t_v) of the 6D rotation output (a1, a2)
 *   scales [5n,2]  = (base_scale_0 exp(S_j0), base_scale_1 exp(S_j1))
 *   opacities [5n] = sigmoid(.)
 *   camera: sh [5n,1,3] = (sigmoid(colour) - 1/2) / C0 (degree-0 SH, so that
 *           gs_project's colour is the decoded colour); intensity/raydrop unused
 *   LiDAR : intensity [5n] = sigmoid(.), raydrop_logit [5n] = raw output; sh unused
 * Arithmetic: fp16 tensor-core MMAs (tcgen05) with fp32 accumulation; hidden
 * activations and d are rounded to fp16 (parity tolerance: DESIGN.md §12).
 * Errors: GS_ERR_CONFIG for a NULL required pointer, an unknown modality,
 * n < 0 or a feature pointer not 16-byte aligned.  n = 0 launches nothing.
 */
gs_status gs_decode_anchors(const gs_anchors *anchors, const gs_decoder *decoder, const float view_origin[3],
                            float *means, float *quats, float *scales, float *opacities, float *sh,
                            float *intensity, float *raydrop_logit, gs_stream stream);

/* ------------------------------------------------------------------------
 * Pixel-partitioned rendering of one frame over several GPUs (SURVEY.md
 * §8(f) NEXT-4; §III-A "Paralleled training": continuous
 * image regions per GPU and "a sparse all-to-all communication scheme to
 * transfer the required Gaussian data to corresponding pixel partitions").
 * Each rank owns a contiguous shard of the surfels and one band of tile
 * rows.  A rank projects its shard for the frame (gs_project), routes every
 * visible surfel to the bands its tile rect overlaps (gs_band_route), packs
 * the routed surfels' attributes per band (gs_pack_surfels) for the
 * all-to-all, and renders its band from the received surfels (unpacked in
 * source-rank order = global index order, so depth ties keep their order)
 * with the band's cropped sensor (paper_2503_11731_b200/pixdist.py).
 */
#define GS_MAX_BANDS 64

size_t gs_band_route_workspace_bytes(int64_t n, int32_t n_bands);

/* band_rows: HOST [n_bands+1] tile-row boundaries, band_rows[0] = 0 <
 * band_rows[1] < ... < band_rows[n_bands] = tile rows of the sensor under
 * opts.  d_counts: device [n_bands] u32 (out): surfels routed to each band.
 * d_index: device [n_bands, n] u32 (out): band b's surfel indices, ascending,
 * in d_index[b*n .. b*n + d_counts[b]).  GS_ERR_RANGE for a bad band table. */
gs_status gs_band_route(const void *projected, int64_t n, const gs_sensor *sensor, const gs_opts *opts,
                        const int32_t *band_rows, int32_t n_bands, uint32_t *d_counts, uint32_t *d_index,
                        void *workspace, size_t workspace_bytes, gs_stream stream);

/* floats per packed surfel: mean 3, quat 4, scale 2, opacity 1, SH
 * (sh_degree+1)^2*3 (sh_degree < 0: none), intensity 1 and ray-drop logit 1
 * if present */
int32_t gs_payload_floats(int32_t sh_degree, int32_t has_intensity, int32_t has_raydrop);

/* payload [m, gs_payload_floats] (device, out) <- the attributes of surfels
 * d_index[0..m) of src; src->sh may be NULL (no SH packed) */
gs_status gs_pack_surfels(const gs_surfels *src, const uint32_t *d_index, int64_t m, float *payload,
                          gs_stream stream);

/* device SoA arrays (out, [m,...]) <- payload [m, gs_payload_floats]; sh,
 * intensity and raydrop_logit are written only if present in the payload */
gs_status gs_unpack_surfels(const float *payload, int64_t m, int32_t sh_degree, int32_t has_intensity,
                            int32_t has_raydrop, float *means, float *quats, float *scales, float *opacities,
                            float *sh, float *intensity, float *raydrop_logit, gs_stream stream);

/* ------------------------------------------------------------------------
 * gs_render_backward -- backward pass of the compositing (SURVEY.md §8(f)
 * NEXT-2; training: PAPER.md:167, :214): the gradients of
 *     L = sum_{channel c, sample p} grad_out[c, p] * out[c, p]
 * (out = the frame gs_render_camera / gs_render_lidar produces: camera
 * r,g,b,depth,nx,ny,nz,alpha; LiDAR range,intensity,raydrop,alpha) with
 * respect to the surfel attributes, for GS_PINHOLE and GS_LIDAR_SPINNING
 * (GS_ERR_UNSUPPORTED for the fisheye kinds).  Uses the forward frame's
 * projected buffer, values and tile_ranges (same surfels, sensor and opts;
 * no overflow).  The backward recomposites every sample in fp32 from the
 * Eq. 1 splat matrix and differentiates the front-to-back recurrence (two
 * walks of each tile list).
 *   grad_out   device [C,H,W] fp32 (C = 8 camera, 4 LiDAR)
 *   workspace  device, >= gs_backward_workspace_bytes(n)
 * Outputs (device, overwritten, zero for surfels that meet no sample):
 *   d_means [n,3], d_quats [n,4] (w.r.t. the unnormalised input quaternion),
 *   d_scales [n,2], d_opacities [n], camera: d_sh [n,(d+1)^2,3] (may be NULL);
 *   LiDAR: d_intensity [n], d_raydrop_logit [n] (may be NULL).
 * Per-surfel sums use fp32 atomics: results are not bitwise reproducible.
 */
size_t gs_backward_workspace_bytes(int64_t n);

gs_status gs_render_backward(const gs_surfels *surfels, const gs_sensor *sensor, const gs_opts *opts,
                             const void *projected, const uint32_t *values, const uint32_t *tile_ranges,
                             const float *grad_out, void *workspace, size_t workspace_bytes, float *d_means,
                             float *d_quats, float *d_scales, float *d_opacities, float *d_sh,
                             float *d_intensity, float *d_raydrop_logit, gs_stream stream);

const char *gs_status_string(gs_status status);
const char *gs_last_error(void);

/* Cumulative number of CUDA kernels this library has launched in the process
 * (all entry points, all streams; memsets are not counted).  Diagnostic: the
 * difference across a region counts the library's launches in it. */
uint64_t gs_kernel_launches(void);

/* Bytes of one projected surfel record for this sensor kind (debug/tests). */
int32_t gs_record_bytes(int32_t kind);

/* Byte offsets inside the projected buffer (debug/tests): offs[0] records
 * [n, gs_record_bytes], offs[1] tile rects [n] int16x4 (x0,y0,x1,y1; x1 may
 * exceed the tile columns for LiDAR azimuth wrap), offs[2] depth keys [n] u32
 * (fp32 bits), offs[3] pair counts [n] u32 (0 for every culled surfel),
 * offs[4] total bytes.  Rects and keys are defined where the count is > 0
 * (surfels dropped by the conservative pre-cull keep whatever was there).  The header at offset 0 holds u32 n_visible at +0 and int64
 * num_pairs at +8. */
void gs_projected_offsets(int64_t n, int32_t kind, size_t offs[5]);

#ifdef __cplusplus
}
#endif
#endif /* GSR_H */
