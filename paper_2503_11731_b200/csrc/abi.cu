// abi.cu -- the C-ABI of include/gsr.h: host-side validation, parameter
// packing and launches.  Stateless: no allocation, no globals besides the
// thread-local error message.
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <atomic>

#include "gsr_internal.cuh"

namespace gsr {
cudaError_t launch_bounds(const DevSurfels &, float *, cudaStream_t);
cudaError_t launch_project(const DevSurfels &, const DevSensor &, const DevOpts &, void *, int64_t *,
                           cudaStream_t);
size_t sort_workspace_bytes(int64_t n, int64_t cap, int64_t ntiles);
cudaError_t launch_bin_sort(const void *proj, int64_t n, const DevSensor &se, int64_t ntiles,
                            uint64_t *keys, uint32_t *values, int64_t cap, uint32_t *ranges, void *ws,
                            int32_t *d_overflow, cudaStream_t st);
size_t render_workspace_bytes(int64_t cap, int64_t ntiles, int32_t split_len, int npix);
size_t band_route_workspace_bytes(int64_t n, int32_t nb);
cudaError_t launch_band_route(const void *proj, int64_t n, int kind, const int32_t *band_rows, int32_t nb,
                              uint32_t *d_counts, uint32_t *d_index, void *ws, cudaStream_t st);
int32_t payload_floats(int sh_floats, int has_int, int has_drop);
cudaError_t launch_pack(const DevSurfels &s, int sh_floats, const uint32_t *index, int64_t m, float *out,
                        cudaStream_t st);
cudaError_t launch_unpack(const float *in, int64_t m, int sh_floats, int has_int, int has_drop, float *means,
                          float *quats, float *scales, float *opac, float *sh, float *inten, float *drop,
                          cudaStream_t st);
size_t backward_workspace_bytes(int64_t n);
cudaError_t launch_backward(const DevSurfels &s, const DevSensor &se, const DevOpts &op, const void *proj,
                            const uint32_t *values, const uint32_t *ranges, const float *gout, void *ws,
                            float *d_means, float *d_quats, float *d_scales, float *d_opac, float *d_sh,
                            float *d_int, float *d_drop, cudaStream_t st);
cudaError_t launch_decode(const gs_anchors *, const gs_decoder *, const float[3], float *, float *, float *,
                          float *, float *, float *, float *, cudaStream_t);
cudaError_t launch_render_camera(const void *, int64_t, const uint32_t *, const uint32_t *,
                                 const int32_t *, const DevSensor &, const DevOpts &, int32_t, void *,
                                 size_t, float *, float *, float *, float *, uint32_t *, cudaStream_t);
cudaError_t launch_render_lidar(const void *, int64_t, const uint32_t *, const uint32_t *,
                                const int32_t *, const DevSensor &, const DevOpts &, int32_t, void *,
                                size_t, float *, float *, float *, float *, uint32_t *, cudaStream_t);
}  // namespace gsr

using namespace gsr;

static thread_local char g_err[512];
static std::atomic<unsigned long long> g_launches{0};

namespace gsr {
void note_launch(int k) { g_launches.fetch_add((unsigned long long)k, std::memory_order_relaxed); }
}  // namespace gsr

extern "C" uint64_t gs_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

static gs_status fail(gs_status s, const char *fmt, const char *arg = "") {
    snprintf(g_err, sizeof(g_err), fmt, arg);
    return s;
}
static gs_status cuda_fail(cudaError_t e, const char *where) {
    snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
    return GS_ERR_CUDA;
}

extern "C" void gs_default_opts(gs_opts *o) {
    if (!o) return;
    o->tile_w = 16;
    o->tile_h = 8;
    o->split_len = 0;
    o->near_plane = 0.2f;
    o->alpha_max = 0.99f;
    o->alpha_min = 1.0f / 255.0f;
    o->t_min = 1e-4f;
    o->support_rho = 9.0f;
    o->lowpass_sigma_px = 0.70710678118654752f;
    o->bg_rgb[0] = o->bg_rgb[1] = o->bg_rgb[2] = 0.f;
    o->bg_range = 0.f;
    o->bg_raydrop = 1.f;
    o->grid_share = 0.f;
}

extern "C" int32_t gs_record_bytes(int32_t kind) { return record_floats(kind) * 4; }

extern "C" size_t gs_projected_bytes(int64_t n, int32_t kind) { return ProjLayout(n, kind).total; }

extern "C" void gs_projected_offsets(int64_t n, int32_t kind, size_t offs[5]) {
    const ProjLayout L(n, kind);
    offs[0] = L.rec;
    offs[1] = L.rect;
    offs[2] = L.key;
    offs[3] = L.cnt;
    offs[4] = L.total;
}

static gs_status check_opts(const gs_opts *o) {
    if (!o) return fail(GS_ERR_CONFIG, "opts is NULL");
    if (o->tile_w < 1 || o->tile_h < 1 || (int64_t)o->tile_w * o->tile_h > 512)
        return fail(GS_ERR_RANGE, "tile shape must hold 32..512 samples");
    if (o->split_len < 0) return fail(GS_ERR_RANGE, "split_len must be >= 0");
    if (!(o->grid_share >= 0.f && o->grid_share <= 1.f)) return fail(GS_ERR_RANGE, "grid_share outside [0, 1]");
    if (!(o->near_plane > 0.f) || !(o->alpha_max > 0.f) || !(o->alpha_max <= 1.f) ||
        !(o->alpha_min >= 0.f) || !(o->t_min >= 0.f) || !(o->support_rho > 0.f) ||
        !(o->lowpass_sigma_px > 0.f))
        return fail(GS_ERR_RANGE, "compositing constants out of range");
    return GS_OK;
}

static gs_status check_sensor(const gs_sensor *s) {
    if (!s) return fail(GS_ERR_CONFIG, "sensor is NULL");
    if (s->kind < 0 || s->kind > 3) return fail(GS_ERR_CONFIG, "unknown sensor kind");
    if (s->width < 1 || s->height < 1) return fail(GS_ERR_CONFIG, "width/height < 1");
    // pixel boxes are packed as two u16 pairs (0xffff = empty); LiDAR column
    // bounds run to 2W-1 across the azimuth seam
    if (s->kind != GS_LIDAR_SPINNING && (s->width > 65535 || s->height > 65535))
        return fail(GS_ERR_RANGE, "camera image wider or taller than 65535 px");
    if (s->kind == GS_LIDAR_SPINNING && s->width > 32767)
        return fail(GS_ERR_RANGE, "LiDAR wider than 32767 columns");
    if (s->kind != GS_LIDAR_SPINNING) {
        if (!(s->fx > 0.f) || !(s->fy > 0.f)) return fail(GS_ERR_RANGE, "focal length must be > 0");
        if (!std::isfinite(s->cx) || !std::isfinite(s->cy)) return fail(GS_ERR_RANGE, "principal point not finite");
        if (s->kind == GS_FISHEYE_CYLINDRICAL) {
            // the columns' azimuths (p_x - c_x) / f_x, p_x in [0, W], must lie in [-pi, pi]
            if (!((double)s->cx / (double)s->fx <= M_PI && ((double)s->width - (double)s->cx) / (double)s->fx <= M_PI))
                return fail(GS_ERR_RANGE, "cylindrical image spans azimuths outside [-pi, pi]");
        }
        if (s->kind == GS_FISHEYE_EQUIDISTANT) {
            if (!(s->theta_max > 0.f && s->theta_max < (float)M_PI))
                return fail(GS_ERR_RANGE, "theta_max outside (0, pi)");
            // the KB lens must be invertible on [0, theta_max] (DESIGN reading R12):
            // theta_d' = 1 + 3k1 t^2 + 5k2 t^4 + 7k3 t^6 + 9k4 t^8 > 0 on a 10^4-point
            // grid and theta_d(theta_max) > 0
            const double k1 = s->k[0], k2 = s->k[1], k3 = s->k[2], k4 = s->k[3];
            if (!std::isfinite(k1 + k2 + k3 + k4)) return fail(GS_ERR_RANGE, "fisheye k not finite");
            const double tm = s->theta_max;
            for (int i = 0; i <= 10000; ++i) {
                const double t = tm * i / 10000.0, t2 = t * t;
                const double dd = 1.0 + t2 * (3.0 * k1 + t2 * (5.0 * k2 + t2 * (7.0 * k3 + t2 * 9.0 * k4)));
                if (!(dd > 0.0)) return fail(GS_ERR_RANGE, "fisheye lens not monotone on [0, theta_max]");
            }
            const double t2 = tm * tm;
            if (!(tm * (1.0 + t2 * (k1 + t2 * (k2 + t2 * (k3 + t2 * k4)))) > 0.0))
                return fail(GS_ERR_RANGE, "fisheye theta_d(theta_max) <= 0");
        }
    } else {
        if (!s->beam_elevation) return fail(GS_ERR_CONFIG, "beam_elevation is NULL");
        if (s->height > GS_MAX_BEAMS) return fail(GS_ERR_RANGE, "more than GS_MAX_BEAMS beams");
        for (int r = 1; r < s->height; ++r)
            if (!(s->beam_elevation[r] < s->beam_elevation[r - 1]))
                return fail(GS_ERR_RANGE, "beam elevations must be strictly decreasing");
        if (!std::isfinite(s->azimuth0)) return fail(GS_ERR_RANGE, "azimuth0 not finite");
        const double span = (double)s->width * (double)s->azimuth_step;
        if (!(s->azimuth_step > 0.f) || !(span <= 2.0 * M_PI * (1.0 + 1e-6)))
            return fail(GS_ERR_RANGE, "azimuth span outside (0, 2pi]");
    }
    return GS_OK;
}

// Warp sub-tile of a binning tile: 32 samples, 8x4 / 16x2 / 32x1, the first
// that divides the tile in the kind's order of preference (LiDAR rows are
// beams: prefer one beam per warp).  Returns false if none divides it.
static bool warp_subtile(int32_t kind, int32_t tw, int32_t th, int32_t *sw, int32_t *sh) {
    static const int32_t cam[3] = {8, 16, 32}, lid[3] = {32, 16, 8};
    const int32_t *pref = kind == GS_LIDAR_SPINNING ? lid : cam;
    for (int i = 0; i < 3; ++i) {
        const int32_t w = pref[i], h = 32 / pref[i];
        if (tw % w == 0 && th % h == 0) { *sw = w; *sh = h; return true; }
    }
    return false;
}

static gs_status check_tiles(const gs_sensor *s, const gs_opts *o) {
    int32_t sw, sh;
    if (!warp_subtile(s->kind, o->tile_w, o->tile_h, &sw, &sh))
        return fail(GS_ERR_RANGE, "tile shape must be a multiple of a 32-sample warp sub-tile (8x4, 16x2, 32x1)");
    return GS_OK;
}

static DevSensor make_dev_sensor(const gs_sensor *s, const gs_opts *o) {
    DevSensor d;
    memset(&d, 0, sizeof(d));
    d.kind = s->kind;
    d.width = s->width;
    d.height = s->height;
    d.tw = o->tile_w;
    d.th = o->tile_h;
    d.mtw = (uint32_t)(((1ull << 32) + (uint64_t)d.tw - 1) / (uint64_t)d.tw);
    d.mth = (uint32_t)(((1ull << 32) + (uint64_t)d.th - 1) / (uint64_t)d.th);
    d.ntx = (s->width + o->tile_w - 1) / o->tile_w;
    d.nty = (s->height + o->tile_h - 1) / o->tile_h;
    warp_subtile(s->kind, o->tile_w, o->tile_h, &d.sw, &d.sh);
    for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) d.R[3 * r + c] = s->world_to_sensor[4 * r + c];
        d.t[r] = s->world_to_sensor[4 * r + 3];
    }
    for (int c = 0; c < 3; ++c) {   // origin o = -R^T t (fp64, rounded once)
        double acc = 0.0;
        for (int r = 0; r < 3; ++r) acc -= (double)d.R[3 * r + c] * (double)d.t[r];
        d.ow[c] = (float)acc;
    }
    d.fx = s->fx; d.fy = s->fy; d.cx = s->cx; d.cy = s->cy;
    for (int k = 0; k < 4; ++k) d.k[k] = s->k[k];
    d.theta_max = s->theta_max;
    {
        const double th = s->theta_max, t2 = th * th;
        d.tdmax = th * (1.0 + (double)s->k[0] * t2 + (double)s->k[1] * t2 * t2 +
                        (double)s->k[2] * t2 * t2 * t2 + (double)s->k[3] * t2 * t2 * t2 * t2);
    }
    d.az0 = s->azimuth0;
    d.az_step = s->azimuth_step;
    if (s->kind == GS_LIDAR_SPINNING) {
        d.nbeams = s->height;
        for (int r = 0; r < s->height; ++r) {
            d.beam[r] = s->beam_elevation[r];
            d.sbeam[r] = (float)sin((double)s->beam_elevation[r]);
        }
        d.full_turn = fabs((double)s->width * (double)s->azimuth_step - 2.0 * M_PI) < 1e-5;
    }
    return d;
}

static DevOpts make_dev_opts(const gs_opts *o) {
    DevOpts d;
    d.near_plane = o->near_plane;
    d.alpha_max = o->alpha_max;
    d.alpha_min = o->alpha_min;
    d.t_min = o->t_min;
    d.support = o->support_rho;
    d.sigma2 = o->lowpass_sigma_px * o->lowpass_sigma_px;
    d.inv_sigma2 = 1.0f / d.sigma2;
    for (int c = 0; c < 3; ++c) d.bg[c] = o->bg_rgb[c];
    d.bg_range = o->bg_range;
    d.bg_raydrop = o->bg_raydrop;
    d.grid_share = o->grid_share > 0.f ? o->grid_share : 1.f;
    return d;
}

extern "C" int64_t gs_num_tiles(const gs_sensor *s, const gs_opts *o) {
    if (check_sensor(s) != GS_OK || check_opts(o) != GS_OK || check_tiles(s, o) != GS_OK) return -1;
    return (int64_t)((s->width + o->tile_w - 1) / o->tile_w) * ((s->height + o->tile_h - 1) / o->tile_h);
}

extern "C" size_t gs_sort_workspace_bytes(int64_t n, int64_t cap, const gs_sensor *s, const gs_opts *o) {
    const int64_t nt = gs_num_tiles(s, o);
    if (nt < 0) return 0;
    return sort_workspace_bytes(n, cap, nt);
}

extern "C" gs_status gs_project(const gs_surfels *sf, const gs_sensor *s, const gs_opts *o, void *projected,
                                size_t projected_bytes, int64_t *d_num_pairs, gs_stream stream) {
    gs_status st;
    if ((st = check_sensor(s)) != GS_OK) return st;
    if ((st = check_opts(o)) != GS_OK) return st;
    if ((st = check_tiles(s, o)) != GS_OK) return st;
    if (!sf) return fail(GS_ERR_CONFIG, "surfels is NULL");
    if (sf->n < 0 || sf->n >= (1ll << 30)) return fail(GS_ERR_RANGE, "surfel count outside [0, 2^30)");
    if (!projected) return fail(GS_ERR_CONFIG, "projected is NULL");
    if (projected_bytes < gs_projected_bytes(sf->n, s->kind))
        return fail(GS_ERR_CONFIG, "projected buffer too small");
    if (sf->n > 0) {
        if (!sf->means || !sf->quats || !sf->scales || !sf->opacities)
            return fail(GS_ERR_CONFIG, "null surfel attribute pointer");
        if (s->kind != GS_LIDAR_SPINNING) {
            if (!sf->sh) return fail(GS_ERR_CONFIG, "cameras need SH coefficients");
            if (sf->sh_degree < 0 || sf->sh_degree > 3) return fail(GS_ERR_CONFIG, "sh_degree outside 0..3");
        }
        if (((uintptr_t)sf->quats & 15) != 0) return fail(GS_ERR_CONFIG, "quats must be 16-byte aligned");
        if (((uintptr_t)sf->scales & 7) != 0) return fail(GS_ERR_CONFIG, "scales must be 8-byte aligned");
        if (sf->sh && ((uintptr_t)sf->sh & 15) != 0) return fail(GS_ERR_CONFIG, "sh must be 16-byte aligned");
    }
    if (((uintptr_t)projected & 255) != 0) return fail(GS_ERR_CONFIG, "projected must be 256-byte aligned");
    DevSurfels ds;
    ds.n = sf->n;
    ds.means = sf->means; ds.quats = sf->quats; ds.scales = sf->scales; ds.opac = sf->opacities;
    ds.sh = sf->sh; ds.inten = sf->intensity; ds.drop = sf->raydrop_logit;
    ds.sh_degree = sf->sh_degree;
    ds.bounds = sf->cull_bounds;
    if (ds.bounds && ((uintptr_t)ds.bounds & 15) != 0) return fail(GS_ERR_CONFIG, "cull_bounds must be 16-byte aligned");
    const DevSensor se = make_dev_sensor(s, o);
    const DevOpts op = make_dev_opts(o);
    cudaError_t e = launch_project(ds, se, op, projected, d_num_pairs, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "gs_project");
    return GS_OK;
}

extern "C" int64_t gs_cull_blocks(int64_t n) { return n > 0 ? (n + SCAN_TILE - 1) / SCAN_TILE : 0; }
static_assert(GS_CULL_BLOCK == SCAN_TILE, "gsr.h block size");

extern "C" gs_status gs_cull_bounds(const gs_surfels *sf, float *bounds, gs_stream stream) {
    if (!sf) return fail(GS_ERR_CONFIG, "surfels is NULL");
    if (sf->n < 0 || sf->n >= (1ll << 30)) return fail(GS_ERR_RANGE, "surfel count outside [0, 2^30)");
    if (sf->n == 0) return GS_OK;
    if (!sf->means || !sf->scales || !bounds) return fail(GS_ERR_CONFIG, "null pointer");
    if (((uintptr_t)sf->scales & 7) != 0) return fail(GS_ERR_CONFIG, "scales must be 8-byte aligned");
    if (((uintptr_t)bounds & 15) != 0) return fail(GS_ERR_CONFIG, "bounds must be 16-byte aligned");
    DevSurfels ds{};
    ds.n = sf->n; ds.means = sf->means; ds.scales = sf->scales;
    const cudaError_t e = launch_bounds(ds, bounds, (cudaStream_t)stream);
    return e == cudaSuccess ? GS_OK : cuda_fail(e, "gs_cull_bounds");
}

extern "C" gs_status gs_bin_sort(const void *projected, int64_t n, const gs_sensor *s, const gs_opts *o,
                                 uint64_t *keys, uint32_t *values, int64_t cap, uint32_t *tile_ranges,
                                 void *workspace, size_t workspace_bytes, int32_t *d_overflow,
                                 gs_stream stream) {
    gs_status st;
    if ((st = check_sensor(s)) != GS_OK) return st;
    if ((st = check_opts(o)) != GS_OK) return st;
    if ((st = check_tiles(s, o)) != GS_OK) return st;
    if (n < 0 || n >= (1ll << 30)) return fail(GS_ERR_RANGE, "surfel count outside [0, 2^30)");
    if (cap < 0 || cap >= (1ll << 30)) return fail(GS_ERR_RANGE, "pair capacity outside [0, 2^30)");
    if (!projected || !tile_ranges || !d_overflow || !workspace || (cap > 0 && !values))
        return fail(GS_ERR_CONFIG, "null buffer");
    const int64_t nt = gs_num_tiles(s, o);
    if (nt >= (1ll << 24)) return fail(GS_ERR_RANGE, "too many tiles");
    if (workspace_bytes < sort_workspace_bytes(n, cap, nt)) return fail(GS_ERR_CONFIG, "workspace too small");
    const DevSensor se = make_dev_sensor(s, o);
    cudaError_t e = launch_bin_sort(projected, n, se, nt, keys, values, cap, tile_ranges, workspace,
                                    d_overflow, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "gs_bin_sort");
    return GS_OK;
}

extern "C" size_t gs_render_workspace_bytes(int64_t cap, const gs_sensor *s, const gs_opts *o) {
    const int64_t nt = gs_num_tiles(s, o);
    if (nt < 0 || cap < 0) return 0;
    return render_workspace_bytes(cap, nt, o->split_len, o->tile_w * o->tile_h);
}

static gs_status check_render(const void *projected, const uint32_t *tile_ranges, const float *alpha,
                              const gs_sensor *s, const gs_opts *o, void *ws, size_t ws_bytes) {
    if (!projected || !tile_ranges || !alpha || !ws) return fail(GS_ERR_CONFIG, "null buffer");
    if (ws_bytes < render_workspace_bytes(0, gs_num_tiles(s, o), o->split_len, o->tile_w * o->tile_h))
        return fail(GS_ERR_CONFIG, "render workspace too small");
    return GS_OK;
}

extern "C" gs_status gs_render_camera(const void *projected, int64_t n, const uint32_t *values,
                                      const uint32_t *tile_ranges, const int32_t *d_overflow,
                                      const gs_sensor *s, const gs_opts *o, void *workspace,
                                      size_t workspace_bytes, float *rgb, float *depth, float *normal,
                                      float *alpha, uint32_t *stats, gs_stream stream) {
    gs_status st;
    if ((st = check_sensor(s)) != GS_OK) return st;
    if ((st = check_opts(o)) != GS_OK) return st;
    if ((st = check_tiles(s, o)) != GS_OK) return st;
    if (s->kind == GS_LIDAR_SPINNING) return fail(GS_ERR_CONFIG, "gs_render_camera called with a LiDAR sensor");
    if ((st = check_render(projected, tile_ranges, alpha, s, o, workspace, workspace_bytes)) != GS_OK) return st;
    const DevSensor se = make_dev_sensor(s, o);
    const DevOpts op = make_dev_opts(o);
    cudaError_t e = launch_render_camera(projected, n, values, tile_ranges, d_overflow, se, op, o->split_len,
                                         workspace, workspace_bytes, rgb, depth, normal, alpha, stats,
                                         (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "gs_render_camera");
    return GS_OK;
}

extern "C" gs_status gs_render_lidar(const void *projected, int64_t n, const uint32_t *values,
                                     const uint32_t *tile_ranges, const int32_t *d_overflow,
                                     const gs_sensor *s, const gs_opts *o, void *workspace,
                                     size_t workspace_bytes, float *range, float *intensity, float *raydrop,
                                     float *alpha, uint32_t *stats, gs_stream stream) {
    gs_status st;
    if ((st = check_sensor(s)) != GS_OK) return st;
    if ((st = check_opts(o)) != GS_OK) return st;
    if ((st = check_tiles(s, o)) != GS_OK) return st;
    if (s->kind != GS_LIDAR_SPINNING) return fail(GS_ERR_CONFIG, "gs_render_lidar called with a camera sensor");
    if ((st = check_render(projected, tile_ranges, alpha, s, o, workspace, workspace_bytes)) != GS_OK) return st;
    const DevSensor se = make_dev_sensor(s, o);
    const DevOpts op = make_dev_opts(o);
    cudaError_t e = launch_render_lidar(projected, n, values, tile_ranges, d_overflow, se, op, o->split_len,
                                        workspace, workspace_bytes, range, intensity, raydrop, alpha, stats,
                                        (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "gs_render_lidar");
    return GS_OK;
}

extern "C" gs_status gs_decode_anchors(const gs_anchors *an, const gs_decoder *de, const float view_origin[3],
                                       float *means, float *quats, float *scales, float *opacities, float *sh,
                                       float *intensity, float *raydrop_logit, gs_stream stream) {
    if (!an || !de || !view_origin) return fail(GS_ERR_CONFIG, "anchors, decoder or view_origin is NULL");
    if (an->n < 0) return fail(GS_ERR_CONFIG, "anchor count < 0");
    if (de->modality != GS_DECODE_CAMERA && de->modality != GS_DECODE_LIDAR)
        return fail(GS_ERR_CONFIG, "unknown decode modality");
    if (!(std::isfinite(view_origin[0]) && std::isfinite(view_origin[1]) && std::isfinite(view_origin[2])))
        return fail(GS_ERR_RANGE, "view_origin not finite");
    if (an->n == 0) return GS_OK;
    if (!an->position || !an->feature || !an->base_scale) return fail(GS_ERR_CONFIG, "anchor array is NULL");
    if (((uintptr_t)an->feature & 15u) != 0) return fail(GS_ERR_CONFIG, "feature pointer not 16-byte aligned");
    const int H = de->modality == GS_DECODE_LIDAR ? 6 : 5;
    for (int h = 0; h < H; ++h) {
        const gs_mlp &m = de->head[h];
        if (!m.w1 || !m.b1 || !m.w2 || !m.b2 || !m.w3 || !m.b3) return fail(GS_ERR_CONFIG, "decoder weight is NULL");
    }
    if (!means || !quats || !scales || !opacities) return fail(GS_ERR_CONFIG, "output array is NULL");
    if (de->modality == GS_DECODE_CAMERA && !sh) return fail(GS_ERR_CONFIG, "camera decode needs sh");
    if (de->modality == GS_DECODE_LIDAR && (!intensity || !raydrop_logit))
        return fail(GS_ERR_CONFIG, "LiDAR decode needs intensity and raydrop_logit");
    if (((uintptr_t)quats & 15u) != 0) return fail(GS_ERR_CONFIG, "quats pointer not 16-byte aligned");
    const cudaError_t e = launch_decode(an, de, view_origin, means, quats, scales, opacities, sh, intensity,
                                        raydrop_logit, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "gs_decode_anchors");
    return GS_OK;
}

extern "C" size_t gs_band_route_workspace_bytes(int64_t n, int32_t n_bands) {
    return band_route_workspace_bytes(n, n_bands < 1 ? 1 : n_bands);
}

extern "C" gs_status gs_band_route(const void *projected, int64_t n, const gs_sensor *s, const gs_opts *o,
                                   const int32_t *band_rows, int32_t n_bands, uint32_t *d_counts,
                                   uint32_t *d_index, void *workspace, size_t workspace_bytes, gs_stream stream) {
    gs_status st = check_sensor(s);
    if (st != GS_OK) return st;
    if ((st = check_opts(o)) != GS_OK) return st;
    if (n < 0) return fail(GS_ERR_CONFIG, "n < 0");
    if (!band_rows || n_bands < 1 || n_bands > GS_MAX_BANDS) return fail(GS_ERR_RANGE, "band table: 1..GS_MAX_BANDS bands");
    const int32_t ty = (s->height + o->tile_h - 1) / o->tile_h;
    if (band_rows[0] != 0 || band_rows[n_bands] != ty) return fail(GS_ERR_RANGE, "band table must cover the tile rows");
    for (int b = 0; b < n_bands; ++b)
        if (!(band_rows[b + 1] > band_rows[b])) return fail(GS_ERR_RANGE, "band table not strictly increasing");
    if (!d_counts || (n > 0 && (!projected || !d_index || !workspace)))
        return fail(GS_ERR_CONFIG, "NULL buffer");
    if (workspace_bytes < band_route_workspace_bytes(n, n_bands)) return fail(GS_ERR_CONFIG, "workspace too small");
    if (n == 0) {
        const cudaError_t e = cudaMemsetAsync(d_counts, 0, 4 * (size_t)n_bands, (cudaStream_t)stream);
        return e == cudaSuccess ? GS_OK : cuda_fail(e, "gs_band_route");
    }
    const cudaError_t e = launch_band_route(projected, n, s->kind, band_rows, n_bands, d_counts, d_index, workspace,
                                            (cudaStream_t)stream);
    return e == cudaSuccess ? GS_OK : cuda_fail(e, "gs_band_route");
}

extern "C" int32_t gs_payload_floats(int32_t sh_degree, int32_t has_intensity, int32_t has_raydrop) {
    const int nsh = sh_degree < 0 ? 0 : (sh_degree + 1) * (sh_degree + 1) * 3;
    return payload_floats(nsh, has_intensity != 0, has_raydrop != 0);
}

extern "C" gs_status gs_pack_surfels(const gs_surfels *src, const uint32_t *d_index, int64_t m, float *payload,
                                     gs_stream stream) {
    if (!src || m < 0) return fail(GS_ERR_CONFIG, "src is NULL or m < 0");
    if (m == 0) return GS_OK;
    if (!d_index || !payload || !src->means || !src->quats || !src->scales || !src->opacities)
        return fail(GS_ERR_CONFIG, "NULL buffer");
    if (src->sh && (src->sh_degree < 0 || src->sh_degree > 3)) return fail(GS_ERR_CONFIG, "sh_degree outside 0..3");
    DevSurfels d;
    d.n = src->n; d.means = src->means; d.quats = src->quats; d.scales = src->scales; d.opac = src->opacities;
    d.sh = src->sh; d.sh_degree = src->sh_degree; d.inten = src->intensity; d.drop = src->raydrop_logit;
    d.bounds = nullptr;
    const int nsh = src->sh ? (src->sh_degree + 1) * (src->sh_degree + 1) * 3 : 0;
    const cudaError_t e = launch_pack(d, nsh, d_index, m, payload, (cudaStream_t)stream);
    return e == cudaSuccess ? GS_OK : cuda_fail(e, "gs_pack_surfels");
}

extern "C" gs_status gs_unpack_surfels(const float *payload, int64_t m, int32_t sh_degree, int32_t has_intensity,
                                       int32_t has_raydrop, float *means, float *quats, float *scales,
                                       float *opacities, float *sh, float *intensity, float *raydrop_logit,
                                       gs_stream stream) {
    if (m < 0) return fail(GS_ERR_CONFIG, "m < 0");
    if (m == 0) return GS_OK;
    if (sh_degree > 3) return fail(GS_ERR_CONFIG, "sh_degree outside 0..3");
    if (!payload || !means || !quats || !scales || !opacities || (sh_degree >= 0 && !sh) ||
        (has_intensity && !intensity) || (has_raydrop && !raydrop_logit))
        return fail(GS_ERR_CONFIG, "NULL buffer");
    const int nsh = sh_degree < 0 ? 0 : (sh_degree + 1) * (sh_degree + 1) * 3;
    const cudaError_t e = launch_unpack(payload, m, nsh, has_intensity != 0, has_raydrop != 0, means, quats, scales,
                                        opacities, sh, intensity, raydrop_logit, (cudaStream_t)stream);
    return e == cudaSuccess ? GS_OK : cuda_fail(e, "gs_unpack_surfels");
}

extern "C" size_t gs_backward_workspace_bytes(int64_t n) { return backward_workspace_bytes(n); }

extern "C" gs_status gs_render_backward(const gs_surfels *sf, const gs_sensor *s, const gs_opts *o,
                                        const void *projected, const uint32_t *values, const uint32_t *tile_ranges,
                                        const float *grad_out, void *workspace, size_t workspace_bytes,
                                        float *d_means, float *d_quats, float *d_scales, float *d_opacities,
                                        float *d_sh, float *d_intensity, float *d_raydrop_logit, gs_stream stream) {
    gs_status st;
    if ((st = check_sensor(s)) != GS_OK) return st;
    if ((st = check_opts(o)) != GS_OK) return st;
    if ((st = check_tiles(s, o)) != GS_OK) return st;
    if (s->kind != GS_PINHOLE && s->kind != GS_LIDAR_SPINNING)
        return fail(GS_ERR_UNSUPPORTED, "gs_render_backward supports pinhole cameras and LiDAR");
    if (!sf) return fail(GS_ERR_CONFIG, "surfels is NULL");
    if (sf->n < 0) return fail(GS_ERR_CONFIG, "n < 0");
    if (sf->n > 0 && (!sf->means || !sf->quats || !sf->scales || !sf->opacities || !projected || !values ||
                      !tile_ranges || !grad_out || !workspace || !d_means || !d_quats || !d_scales || !d_opacities))
        return fail(GS_ERR_CONFIG, "NULL buffer");
    if (s->kind == GS_PINHOLE && sf->n > 0 && (!sf->sh || sf->sh_degree < 0 || sf->sh_degree > 3))
        return fail(GS_ERR_CONFIG, "cameras need SH coefficients of degree 0..3");
    if (workspace_bytes < backward_workspace_bytes(sf->n)) return fail(GS_ERR_CONFIG, "workspace too small");
    DevSurfels ds;
    ds.n = sf->n;
    ds.means = sf->means; ds.quats = sf->quats; ds.scales = sf->scales; ds.opac = sf->opacities;
    ds.sh = sf->sh; ds.inten = sf->intensity; ds.drop = sf->raydrop_logit;
    ds.sh_degree = sf->sh_degree;
    ds.bounds = nullptr;
    const DevSensor se = make_dev_sensor(s, o);
    const DevOpts op = make_dev_opts(o);
    const cudaError_t e = launch_backward(ds, se, op, projected, values, tile_ranges, grad_out, workspace, d_means,
                                          d_quats, d_scales, d_opacities, d_sh, d_intensity, d_raydrop_logit,
                                          (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "gs_render_backward");
    return GS_OK;
}

extern "C" const char *gs_status_string(gs_status s) {
    switch (s) {
        case GS_OK: return "ok";
        case GS_ERR_CONFIG: return "configuration error";
        case GS_ERR_RANGE: return "argument out of range";
        case GS_ERR_CAPACITY: return "pair capacity exceeded";
        case GS_ERR_CUDA: return "CUDA error";
        case GS_ERR_UNSUPPORTED: return "unsupported";
    }
    return "unknown status";
}

extern "C" const char *gs_last_error(void) { return g_err; }
