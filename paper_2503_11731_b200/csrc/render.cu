// render.cu -- front-to-back compositing (gs_render_camera, gs_render_lidar).
//
// PAPER.md Eq. 2 ray-splat intersection with the unified plane pair
// (Eq. 3 pinhole, Eq. 5 LiDAR, equidistant fisheye per DESIGN R4); 2DGS
// low-pass floor for cameras; north_star rule alpha = min(alpha_max,
// o G), skip alpha < alpha_min, stop before T < t_min.
//
// Work decomposition (B200): one CTA composites one binning
// tile (opts tile_w x tile_h samples); each of its consumer warps owns a
// 32-sample sub-tile (8x4 pixels for cameras, 32x1 LiDAR columns of one beam)
// and one producer warp streams the tile's depth-sorted surfel records into a
// shared-memory ring with cp.async copies completing on mbarriers, so every
// record is fetched from L2/HBM once per tile and the consumer warps drift up
// to a ring's length apart instead of meeting at a barrier per batch.  Each
// consumer ballots which records of a slot touch its sub-tile (conservative
// pixel box) and walks only those, in list order, with warp-vote early
// termination; the producer stops when all consumers are done.  CTAs are
// persistent and pull work items (tile, segment) from a longest-first
// schedule built on the device.  Lists longer than split_len are cut into
// segments composited in parallel; a merge kernel combines the segment
// composites with the transmittance prefix and re-walks the one segment in
// which a ray stops, so the stop rule stays exact.  No atomics touch the
// outputs: results are bitwise deterministic and, for unsplit lists,
// independent of the tile shape.
//
// The plane pair of a sample meets the surfel where
// (M^T h_u) x (M^T h_v) = det(M) M^{-1} (h_u x h_v): the kernels evaluate the
// adjugate of the surfel map on the ray direction.  Records are written
// relative to the surfel centre so that fp32 suffices here.
#include <cuda.h>   // CUtensorMap (the TMA descriptor type; encoded through the runtime's driver entry point)
#include <string.h>

#include <algorithm>
#include <mutex>

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

// Packed fp32 pairs (sm_100 f32x2 add / sub / mul / fma: two independent
// IEEE fp32 operations per instruction, the same roundings as the scalar ones).
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk(float a, float b) {
    f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk(f2 r, float &a, float &b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); }
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
    f2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
    f2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
    f2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

constexpr float LOG2E_HALF = 0.72134752044448170368f;   // 0.5 * log2(e)
constexpr int NB = 32;                                   // schedule buckets
constexpr int NPART = 10;                                // floats per partial composite
constexpr uint32_t LMIN = 1024;   // shortest segment of the adaptive split (workspace sizing)
#ifndef GSR_NCP
#define GSR_NCP 4
#endif
constexpr int NCP = GSR_NCP;      // checkpoints per split segment (the re-walk covers one fifth)
constexpr uint32_t NO_STOP = 0xffffffffu;
constexpr unsigned FULL = 0xffffffffu;

// F: floats per record; BB: float index of the packed pixel box; S4: record
// stride in shared memory in 16-byte units (all lanes of a warp read the same
// record: broadcast, no bank conflicts).
template <int KIND> struct Rec;
template <> struct Rec<GS_PINHOLE> { static constexpr int F = PH_FLOATS, BB = PH_BBX, S4 = PH_FLOATS / 4; };
template <> struct Rec<GS_FISHEYE_EQUIDISTANT> { static constexpr int F = FE_FLOATS, BB = FE_BBX, S4 = FE_FLOATS / 4; };
template <> struct Rec<GS_LIDAR_SPINNING> { static constexpr int F = LI_FLOATS, BB = LI_BBX, S4 = LI_FLOATS / 4; };
template <> struct Rec<GS_FISHEYE_CYLINDRICAL> : Rec<GS_FISHEYE_EQUIDISTANT> {};

// ---------------------------------------------------------------- workspace
struct SchedHdr {
    uint32_t counter;        // persistent work counter
    uint32_t n_items;
    uint32_t n_split;        // tiles whose list was split
    uint32_t slot_cursor;    // partial-slot allocator
    uint32_t rw_count;       // re-walk items (split tile, segment) appended by k_merge_plan
    uint32_t rw_counter;     // persistent work counter of k_rewalk
    uint32_t P;              // total pairs (max tile range end)
    uint32_t ovf;            // P exceeds the capacity the workspace was sized for: render background
    uint32_t bucket_cnt[NB];
    uint32_t bucket_cur[NB];
    uint32_t pad1[24];
};
static_assert(sizeof(SchedHdr) == 384, "hdr");

struct RenderWs {
    size_t hdr, items, split_base, split_list, partials, mstate, rw_items, ckpt, total;
    uint32_t max_items, max_split, max_slots, L;
    RenderWs(int64_t cap, int64_t ntiles, int32_t split_len, int npix) {
        L = split_len > 0 ? (uint32_t)split_len : LMIN;
        const uint64_t c = (uint64_t)(cap > 0 ? cap : 0);
        max_items = (uint32_t)(ntiles + c / L + 1);
        max_split = (uint32_t)std::min<uint64_t>((uint64_t)ntiles, c / L + 1);
        max_slots = (uint32_t)(2 * (c / L) + 2);
        size_t o = 0;
        hdr = o; o += 512;
        items = o; o += align256((size_t)max_items * 8);
        split_base = o; o += align256((size_t)ntiles * 4);
        split_list = o; o += align256((size_t)max_split * 4);
        partials = o; o += align256((size_t)max_slots * NPART * npix * 4);
        mstate = o; o += align256((size_t)max_split * NPART * npix * 4);
        rw_items = o; o += align256((size_t)max_slots * 8);
        ckpt = o; o += align256((size_t)max_slots * NCP * NPART * npix * 4);
        total = o;
    }
};

// ---------------------------------------------------------------- per-sample state
struct Ray {
    float px, py;            // pixel centre (cameras)
    int pxi, pyi, pxw;       // integer sample coordinates, wrapped column (LiDAR seam)
    float dh[3], dl[3];      // unit ray direction, hi + lo (fisheye, LiDAR)
    bool inside, valid;
};

struct Acc {
    float T, A, c0, c1, c2, d, n0, n1, n2;
};

// The 32 samples of one warp: an sw x sh block of its tile (compact sub-tiles
// keep small surfels inside few warps; measured faster than interleaving the
// warps' rows, which balances the warps of a tile but spreads each surfel
// over more of them).
struct SubTile {
    int x0, y0, x1, y1;   // inclusive
};

// Bounding rectangle of the warp's samples whose rays are still running: the
// warp-level record test shrinks to it as samples stop (a record that only
// covers stopped samples is skipped).  Not called when every lane is done.
// Cameras only: LiDAR sub-tiles are one beam row whose rays stop in no
// particular column order, and the recomputation cost more than it saved
// there (tools/sweep.py).
template <int KIND>
constexpr bool ACTIVE_RECT = KIND != GS_LIDAR_SPINNING;
__device__ __forceinline__ SubTile active_rect(const Ray &ry, bool done) {
    SubTile a;
    a.x0 = __reduce_min_sync(0xffffffffu, done ? 0x7fffffff : ry.pxi);
    a.x1 = __reduce_max_sync(0xffffffffu, done ? (int)0x80000000 : ry.pxi);
    a.y0 = __reduce_min_sync(0xffffffffu, done ? 0x7fffffff : ry.pyi);
    a.y1 = __reduce_max_sync(0xffffffffu, done ? (int)0x80000000 : ry.pyi);
    return a;
}

__device__ __forceinline__ SubTile sub_tile(const DevSensor &se, int tile, int warp) {
    const int tyi = tile / se.ntx, txi = tile - tyi * se.ntx;
    const int nsx = se.tw / se.sw;
    SubTile st;
    st.x0 = txi * se.tw + (warp % nsx) * se.sw;
    st.y0 = tyi * se.th + (warp / nsx) * se.sh;
    st.x1 = st.x0 + se.sw - 1;
    st.y1 = st.y0 + se.sh - 1;
    return st;
}

template <int KIND>
__device__ __forceinline__ Ray make_ray(const DevSensor &se, const SubTile &st, int lane) {
    Ray ry;
    ry.pxi = st.x0 + lane % se.sw;
    ry.pyi = st.y0 + lane / se.sw;
    ry.pxw = ry.pxi + se.width;
    ry.inside = ry.pxi < se.width && ry.pyi < se.height;
    ry.px = (float)ry.pxi + 0.5f;
    ry.py = (float)ry.pyi + 0.5f;
    ry.valid = ry.inside;
    for (int k = 0; k < 3; ++k) ry.dh[k] = ry.dl[k] = 0.f;
    if (KIND == GS_FISHEYE_EQUIDISTANT && ry.inside) {
        // invert theta_d = theta (1 + k1 t^2 + k2 t^4 + k3 t^6 + k4 t^8) (Newton, fp64)
        const double mx = __ddiv_rn(__dadd_rn((double)ry.px, -(double)se.cx), (double)se.fx);
        const double my = __ddiv_rn(__dadd_rn((double)ry.py, -(double)se.cy), (double)se.fy);
        const double td = __dsqrt_rn(__dadd_rn(__dmul_rn(mx, mx), __dmul_rn(my, my)));
        ry.valid = td <= se.tdmax;
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
        double st_, ct;
        sincos(th, &st_, &ct);
        split_hilo(st_ * cp, ry.dh[0], ry.dl[0]);
        split_hilo(st_ * sp, ry.dh[1], ry.dl[1]);
        split_hilo(ct, ry.dh[2], ry.dl[2]);
    }
    if (KIND == GS_FISHEYE_CYLINDRICAL && ry.inside) {
        // Eq. 4 (reading R20): column -> azimuth phi about the camera y axis, row ->
        // y / sqrt(x^2 + z^2) = (p_y - c_y) / f_y; unit ray (sin phi, yh, cos phi) / sqrt(1 + yh^2)
        const double ph = __ddiv_rn(__dadd_rn((double)ry.px, -(double)se.cx), (double)se.fx);
        const double yh = __ddiv_rn(__dadd_rn((double)ry.py, -(double)se.cy), (double)se.fy);
        double sp, cp;
        sincos(ph, &sp, &cp);
        const double inv = 1.0 / sqrt(1.0 + yh * yh);
        split_hilo(sp * inv, ry.dh[0], ry.dl[0]);
        split_hilo(yh * inv, ry.dh[1], ry.dl[1]);
        split_hilo(cp * inv, ry.dh[2], ry.dl[2]);
    }
    if (KIND == GS_LIDAR_SPINNING && ry.inside) {   // Eq. 5: theta = elevation (row), phi = azimuth (column)
        const double th = (double)se.beam[ry.pyi];
        const double ph = (double)se.az0 + (double)ry.pxi * (double)se.az_step;
        double st_, ct, sf, cf;
        sincos(th, &st_, &ct);
        sincos(ph, &sf, &cf);
        split_hilo(ct * cf, ry.dh[0], ry.dl[0]);
        split_hilo(ct * sf, ry.dh[1], ry.dl[1]);
        split_hilo(st_, ry.dh[2], ry.dl[2]);
    }
    return ry;
}

__device__ __forceinline__ bool in_box(uint32_t bx, uint32_t by, int x, int xw, int y) {
    const int x0 = (int)(bx & 0xffffu), x1 = (int)(bx >> 16);
    const int y0 = (int)(by & 0xffffu), y1 = (int)(by >> 16);
    const uint32_t wx = (uint32_t)(x1 - x0);
    const bool okx = (uint32_t)(x - x0) <= wx || (uint32_t)(xw - x0) <= wx;
    return okx && (uint32_t)(y - y0) <= (uint32_t)(y1 - y0);
}

// Does a record's conservative pixel box (packed u16 pairs; LiDAR columns may
// run past width-1 = azimuth wrap) touch the sub-tile?
template <bool WRAP>
__device__ __forceinline__ bool box_hits(uint32_t bx, uint32_t by, const SubTile &st, int W) {
    const int x0 = (int)(bx & 0xffffu), x1 = (int)(bx >> 16);
    const int y0 = (int)(by & 0xffffu), y1 = (int)(by >> 16);
    bool okx = x0 <= st.x1 && x1 >= st.x0;
    if (WRAP) okx = okx || (x0 <= st.x1 + W && x1 >= st.x0 + W);   // LiDAR azimuth seam
    return okx && y0 <= st.y1 && y1 >= st.y0;
}

// Can the record contribute to any sample of the sub-tile?  Pinhole: the
// 3-sigma disk's pixel box or the low-pass disc (circle about the projected
// centre, radius^2 = RCUT2, widened by 1e-3 px for the fp32 centre) reaches a
// pixel centre of the sub-tile.  Others: the pixel box.
constexpr int ELL_MIN = 4;   // boxes spanning <= this many px (width + height) skip the ellipse test
// Pinhole: can the 3-sigma region {Q <= 0} reach the sub-tile's pixel-centre
// rectangle?  Q(d) = |A01 d|^2 - R (a2.d + qc)^2 (d = pixel - centre) is the
// compositor's own support test; when its quadratic part is well-conditioned
// positive definite (a bounded ellipse) the minimum of Q over the rectangle
// is at the ellipse centre if that lies inside, else on an edge at the
// clamped vertex of a 1-D quadratic.  The rectangle is widened by 0.01 px and
// the threshold by 2e-3 R w_max^2 (fp32 slack); otherwise "yes".
__device__ __forceinline__ bool ellipse_hits(const float4 *__restrict__ r, float cx, float cy, const SubTile &st) {
    const float4 g0 = r[0], g1 = r[1];
    const float R = g1.w, qc = g1.z;
    // g0 = (A00, A10, A01, A11)
    const float M00 = fmaf(g0.x, g0.x, fmaf(g0.y, g0.y, -R * g1.x * g1.x));
    const float M11 = fmaf(g0.z, g0.z, fmaf(g0.w, g0.w, -R * g1.y * g1.y));
    const float M01 = fmaf(g0.x, g0.z, fmaf(g0.y, g0.w, -R * g1.x * g1.y));
    const float det = fmaf(M00, M11, -M01 * M01);
    // well-conditioned only: no cancellation in M00, M11 or det beyond 1e-3 of their terms
    const float t00 = fmaf(g0.x, g0.x, fmaf(g0.y, g0.y, R * g1.x * g1.x));
    const float t11 = fmaf(g0.z, g0.z, fmaf(g0.w, g0.w, R * g1.y * g1.y));
    if (!(M00 > 1e-3f * t00) || !(M11 > 1e-3f * t11) || !(det > 1e-3f * M00 * M11)) return true;
    const float B0 = -R * qc * g1.x, B1 = -R * qc * g1.y, C = -R * qc * qc;
    const float X0 = (float)st.x0 + 0.49f - cx, X1 = (float)st.x1 + 0.51f - cx;
    const float Y0 = (float)st.y0 + 0.49f - cy, Y1 = (float)st.y1 + 0.51f - cy;
    const float idet = __fdividef(1.f, det);   // approximate: it only places the test points
    const float sx = (M01 * B1 - M11 * B0) * idet, sy = (M01 * B0 - M00 * B1) * idet;
    if (sx >= X0 && sx <= X1 && sy >= Y0 && sy <= Y1) return true;
    // slack 2e-3 R w_max^2, w_max bounding |a2.d + qc| over the rectangle (Q's terms there)
    const float wmax = fabsf(qc) + fabsf(g1.x) * fmaxf(fabsf(X0), fabsf(X1)) + fabsf(g1.y) * fmaxf(fabsf(Y0), fabsf(Y1));
    const float tol = 2e-3f * R * wmax * wmax;
    auto q = [&](float x, float y) {
        return fmaf(x, fmaf(M00, x, 2.f * fmaf(M01, y, B0)), fmaf(y, fmaf(M11, y, 2.f * B1), C));
    };
    const float i00 = __fdividef(1.f, M00), i11 = __fdividef(1.f, M11);
    const float xa = fminf(fmaxf(-(M01 * Y0 + B0) * i00, X0), X1);
    const float xb = fminf(fmaxf(-(M01 * Y1 + B0) * i00, X0), X1);
    const float ya = fminf(fmaxf(-(M01 * X0 + B1) * i11, Y0), Y1);
    const float yb = fminf(fmaxf(-(M01 * X1 + B1) * i11, Y0), Y1);
    const float m = fminf(fminf(q(xa, Y0), q(xb, Y1)), fminf(q(X0, ya), q(X1, yb)));
    return m <= tol;
}

template <int KIND>
__device__ __forceinline__ bool rec_hits(const float4 *__restrict__ r, const SubTile &st, int W) {
    constexpr int BB4 = Rec<KIND>::BB / 4;
    const float4 bb = r[BB4];
    const bool box = box_hits<KIND == GS_LIDAR_SPINNING>(__float_as_uint(bb.z), __float_as_uint(bb.w), st, W);
    if (KIND != GS_PINHOLE) return box;
    const float4 c = r[2];
    const float cx = c.x + c.z, cy = c.y + c.w, r2 = r[3].x;
    if (box) {
        // small boxes (<= ELL_MIN px across, summed) are already tight: skip the ellipse test
        const uint32_t bx = __float_as_uint(bb.z), by = __float_as_uint(bb.w);
        const int span = (int)(bx >> 16) - (int)(bx & 0xffffu) + (int)(by >> 16) - (int)(by & 0xffffu);
        if (span <= ELL_MIN || ellipse_hits(r, cx, cy, st)) return true;
    }
    const float ddx = fmaxf(fmaxf((float)st.x0 + 0.5f - cx, cx - ((float)st.x1 + 0.5f)), 0.f);
    const float ddy = fmaxf(fmaxf((float)st.y0 + 0.5f - cy, cy - ((float)st.y1 + 0.5f)), 0.f);
    return fmaf(ddx, ddx, ddy * ddy) <= fmaf(r2, 1.0001f, 1e-3f);
}

// A staged record addressed by its 32-bit shared-memory address: the walk
// keeps one base register per slot and forms each record's address with one
// multiply-add (with a generic pointer the compiler re-derived it from the
// slot and bit index on every iteration).
struct SmemRec {
    uint32_t a;
    __device__ __forceinline__ float4 operator[](int k) const {
        float4 v;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                     : "r"(a + 16u * (uint32_t)k));
        return v;
    }
};

// One (sample, surfel) evaluation in list order.  Returns false once the ray
// stops (the surfel that would push T below t_min is not composited, R3).
template <int KIND, bool STATS, typename RP>
__device__ __forceinline__ bool eval_record(const RP r, const Ray &ry, const DevOpts &op,
                                            Acc &a, uint32_t &n_eval, uint32_t &n_comp) {
    if (STATS) {   // the sample lies in the record's conservative support region
        constexpr int BB4 = Rec<KIND>::BB / 4;
        const float4 bb = r[BB4];
        bool in = in_box(__float_as_uint(bb.z), __float_as_uint(bb.w), ry.pxi, ry.pxw, ry.pyi);
        if (KIND == GS_PINHOLE && !in) {
            const float4 c = r[2];
            const float ex = ry.px - (c.x + c.z), ey = ry.py - (c.y + c.w);
            in = fmaf(ex, ex, ey * ey) <= r[3].x;
        }
        if (in) ++n_eval;
    }
    float rho, dep, o;
    if (KIND == GS_PINHOLE) {
        const float4 g0 = r[0], g1 = r[1], g2 = r[2], g3 = r[3];
        // (dx, dy) = (p - c_hi) - c_lo; (q0, q1) = A01 (dx, dy), A column-major in g0
        float dx, dy, q0, q1;
        upk(sub2(sub2(pk(ry.px, ry.py), pk(g2.x, g2.y)), pk(g2.z, g2.w)), dx, dy);
        upk(fma2(pk(g0.x, g0.y), pk(dx, dx), mul2(pk(g0.z, g0.w), pk(dy, dy))), q0, q1);
        const float s2 = fmaf(dx, dx, dy * dy);
        const float q2 = fmaf(g1.x, dx, fmaf(g1.y, dy, g1.z));
        const float n3 = fmaf(q0, q0, q1 * q1);
        if ((n3 > g1.w * q2 * q2) && (s2 > g3.x)) return true;
        const float ir = fast_rcp(q2);
        const float rho3 = n3 * ir * ir;
        const float rho2 = s2 * op.inv_sigma2;
        const bool use3 = rho3 <= rho2;
        rho = use3 ? rho3 : rho2;
        dep = use3 ? g3.z * ir : g3.w;
        o = g3.y;
    } else {
        float rho3, rho2, ir, dep3, depc;
        const float4 g0 = r[0], g1 = r[1], g2 = r[2], g3 = r[3], g4 = r[4];
        const float ex = (ry.dh[0] - g0.x) + (ry.dl[0] - g1.x);
        const float ey = (ry.dh[1] - g0.y) + (ry.dl[1] - g1.y);
        const float ez = (ry.dh[2] - g0.z) + (ry.dl[2] - g1.z);
        const float hu = fmaf(g2.x, ex, fmaf(g2.y, ey, g2.z * ez));
        const float hv = fmaf(g3.x, ex, fmaf(g3.y, ey, g3.z * ez));
        const float Dd = fmaf(g4.x, ex, fmaf(g4.y, ey, fmaf(g4.z, ez, g1.w)));
        const float n3 = fmaf(hu, hu, hv * hv);
        if (dir_camera(KIND)) {
            const float4 g5 = r[5], g6 = r[6];
            const float dx = (ry.px - g5.x) - g5.z, dy = (ry.py - g5.y) - g5.w;
            const float s2 = fmaf(dx, dx, dy * dy);
            if ((n3 > g0.w * Dd * Dd) && (s2 > g6.x)) return true;
            rho2 = s2 * op.inv_sigma2;
        } else {
            if (n3 > g0.w * Dd * Dd) return true;
            rho2 = __int_as_float(0x7f800000);   // no low-pass for LiDAR (R6)
        }
        ir = fast_rcp(Dd);
        rho3 = n3 * ir * ir;
        dep3 = g3.w * ir;
        depc = g4.w;
        o = g2.w;
        const bool use3 = rho3 <= rho2;
        rho = use3 ? rho3 : rho2;
        dep = use3 ? dep3 : depc;
    }
    if (!(rho <= op.support) || !(dep >= op.near_plane)) return true;
    const float al = fminf(op.alpha_max, o * fast_ex2(-LOG2E_HALF * rho));
    if (!(al >= op.alpha_min)) return true;
    const float Tn = a.T * (1.f - al);
    if (Tn < op.t_min) return false;
    const float w = al * a.T;
    if (KIND == GS_LIDAR_SPINNING) {
        const float4 p = r[5];
        a.c0 = fmaf(w, p.x, a.c0);   // intensity
        a.c1 = fmaf(w, p.y, a.c1);   // ray-drop probability
    } else if (KIND == GS_PINHOLE) {   // packed: (c0,c1) (c2,n0) (n1,n2) += w (r,g) (b,nx) (ny,nz)
        const float4 c0 = r[4], c1 = r[5];
        const f2 ww = pk(w, w);
        upk(fma2(ww, pk(c0.x, c0.y), pk(a.c0, a.c1)), a.c0, a.c1);
        upk(fma2(ww, pk(c0.z, c0.w), pk(a.c2, a.n0)), a.c2, a.n0);
        upk(fma2(ww, pk(c1.x, c1.y), pk(a.n1, a.n2)), a.n1, a.n2);
    } else {
        const float4 c0 = r[7], c1 = r[8];
        a.c0 = fmaf(w, c0.x, a.c0); a.c1 = fmaf(w, c0.y, a.c1); a.c2 = fmaf(w, c0.z, a.c2);
        a.n0 = fmaf(w, c0.w, a.n0); a.n1 = fmaf(w, c1.x, a.n1); a.n2 = fmaf(w, c1.y, a.n2);
    }
    a.d = fmaf(w, dep, a.d);
    a.A += w;
    a.T = Tn;
    if (STATS) ++n_comp;
    return true;
}

// Segment checkpoints: a split segment's walk leaves its local composite after
// every CB batches (NCP of them, SoA like the partials) so that the exact-stop
// re-walk can start from the last checkpoint before the stop instead of the
// segment start.  The slot's last float is unused (the stop batch lives in
// the partial).
struct Ckpt {
    float *base;     // this segment's NCP checkpoint blocks, or nullptr
    uint32_t cb;     // batches between checkpoints
    int npix, t;     // samples per tile, this thread's sample
    uint32_t next;   // batches walked when checkpoint c is due (~0u: none)
    uint32_t c;      // next checkpoint, 1..NCP
};

__device__ __forceinline__ Ckpt make_ckpt(float *base, uint32_t cb, int npix, int t) {
    return Ckpt{base, cb, npix, t, base ? cb : ~0u, 1u};
}

__device__ __forceinline__ void ckpt_store(Ckpt &ck, uint32_t b_done, uint32_t nb, const Acc &a) {
    // b_done batches have been walked; checkpoint c sits at c * cb batches
    if (b_done != ck.next) return;
    const uint32_t c = ck.c++;
    ck.next = ck.c <= (uint32_t)NCP ? ck.next + ck.cb : ~0u;
    if (b_done >= nb) return;
    float *p = ck.base + (size_t)(c - 1) * NPART * ck.npix + ck.t;
    const int n = ck.npix;
    p[0 * n] = a.T; p[1 * n] = a.A; p[2 * n] = a.c0; p[3 * n] = a.c1; p[4 * n] = a.c2;
    p[5 * n] = a.d; p[6 * n] = a.n0; p[7 * n] = a.n1; p[8 * n] = a.n2;
}

__device__ __forceinline__ uint32_t ckpt_batches(uint32_t L) {   // cb for segment length L
    const uint32_t nb = (L + 31) >> 5;
    return (nb + NCP) / (NCP + 1);
}

// ---------------------------------------------------------------- staging pipeline
// Warp-specialised: the last warp of the CTA is the producer -- it copies the
// depth-sorted records of the tile list into a ring of KSLOTS slots (32
// records each, one record per lane as 16-byte cp.async ops whose completion
// arrives on the slot's `full` mbarrier; measured faster than one TMA bulk
// copy per 96-byte record, which are too small to amortise); the other warps are
// consumers, one per 32-sample sub-tile, and release a slot on its `empty`
// mbarrier.  Consumers run up to KSLOTS batches apart instead of meeting at a
// CTA barrier per batch.  When every consumer's samples have stopped, the
// producer publishes a STOP slot instead of more records.
constexpr int KSLOTS = 8;
struct Pipe {
    unsigned long long full[KSLOTS], empty[KSLOTS];
    uint32_t stop_seq[KSLOTS];   // batch clock of a STOP slot
    int n_done;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(void *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
// try_wait with a suspend-time hint: the warp sleeps in hardware until the
// phase completes (or the hint expires) instead of re-issuing the probe --
// without it ncu counted ~45 % of the compositor's issued instructions in
// this spin loop.
__device__ __forceinline__ void mbar_wait(void *b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(smem_u32(b)),
        "r"(parity), "r"(0x989680u)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(void *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void cp_async_arrive(void *b) {   // arrive when this thread's cp.async ops land
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
}

// TMA gather4 staging (sm_100a): the pinhole producer fills a 32-record slot
// with eight cp.async.bulk.tensor.2d ... tile::gather4 copies (four 96-byte
// record rows each, rows addressed by surfel id through a 2-D tensor map
// over the record array) that complete on the slot's `full` mbarrier by
// transaction count, instead of 192 16-byte cp.async ops.  The group
// destinations (4 x 96 B) stay 128-byte aligned; the fisheye's 144-byte
// records would not, so they keep cp.async.
#ifndef GSR_TMA_GATHER
#define GSR_TMA_GATHER 0   // 1: lanes 0-7 issue one gather4 each; 2: lane 0 issues all eight
#endif
#ifndef GSR_TMA_L2PROMO
#define GSR_TMA_L2PROMO 1   // the tensor map's L2 promotion: 0 none, 1 128 B, 2 256 B
#endif
template <int KIND>
constexpr bool TMA_STAGE = GSR_TMA_GATHER != 0 && KIND == GS_PINHOLE;
__device__ __forceinline__ void mbar_arrive_expect_tx(void *b, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void tma_gather4(void *dst, const CUtensorMap *tm, int r0, int r1, int r2, int r3,
                                            void *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"((uint64_t)tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void pipe_init(Pipe &pp, int nw, uint32_t full_count) {
    if (threadIdx.x == 0) {
        for (int k = 0; k < KSLOTS; ++k) {
            mbar_init(&pp.full[k], full_count);   // the 32 producer lanes (cp.async) or one (TMA)
            mbar_init(&pp.empty[k], (uint32_t)nw);
            pp.stop_seq[k] = 0xffffffffu;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
}

// Evaluate the records of `buf` whose bit is set in the (warp-uniform) mask,
// in order, for this lane's sample; stop at the first that ends the ray.
// Pinhole masks are sparse after the ellipse test (≈3 records of 32 on the
// Chunked forward camera): a find-first-set loop.  Fisheye and LiDAR masks
// are denser: records in groups of four with compile-time offsets (empty
// groups skipped), fewer instructions per record there (tools/sweep.py).
template <int KIND, bool STATS>
__device__ __forceinline__ void eval_bits(uint32_t bits, const float4 *__restrict__ buf, const Ray &ry,
                                          const DevOpts &op, Acc &a, bool &done, bool &stopped,
                                          uint32_t &n_eval, uint32_t &n_comp) {
    constexpr int S4 = Rec<KIND>::S4;
    if constexpr (KIND == GS_PINHOLE) {   // sparse masks (after the ellipse test): one set bit at a time
        uint32_t base = (uint32_t)__cvta_generic_to_shared(buf);
        asm("" : "+r"(base));   // keep the slot base in a register
        bool stop = false;
#pragma unroll 1
        while (bits) {
            const uint32_t u = (uint32_t)__ffs(bits) - 1u;
            bits &= bits - 1;
            if (!eval_record<KIND, STATS>(SmemRec{base + u * (uint32_t)(S4 * 16)}, ry, op, a, n_eval, n_comp)) {
                stop = true;
                break;
            }
        }
        if (stop) {
            done = true;
            stopped = true;
        }
    } else {
#pragma unroll 1
        for (int jj = 0; jj < 32; jj += 4) {
            const uint32_t nib = (bits >> jj) & 0xfu;
            if (!nib) continue;
            const float4 *b4 = buf + jj * S4;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (nib & (1u << u)) {
                    if (!eval_record<KIND, STATS>(b4 + u * S4, ry, op, a, n_eval, n_comp)) {
                        done = true;
                        stopped = true;
                        return;
                    }
                }
            }
        }
    }
}

// CTA walk of list entries [s, e) of `values`; every thread of the CTA calls
// it.  Consumer thread: its sample `ry` in its warp's sub-tile `st`; `done`
// lanes skip work and a lane becomes done when its ray stops (`stopped`).
// g: batches used so far by this CTA (the ring's phase clock, equal in all
// threads).
template <int KIND, bool STATS>
__device__ __forceinline__ void walk_pipe(const float4 *__restrict__ rec, const CUtensorMap *tm,
                                     const uint32_t *__restrict__ values,
                                     uint32_t s, uint32_t e, float4 *ring, Pipe &pp, uint32_t &g,
                                     const SubTile &st, const Ray &ry, const DevSensor &se, const DevOpts &op,
                                     Acc &a, bool &done, bool &stopped, uint32_t &stop_b, Ckpt &ck,
                                     uint32_t &n_eval, uint32_t &n_comp) {
    constexpr int R4 = Rec<KIND>::F / 4, S4 = Rec<KIND>::S4;
    constexpr int BB4 = Rec<KIND>::BB / 4;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5) - 1;
    const uint32_t nb = s < e ? (e - s + 31) >> 5 : 0u;
    if (threadIdx.x == 0) pp.n_done = 0;
    __syncthreads();
    bool wdone = true;
    if (warp < nw) {
        wdone = __all_sync(FULL, done);
        if (wdone && lane == 0) atomicAdd(&pp.n_done, 1);
    }
    __syncthreads();
    uint32_t used = nb;
    if (warp == nw) {   // producer
        for (uint32_t b = 0; b < nb; ++b) {
            const uint32_t gg = g + b, slot = gg % KSLOTS;
            if (gg >= KSLOTS) mbar_wait(&pp.empty[slot], ((gg / KSLOTS) & 1u) ^ 1u);
            // one read, broadcast: the lanes must agree on STOP
            const bool stop = __shfl_sync(FULL, *(volatile int *)&pp.n_done, 0) >= nw;
            if (stop) {
                if (lane == 0) pp.stop_seq[slot] = gg;
                __syncwarp();
                if (!TMA_STAGE<KIND> || lane == 0)
                    mbar_arrive(&pp.full[slot]);   // release: the STOP mark is visible to the waiters
                used = b + 1;
                break;
            }
            const uint32_t first = s + b * 32;
            if constexpr (TMA_STAGE<KIND>) {
                // lane q < 8 gathers records 4q..4q+3 of the batch (a short last batch
                // repeats its last record; consumers ignore lanes >= cnt)
                const uint32_t id = __ldg(values + min(first + lane, e - 1));
                if (GSR_TMA_GATHER == 2) {   // lane 0 issues all eight
                    if (lane == 0) mbar_arrive_expect_tx(&pp.full[slot], 32u * R4 * 16u);
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int r0 = (int)__shfl_sync(FULL, id, 4 * q), r1 = (int)__shfl_sync(FULL, id, 4 * q + 1);
                        const int r2 = (int)__shfl_sync(FULL, id, 4 * q + 2), r3 = (int)__shfl_sync(FULL, id, 4 * q + 3);
                        if (lane == 0) tma_gather4(ring + (slot * 32 + 4 * q) * S4, tm, r0, r1, r2, r3, &pp.full[slot]);
                    }
                    continue;
                }
                const int q4 = (lane & 7) * 4;
                const int r0 = (int)__shfl_sync(FULL, id, q4), r1 = (int)__shfl_sync(FULL, id, q4 + 1);
                const int r2 = (int)__shfl_sync(FULL, id, q4 + 2), r3 = (int)__shfl_sync(FULL, id, q4 + 3);
                if (lane == 0) mbar_arrive_expect_tx(&pp.full[slot], 32u * R4 * 16u);
                __syncwarp();
                if (lane < 8)
                    tma_gather4(ring + (slot * 32 + q4) * S4, tm, r0, r1, r2, r3, &pp.full[slot]);
                continue;
            }
            if (first + lane < e) {
                const uint32_t id = __ldg(values + first + lane);
                const float4 *src = rec + (size_t)id * R4;
                float4 *dst = ring + (slot * 32 + lane) * S4;
#pragma unroll
                for (int k = 0; k < R4; ++k) cp_async16(dst + k, src + k);
            }
            cp_async_arrive(&pp.full[slot]);
        }
    } else {   // consumers
        uint32_t dmask = __ballot_sync(FULL, done);
        SubTile ast = (wdone || !ACTIVE_RECT<KIND>) ? st : active_rect(ry, done);
        for (uint32_t b = 0; b < nb; ++b) {
            const uint32_t gg = g + b, slot = gg % KSLOTS;
            mbar_wait(&pp.full[slot], (gg / KSLOTS) & 1u);
            const int cnt = *(volatile uint32_t *)&pp.stop_seq[slot] == gg ? -1 : (int)min(32u, e - (s + b * 32));
            if (cnt >= 0 && !wdone) {
                const float4 *buf = ring + slot * 32 * S4;
                const bool hit = lane < cnt && rec_hits<KIND>(buf + lane * S4, ast, se.width);
                const uint32_t bits = __ballot_sync(FULL, hit);
                if (bits && !done) {
                    eval_bits<KIND, STATS>(bits, buf, ry, op, a, done, stopped, n_eval, n_comp);
                    if (stopped && stop_b == NO_STOP) stop_b = b;
                }
                const uint32_t dm = __ballot_sync(FULL, done);
                if (dm == FULL) {
                    wdone = true;
                    if (lane == 0) atomicAdd(&pp.n_done, 1);
                } else if (ACTIVE_RECT<KIND> && dm != dmask) {
                    dmask = dm;
                    ast = active_rect(ry, done);
                }
            }
            if (cnt >= 0) ckpt_store(ck, b + 1, nb, a);
            __syncwarp();
            if (lane == 0) mbar_arrive(&pp.empty[slot]);
            if (cnt < 0) { used = b + 1; break; }
        }
    }
    g += used;
    __syncthreads();
}

// One-warp tiles (LiDAR 32x1): no producer warp -- the warp stages its own
// list into a double buffer of 2 x 32 records with cp.async and walks it.
template <int KIND, bool STATS>
__device__ __forceinline__ void walk_self(const float4 *__restrict__ rec, const uint32_t *__restrict__ values,
                                          uint32_t s, uint32_t e, float4 *buf2, const SubTile &st, const Ray &ry,
                                          const DevSensor &se, const DevOpts &op, Acc &a, bool &done,
                                          bool &stopped, uint32_t &stop_b, Ckpt &ck, uint32_t &n_eval,
                                          uint32_t &n_comp) {
    constexpr int R4 = Rec<KIND>::F / 4, S4 = Rec<KIND>::S4;
    constexpr int BB4 = Rec<KIND>::BB / 4;
    const int lane = threadIdx.x & 31;
    if (__all_sync(FULL, done) || s >= e) return;
    auto stage = [&](uint32_t first, float4 *dst) {
        if (first + lane < e) {
            const uint32_t id = __ldg(values + first + lane);
            const float4 *src = rec + (size_t)id * R4;
            float4 *d = dst + lane * S4;
#pragma unroll
            for (int k = 0; k < R4; ++k) cp_async16(d + k, src + k);
        }
        cp_async_commit();
    };
    const uint32_t nb = (e - s + 31) >> 5;
    stage(s, buf2);
    uint32_t dmask = __ballot_sync(FULL, done);
    SubTile ast = ACTIVE_RECT<KIND> ? active_rect(ry, done) : st;
    for (uint32_t b = 0; b < nb; ++b) {
        if (b + 1 < nb) {
            stage(s + (b + 1) * 32, buf2 + ((b + 1) & 1) * 32 * S4);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncwarp();
        const float4 *buf = buf2 + (b & 1) * 32 * S4;
        const int cnt = (int)min(32u, e - (s + b * 32));
        const bool hit = lane < cnt && rec_hits<KIND>(buf + lane * S4, ast, se.width);
        const uint32_t bits = __ballot_sync(FULL, hit);
        if (bits && !done) {
            eval_bits<KIND, STATS>(bits, buf, ry, op, a, done, stopped, n_eval, n_comp);
            if (stopped && stop_b == NO_STOP) stop_b = b;
        }
        const uint32_t dm = __ballot_sync(FULL, done);
        if (dm == FULL) break;   // every later checkpoint is past every stop: never read
        if (ACTIVE_RECT<KIND> && dm != dmask) { dmask = dm; ast = active_rect(ry, done); }
        ckpt_store(ck, b + 1, nb, a);
        __syncwarp();
    }
    cp_async_wait<0>();
    __syncwarp();
}

template <int KIND, bool STATS>
__device__ __forceinline__ void walk(bool piped, const float4 *__restrict__ rec, const CUtensorMap *tm,
                                     const uint32_t *__restrict__ values,
                                     uint32_t s, uint32_t e, float4 *smem, Pipe &pp, uint32_t &g,
                                     const SubTile &st, const Ray &ry, const DevSensor &se, const DevOpts &op,
                                     Acc &a, bool &done, bool &stopped, uint32_t &stop_b, Ckpt &ck,
                                     uint32_t &n_eval, uint32_t &n_comp) {
    if (piped)
        walk_pipe<KIND, STATS>(rec, tm, values, s, e, smem, pp, g, st, ry, se, op, a, done, stopped, stop_b, ck,
                               n_eval, n_comp);
    else
        walk_self<KIND, STATS>(rec, values, s, e, smem, st, ry, se, op, a, done, stopped, stop_b, ck, n_eval,
                               n_comp);
}

template <int KIND>
__device__ __forceinline__ void write_final(const DevSensor &se, const DevOpts &op, const Ray &ry,
                                            const Acc &a, float *o0, float *o1, float *o2, float *o3) {
    if (!ry.inside) return;
    const size_t HW = (size_t)se.width * se.height, pix = (size_t)ry.pyi * se.width + ry.pxi;
    if (KIND == GS_LIDAR_SPINNING) {   // o0 range, o1 intensity, o2 raydrop, o3 alpha
        if (o0) o0[pix] = a.A > 0.f ? a.d / a.A : op.bg_range;
        if (o1) o1[pix] = a.c0;
        if (o2) o2[pix] = fmaf(a.T, op.bg_raydrop, a.c1);
        o3[pix] = a.A;
        return;
    }
    // cameras: o0 rgb [3,H,W], o1 depth, o2 normal [3,H,W], o3 alpha
    if (!ry.valid) {
        if (o0) { o0[pix] = op.bg[0]; o0[HW + pix] = op.bg[1]; o0[2 * HW + pix] = op.bg[2]; }
        if (o1) o1[pix] = 0.f;
        if (o2) { o2[pix] = 0.f; o2[HW + pix] = 0.f; o2[2 * HW + pix] = 0.f; }
        o3[pix] = 0.f;
        return;
    }
    if (o0) {
        o0[pix] = fmaf(a.T, op.bg[0], a.c0);
        o0[HW + pix] = fmaf(a.T, op.bg[1], a.c1);
        o0[2 * HW + pix] = fmaf(a.T, op.bg[2], a.c2);
    }
    if (o1) o1[pix] = a.A > 0.f ? a.d / a.A : 0.f;
    if (o2) { o2[pix] = a.n0; o2[HW + pix] = a.n1; o2[2 * HW + pix] = a.n2; }
    o3[pix] = a.A;
}

__device__ __forceinline__ uint32_t seg_count(uint32_t len, uint32_t L) { return len <= L ? 1u : (len + L - 1) / L; }
__device__ __forceinline__ uint32_t bucket_of(uint32_t len, uint32_t L) {
    if (len == 0) return 0;
    const uint32_t b = 32 - __clz(min(len, L));
    return b >= NB ? NB - 1 : b;
}

// Segment length: fixed (opts split_len > 0), else adaptive -- a quarter of a
// fair share of the frame's pairs per resident CTA (at least LMIN), so the
// longest-first schedule keeps every SM busy to the end while the exact-stop
// re-walk (one checkpoint interval) stays short (measured on the Chunked
// forward camera, fisheye and LiDAR frames with tools/sweep.py).
__device__ __forceinline__ uint32_t seg_len(const SchedHdr *h, uint32_t lfix, uint32_t ctas) {
    if (lfix) return lfix;
    const uint32_t share = (h->P / (4u * ctas) + 255u) & ~255u;
    return share > LMIN ? share : LMIN;
}

// ---------------------------------------------------------------- schedule
// d_overflow (gs_bin_sort's flag) or a pair count above the capacity the
// render workspace was sized for: the frame renders as background (nothing
// below reads past the workspace)
__device__ __forceinline__ bool frame_ovf(const int32_t *d_overflow, const SchedHdr *h) {
    return (d_overflow && *d_overflow) || h->ovf;
}

__global__ void k_sched_total(const uint2 *__restrict__ ranges, int ntiles, const int32_t *d_overflow, SchedHdr *h,
                              uint64_t cap) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntiles || (d_overflow && *d_overflow)) return;
    const uint32_t e = ranges[t].y;
    if (e) atomicMax(&h->P, e);
    if (e > cap) h->ovf = 1u;
}

__global__ void k_sched_count(const uint2 *__restrict__ ranges, int ntiles, const int32_t *d_overflow,
                              SchedHdr *h, uint32_t lfix, uint32_t ctas) {
    const uint32_t L = seg_len(h, lfix, ctas);
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntiles) return;
    const bool ovf = frame_ovf(d_overflow, h);
    const uint2 rg = ranges[t];
    const uint32_t len = ovf ? 0u : rg.y - rg.x;
    atomicAdd(&h->bucket_cnt[bucket_of(len, L)], seg_count(len, L));
}

__global__ void k_sched_scan(SchedHdr *h) {   // one warp: descending-bucket exclusive scan
    const int lane = threadIdx.x;
    const uint32_t c = h->bucket_cnt[NB - 1 - lane];
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
    }
    h->bucket_cur[NB - 1 - lane] = x - c;
    if (lane == 31) h->n_items = x;
}

__global__ void k_sched_fill(const uint2 *__restrict__ ranges, int ntiles, const int32_t *d_overflow,
                             SchedHdr *h, uint2 *__restrict__ items, uint32_t *__restrict__ split_base,
                             uint32_t *__restrict__ split_list, uint32_t lfix, uint32_t ctas) {
    const uint32_t L = seg_len(h, lfix, ctas);
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntiles) return;
    const bool ovf = frame_ovf(d_overflow, h);
    const uint2 rg = ranges[t];
    const uint32_t len = ovf ? 0u : rg.y - rg.x;
    const uint32_t ns = seg_count(len, L);
    const uint32_t pos = atomicAdd(&h->bucket_cur[bucket_of(len, L)], ns);
    for (uint32_t k = 0; k < ns; ++k) items[pos + k] = make_uint2((uint32_t)t, k);
    if (ns > 1) {
        split_base[t] = atomicAdd(&h->slot_cursor, ns);
        split_list[atomicAdd(&h->n_split, 1u)] = (uint32_t)t;
    }
}

// ---------------------------------------------------------------- composite
// Persistent CTAs (blockDim = samples per tile); one work item = (tile,
// segment).  Unsplit tiles are written out; segments of split tiles leave
// their local composite (T = 1 at the segment start) in `partials` (SoA).
template <int KIND, bool STATS>
__device__ __forceinline__ void render_body(
    const float4 *__restrict__ rec, const CUtensorMap *tm, const uint32_t *__restrict__ values,
    const uint2 *__restrict__ ranges, const int32_t *__restrict__ d_overflow,
    const DevSensor &se, const DevOpts op, SchedHdr *h,
    const uint2 *__restrict__ items, const uint32_t *__restrict__ split_base,
    float *__restrict__ partials, float *__restrict__ ckpt, float *__restrict__ o0, float *__restrict__ o1,
    float *__restrict__ o2, float *__restrict__ o3, uint32_t *__restrict__ out_stats, uint32_t lfix, uint32_t ctas) {
    const uint32_t L = seg_len(h, lfix, ctas);
    const uint32_t cb = ckpt_batches(L);
    extern __shared__ __align__(128) float4 smem[];   // TMA destinations: 128-byte aligned
    __shared__ uint32_t s_item;
    __shared__ Pipe pp;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const bool piped = blockDim.x > 32;   // one-warp tiles stage for themselves
    const int nw = piped ? (int)(blockDim.x >> 5) - 1 : 1, npix = nw * 32;
    const bool cons = warp < nw;
    const bool ovf = frame_ovf(d_overflow, h);
    const uint32_t n_items = h->n_items;
    if (piped) pipe_init(pp, nw, TMA_STAGE<KIND> ? 1u : 32u);
    uint32_t g = 0;
    while (true) {
        if (t == 0) s_item = atomicAdd(&h->counter, 1u);
        __syncthreads();
        const uint32_t item = s_item;
        __syncthreads();
        if (item >= n_items) break;
        const uint2 it = items[item];
        const int tile = (int)it.x;
        const uint32_t seg = it.y;
        uint2 rg = ranges[tile];
        if (ovf) rg.y = rg.x;
        const uint32_t len = rg.y - rg.x, ns = seg_count(len, L);
        const uint32_t s = rg.x + seg * L, e = min(rg.y, s + L);
        const SubTile st = sub_tile(se, tile, warp);
        const Ray ry = make_ray<KIND>(se, st, lane);
        Acc a = {1.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        bool done = !ry.valid, stopped = false;
        uint32_t n_eval = 0, n_comp = 0, stop_b = NO_STOP;
        Ckpt ck = make_ckpt(ns > 1 && cons ? ckpt + (size_t)(split_base[tile] + seg) * NCP * NPART * npix : nullptr,
                            cb, npix, t);
        walk<KIND, STATS>(piped, rec, tm, values, s, e, smem, pp, g, st, ry, se, op, a, done, stopped, stop_b, ck,
                          n_eval, n_comp);
        if (!cons) continue;
        if (ns == 1) {
            write_final<KIND>(se, op, ry, a, o0, o1, o2, o3);
            if (STATS && ry.inside) {
                const size_t HW = (size_t)se.width * se.height, pix = (size_t)ry.pyi * se.width + ry.pxi;
                out_stats[pix] = n_comp;
                out_stats[HW + pix] = n_eval;
            }
        } else {
            float *p = partials + (size_t)(split_base[tile] + seg) * NPART * npix + t;
            p[0 * npix] = a.T; p[1 * npix] = a.A; p[2 * npix] = a.c0; p[3 * npix] = a.c1;
            p[4 * npix] = a.c2; p[5 * npix] = a.d; p[6 * npix] = a.n0; p[7 * npix] = a.n1;
            p[8 * npix] = a.n2; p[9 * npix] = __uint_as_float(stopped ? stop_b + 1u : 0u);   // 0 = no local stop
        }
    }
}

// The north_star compositing constants (gs_default_opts) as compile-time
// literals: the DEF kernels fold them into immediates instead of reloading
// six uniform registers in every record evaluation.  Chosen on the host when
// the options equal the defaults bit for bit (is_default_ops).
constexpr float DEF_LP_SIGMA = 0.70710678118654752f;
constexpr float DEF_SIGMA2 = DEF_LP_SIGMA * DEF_LP_SIGMA;
__device__ __forceinline__ DevOpts default_ops(DevOpts o) {
    o.near_plane = 0.2f;
    o.alpha_max = 0.99f;
    o.alpha_min = 1.0f / 255.0f;
    o.t_min = 1e-4f;
    o.support = 9.0f;
    o.sigma2 = DEF_SIGMA2;
    o.inv_sigma2 = 1.0f / DEF_SIGMA2;
    return o;
}
static bool is_default_ops(const DevOpts &o) {
    auto same = [](float a, float b) { return memcmp(&a, &b, 4) == 0; };
    return same(o.near_plane, 0.2f) && same(o.alpha_max, 0.99f) && same(o.alpha_min, 1.0f / 255.0f) &&
           same(o.t_min, 1e-4f) && same(o.support, 9.0f) && same(o.sigma2, DEF_SIGMA2) &&
           same(o.inv_sigma2, 1.0f / DEF_SIGMA2);
}

// Register budgets (measured, tools/sweep.py): the pinhole compositor at 48
// registers per thread (eight 5-warp CTAs per SM; 64 / 56 were 5-6 % slower
// once the packed evaluation had lowered its pressure), fisheye and LiDAR at
// 64.
#ifndef GSR_PH_REGS
#define GSR_PH_REGS 48
#endif
#ifndef GSR_RAY_REGS
#define GSR_RAY_REGS 64
#endif
#ifndef GSR_RW_REGS
#define GSR_RW_REGS 80   // the exact-stop re-walk of split lists
#endif
template <bool STATS, bool DEF>
__global__ void __maxnreg__(GSR_PH_REGS) k_render_pinhole(
    const float4 *__restrict__ rec, const __grid_constant__ CUtensorMap tmap, const uint32_t *__restrict__ values,
    const uint2 *__restrict__ ranges, const int32_t *__restrict__ d_overflow,
    const __grid_constant__ DevSensor se, const DevOpts op, SchedHdr *h,
    const uint2 *__restrict__ items, const uint32_t *__restrict__ split_base,
    float *__restrict__ partials, float *__restrict__ ckpt, float *__restrict__ o0, float *__restrict__ o1,
    float *__restrict__ o2, float *__restrict__ o3, uint32_t *__restrict__ out_stats, uint32_t lfix, uint32_t ctas) {
    render_body<GS_PINHOLE, STATS>(rec, &tmap, values, ranges, d_overflow, se, DEF ? default_ops(op) : op, h, items, split_base,
                                   partials, ckpt, o0, o1, o2, o3, out_stats, lfix, ctas);
}

template <int KIND, bool STATS, bool DEF>
__global__ void __maxnreg__(GSR_RAY_REGS) k_render(
    const float4 *__restrict__ rec, const __grid_constant__ CUtensorMap tmap, const uint32_t *__restrict__ values,
    const uint2 *__restrict__ ranges, const int32_t *__restrict__ d_overflow,
    const __grid_constant__ DevSensor se, const DevOpts op, SchedHdr *h,
    const uint2 *__restrict__ items, const uint32_t *__restrict__ split_base,
    float *__restrict__ partials, float *__restrict__ ckpt, float *__restrict__ o0, float *__restrict__ o1,
    float *__restrict__ o2, float *__restrict__ o3, uint32_t *__restrict__ out_stats, uint32_t lfix, uint32_t ctas) {
    render_body<KIND, STATS>(rec, &tmap, values, ranges, d_overflow, se, DEF ? default_ops(op) : op, h, items, split_base,
                             partials, ckpt, o0, o1, o2, o3, out_stats, lfix, ctas);
}

// ---------------------------------------------------------------- merge of split lists
// k_merge_plan: one CTA per split tile, one thread per sample.  Each sample
// walks its segment composites in order, C += T_run C_k, T_run *= T_k, while
// no stop can have happened (no local stop and T_run T_k >= t_min).  Samples
// that never stop inside a later segment are final and written out; for the
// others the first segment k* in which the ray stops with T_run < 1 must be
// re-walked from T_run with the exact stop rule: their prefix composite and
// k* are kept in `mstate` (SoA) and one re-walk item (split tile, k*) is
// appended per distinct k*.  k_rewalk then walks those items in parallel.
template <int KIND>
__global__ void __launch_bounds__(512) k_merge_plan(
    const uint2 *__restrict__ ranges, const __grid_constant__ DevSensor se, const DevOpts op,
    SchedHdr *h, const uint32_t *__restrict__ split_base, const uint32_t *__restrict__ split_list,
    const float *__restrict__ partials, const float *__restrict__ ckpt, float *__restrict__ mstate,
    uint2 *__restrict__ rw_items, float *__restrict__ o0, float *__restrict__ o1, float *__restrict__ o2,
    float *__restrict__ o3, uint32_t lfix, uint32_t ctas) {
    const uint32_t L = seg_len(h, lfix, ctas);
    const uint32_t cb = ckpt_batches(L);
    if (blockIdx.x >= h->n_split) return;
    const int tile = (int)split_list[blockIdx.x];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31, npix = blockDim.x;
    const uint2 rg = ranges[tile];
    const uint32_t ns = seg_count(rg.y - rg.x, L), base = split_base[tile];
    const SubTile st = sub_tile(se, tile, warp);
    const Ray ry = make_ray<KIND>(se, st, lane);
    Acc a = {1.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int kstar = -1;
    for (uint32_t k = 0; k < ns; ++k) {
        const float *p = partials + (size_t)(base + k) * NPART * npix + t;
        const float Tk = p[0];
        const bool stop_k = __float_as_uint(p[9 * npix]) != 0u;
        if (!stop_k && a.T * Tk >= op.t_min) {
            const float Tr = a.T;
            a.A = fmaf(Tr, p[1 * npix], a.A); a.c0 = fmaf(Tr, p[2 * npix], a.c0);
            a.c1 = fmaf(Tr, p[3 * npix], a.c1); a.c2 = fmaf(Tr, p[4 * npix], a.c2);
            a.d = fmaf(Tr, p[5 * npix], a.d); a.n0 = fmaf(Tr, p[6 * npix], a.n0);
            a.n1 = fmaf(Tr, p[7 * npix], a.n1); a.n2 = fmaf(Tr, p[8 * npix], a.n2);
            a.T = Tr * Tk;
        } else if (a.T == 1.f) {   // nothing composited before: the local composite is exact
            a.T = Tk; a.A = p[1 * npix]; a.c0 = p[2 * npix]; a.c1 = p[3 * npix]; a.c2 = p[4 * npix];
            a.d = p[5 * npix]; a.n0 = p[6 * npix]; a.n1 = p[7 * npix]; a.n2 = p[8 * npix];
            break;
        } else {
            kstar = (int)k;
            break;
        }
    }
    if (!ry.valid) kstar = -1;
    int tag = -1;   // (k*, c): re-walk segment k* from its checkpoint c (0 = the segment start)
    if (kstar < 0) {
        write_final<KIND>(se, op, ry, a, o0, o1, o2, o3);
    } else {
        // advance to the last checkpoint c of segment k* that precedes both the local stop
        // (c cb <= stop batch) and the global one (T_run T_c >= t_min): the ray is still
        // running there, so the prefix composite extends exactly to it
        const uint32_t k = (uint32_t)kstar;
        const float *p = partials + (size_t)(base + k) * NPART * npix + t;
        const uint32_t sb = __float_as_uint(p[9 * npix]);   // local stop batch + 1, 0 = none
        const uint32_t seg_s = rg.x + k * L, seg_e = min(rg.y, seg_s + L), nb = (seg_e - seg_s + 31) >> 5;
        const float Tr = a.T;
        int c = 0;
        for (int cc = 1; cc <= NCP; ++cc) {
            const uint32_t at = (uint32_t)cc * cb;
            if (at >= nb || (sb != 0u && at > sb - 1u)) break;
            const float *q = ckpt + ((size_t)(base + k) * NCP + (cc - 1)) * NPART * npix + t;
            if (!(Tr * q[0] >= op.t_min)) break;
            c = cc;
        }
        if (c > 0) {
            const float *q = ckpt + ((size_t)(base + k) * NCP + (c - 1)) * NPART * npix + t;
            a.A = fmaf(Tr, q[1 * npix], a.A); a.c0 = fmaf(Tr, q[2 * npix], a.c0);
            a.c1 = fmaf(Tr, q[3 * npix], a.c1); a.c2 = fmaf(Tr, q[4 * npix], a.c2);
            a.d = fmaf(Tr, q[5 * npix], a.d); a.n0 = fmaf(Tr, q[6 * npix], a.n0);
            a.n1 = fmaf(Tr, q[7 * npix], a.n1); a.n2 = fmaf(Tr, q[8 * npix], a.n2);
            a.T = Tr * q[0];
        }
        tag = kstar | (c << 24);
    }
    float *m = mstate + (size_t)blockIdx.x * NPART * npix + t;
    m[0 * npix] = a.T; m[1 * npix] = a.A; m[2 * npix] = a.c0; m[3 * npix] = a.c1; m[4 * npix] = a.c2;
    m[5 * npix] = a.d; m[6 * npix] = a.n0; m[7 * npix] = a.n1; m[8 * npix] = a.n2;
    m[9 * npix] = __int_as_float(tag);
    for (uint32_t k = 0; k < ns; ++k)
        for (int c = 0; c <= NCP; ++c)
            if (__syncthreads_or(tag == (int)(k | ((uint32_t)c << 24))) && t == 0)
                rw_items[atomicAdd(&h->rw_count, 1u)] = make_uint2(blockIdx.x, k | ((uint32_t)c << 24));
}

// Persistent CTAs over the re-walk items: segment k of split tile s is walked
// from each stopping sample's prefix transmittance; the segment's result is
// added to the prefix composite and the sample written out.
template <int KIND>
__global__ void __maxnreg__(GSR_RW_REGS) k_rewalk(
    const float4 *__restrict__ rec, const __grid_constant__ CUtensorMap tmap, const uint32_t *__restrict__ values,
    const uint2 *__restrict__ ranges, const __grid_constant__ DevSensor se, const DevOpts op,
    SchedHdr *h, const uint32_t *__restrict__ split_list, const float *__restrict__ mstate,
    const uint2 *__restrict__ rw_items, float *__restrict__ o0, float *__restrict__ o1,
    float *__restrict__ o2, float *__restrict__ o3, uint32_t lfix, uint32_t ctas) {
    const uint32_t L = seg_len(h, lfix, ctas);
    const uint32_t cb = ckpt_batches(L);
    extern __shared__ __align__(128) float4 smem[];   // TMA destinations: 128-byte aligned
    __shared__ uint32_t s_item;
    __shared__ Pipe pp;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const bool piped = blockDim.x > 32;
    const int nw = piped ? (int)(blockDim.x >> 5) - 1 : 1, npix = nw * 32;
    const bool cons = warp < nw;
    const uint32_t n_items = h->rw_count;
    const CUtensorMap *tm = &tmap;
    if (piped) pipe_init(pp, nw, TMA_STAGE<KIND> ? 1u : 32u);
    uint32_t g = 0;
    while (true) {
        if (t == 0) s_item = atomicAdd(&h->rw_counter, 1u);
        __syncthreads();
        const uint32_t item = s_item;
        __syncthreads();
        if (item >= n_items) break;
        const uint2 it = rw_items[item];
        const int tile = (int)split_list[it.x];
        const uint32_t k = it.y & 0xffffffu, c = it.y >> 24;
        const uint2 rg = ranges[tile];
        const SubTile st = sub_tile(se, tile, warp);
        const Ray ry = make_ray<KIND>(se, st, lane);
        const float *m = mstate + (size_t)it.x * NPART * npix + (cons ? t : 0);
        const bool mine = cons && __float_as_uint(m[9 * npix]) == it.y;
        Acc r = {m[0], 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        bool done = !mine, stopped = false;
        uint32_t ne = 0, nc = 0, sb = NO_STOP;
        Ckpt ck = make_ckpt(nullptr, 1u, npix, t);
        // the chunk between checkpoints c and c+1 of segment k (the ray stops inside it)
        const uint32_t seg_s = rg.x + k * L, seg_e = min(rg.y, seg_s + L);
        const uint32_t s = min(seg_e, seg_s + c * cb * 32u), e = min(seg_e, seg_s + (c + 1u) * cb * 32u);
        walk<KIND, false>(piped, rec, tm, values, s, e, smem, pp, g, st, ry, se, op, r, done, stopped, sb, ck, ne, nc);
        if (mine) {
            Acc a = {r.T, m[1 * npix] + r.A, m[2 * npix] + r.c0, m[3 * npix] + r.c1, m[4 * npix] + r.c2,
                     m[5 * npix] + r.d, m[6 * npix] + r.n0, m[7 * npix] + r.n1, m[8 * npix] + r.n2};
            write_final<KIND>(se, op, ry, a, o0, o1, o2, o3);
        }
    }
}

// ---------------------------------------------------------------- host
// The record array as a 2-D fp32 tensor [n rows][F columns] for the gather4
// staging: box = one full row, no swizzle / interleave, row stride F*4 bytes.
// cuTensorMapEncodeTiled is reached through the runtime's driver entry point
// (no link against libcuda); the descriptor travels as a __grid_constant__
// kernel parameter, so it is captured with the launch in a CUDA graph.
typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                     const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                                     CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                     CUtensorMapFloatOOBfill);
static cudaError_t record_tmap(CUtensorMap *m, const float4 *rec, int64_t n, int F) {
    static PFN_encodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_encodeTiled)p;
    });
    if (!fn) return cudaErrorNotSupported;
    const cuuint64_t dims[2] = {(cuuint64_t)F, (cuuint64_t)n};
    const cuuint64_t strides[1] = {(cuuint64_t)F * 4u};
    const cuuint32_t box[2] = {(cuuint32_t)F, 1u}, estr[2] = {1u, 1u};
    const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)rec, dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          GSR_TMA_L2PROMO == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                          : GSR_TMA_L2PROMO == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                                                 : CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

size_t render_workspace_bytes(int64_t cap, int64_t ntiles, int32_t split_len, int npix) {
    return RenderWs(cap, ntiles, split_len, npix).total;
}

template <int KIND, bool STATS>
static cudaError_t launch(const void *proj, int64_t n, const uint32_t *values, const uint32_t *ranges,
                          const int32_t *d_overflow, const DevSensor &se, const DevOpts &op, int32_t split_len,
                          void *ws, size_t ws_bytes, float *o0, float *o1, float *o2, float *o3,
                          uint32_t *stats, cudaStream_t st) {
    const ProjLayout PL(n, se.kind);
    const float4 *rec = (const float4 *)((const char *)proj + PL.rec);
    const int ntiles = se.ntx * se.nty;
    const int npix = se.tw * se.th;
    CUtensorMap tmap;
    memset(&tmap, 0, sizeof(tmap));
    if (TMA_STAGE<KIND> && npix > 32 && n > 0) {
        cudaError_t te = record_tmap(&tmap, rec, n, Rec<KIND>::F);
        if (te != cudaSuccess) return te;
    }
    // capacity implied by the workspace size (the pair capacity of gs_bin_sort)
    int64_t cap = 0;
    {
        int64_t lo = 0, hi = (int64_t)1 << 31;
        while (lo < hi) {   // largest cap whose layout fits
            const int64_t mid = (lo + hi + 1) / 2;
            if (RenderWs(mid, ntiles, split_len, npix).total <= ws_bytes) lo = mid; else hi = mid - 1;
        }
        cap = lo;
    }
    const RenderWs W(cap, ntiles, split_len, npix);
    char *wb = (char *)ws;
    SchedHdr *h = (SchedHdr *)(wb + W.hdr);
    uint2 *items = (uint2 *)(wb + W.items);
    uint32_t *split_base = (uint32_t *)(wb + W.split_base), *split_list = (uint32_t *)(wb + W.split_list);
    float *partials = (float *)(wb + W.partials);
    float *ckpt = (float *)(wb + W.ckpt);
    // instrumented runs are never split; split_len > 0 fixes the segment length
    const uint32_t lfix = STATS ? 0x7fffffffu : (split_len > 0 ? (uint32_t)split_len : 0u);
    cudaError_t e = cudaMemsetAsync(h, 0, sizeof(SchedHdr), st);
    if (e != cudaSuccess) return e;
    const bool piped = npix > 32;   // multi-warp tiles: a producer warp + the staging ring
    const size_t sm = (size_t)(piped ? KSLOTS : 2) * 32 * Rec<KIND>::S4 * 16;
    const int nthr = piped ? npix + 32 : npix;
    const bool def = is_default_ops(op);
    auto *kern = KIND == GS_PINHOLE ? (def ? k_render_pinhole<STATS, true> : k_render_pinhole<STATS, false>)
                                    : (def ? k_render<KIND, STATS, true> : k_render<KIND, STATS, false>);
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, nthr, sm);
    const unsigned ctas = (unsigned)std::max(1, (int)((float)(nsm * std::max(per, 1)) * op.grid_share));
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ctas, (int64_t)W.max_items));
    const unsigned gt = (unsigned)((ntiles + 255) / 256);
    note_launch(4);
    k_sched_total<<<gt, 256, 0, st>>>((const uint2 *)ranges, ntiles, d_overflow, h, (uint64_t)cap);
    k_sched_count<<<gt, 256, 0, st>>>((const uint2 *)ranges, ntiles, d_overflow, h, lfix, ctas);
    k_sched_scan<<<1, 32, 0, st>>>(h);
    k_sched_fill<<<gt, 256, 0, st>>>((const uint2 *)ranges, ntiles, d_overflow, h, items, split_base, split_list,
                                     lfix, ctas);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    note_launch();
    kern<<<grid, nthr, sm, st>>>(rec, tmap, values, (const uint2 *)ranges, d_overflow, se, op, h,
                                                  items, split_base, partials, ckpt, o0, o1, o2, o3, stats, lfix,
                                                  ctas);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (!STATS && W.max_split > 0) {
        float *mstate = (float *)(wb + W.mstate);
        uint2 *rw_items = (uint2 *)(wb + W.rw_items);
        note_launch(2);
        k_merge_plan<KIND><<<W.max_split, npix, 0, st>>>((const uint2 *)ranges, se, op, h, split_base, split_list,
                                                         partials, ckpt, mstate, rw_items, o0, o1, o2, o3, lfix, ctas);
        e = cudaFuncSetAttribute(k_rewalk<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
        int per_rw = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_rw, k_rewalk<KIND>, nthr, sm);
        const unsigned grid_rw = (unsigned)std::max<int64_t>(
            1, std::min<int64_t>((int64_t)((float)(nsm * std::max(per_rw, 1)) * op.grid_share), (int64_t)W.max_slots));
        k_rewalk<KIND><<<grid_rw, nthr, sm, st>>>(rec, tmap, values, (const uint2 *)ranges, se, op, h, split_list,
                                                  mstate, rw_items, o0, o1, o2, o3, lfix, ctas);
        e = cudaGetLastError();
    }
    return e;
}

cudaError_t launch_render_camera(const void *proj, int64_t n, const uint32_t *values,
                                 const uint32_t *ranges, const int32_t *d_overflow,
                                 const DevSensor &se, const DevOpts &op, int32_t split_len, void *ws,
                                 size_t ws_bytes, float *rgb, float *depth, float *normal, float *alpha,
                                 uint32_t *stats, cudaStream_t st) {
    if (se.kind == GS_PINHOLE)
        return stats ? launch<GS_PINHOLE, true>(proj, n, values, ranges, d_overflow, se, op, split_len, ws, ws_bytes, rgb, depth, normal, alpha, stats, st)
                     : launch<GS_PINHOLE, false>(proj, n, values, ranges, d_overflow, se, op, split_len, ws, ws_bytes, rgb, depth, normal, alpha, stats, st);
    if (se.kind == GS_FISHEYE_CYLINDRICAL)
        return stats ? launch<GS_FISHEYE_CYLINDRICAL, true>(proj, n, values, ranges, d_overflow, se, op, split_len, ws, ws_bytes, rgb, depth, normal, alpha, stats, st)
                     : launch<GS_FISHEYE_CYLINDRICAL, false>(proj, n, values, ranges, d_overflow, se, op, split_len, ws, ws_bytes, rgb, depth, normal, alpha, stats, st);
    return stats ? launch<GS_FISHEYE_EQUIDISTANT, true>(proj, n, values, ranges, d_overflow, se, op, split_len, ws, ws_bytes, rgb, depth, normal, alpha, stats, st)
                 : launch<GS_FISHEYE_EQUIDISTANT, false>(proj, n, values, ranges, d_overflow, se, op, split_len, ws, ws_bytes, rgb, depth, normal, alpha, stats, st);
}

cudaError_t launch_render_lidar(const void *proj, int64_t n, const uint32_t *values,
                                const uint32_t *ranges, const int32_t *d_overflow,
                                const DevSensor &se, const DevOpts &op, int32_t split_len, void *ws,
                                size_t ws_bytes, float *range, float *inten, float *drop, float *alpha,
                                uint32_t *stats, cudaStream_t st) {
    return stats ? launch<GS_LIDAR_SPINNING, true>(proj, n, values, ranges, d_overflow, se, op, split_len, ws, ws_bytes, range, inten, drop, alpha, stats, st)
                 : launch<GS_LIDAR_SPINNING, false>(proj, n, values, ranges, d_overflow, se, op, split_len, ws, ws_bytes, range, inten, drop, alpha, stats, st);
}

}  // namespace gsr
