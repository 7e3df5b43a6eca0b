// scan.cuh -- single-pass decoupled look-back primitives (device-wide scans
// without a host round trip; the element counts live in device memory).
#pragma once
#include <stdint.h>

namespace gsr {

constexpr unsigned FULL_MASK = 0xffffffffu;

// 64-bit status word: [63:62] flag (1 = aggregate, 2 = inclusive prefix), [61:0] value.
constexpr unsigned long long LB_AGG = 1ull << 62;
constexpr unsigned long long LB_PRE = 2ull << 62;
constexpr unsigned long long LB_VAL = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile_u32(uint32_t *p, uint32_t v) {
    asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Publish `aggregate` for tile `tile` and return the exclusive prefix of all
// earlier tiles.  Called by ONE thread.  Tiles must be numbered in the order
// their CTAs started (dynamic tile ids), so the spin always terminates.
__device__ __forceinline__ unsigned long long lookback_u64(unsigned long long *st, uint32_t tile,
                                                          unsigned long long aggregate) {
    if (tile == 0) {
        st_volatile_u64(&st[0], LB_PRE | aggregate);
        return 0;
    }
    st_volatile_u64(&st[tile], LB_AGG | aggregate);
    unsigned long long excl = 0;
    int64_t t = (int64_t)tile - 1;
    while (true) {
        const unsigned long long s = ld_volatile_u64(&st[t]);
        const unsigned long long f = s >> 62;
        if (f == 0) continue;
        excl += s & LB_VAL;
        if (f == 2) break;
        --t;
    }
    st_volatile_u64(&st[tile], LB_PRE | (excl + aggregate));
    return excl;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
    return v;
}

// Warp-parallel decoupled look-back: called by all 32 lanes of one warp with
// the same `aggregate`.  Lane l inspects predecessors tile - 1 - l - 32 k,
// k < LB_K, so each step covers 32 LB_K predecessors in one L2 round trip.
// LB_K = 4 (a 128-tile window) measured equal to LB_K = 1 on the Chunked
// frames (k_cull / k_compact / k_pair_offsets: projection 0.785 vs 0.789 ms,
// binning 0.979 vs 0.975 ms), so the window is not what holds these scans to
// ~22 ns per 2048-item tile; the default stays 1.  Returns the exclusive
// prefix (all lanes) and publishes the inclusive prefix.
#ifndef GSR_LB_K
#define GSR_LB_K 1
#endif
constexpr int LB_K = GSR_LB_K;
__device__ __forceinline__ unsigned long long lookback_warp_u64(unsigned long long *st, uint32_t tile,
                                                               unsigned long long aggregate) {
    const int lane = (int)(threadIdx.x & 31);
    if (tile == 0) {
        if (lane == 0) st_volatile_u64(&st[0], LB_PRE | aggregate);
        return 0;
    }
    if (lane == 0) st_volatile_u64(&st[tile], LB_AGG | aggregate);
    unsigned long long acc = 0;   // this lane's share of the exclusive prefix
    int64_t base = (int64_t)tile - 1;
    bool found = false;
    while (!found) {
        unsigned long long s[LB_K];
#pragma unroll
        for (int k = 0; k < LB_K; ++k) {
            const int64_t idx = base - lane - 32 * k;
            s[k] = idx >= 0 ? ld_volatile_u64(&st[idx]) : LB_PRE;
        }
#pragma unroll
        for (int k = 0; k < LB_K; ++k) {
            if (found) break;
            const int64_t idx = base - lane - 32 * k;
            while (__any_sync(FULL_MASK, (s[k] >> 62) == 0))
                if ((s[k] >> 62) == 0) s[k] = ld_volatile_u64(&st[idx]);
            const uint32_t pre = __ballot_sync(FULL_MASK, (s[k] >> 62) == 2);
            unsigned long long v = s[k] & LB_VAL;
            if (pre) {
                const int stop = __ffs(pre) - 1;   // nearest predecessor that holds an inclusive prefix
                if (lane > stop) v = 0;
                found = true;
            }
            acc += v;
        }
        base -= 32 * LB_K;
    }
    const unsigned long long excl = warp_sum_u64(acc);
    if (lane == 0) st_volatile_u64(&st[tile], LB_PRE | (excl + aggregate));
    return excl;
}

// Exclusive scan of n <= 32 values v[0..n) held in shared memory, done by one
// warp in place; returns the total (all lanes).
__device__ __forceinline__ unsigned long long warp_excl_scan_smem(unsigned long long *v, int n) {
    const int lane = (int)(threadIdx.x & 31);
    const unsigned long long x = lane < n ? v[lane] : 0ull;
    unsigned long long inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(FULL_MASK, inc, o);
        if (lane >= o) inc += y;
    }
    const unsigned long long tot = __shfl_sync(FULL_MASK, inc, 31);
    __syncwarp();
    if (lane < n) v[lane] = inc - x;
    __syncwarp();
    return tot;
}
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T x) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T y = __shfl_up_sync(FULL_MASK, x, o);
        if ((int)lane_id() >= o) x += y;
    }
    return x;
}

}  // namespace gsr
