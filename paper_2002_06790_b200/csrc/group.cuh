// Lane-group reductions shared by the warp-per-group engines (fused.cu, simulate_large.cu).
#pragma once

#include "internal.cuh"

// Reductions over one lane group: kGS = 32 is the warp, kGS = 16 a half-warp (two
// candidates per warp), kGS = 10 a third (three candidates per warp; lanes 30-31 idle).
// redux.sync reduces over the whole warp, so each group's reduction runs with the other
// lanes contributing the identity (one REDUX per group).
template <int kGS>
constexpr int kGroupsOf = 32 / kGS;

template <int kGS>
static __device__ __forceinline__ unsigned group_min_u32(unsigned x, int grp) {
    if constexpr (kGS == 32) {
        return __reduce_min_sync(DFSIM_FULL_MASK, x);
    } else {
        unsigned r = 0xffffffffu;
#pragma unroll
        for (int g = 0; g < kGroupsOf<kGS>; g++) {
            const unsigned t = __reduce_min_sync(DFSIM_FULL_MASK, grp == g ? x : 0xffffffffu);
            if (grp == g) r = t;
        }
        return r;
    }
}

template <int kGS>
static __device__ __forceinline__ unsigned group_max_u32(unsigned x, int grp) {
    if constexpr (kGS == 32) {
        return __reduce_max_sync(DFSIM_FULL_MASK, x);
    } else {
        unsigned r = 0u;
#pragma unroll
        for (int g = 0; g < kGroupsOf<kGS>; g++) {
            const unsigned t = __reduce_max_sync(DFSIM_FULL_MASK, grp == g ? x : 0u);
            if (grp == g) r = t;
        }
        return r;
    }
}

template <int kGS>
static __device__ __forceinline__ unsigned group_add_u32(unsigned x, int grp) {
    if constexpr (kGS == 32) {
        return __reduce_add_sync(DFSIM_FULL_MASK, x);
    } else {
        unsigned r = 0u;
#pragma unroll
        for (int g = 0; g < kGroupsOf<kGS>; g++) {
            const unsigned t = __reduce_add_sync(DFSIM_FULL_MASK, grp == g ? x : 0u);
            if (grp == g) r = t;
        }
        return r;
    }
}

template <int kGS>
static __device__ __forceinline__ unsigned group_bits(unsigned b, int grp) {
    if constexpr (kGS == 32) {
        return b;
    } else {
        return (b >> (grp * kGS)) & ((1u << kGS) - 1u);
    }
}

template <int kGS>
static __device__ __forceinline__ bool group_any(bool p, int grp) {
    return group_bits<kGS>(__ballot_sync(DFSIM_FULL_MASK, p), grp) != 0;
}

// finishes are >= +0.0, so their IEEE bits order like unsigned integers
template <int kGS>
static __device__ __forceinline__ double group_min_nonneg(double x, int grp) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    const unsigned hi = group_min_u32<kGS>(static_cast<unsigned>(b >> 32), grp);
    const unsigned lo = group_min_u32<kGS>(static_cast<unsigned>(b >> 32) == hi ? static_cast<unsigned>(b) : 0xffffffffu, grp);
    return __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(hi) << 32) | lo));
}

template <int kGS>
static __device__ __forceinline__ double group_max_nonneg(double x, int grp) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    const unsigned hi = group_max_u32<kGS>(static_cast<unsigned>(b >> 32), grp);
    const unsigned lo = group_max_u32<kGS>(static_cast<unsigned>(b >> 32) == hi ? static_cast<unsigned>(b) : 0u, grp);
    return __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(hi) << 32) | lo));
}

