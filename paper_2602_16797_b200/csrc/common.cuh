// Device-side helpers shared by every msvd kernel (sm_100a only).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#ifndef __CUDACC__
#error "common.cuh is CUDA-only"
#endif

namespace msvd {

constexpr unsigned kFull = 0xffffffffu;
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier (CTA scope) -------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "MSVD_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra MSVD_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// ---- TMA bulk copy global -> shared (1-D, UBLKCP), streaming L2 policy ----
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// 8-byte cp.async (LDGSTS) global -> shared, grouped completion
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// named barrier among `nthreads` threads (id 1..15; 0 is __syncthreads)
// order this thread's earlier generic shared-memory accesses before later
// async-proxy (bulk copy) writes to the same buffer
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, o));
    return v;
}

// Transpose-reduce over NV (16 or 32) slots: every lane holds v[0..NV); on
// return v[0] on lane l is the warp-wide sum of slot l % NV.
// NV-1 shuffles for the transpose plus one per remaining lane bit.
template <int NV>
__device__ __forceinline__ double warp_transpose_reduce(double (&v)[NV]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int s = NV / 2; s >= 1; s >>= 1) {
        const bool upper = (lane & s) != 0;
#pragma unroll
        for (int i = 0; i < s; ++i) {
            const double send = upper ? v[i] : v[i + s];
            const double keep = upper ? v[i + s] : v[i];
            v[i] = keep + __shfl_xor_sync(kFull, send, s);
        }
    }
#pragma unroll
    for (int o = NV; o < 32; o <<= 1) v[0] += __shfl_xor_sync(kFull, v[0], o);
    return v[0];
}
__device__ __forceinline__ double warp_transpose_reduce32(double (&v)[32]) {
    return warp_transpose_reduce<32>(v);
}

// ---- SplitMix64 (rng.hpp:13-64) -------------------------------------------
__device__ __forceinline__ uint64_t sm_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t sm_keyed_state(uint64_t seed, uint64_t key) {
    return sm_mix(seed + kGolden * (key + 1));
}

__device__ __forceinline__ double atomic_max_pos(double* addr, double v) {
    // valid for non-negative doubles: their bit patterns order like int64
    unsigned long long* a = reinterpret_cast<unsigned long long*>(addr);
    unsigned long long old = atomicMax(a, static_cast<unsigned long long>(__double_as_longlong(v)));
    return __longlong_as_double(static_cast<long long>(old));
}

}  // namespace msvd
