// common.cuh -- shared device helpers of the sm_100a IIR kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

namespace iirg {

#ifndef IIRG_NT
#define IIRG_NT 128
#endif
constexpr int NT = IIRG_NT;      // threads per CTA (4 warps)
constexpr int NW = NT / 32;      // warps per CTA
constexpr int LOG_NW = NW == 2 ? 1 : NW == 4 ? 2 : NW == 8 ? 3 : NW == 16 ? 4 : 5;

constexpr int HALO = 8;          // u-history halo of the DF backward tile (>= M)
#ifndef IIRG_DF_GU
#define IIRG_DF_GU 2                 // unroll of the DF backward's per-chunk group loops (I-cache)
#endif

// Samples per thread chunk (L) by data type; a tile is NT * L samples.
// High orders use twice the chunk length: the fp64 carry scans cost M^2 per
// chunk, so longer chunks halve that work per sample (the per-thread recursion
// they lengthen is cheap in comparison).
#ifndef IIRG_LONG_CHUNK_M
#define IIRG_LONG_CHUNK_M 4
#endif
template <typename T, int M> struct Chunk {
    static constexpr int L = (sizeof(T) == 4 ? 32 : 16) * (M >= IIRG_LONG_CHUNK_M ? 2 : 1);
};

// Shared-memory tile layout: 16 B of padding after every 128 B row, so that the
// 128-bit reads of 8 consecutive threads (each owning one or more whole rows)
// fall into distinct banks.
template <typename T> __host__ __device__ constexpr int pidx(int e) {
    return e + (e / (128 / (int)sizeof(T))) * (16 / (int)sizeof(T));
}

template <typename T> struct Vec;
template <> struct Vec<float>  { using type = float4;  static constexpr int W = 4; };
template <> struct Vec<double> { using type = double2; static constexpr int W = 2; };

__device__ __forceinline__ float  vget(const float4& v, int i)  { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }
__device__ __forceinline__ double vget(const double2& v, int i) { return i == 0 ? v.x : v.y; }
__device__ __forceinline__ void vset(float4& v, int i, float s)   { if (i == 0) v.x = s; else if (i == 1) v.y = s; else if (i == 2) v.z = s; else v.w = s; }
__device__ __forceinline__ void vset(double2& v, int i, double s) { if (i == 0) v.x = s; else v.y = s; }

// Blackwell paired fp32 FMA (fma.rn.f32x2 -> FFMA2): two lanes of a 64-bit
// register pair per instruction; a pair built from one scalar (pk2(s, s)) is
// folded by ptxas into the instruction's scalar-broadcast operand form.
__device__ __forceinline__ unsigned long long pk2(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ float lo2(unsigned long long v) { return __uint_as_float((unsigned)(v & 0xffffffffull)); }
__device__ __forceinline__ float hi2(unsigned long long v) { return __uint_as_float((unsigned)(v >> 32)); }

// Streaming global accesses (no L1 allocation; inputs are read exactly once).
__device__ __forceinline__ float4 ldg_stream(const float4* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ double2 ldg_stream(const double2* p) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ void stg_stream(float4* p, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ void stg_stream(double2* p, double2 v) {
    asm volatile("st.global.cs.v2.f64 [%0], {%1,%2};" :: "l"(p), "d"(v.x), "d"(v.y) : "memory");
}

// Loads of data another pass just pulled into L2 (no L1 allocation).
__device__ __forceinline__ float4 ldg_l2(const float4* p) {
    float4 r;
    asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ double2 ldg_l2(const double2* p) {
    double2 r;
    asm volatile("ld.global.cg.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}
// Bulk prefetch of [p, p + bytes) into L2 (16 B aligned, bytes a multiple of 16).
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(p), "r"(bytes) : "memory");
}

// Look-back status words: release / acquire at GPU scope.
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Look-back payload slots: every fp64 slot starts as the all-ones NaN sentinel
// (never produced by arithmetic: NVIDIA GPUs return a canonical NaN), so a
// reader needs one round trip and no separate flag: it re-reads until no
// element is the sentinel.  8-byte stores / loads are single-copy atomic.
__device__ __forceinline__ double ld_relaxed(const double* p) {
    double v;   // volatile: performed every time (a .cv cache hint alone may be hoisted by ptxas)
    asm volatile("ld.volatile.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ bool is_sentinel(double v) { return __double_as_longlong(v) == -1LL; }
__device__ __forceinline__ double sentinel() { return __longlong_as_double(-1LL); }

__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// Debug phase tracing (globaltimer ns); disabled when the pointer is null.
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// Kernel spans (debug): slots [base + 2 kind] = first CTA entry, [+1] = last CTA exit.
__device__ __forceinline__ void span_enter(unsigned long long* sp) {
    if (sp != nullptr && threadIdx.x == 0) atomicMin(sp, gtimer());
}
__device__ __forceinline__ void span_exit(unsigned long long* sp) {
    if (sp != nullptr && threadIdx.x == 0) atomicMax(sp + 1, gtimer());
}
#define IIRG_TRACE(ptr, slot, k) \
    do { if ((ptr) != nullptr && threadIdx.x == 0) (ptr)[(size_t)(slot) * 16 + (k)] = gtimer(); } while (0)

__device__ __forceinline__ double shfl_up_d(double v, int d) { return __shfl_up_sync(0xffffffffu, v, d); }
__device__ __forceinline__ double shfl_d(double v, int s) { return __shfl_sync(0xffffffffu, v, s); }

// Copy global [p0, p0+n) of a row of length Tlen into a padded smem tile;
// positions outside [0, Tlen) read as zero.  vec: rows and p0 are 16 B aligned.
template <typename T, int N>
__device__ __forceinline__ void tile_load(T* __restrict__ sm, const T* __restrict__ row, int64_t p0,
                                          int64_t Tlen, bool vec) {
    using V = typename Vec<T>::type;
    constexpr int W = Vec<T>::W;
    if (vec) {
#pragma unroll 4
        for (int q = threadIdx.x; q < N / W; q += NT) {
            const int64_t pos = p0 + (int64_t)q * W;
            V v;
            if (pos >= 0 && pos < Tlen) v = ldg_stream(reinterpret_cast<const V*>(row + pos));
            else { v = V{}; }
            *reinterpret_cast<V*>(sm + pidx<T>(q * W)) = v;
        }
    } else {
        for (int e = threadIdx.x; e < N; e += NT) {
            const int64_t pos = p0 + e;
            sm[pidx<T>(e)] = (pos >= 0 && pos < Tlen) ? row[pos] : T(0);
        }
    }
}

// Store the smem tile [0, N) to global positions [p0, p0+N) clipped to [0, Tlen).
template <typename T, int N>
__device__ __forceinline__ void tile_store(T* __restrict__ row, const T* __restrict__ sm, int64_t p0,
                                           int64_t Tlen, bool vec) {
    using V = typename Vec<T>::type;
    constexpr int W = Vec<T>::W;
    if (vec && p0 >= 0 && p0 + N <= Tlen) {        // interior tile: no clipping
        T* dst = row + p0;
#pragma unroll
        for (int q = threadIdx.x; q < N / W; q += NT)
            stg_stream(reinterpret_cast<V*>(dst + q * W), *reinterpret_cast<const V*>(sm + pidx<T>(q * W)));
    } else if (vec) {
#pragma unroll 4
        for (int q = threadIdx.x; q < N / W; q += NT) {
            const int64_t pos = p0 + (int64_t)q * W;
            if (pos >= 0 && pos < Tlen)
                stg_stream(reinterpret_cast<V*>(row + pos), *reinterpret_cast<const V*>(sm + pidx<T>(q * W)));
        }
    } else {
        for (int e = threadIdx.x; e < N; e += NT) {
            const int64_t pos = p0 + e;
            if (pos >= 0 && pos < Tlen) row[pos] = sm[pidx<T>(e)];
        }
    }
}


// ---- cp.async (Ampere+ LDGSTS; 16 B, L2 only, zero-fill when src_bytes = 0) ----
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, unsigned src_bytes) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" :: "r"(s), "l"(gmem), "r"(src_bytes) : "memory");
}
// 16 B through L1 (.ca): data every CTA of an SM reads (the power tables)
__device__ __forceinline__ void cp_async16_ca(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" :: "r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(s), "l"(gmem) : "memory");
}
// one 4 / 8 byte element (the size of T)
template <typename T>
__device__ __forceinline__ void cp_async_elem(T* smem, const T* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    if constexpr (sizeof(T) == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(s), "l"(gmem) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(s), "l"(gmem) : "memory");
}
// the mbarrier tracks this thread's prior cp.async copies: its pending count is raised by one
// now and lowered when they have landed (no .noinc)
__device__ __forceinline__ void cp_async_mbar_arrive(unsigned long long* bar) {
    asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];"
                 :: "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }

// Asynchronous version of tile_load (vector path via cp.async; the scalar path
// is synchronous).  The caller commits / waits.
template <typename T, int N>
__device__ __forceinline__ void tile_load_async(T* __restrict__ sm, const T* __restrict__ row, int64_t p0,
                                                int64_t Tlen, bool vec) {
    constexpr int W = Vec<T>::W;
    if (vec && p0 >= 0 && p0 + N <= Tlen) {        // interior tile: no clipping
        const T* src = row + p0;
#pragma unroll
        for (int q = threadIdx.x; q < N / W; q += NT) cp_async16(sm + pidx<T>(q * W), src + q * W, 16u);
    } else if (vec) {
#pragma unroll 4
        for (int q = threadIdx.x; q < N / W; q += NT) {
            const int64_t pos = p0 + (int64_t)q * W;
            const bool in = pos >= 0 && pos < Tlen;
            cp_async16(sm + pidx<T>(q * W), in ? (const void*)(row + pos) : (const void*)row, in ? 16u : 0u);
        }
    } else {
        for (int e = threadIdx.x; e < N; e += NT) {
            const int64_t pos = p0 + e;
            sm[pidx<T>(e)] = (pos >= 0 && pos < Tlen) ? row[pos] : T(0);
        }
    }
}


// ---- TMA bulk copies (cp.async.bulk, no tensor map) + mbarrier -------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
// global -> shared, completion counted on `bar` (bytes: multiple of 16, both 16 B aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// shared -> global (bulk group)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 :: "l"(dst), "r"(smem_u32(src)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

}  // namespace iirg
