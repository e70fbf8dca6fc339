// tv.cuh -- per-sample ("parameter-varying") all-pole DF filter:
//   y(n) = x(n) - sum_{i=1..M} a_i(n) y(n-i),   v(n) = [y(n-1) .. y(n-M)],  v(0) = zi
// and its closed-form backward (Eq.7 with time-varying A(n) = companion(a(n)),
// C(n) = -a(n), D = 1; readings R10/R11):
//   g(n) = dz(n)[0] + dy(n)        (= grad_x(n), Eq.8)
//   dz(n-1)[i] = dz(n)[i+1] - a_{i+1}(n) g(n),   dz(N-1) = grad_zf,  grad_zi = dz(-1)
//   grad_a_i(n) = -g(n) y(n-i)     (Eq.9's dA(n) = dz(n) v(n)^T and Eq.6's dC)
//
// Time parallelism (Eq.10) with time-varying transitions: the sequence is cut
// into segments of TV_SEG samples.  Segment k's transition Phi_k = A(n1-1)..A(n0)
// and zero-state response w_k are built by one warp, lane j propagating the
// basis state e_j (lane M propagates x from the zero state): M^2 FMA per sample,
// the price of a matrix-valued scan element.  A per-sequence fp64
// chain s_{k+1} = Phi_k s_k + w_k (two-level: groups of TV_GS segments) gives
// every segment's entering state, and one
// thread per segment re-runs the plain recursion from it.  The backward reuses
// Phi_k^T from the tape (the adjoint segment map is exactly Phi_k^T).
#pragma once
#include "common.cuh"

namespace iirg {

#ifndef IIRG_TV_SEG
#define IIRG_TV_SEG 512
#endif
constexpr int TV_SEG = IIRG_TV_SEG;  // samples per segment
constexpr int TV_THREADS = 128;      // thread-per-segment kernels
constexpr int TV_PHI_WARPS = 4;      // warps (segments) per CTA of the Phi kernel
template <typename T> constexpr int tv_ch() { return sizeof(T) == 4 ? 32 : 16; }   // staged chunk (Phi kernel)
constexpr int TV_U = 8;              // unroll of the sequential recursions

#ifndef IIRG_TV_GS
#define IIRG_TV_GS 16
#endif
constexpr int TV_GS = IIRG_TV_GS;    // segments per group of the two-level chain
constexpr int TV_GRP_WARPS = 2;      // warps (groups) per CTA of the group / expansion kernels

struct TvArgs {
    const void* a; const void* x; const void* zi;     // a: (B, T, M)
    void* y; void* zf;                                // forward outputs
    const void* gy; const void* gzf; const void* yin; // backward inputs (yin = forward y)
    void* gx; void* ga; void* gzi;                    // backward outputs
    void* phi;                                        // tape: [B][nseg][M][M]  (Phi[i][j])
    double* w;                                        // ws: [B][nseg][M] segment aggregates
    double* carry;                                    // ws: [B][nseg][M] entering states
    int64_t B, T; int nseg;
    int vec;                                          // rows 16 B aligned and M % (16 / sizeof(T)) == 0
    double* psi;                                      // ws: [B][ngrp][M][M] group transitions
    double* omega;                                    // ws: [B][ngrp][M] group zero-state responses
    double* sgrp;                                     // ws: [B][ngrp][M] states entering each group
    int ngrp;
};

// ---------------------------------------------------------------------------
// Forward phase 1: one warp per segment builds Phi_k (lanes 0..M-1) and w_k
// (lane M).  Coefficients are staged per chunk of TV_CH samples in shared
// memory and read by broadcast.
// A: accumulation type (fp64 for fp32 data: the basis propagation over a segment
// sees transient, non-normal growth of the time-varying product; fp32 accumulation
// measured 2.7e-5 y error and 2e-4 grad_a error on config 3's 32 sequences).
#ifndef IIRG_PHI_MINB
#define IIRG_PHI_MINB 1
#endif
template <typename T, int M, typename A = T>
__global__ void __launch_bounds__(32 * TV_PHI_WARPS, IIRG_PHI_MINB) tv_phi_kernel(const TvArgs p) {
    static_assert(M <= 32, "orders 1..32");
    // Columns: lane l of column block cb carries column col = 32 cb + l (col < M: basis
    // state e_col, col = M: the input response w).  Orders <= 31 need one block; order 32
    // runs a second block for the input column (the segment's coefficients staged again).
    constexpr int NCB = (M + 1 + 31) / 32;
    // With A wider than T the staged chunk is converted ONCE into an A copy (each lane
    // converts 1/32 of it) instead of every lane converting all M coefficients of every
    // sample: the F2F conversions, not the FMAs, bounded the fp64-accumulating kernel.
    constexpr bool CONV = sizeof(A) != sizeof(T);
    constexpr int TV_CH = CONV ? 16 : tv_ch<T>();
    __shared__ __align__(16) T sa[TV_PHI_WARPS][2][TV_CH * M];
    __shared__ __align__(16) T sx[TV_PHI_WARPS][2][TV_CH];
    __shared__ __align__(16) A sd[TV_PHI_WARPS][CONV ? TV_CH * M : 2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t seg = (int64_t)blockIdx.x * TV_PHI_WARPS + warp;
    if (seg >= p.B * p.nseg) return;
    const int64_t seq = seg / p.nseg;
    const int k = (int)(seg - seq * p.nseg);
    const int64_t n0 = (int64_t)k * TV_SEG, n1 = min(n0 + TV_SEG, p.T);
    const T* arow = static_cast<const T*>(p.a) + seq * p.T * M;
    const T* xrow = static_cast<const T*>(p.x) + seq * p.T;
    constexpr int E = 16 / (int)sizeof(T);
    const bool vec = p.vec != 0 && (TV_CH * M) % E == 0;
    // stage chunk [c, c + TV_CH) into buffer b (zero beyond n1)
    auto stage = [&](int64_t c, int b) {
        const int cnt = (int)min((int64_t)TV_CH, n1 - c);
        if (vec && cnt == TV_CH) {
            for (int e = lane * E; e < TV_CH * M; e += 32 * E) cp_async16(&sa[warp][b][e], arow + c * M + e, 16u);
        } else {
            for (int e = lane; e < TV_CH * M; e += 32) sa[warp][b][e] = (e < cnt * M) ? arow[c * M + e] : T(0);
        }
        if (lane < TV_CH) sx[warp][b][lane] = (lane < cnt) ? xrow[c + lane] : T(0);
    };
#pragma unroll 1
    for (int cb = 0; cb < NCB; ++cb) {
    const int col = 32 * cb + lane;
    A v[M];
#pragma unroll
    for (int i = 0; i < M; ++i) v[i] = (col == i) ? A(1) : A(0);
    __syncwarp();
    stage(n0, 0);
    cp_async_commit();
    int b = 0;
    for (int64_t c = n0; c < n1; c += TV_CH, b ^= 1) {
        const int cnt = (int)min((int64_t)TV_CH, n1 - c);
        __syncwarp();
        if (c + TV_CH < n1) stage(c + TV_CH, b ^ 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncwarp();
        const A* cs;
        if constexpr (CONV) {
#pragma unroll
            for (int e = lane; e < TV_CH * M; e += 32) sd[warp][e] = A(sa[warp][b][e]);
            __syncwarp();
            cs = sd[warp];
        } else {
            cs = reinterpret_cast<const A*>(sa[warp][b]);
        }
        if (cnt == TV_CH) {
#pragma unroll
            for (int s2 = 0; s2 < TV_CH; ++s2) {
                A yn = (col == M) ? A(sx[warp][b][s2]) : A(0);
                A cf[M];
                if constexpr ((M * sizeof(A)) % 16 == 0) {
#pragma unroll
                    for (int q = 0; q < M * (int)sizeof(A) / 16; ++q) {
                        const uint4 t4 = reinterpret_cast<const uint4*>(cs + s2 * M)[q];
                        memcpy(&cf[q * (16 / sizeof(A))], &t4, 16);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < M; ++i) cf[i] = cs[s2 * M + i];
                }
                if constexpr (M >= 8) {
                    // four independent partial sums (terms i = 3 mod 4 ... 0 mod 4) cut the
                    // dependent DFMA chain from M to M/4 + 2 (latency, not the FP64 pipe, bound it)
                    A ps[4] = {yn, A(0), A(0), A(0)};
#pragma unroll
                    for (int i = M - 1; i >= 0; --i) ps[i & 3] = fma(-cf[i], v[i], ps[i & 3]);
                    yn = (ps[0] + ps[1]) + (ps[2] + ps[3]);
                } else {
#pragma unroll
                    for (int i = M - 1; i >= 0; --i) yn = fma(-cf[i], v[i], yn);
                }
#pragma unroll
                for (int i = M - 1; i >= 1; --i) v[i] = v[i - 1];
                v[0] = yn;
            }
        } else {                                   // ragged last chunk: exactly cnt samples
            for (int s2 = 0; s2 < cnt; ++s2) {
                A yn = (col == M) ? A(sx[warp][b][s2]) : A(0);
#pragma unroll
                for (int i = M - 1; i >= 0; --i) yn = fma(-cs[s2 * M + i], v[i], yn);
#pragma unroll
                for (int i = M - 1; i >= 1; --i) v[i] = v[i - 1];
                v[0] = yn;
            }
        }
    }
    if (col < M) {
        T* ph = static_cast<T*>(p.phi) + seg * M * M;
#pragma unroll
        for (int i = 0; i < M; ++i) ph[i * M + col] = (T)v[i];             // column `col`
    } else if (col == M && p.w != nullptr) {                        // (NULL: w comes from TV_FWD_AGG)
#pragma unroll
        for (int i = 0; i < M; ++i) p.w[seg * M + i] = (double)v[i];
    }
    }                                                                    // column blocks
}

// ---------------------------------------------------------------------------
// Two-level chain (replaces the serial per-sequence chain over all segments).
// Segments are grouped by TV_GS in chain order (FWD: increasing k, BWD:
// decreasing k).  (1) tv_group_kernel, one warp per group: the group map
// Psi_g = Phi_last .. Phi_first (BWD: transposes) and zero-state response
// omega_g, fp64;  (2) tv_groupchain_kernel, one warp per sequence:
// S_{g+1} = Psi_g S_g + omega_g over the groups;  (3) tv_expand_kernel, one
// warp per group: carry[k] for the group's segments from S_g.  The serial
// depth drops from nseg hops to nseg / TV_GS + TV_GS hops.
template <typename T, int M>
struct TvPhiBuf {                                       // per-warp double buffer of one Phi_k (T, M x M)
    static constexpr int MM = M * M;
    static constexpr int E = 16 / (int)sizeof(T);
    static constexpr int SLOT = (MM + E - 1) / E * E;   // elements, 16 B multiple
};
template <typename T, int M>
__device__ __forceinline__ void tv_load_phi(T* dst, const T* src, int lane, bool vec) {
    using PB = TvPhiBuf<T, M>;
    if (vec && (PB::MM % PB::E) == 0) {
        for (int e = lane * PB::E; e < PB::MM; e += 32 * PB::E) cp_async16(dst + e, src + e, 16u);
    } else {
        for (int e = lane; e < PB::MM; e += 32) dst[e] = src[e];
    }
}

template <typename T, int M, bool BWD>
__global__ void __launch_bounds__(32 * TV_GRP_WARPS) tv_group_kernel(const TvArgs p) {
    using PB = TvPhiBuf<T, M>;
    constexpr bool CONV = sizeof(T) != sizeof(double);   // fp32 tape: convert each Phi once
    constexpr int SDS = M + 1;                            // padded row stride of the fp64 copy
    __shared__ __align__(16) T sphi[TV_GRP_WARPS][2][PB::SLOT];
    __shared__ __align__(16) double sdp[TV_GRP_WARPS][CONV ? M * SDS : 1];
    __shared__ double som[TV_GRP_WARPS][M];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t gid = (int64_t)blockIdx.x * TV_GRP_WARPS + warp;
    if (gid >= p.B * p.ngrp) return;
    const int64_t seq = gid / p.ngrp;
    const int g = (int)(gid - seq * p.ngrp);
    const int k0 = g * TV_GS, k1 = min(k0 + TV_GS, p.nseg), nk = k1 - k0;
    const T* phi = static_cast<const T*>(p.phi) + seq * p.nseg * PB::MM;
    const double* wv = p.w + seq * p.nseg * M;
    const bool vec = (reinterpret_cast<uintptr_t>(p.phi) & 15u) == 0;
    auto kof = [&](int q) { return BWD ? k1 - 1 - q : k0 + q; };
    double col[M];                                       // lane j: column j of Psi
#pragma unroll
    for (int i = 0; i < M; ++i) col[i] = (i == lane) ? 1.0 : 0.0;
    double om = 0.0;                                     // lane i: omega_i
    tv_load_phi<T, M>(sphi[warp][0], phi + (int64_t)kof(0) * PB::MM, lane, vec);
    cp_async_commit();
    for (int q = 0; q < nk; ++q) {
        const int k = kof(q), b = q & 1;
        if (q + 1 < nk) tv_load_phi<T, M>(sphi[warp][b ^ 1], phi + (int64_t)kof(q + 1) * PB::MM, lane, vec);
        cp_async_commit();
        const double wk = lane < M ? wv[(int64_t)k * M + lane] : 0.0;
        if (lane < M) som[warp][lane] = om;
        cp_async_wait<1>();
        __syncwarp();
        // the segment's transition converted to fp64 ONCE (each lane 1/32 of it; BWD: transposed)
        // instead of one conversion per use by every lane (M^2 conversions per lane and segment)
        if constexpr (CONV) {
            const T* P = sphi[warp][b];
            double* D = sdp[warp];
            for (int e = lane; e < M * M; e += 32) {
                const int r = e / M, c = e - r * M;
                D[BWD ? c * SDS + r : r * SDS + c] = (double)P[e];
            }
        }
        __syncwarp();
        // element (i, l) of Phi (BWD: Phi^T)
        auto el = [&](int i, int l) -> double {
            if constexpr (CONV) return sdp[warp][i * SDS + l];
            else { const T* P = sphi[warp][b]; return (double)(BWD ? P[l * M + i] : P[i * M + l]); }
        };
        if (lane < M) {
            double nc[M];
#pragma unroll
            for (int i = 0; i < M; ++i) {                // Psi <- Phi Psi  (BWD: Phi^T Psi)
                double acc = 0.0;
#pragma unroll
                for (int l = 0; l < M; ++l) acc = fma(el(i, l), col[l], acc);
                nc[i] = acc;
            }
#pragma unroll
            for (int i = 0; i < M; ++i) col[i] = nc[i];
            double a = wk;                               // omega <- Phi omega + w_k
#pragma unroll
            for (int l = 0; l < M; ++l) a = fma(el(lane, l), som[warp][l], a);
            om = a;
        }
        __syncwarp();
    }
    if (lane < M) {
        double* ps = p.psi + gid * PB::MM;
#pragma unroll
        for (int i = 0; i < M; ++i) ps[i * M + lane] = col[i];
        p.omega[gid * M + lane] = om;
    }
}

// one warp per sequence: S_{g+1} = Psi_g S_g + omega_g (chain order), S_0 = zi / grad_zf
template <int M, bool BWD>
__global__ void __launch_bounds__(32) tv_groupchain_kernel(const TvArgs p, const void* x0v, int dsz) {
    constexpr int MM = M * M;
    constexpr int RING = 4;
    __shared__ __align__(16) double ring[RING][MM + (MM & 1)];
    __shared__ double ss[M];
    const int lane = threadIdx.x;
    const int64_t seq = blockIdx.x;
    double s = 0.0;
    if (x0v != nullptr && lane < M)
        s = dsz == 8 ? static_cast<const double*>(x0v)[seq * M + lane]
                     : (double)static_cast<const float*>(x0v)[seq * M + lane];
    const double* psi = p.psi + seq * p.ngrp * MM;
    auto gof = [&](int q) { return BWD ? p.ngrp - 1 - q : q; };
    auto issue = [&](int q) {
        if (q < p.ngrp) {
            const double* src = psi + (int64_t)gof(q) * MM;
            if constexpr (MM % 2 == 0) {                 // 16 B pieces stay aligned
                for (int e = lane * 2; e < MM; e += 64) cp_async16(&ring[q % RING][e], src + e, 16u);
            } else {
                for (int e = lane; e < MM; e += 32) ring[q % RING][e] = src[e];
            }
        }
        cp_async_commit();
    };
    for (int q = 0; q < RING - 1; ++q) issue(q);
    for (int q = 0; q < p.ngrp; ++q) {
        const int g = gof(q);
        __syncwarp();
        issue(q + RING - 1);
        const double og = lane < M ? p.omega[(seq * p.ngrp + g) * M + lane] : 0.0;
        if (lane < M) { p.sgrp[(seq * p.ngrp + g) * M + lane] = s; ss[lane] = s; }
        cp_async_wait<RING - 1>();
        __syncwarp();
        double a0 = og, a1 = 0.0;
        if (lane < M) {
            const double* P = ring[q % RING];
#pragma unroll
            for (int j = 0; j < M; j += 2) {
                a0 = fma(P[lane * M + j], ss[j], a0);
                if (j + 1 < M) a1 = fma(P[lane * M + j + 1], ss[j + 1], a1);
            }
        }
        s = a0 + a1;
    }
}

// one warp per group: carry[k] = state entering segment k, from S_g
template <typename T, int M, bool BWD>
__global__ void __launch_bounds__(32 * TV_GRP_WARPS) tv_expand_kernel(const TvArgs p) {
    using PB = TvPhiBuf<T, M>;
    __shared__ __align__(16) T sphi[TV_GRP_WARPS][2][PB::SLOT];
    __shared__ double ss[TV_GRP_WARPS][M];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t gid = (int64_t)blockIdx.x * TV_GRP_WARPS + warp;
    if (gid >= p.B * p.ngrp) return;
    const int64_t seq = gid / p.ngrp;
    const int g = (int)(gid - seq * p.ngrp);
    const int k0 = g * TV_GS, k1 = min(k0 + TV_GS, p.nseg), nk = k1 - k0;
    const T* phi = static_cast<const T*>(p.phi) + seq * p.nseg * PB::MM;
    const double* wv = p.w + seq * p.nseg * M;
    const bool vec = (reinterpret_cast<uintptr_t>(p.phi) & 15u) == 0;
    auto kof = [&](int q) { return BWD ? k1 - 1 - q : k0 + q; };
    double s = lane < M ? p.sgrp[gid * M + lane] : 0.0;
    tv_load_phi<T, M>(sphi[warp][0], phi + (int64_t)kof(0) * PB::MM, lane, vec);
    cp_async_commit();
    for (int q = 0; q < nk; ++q) {
        const int k = kof(q), b = q & 1;
        if (q + 1 < nk) tv_load_phi<T, M>(sphi[warp][b ^ 1], phi + (int64_t)kof(q + 1) * PB::MM, lane, vec);
        cp_async_commit();
        const double wk = lane < M ? wv[(int64_t)k * M + lane] : 0.0;
        if (lane < M) { p.carry[(seq * p.nseg + k) * M + lane] = s; ss[warp][lane] = s; }
        cp_async_wait<1>();
        __syncwarp();
        double a0 = wk, a1 = 0.0;
        if (lane < M) {
            const T* P = sphi[warp][b];
#pragma unroll
            for (int j = 0; j < M; j += 2) {
                a0 = fma((double)(BWD ? P[j * M + lane] : P[lane * M + j]), ss[warp][j], a0);
                if (j + 1 < M) a1 = fma((double)(BWD ? P[(j + 1) * M + lane] : P[lane * M + j + 1]), ss[warp][j + 1], a1);
            }
        }
        __syncwarp();
        s = a0 + a1;
    }
}

// Coefficient row of sample n (M values).
template <typename T, int M>
__device__ __forceinline__ void load_row(const T* __restrict__ ar, T (&c)[M]) {
    if constexpr (sizeof(T) == 4 && M % 4 == 0) {
#pragma unroll
        for (int q = 0; q < M / 4; ++q) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(ar) + q);
            c[4 * q] = t.x; c[4 * q + 1] = t.y; c[4 * q + 2] = t.z; c[4 * q + 3] = t.w;
        }
    } else if constexpr (sizeof(T) == 8 && M % 2 == 0) {
#pragma unroll
        for (int q = 0; q < M / 2; ++q) {
            const double2 t = __ldg(reinterpret_cast<const double2*>(ar) + q);
            c[2 * q] = t.x; c[2 * q + 1] = t.y;
        }
    } else {
#pragma unroll
        for (int i = 0; i < M; ++i) c[i] = __ldg(ar + i);
    }
}

// ---------------------------------------------------------------------------
// Thread-per-segment recursions (forward emit, backward aggregate, backward
// emit).  Lane l of a warp owns segment 32 w + l, so every lane streams its own
// contiguous 4M bytes/sample of coefficient rows.  Each lane moves its segment's
// chunk of C samples with ONE TMA bulk copy (cp.async.bulk, global -> shared,
// completion counted on a per-buffer mbarrier; double-buffered), and grad_a
// leaves the same way (shared -> global bulk copy), so the 96 B/sample streams
// cost O(1) instructions per chunk instead of one uncoalesced access per 16 B.
// Rows are padded by 16 B in shared memory: the lanes' 128-bit reads of their
// own rows are bank-conflict free.  The short per-sample scalars (x, y, dy, dx)
// are accessed per lane; each 128 B line then serves 32 samples from L1.
// The recursions accumulate in fp64 (R) with T I/O: these kernels are bound by
// the coefficient bytes, and fp64 removes the O(TV_SEG) fp32 rounding growth of
// a long feedback loop ("TV precision").
constexpr int TV_SEQ_WARPS = 2;           // warps per CTA (x 32 segments)
// TV_FWD_AGG: the forward recursion from the zero state over each segment, fp64, writing only
// the segment's zero-state response w_k (no output): the input column of tv_phi in fp64.
enum TvMode { TV_FWD_EMIT = 0, TV_BWD_AGG = 1, TV_BWD_EMIT = 2, TV_FWD_AGG = 3 };
// Samples per staged chunk: the coefficient stream is latency-bound (one
// thread per segment, few warps per SM), so the bytes in flight per lane are
// what sets the bandwidth; the emit-backward also stages grad_a (its TMA
// store beats per-lane row stores), so it keeps smaller chunks to stay at the
// same occupancy.
constexpr int TV_PF = 3;                  // chunks of scalar-stream prefetch in tv_seq_kernel (ring of 4)
#ifndef IIRG_TV_CHF
#define IIRG_TV_CHF 8                        // samples per staged coefficient chunk (forward / aggregate modes)
#endif
#ifndef IIRG_TV_CHB
#define IIRG_TV_CHB 4                        // ... backward emit (three buffers)
#endif
template <typename T, int M, int MODE> constexpr int tv_chunk() {
    return (MODE != TV_BWD_EMIT && M * (int)sizeof(T) <= 128) ? IIRG_TV_CHF : IIRG_TV_CHB;
}
template <typename T, int M, int MODE>
__device__ __forceinline__ int64_t chunk_start_of(int64_t n0, int c, bool bwd) {
    constexpr int C = tv_chunk<T, M, MODE>();
    return bwd ? n0 + (int64_t)(TV_SEG / C - 1 - c) * C : n0 + (int64_t)c * C;
}

template <typename T, int M, int MODE>
struct TvStage {
    static constexpr int PAD = 16 / (int)sizeof(T);
    static constexpr int C = tv_chunk<T, M, MODE>();
    static constexpr int ROW = C * M;                   // elements of one segment's chunk
    static constexpr int STRIDE = ROW + PAD;            // smem row stride (elements), 16 B multiple
    static constexpr int NBUF(int mode) { return 2 + (mode == TV_BWD_EMIT ? 1 : 0); }
    static constexpr size_t bytes(int mode) {           // per CTA (plus static mbarriers)
        return (size_t)TV_SEQ_WARPS * NBUF(mode) * 32 * STRIDE * sizeof(T);
    }
};

template <typename T, int M, int MODE>
__global__ void __launch_bounds__(32 * TV_SEQ_WARPS) tv_seq_kernel(const TvArgs p) {
    using R = double;
    using ST = TvStage<T, M, MODE>;
    constexpr bool BWD = MODE == TV_BWD_AGG || MODE == TV_BWD_EMIT;
    constexpr bool FWD = !BWD;
    constexpr int C = ST::C;
    constexpr int NCH = TV_SEG / C;
    constexpr int RB = M * (int)sizeof(T);                  // bytes of one coefficient row
    extern __shared__ __align__(128) unsigned char tv_raw[];
    __shared__ __align__(8) unsigned long long s_bar[TV_SEQ_WARPS][2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T* sA = reinterpret_cast<T*>(tv_raw) + (size_t)warp * ST::NBUF(MODE) * 32 * ST::STRIDE;   // 2 buffers
    T* sG = sA + 2 * 32 * ST::STRIDE;                                                            // grad_a staging
    unsigned long long* bar = s_bar[warp];
    const bool bulk = p.vec != 0;                            // rows 16 B multiples, aligned bases
    const int64_t nsegtot = p.B * p.nseg;
    const int64_t seg = ((int64_t)blockIdx.x * TV_SEQ_WARPS + warp) * 32 + lane;
    const bool valid = seg < nsegtot;
    const int64_t seq = valid ? seg / p.nseg : 0;
    const int k = valid ? (int)(seg - seq * p.nseg) : 0;
    const int64_t n0 = (int64_t)k * TV_SEG, n1 = valid ? min(n0 + TV_SEG, p.T) : n0;
    const T* a = static_cast<const T*>(p.a);
    T* myA[2] = {sA + lane * ST::STRIDE, sA + 32 * ST::STRIDE + lane * ST::STRIDE};
    T* myG = sG + lane * ST::STRIDE;
    if (lane == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); }
    mbar_fence_init();
    __syncwarp();
    unsigned phase[2] = {0u, 0u};

    // stage chunk c of every lane's segment into buffer b
    auto stage = [&](int c, int b) {
        const int64_t cs = chunk_start_of<T, M, MODE>(n0, c, BWD);
        const int64_t vs = max(cs, n0), ve = min(cs + C, n1);
        const int nv = valid && ve > vs ? (int)(ve - vs) : 0;
        T* dst = myA[b];
        // rows outside the valid range read as zero (ragged last segment only)
        if (nv < C)
            for (int e = 0; e < C * M; ++e) {
                const int64_t n = cs + e / M;
                if (!(n >= vs && n < ve)) dst[e] = T(0);
            }
        if (bulk) {
            fence_proxy_async();                             // generic reads / writes of this buffer done
            const unsigned bytes = (unsigned)(nv * RB);
            const unsigned total = __reduce_add_sync(0xffffffffu, bytes);
            if (lane == 0) mbar_arrive_expect_tx(&bar[b], total);
            __syncwarp();
            if (bytes) bulk_g2s(dst + (vs - cs) * M, a + (seq * p.T + vs) * M, bytes, &bar[b]);
        } else {
            for (int64_t n = vs; n < ve; ++n)
#pragma unroll
                for (int i = 0; i < M; ++i) dst[(n - cs) * M + i] = __ldg(a + (seq * p.T + n) * M + i);
        }
    };

    R v[M];                                      // FWD: v = [y(n-1)..y(n-M)];  BWD: d = dz(n)
    T yw[M];                                     // BWD_EMIT: yw[i] = y(n-1-i) (data type: grad_a = -g y is one product)
    const T* xrow = static_cast<const T*>(p.x) + seq * p.T;
    const T* gyrow = p.gy == nullptr ? nullptr : static_cast<const T*>(p.gy) + seq * p.T;
    const T* yrow = static_cast<const T*>(p.yin) + seq * p.T;
    T* youtrow = MODE == TV_FWD_EMIT ? static_cast<T*>(p.y) + seq * p.T : nullptr;
    T* gxrow = (MODE == TV_BWD_EMIT && p.gx != nullptr) ? static_cast<T*>(p.gx) + seq * p.T : nullptr;
    T* garow = (MODE == TV_BWD_EMIT && p.ga != nullptr) ? static_cast<T*>(p.ga) + seq * p.T * M : nullptr;
    const T* zi = p.zi == nullptr ? nullptr : static_cast<const T*>(p.zi) + seq * M;
    auto yat = [&](int64_t m) -> T {             // y(m), m >= -M; y(-k) = zi[k-1]
        if (m >= 0) return __ldg(yrow + m);
        return zi != nullptr ? zi[-m - 1] : T(0);
    };
#pragma unroll
    for (int i = 0; i < M; ++i) {
        v[i] = (MODE == TV_BWD_AGG || MODE == TV_FWD_AGG || !valid) ? 0.0 : p.carry[seg * M + i];
        yw[i] = (MODE == TV_BWD_EMIT && valid) ? yat(n1 - 2 - i) : T(0);
    }
    // The per-sample scalar streams (x forward; dy and the y window backward) are
    // loaded TV_PF chunks ahead into a register ring: a load issued at the sample
    // that needs it puts one full memory latency on the serial recursion per sample.
    constexpr int NR = TV_PF + 1;
    T ps[NR][C], py[NR][C];
    auto prefetch = [&](int c, int slot) {
        const int64_t cs = chunk_start_of<T, M, MODE>(n0, c, BWD);
#pragma unroll
        for (int u = 0; u < C; ++u) {
            const int s2 = BWD ? C - 1 - u : u;
            const int64_t n = cs + s2;
            const bool in = valid && n >= n0 && n < n1;
            if constexpr (FWD) ps[slot][u] = in ? __ldg(xrow + n) : T(0);
            else ps[slot][u] = (in && gyrow != nullptr) ? __ldg(gyrow + n) : T(0);
            if constexpr (MODE == TV_BWD_EMIT) py[slot][u] = in ? yat(n - 1 - M) : T(0);
        }
    };
#pragma unroll
    for (int c = 0; c < TV_PF; ++c)
        if (c < NCH) prefetch(c, c);
    stage(0, 0);
    static_assert(NCH % NR == 0, "the ring slot must be a compile-time constant in the unrolled loop");
#pragma unroll NR
    for (int c = 0; c < NCH; ++c) {
        const int b = c & 1;
        __syncwarp();
        if (c + 1 < NCH) stage(c + 1, b ^ 1);
        if (c + TV_PF < NCH) prefetch(c + TV_PF, (c + TV_PF) % NR);
        const int slot = c % NR;
        if (bulk) { mbar_wait(&bar[b], phase[b]); phase[b] ^= 1u; }
        __syncwarp();
        const T* my = myA[b];
        const int64_t cs = chunk_start_of<T, M, MODE>(n0, c, BWD);
        if constexpr (MODE == TV_BWD_EMIT) {
            if (bulk) bulk_wait_read0();                 // previous grad_a chunk has left smem
            __syncwarp();
        }
#pragma unroll
        for (int u = 0; u < C; ++u) {
            const int s2 = BWD ? C - 1 - u : u;          // position in the chunk
            const int64_t n = cs + s2;
            const bool in = valid && n >= n0 && n < n1;
            T cf[M];
            if constexpr (RB % 16 == 0) {
#pragma unroll
                for (int q = 0; q < M * (int)sizeof(T) / 16; ++q) {
                    const uint4 t4 = reinterpret_cast<const uint4*>(my + s2 * M)[q];
                    memcpy(&cf[q * (16 / sizeof(T))], &t4, 16);
                }
            } else {
#pragma unroll
                for (int i = 0; i < M; ++i) cf[i] = my[s2 * M + i];
            }
            if constexpr (FWD) {
                if (in) {
                    // four independent partial sums of the older terms; only the
                    // newest term (a_1 y(n-1)) waits on the previous sample
                    R acc[4] = {(R)ps[slot][u], 0.0, 0.0, 0.0};
#pragma unroll
                    for (int i = M - 1; i >= 1; --i) acc[i & 3] = fma(-(R)cf[i], v[i], acc[i & 3]);
                    const R rest = (acc[1] + acc[2]) + (acc[3] + acc[0]);
                    const R yn = fma(-(R)cf[0], v[0], rest);
#pragma unroll
                    for (int i = M - 1; i >= 1; --i) v[i] = v[i - 1];
                    v[0] = yn;
                    if constexpr (MODE == TV_FWD_EMIT) youtrow[n] = (T)yn;
                }
            } else {
                if (in) {
                    const R g = v[0] + (R)ps[slot][u];
                    if constexpr (MODE == TV_BWD_EMIT) {
                        const T gT = (T)g;
                        if (gxrow) gxrow[n] = gT;
                        if constexpr (sizeof(T) == 4 && M % 4 == 0) {   // 16 B stores (rows 16 B aligned)
#pragma unroll
                            for (int q = 0; q < M / 4; ++q)
                                reinterpret_cast<float4*>(myG + s2 * M)[q] =
                                    make_float4(-gT * yw[4 * q], -gT * yw[4 * q + 1], -gT * yw[4 * q + 2],
                                                -gT * yw[4 * q + 3]);
                        } else {
#pragma unroll
                            for (int i = 0; i < M; ++i) myG[s2 * M + i] = -gT * yw[i];
                        }
#pragma unroll
                        for (int i = 0; i < M - 1; ++i) yw[i] = yw[i + 1];
                        yw[M - 1] = py[slot][u];
                    }
#pragma unroll
                    for (int i = 0; i < M - 1; ++i) v[i] = fma(-(R)cf[i], g, v[i + 1]);
                    v[M - 1] = -(R)cf[M - 1] * g;
                }
            }
        }
        if constexpr (MODE == TV_BWD_EMIT) {
            if (garow != nullptr) {
                const int64_t vs = max(cs, n0), ve = min(cs + C, n1);
                if (valid && ve > vs) {
                    if (bulk) {
                        fence_proxy_async();                 // make the generic smem writes visible to TMA
                        bulk_s2g(garow + vs * M, myG + (vs - cs) * M, (unsigned)((ve - vs) * RB));
                        bulk_commit();
                    } else {
                        for (int64_t n = vs; n < ve; ++n)
#pragma unroll
                            for (int i = 0; i < M; ++i) garow[n * M + i] = myG[(n - cs) * M + i];
                    }
                }
            }
        }
    }
    if constexpr (MODE == TV_BWD_EMIT) {
        if (bulk) bulk_wait0();
    }
    if (!valid) return;
    if constexpr (MODE == TV_FWD_EMIT) {
        if (p.zf != nullptr && n1 == p.T) {
            T* zf = static_cast<T*>(p.zf) + seq * M;
#pragma unroll
            for (int i = 0; i < M; ++i) zf[i] = (T)v[i];
        }
    } else if constexpr (MODE == TV_BWD_AGG || MODE == TV_FWD_AGG) {
#pragma unroll
        for (int i = 0; i < M; ++i) p.w[seg * M + i] = v[i];
    } else {
        if (p.gzi != nullptr && k == 0) {
            T* gzi = static_cast<T*>(p.gzi) + seq * M;
#pragma unroll
            for (int i = 0; i < M; ++i) gzi[i] = (T)v[i];
        }
    }
}

}  // namespace iirg
