// ubench.cu -- design microbenchmarks for the round-2 LTI engine (not part of the library).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I. tools/ubench.cu -o /tmp/ubench
// (a) issue rates of FFMA, FFMA2 (fma.rn.f32x2), DFMA per SM per clock;
// (b) streaming read+write bandwidth of (i) a float4 copy kernel, (ii) persistent warp tiles moved by
//     per-lane cp.async.bulk rows into padded shared memory and back (the v2 data path), double buffered.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2511_14390_b200/csrc/common.cuh"
using namespace iirg;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

template <int KIND>
__global__ void alu_kernel(float* out, int iters, float s) {
    float a[8];
    double d[8];
    unsigned long long p[8];
    for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 0.001f + i; d[i] = a[i]; p[i] = pk2(a[i], a[i] + 1.f); }
    const unsigned long long S = pk2(s, s);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (KIND == 0) a[i] = fmaf(a[i], s, 0.5f);
                if (KIND == 1) p[i] = ffma2(p[i], S, p[(i + 1) & 7]);
                if (KIND == 2) d[i] = fma(d[i], (double)s, 0.5);
            }
    }
    float r = 0;
    for (int i = 0; i < 8; ++i) r += a[i] + (float)d[i] + lo2(p[i]) + hi2(p[i]);
    if (r == 12345.f) out[0] = r;
}

__global__ void copy4(const float4* __restrict__ x, float4* __restrict__ y, size_t n4) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
        stg_stream(y + i, ldg_stream(x + i));
}

// persistent warp tiles: tile = 32 rows of L floats; row r of the tile -> smem row at pitch L*4+16.
template <int L, int NWP>
__global__ void __launch_bounds__(NWP * 32) warp_tiles(const float* __restrict__ x, float* __restrict__ y,
                                                      long ntiles, unsigned* ticket, int compute) {
    constexpr int PITCH = L + 4;                  // floats
    constexpr int TILE = 32 * PITCH;
    extern __shared__ __align__(128) float sm[];
    __shared__ unsigned long long bar[NWP][2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* buf[2] = {sm + (warp * 2) * TILE, sm + (warp * 2 + 1) * TILE};
    if (lane == 0) { mbar_init(&bar[warp][0], 1); mbar_init(&bar[warp][1], 1); }
    mbar_fence_init();
    __syncwarp();
    unsigned ph[2] = {0, 0};
    auto fetch = [&](int b, long t) {
        if (lane == 0) mbar_arrive_expect_tx(&bar[warp][b], 32 * L * 4);
        __syncwarp();
        bulk_g2s(buf[b] + lane * PITCH, x + (t * 32 + lane) * L, L * 4, &bar[warp][b]);
    };
    long t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1u);
    t = __shfl_sync(~0u, t, 0);
    int b = 0;
    if (t < ntiles) fetch(0, t);
    while (t < ntiles) {
        long tn = 0;
        if (lane == 0) tn = atomicAdd(ticket, 1u);
        tn = __shfl_sync(~0u, tn, 0);
        if (tn < ntiles) {
            bulk_wait_read0();                   // the store that last read buf[b^1] is done reading
            __syncwarp();
            fetch(b ^ 1, tn);
        }
        mbar_wait(&bar[warp][b], ph[b]);
        ph[b] ^= 1;
        float* row = buf[b] + lane * PITCH;
        if (compute) {
            float s = 0.f;
#pragma unroll
            for (int g = 0; g < L / 4; ++g) {
                float4 v = *reinterpret_cast<float4*>(row + 4 * g);
                s = fmaf(s, 0.5f, v.x); v.x = s; s = fmaf(s, 0.5f, v.y); v.y = s;
                s = fmaf(s, 0.5f, v.z); v.z = s; s = fmaf(s, 0.5f, v.w); v.w = s;
                *reinterpret_cast<float4*>(row + 4 * g) = v;
            }
        }
        fence_proxy_async();
        __syncwarp();
        bulk_s2g(y + (t * 32 + lane) * L, row, L * 4);
        bulk_commit();
        t = tn;
        b ^= 1;
    }
    bulk_wait0();
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    CK(cudaGetDevice(&dev));
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    float* out;
    CK(cudaMalloc(&out, 4));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char* names[3] = {"FFMA", "FFMA2 (2 flop-pairs)", "DFMA"};
    for (int k = 0; k < 3; ++k) {
        const int iters = 2000, blocks = sms * 8, threads = 256;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (k == 0) alu_kernel<0><<<blocks, threads>>>(out, iters, 0.999f);
            if (k == 1) alu_kernel<1><<<blocks, threads>>>(out, iters, 0.999f);
            if (k == 2) alu_kernel<2><<<blocks, threads>>>(out, iters, 0.999f);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double instr = (double)blocks * threads * iters * 16 * 8;   // thread-instructions
        printf("%-22s %.1f thread-instr/clk/SM (at %d MHz nominal), %.2f Tinstr/s\n", names[k],
               instr / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000, instr / (ms * 1e-3) / 1e12);
    }
    const size_t n = (size_t)1 << 28;      // 1 GiB fp32
    float *x, *y;
    CK(cudaMalloc(&x, n * 4));
    CK(cudaMalloc(&y, n * 4));
    CK(cudaMemset(x, 0, n * 4));
    unsigned* ticket;
    CK(cudaMalloc(&ticket, 4));
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        copy4<<<sms * 8, 256>>>((const float4*)x, (float4*)y, n / 4);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("copy4: %.1f GB/s (read+write)\n", 2.0 * n * 4 / (ms * 1e-3) / 1e9);
    auto run_wt = [&](auto kern, int L, int nwp, int compute) {
        const size_t smem = (size_t)nwp * 2 * 32 * (L + 4) * 4;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, nwp * 32, smem);
        const long ntiles = (long)(n / (32 * L));
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemset(ticket, 0, 4);
            cudaEventRecord(e0);
            kern<<<sms * per, nwp * 32, smem>>>(x, y, ntiles, ticket, compute);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
        }
        cudaEventElapsedTime(&ms, e0, e1);
        printf("warp_tiles L=%d warps/CTA=%d CTAs/SM=%d compute=%d: %.1f GB/s\n", L, nwp, per, compute,
               2.0 * n * 4 / (ms * 1e-3) / 1e9);
    };
    for (int c = 0; c < 2; ++c) {
        run_wt(warp_tiles<32, 4>, 32, 4, c);
        run_wt(warp_tiles<64, 4>, 64, 4, c);
        run_wt(warp_tiles<64, 2>, 64, 2, c);
        run_wt(warp_tiles<128, 2>, 128, 2, c);
        run_wt(warp_tiles<64, 8>, 64, 8, c);
    }
    return 0;
}
