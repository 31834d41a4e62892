// MUFU.RCP throughput on B200, alone and interleaved with packed FP32 at the
// ratios of the sum loops (Gram loop: 2 MUFU per 11 packed; TMEM-drain
// epilogue with paired reciprocals: 2 MUFU per 3 packed).  Independent chains,
// 16 warps per sub-partition, so latency is hidden and the pipes are the bound.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mbm scripts/microbench_mufu.cu && ./mbm
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// per iteration and chain: MU reciprocals and PK packed FFMA2
template <int MU, int PK>
__global__ void __launch_bounds__(512, 2) k(float* out, int iters, float c) {
    constexpr int CH = 8;
    float a[CH];
    float2 b[CH];
#pragma unroll
    for (int q = 0; q < CH; ++q) {
        a[q] = 1.f + threadIdx.x * 1e-4f + q;
        b[q] = make_float2(a[q], a[q] * 0.5f);
    }
    const float2 m = make_float2(c, c), d = make_float2(1e-7f, 2e-7f);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < CH; ++q) {
#pragma unroll
            for (int u = 0; u < MU; ++u) a[q] = rcp_approx(a[q] + 1.0f) ;
#pragma unroll
            for (int u = 0; u < PK; ++u) b[q] = __ffma2_rn(b[q], m, d);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < CH; ++q) s += a[q] + b[q].x + b[q].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MU, int PK>
void run(float* d, int sms) {
    const int iters = 4096, grid = 2 * sms, threads = 512;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<MU, PK><<<grid, threads>>>(d, 64, 0.999f);
    cudaEventRecord(e0);
    k<MU, PK><<<grid, threads>>>(d, iters, 0.999f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = (double)grid * threads / 32, per = (double)iters * 8;
    const double clk = ms * 1e-3 * 1.965e9;
    // MU also carries one FADD per reciprocal (the +1 keeps the chain finite)
    printf("MUFU %d : FFMA2 %2d (+%d FADD): %.3f ms  MUFU %.2f /clk/SM (lanes)  packed %.2f warp-instr/clk/SMSP\n", MU, PK,
           MU, ms, warps * per * MU * 32 / clk / sms, warps * per * PK / clk / sms / 4);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* d;
    cudaMalloc(&d, (size_t)2 * sms * 512 * 4);
    run<1, 0>(d, sms);
    run<2, 0>(d, sms);
    run<0, 4>(d, sms);
    run<2, 3>(d, sms);
    run<2, 6>(d, sms);
    run<2, 11>(d, sms);
    run<1, 11>(d, sms);
    run<1, 8>(d, sms);
    return 0;
}
