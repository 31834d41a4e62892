// Instruction-mix micro-benchmark for the all-pairs inner loop on B200.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mb scripts/microbench_mix.cu && ./mb
// Prints pairs/s (or lane-ops/s) for several formulations of the per-pair work.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float max3f(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

template <int MODE, int R>
__global__ void __launch_bounds__(128) k(float* out, int iters, float4 c0, float4 c1) {
    float rx[R], ry[R], rz[R], m[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        rx[r] = threadIdx.x * 1e-3f + r;
        ry[r] = rx[r] * 0.5f;
        rz[r] = rx[r] * 0.25f;
        m[r] = -1e30f;
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            float t0 = fmaf(rx[r], c0.x, c0.w), t1 = fmaf(rx[r], c1.x, c1.w);
            t0 = fmaf(ry[r], c0.y, t0);
            t1 = fmaf(ry[r], c1.y, t1);
            t0 = fmaf(rz[r], c0.z, t0);
            t1 = fmaf(rz[r], c1.z, t1);
            if (MODE == 0) m[r] = max3f(m[r], t0, t1);          // 3 FFMA + 1/2 FMNMX3
            if (MODE == 1) m[r] = fmaxf(fmaxf(m[r], t0), t1);   // 3 FFMA + 1 FMNMX
            if (MODE == 2) m[r] = m[r] + t0 + t1;                // 3 FFMA + 1 FADD
            if (MODE == 3) m[r] = fmaf(t0, t1, m[r]);            // 3.5 FFMA
        }
        c0.w += 1e-7f;
        c1.w -= 1e-7f;
    }
    float s = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r) s += m[r];
    if (s == 1234.5f) out[0] = s;
}

template <int MODE, int R>
void run(const char* name, int blocks_per_sm) {
    float* out;
    cudaMalloc(&out, 64);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * blocks_per_sm, iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k<MODE, R><<<blocks, 128>>>(out, iters, make_float4(0.1f, 0.2f, 0.3f, -1e6f), make_float4(0.3f, 0.2f, 0.1f, -1e6f));
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double pairs = (double)blocks * 128 * iters * R * 2;
    printf("%-34s blocks/SM=%2d  %.3f Tpair/s\n", name, blocks_per_sm, pairs / (ms * 1e-3) / 1e12);
    cudaFree(out);
}

int main() {
    for (int b : {4, 8, 16}) {
        run<0, 8>("3FFMA+0.5FMNMX3 R=8", b);
        run<1, 8>("3FFMA+1FMNMX R=8", b);
        run<2, 8>("3FFMA+1FADD R=8", b);
        run<3, 8>("3.5FFMA R=8", b);
        run<0, 4>("3FFMA+0.5FMNMX3 R=4", b);
        run<0, 16>("3FFMA+0.5FMNMX3 R=16", b);
    }
    return 0;
}
