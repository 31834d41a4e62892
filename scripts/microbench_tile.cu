// Micro-tile shape sweep for the Gram filter loop (columns from shared memory).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mbt scripts/microbench_tile.cu && ./mbt
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float max3f(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

constexpr int W = 256;

template <int R, int C>
__global__ void __launch_bounds__(128) k(const float4* __restrict__ cols, float* out, int reps) {
    __shared__ float4 s[W];
    for (int q = threadIdx.x; q < W; q += blockDim.x) s[q] = cols[q];
    __syncthreads();
    float rx[R], ry[R], rz[R], m[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        rx[r] = threadIdx.x * 1e-3f + r;
        ry[r] = rx[r] * 0.5f;
        rz[r] = rx[r] * 0.25f;
        m[r] = -1e30f;
    }
    for (int it = 0; it < reps; ++it) {
#pragma unroll 2
        for (int kk = 0; kk < W; kk += C) {
            float4 c[C];
#pragma unroll
            for (int q = 0; q < C; ++q) c[q] = s[kk + q];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                float t[C];
#pragma unroll
                for (int q = 0; q < C; ++q) t[q] = fmaf(rz[r], c[q].z, fmaf(ry[r], c[q].y, fmaf(rx[r], c[q].x, c[q].w)));
#pragma unroll
                for (int q = 0; q < C; q += 2) m[r] = max3f(m[r], t[q], t[q + 1]);
            }
        }
    }
    float sum = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r) sum += m[r];
    if (sum == 1234.5f) out[0] = sum;
}

template <int R, int C>
void run(int bps) {
    float4* cols;
    float* out;
    cudaMalloc(&cols, W * sizeof(float4));
    cudaMemset(cols, 0, W * sizeof(float4));
    cudaMalloc(&out, 64);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k<R, C>, 128, 0);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k<R, C>);
    const int blocks = sms * bps, reps = 64;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k<R, C><<<blocks, 128>>>(cols, out, reps);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double pairs = (double)blocks * 128 * reps * W * R;
    printf("R=%2d C=%d regs=%3d occ=%2d blocks/SM=%2d  %.3f Tpair/s\n", R, C, fa.numRegs, occ, bps,
           pairs / (ms * 1e-3) / 1e12);
    cudaFree(cols);
    cudaFree(out);
}

int main() {
    for (int b : {4, 8}) {
        run<8, 2>(b);
        run<4, 2>(b);
        run<4, 4>(b);
        run<8, 4>(b);
        run<2, 8>(b);
        run<6, 2>(b);
        run<12, 2>(b);
        run<16, 2>(b);
        run<2, 4>(b);
        run<1, 8>(b);
    }
    return 0;
}
