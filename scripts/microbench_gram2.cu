// Shape sweep for the packed Gram filter loop (FFMA2 + FMNMX3), columns from shared memory.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mbg scripts/microbench_gram2.cu && ./mbg
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float max3f(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

constexpr int W = 256;

// R rows per thread, P column pairs per k-step; MODE 0: FMNMX3 per pair-of-pairs,
// MODE 1: FMNMX3 over (m, t0.x, t0.y) then (m, t1.x, t1.y)..., MODE 2: max over two col-pairs first
template <int R, int P, int MODE, int MINB>
__global__ void __launch_bounds__(128, MINB) k(const float4* __restrict__ cols, float* out, int reps) {
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
        for (int kk = 0; kk < W; kk += 2 * P) {
            float2 cx[P], cy[P], cz[P], cw[P];
#pragma unroll
            for (int p = 0; p < P; ++p) {
                const float4 A = s[kk + 2 * p], B = s[kk + 2 * p + 1];
                cx[p] = make_float2(A.x, A.y); cy[p] = make_float2(A.z, A.w);
                cz[p] = make_float2(B.x, B.y); cw[p] = make_float2(B.z, B.w);
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                float2 t[P];
#pragma unroll
                for (int p = 0; p < P; ++p) t[p] = __ffma2_rn(make_float2(rx[r], rx[r]), cx[p], cw[p]);
#pragma unroll
                for (int p = 0; p < P; ++p) t[p] = __ffma2_rn(make_float2(ry[r], ry[r]), cy[p], t[p]);
#pragma unroll
                for (int p = 0; p < P; ++p) t[p] = __ffma2_rn(make_float2(rz[r], rz[r]), cz[p], t[p]);
                if (MODE == 0 || P == 1) {
#pragma unroll
                    for (int p = 0; p < P; ++p) m[r] = max3f(m[r], t[p].x, t[p].y);
                } else {
#pragma unroll
                    for (int p = 0; p < P; p += 2) {
                        const float u = max3f(t[p].x, t[p].y, t[p + 1].x);
                        m[r] = max3f(m[r], u, t[p + 1].y);
                    }
                }
            }
        }
    }
    float sum = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r) sum += m[r];
    if (sum == 1234.5f) out[0] = sum;
}

template <int R, int P, int MODE, int MINB>
void run(int bps) {
    float4* cols;
    float* out;
    cudaMalloc(&cols, W * sizeof(float4));
    cudaMemset(cols, 0, W * sizeof(float4));
    cudaMalloc(&out, 64);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k<R, P, MODE, MINB>);
    const int blocks = sms * bps, reps = 64;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k<R, P, MODE, MINB><<<blocks, 128>>>(cols, out, reps);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double pairs = (double)blocks * 128 * reps * W * R;
    printf("R=%2d P=%d mode=%d minB=%d regs=%3d b/SM=%2d  %.3f Tpair/s  (FMA pipe %.0f%%)\n", R, P, MODE, MINB,
           fa.numRegs, bps, pairs / (ms * 1e-3) / 1e12, 100.0 * 3.0 * pairs / (ms * 1e-3) / 36.3e12);
    cudaFree(cols);
    cudaFree(out);
}

int main() {
    for (int b : {4, 8}) {
        run<8, 1, 0, 4>(b);
        run<8, 2, 0, 4>(b);
        run<8, 2, 1, 4>(b);
        run<4, 4, 1, 4>(b);
        run<4, 2, 0, 4>(b);
        run<6, 2, 1, 4>(b);
        run<8, 4, 1, 2>(b);
        run<16, 1, 0, 2>(b);
        run<4, 4, 1, 8>(b);
    }
    return 0;
}
