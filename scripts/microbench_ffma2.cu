// Packed-FP32 (FFMA2, sm_100) throughput and the packed all-pairs loops.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mb2 scripts/microbench_ffma2.cu && ./mb2
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float max3f(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__global__ void ffma_peak(float* out, int iters, float b, float c) {
    float v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = threadIdx.x * 1e-3f + k;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = fmaf(v[k], c, b);
    float s = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += v[k];
    if (s == 1234.5f) out[0] = s;
}

__global__ void ffma2_peak(float* out, int iters, float b, float c) {
    float2 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = make_float2(threadIdx.x * 1e-3f + k, k * 0.5f);
    const float2 bb = make_float2(b, b * 0.5f), cc = make_float2(c, c);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __ffma2_rn(v[k], cc, bb);
    float s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k].x + v[k].y;
    if (s == 1234.5f) out[0] = s;
}

constexpr int W = 256;  // columns per chunk, interleaved in pairs: (x0,x1,y0,y1)(z0,z1,w0,w1)

template <int R>
__global__ void __launch_bounds__(128) gram2(const float4* __restrict__ cols, float* out, int reps) {
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
#pragma unroll 4
        for (int kk = 0; kk < W; kk += 2) {
            const float4 a = s[kk], b = s[kk + 1];
            const float2 X = make_float2(a.x, a.y), Y = make_float2(a.z, a.w), Z = make_float2(b.x, b.y),
                         Wc = make_float2(b.z, b.w);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                float2 t = __ffma2_rn(make_float2(rx[r], rx[r]), X, Wc);
                t = __ffma2_rn(make_float2(ry[r], ry[r]), Y, t);
                t = __ffma2_rn(make_float2(rz[r], rz[r]), Z, t);
                m[r] = max3f(m[r], t.x, t.y);
            }
        }
    }
    float sum = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r) sum += m[r];
    if (sum == 1234.5f) out[0] = sum;
}

// packed direct formula: negated columns (-x0,-x1,-y0,-y1)(-z0,-z1,*,*), two column pairs per step
template <int R>
__global__ void __launch_bounds__(128) direct2(const float4* __restrict__ cols, float* out, int reps) {
    __shared__ float4 s[W];
    for (int q = threadIdx.x; q < W; q += blockDim.x) s[q] = cols[q];
    __syncthreads();
    float rx[R], ry[R], rz[R];
    float2 acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        rx[r] = threadIdx.x * 1e-3f + r;
        ry[r] = rx[r] * 0.5f;
        rz[r] = rx[r] * 0.25f;
        acc[r] = make_float2(0.f, 0.f);
    }
    const float2 one = make_float2(1.f, 1.f);
    for (int it = 0; it < reps; ++it) {
#pragma unroll 2
        for (int kk = 0; kk < W; kk += 4) {
            const float4 a0 = s[kk], b0 = s[kk + 1], a1 = s[kk + 2], b1 = s[kk + 3];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                float2 dx = __fadd2_rn(make_float2(rx[r], rx[r]), make_float2(a0.x, a0.y));
                float2 dy = __fadd2_rn(make_float2(ry[r], ry[r]), make_float2(a0.z, a0.w));
                float2 dz = __fadd2_rn(make_float2(rz[r], rz[r]), make_float2(b0.x, b0.y));
                float2 p0 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __ffma2_rn(dx, dx, one)));
                dx = __fadd2_rn(make_float2(rx[r], rx[r]), make_float2(a1.x, a1.y));
                dy = __fadd2_rn(make_float2(ry[r], ry[r]), make_float2(a1.z, a1.w));
                dz = __fadd2_rn(make_float2(rz[r], rz[r]), make_float2(b1.x, b1.y));
                float2 p1 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __ffma2_rn(dx, dx, one)));
                const float2 pr = __fmul2_rn(p0, p1), sm = __fadd2_rn(p0, p1);
                acc[r] = __ffma2_rn(sm, make_float2(rcp_approx(pr.x), rcp_approx(pr.y)), acc[r]);
            }
        }
    }
    float sum = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r) sum += acc[r].x + acc[r].y;
    if (sum == 1234.5f) out[0] = sum;
}

template <typename K>
double timeit(K kern, int blocks, int threads, float4* cols, float* out, int reps) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        kern<<<blocks, threads>>>(cols, out, reps);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
    }
    return ms * 1e-3;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    float4* cols;
    cudaMalloc(&out, 64);
    cudaMalloc(&cols, W * sizeof(float4));
    cudaMemset(cols, 0, W * sizeof(float4));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    const int blocks = sms * 8, iters = 65536;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        ffma_peak<<<blocks, 256>>>(out, iters, 0.5f, 0.999f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA   lane-FMA/s  %.2f T\n", (double)blocks * 256 * iters * 16 / (ms * 1e-3) / 1e12);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        ffma2_peak<<<blocks, 256>>>(out, iters, 0.5f, 0.999f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA2  lane-FMA/s  %.2f T\n", (double)blocks * 256 * iters * 16 / (ms * 1e-3) / 1e12);
    for (int bps : {4, 8}) {
        const int reps = 64;
        double s8 = timeit(gram2<8>, sms * bps, 128, cols, out, reps);
        printf("gram2   R=8  b/SM=%d  %.3f Tpair/s\n", bps, (double)sms * bps * 128 * reps * W * 8 / s8 / 1e12);
        double s4 = timeit(gram2<4>, sms * bps, 128, cols, out, reps);
        printf("gram2   R=4  b/SM=%d  %.3f Tpair/s\n", bps, (double)sms * bps * 128 * reps * W * 4 / s4 / 1e12);
        double s16 = timeit(gram2<16>, sms * bps, 128, cols, out, reps);
        printf("gram2   R=16 b/SM=%d  %.3f Tpair/s\n", bps, (double)sms * bps * 128 * reps * W * 16 / s16 / 1e12);
        double d8 = timeit(direct2<8>, sms * bps, 128, cols, out, reps);
        printf("direct2 R=8  b/SM=%d  %.3f Tpair/s\n", bps, (double)sms * bps * 128 * reps * W * 8 / d8 / 1e12);
        double d4 = timeit(direct2<4>, sms * bps, 128, cols, out, reps);
        printf("direct2 R=4  b/SM=%d  %.3f Tpair/s\n", bps, (double)sms * bps * 128 * reps * W * 4 / d4 / 1e12);
    }
    return 0;
}
