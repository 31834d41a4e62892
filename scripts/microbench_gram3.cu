// Which reduction instruction can ride alongside FFMA2 without stealing FMA-pipe cycles?
// The Gram filter loop is 3 FFMA2 + 1 reduction per two pairs; this sweeps the reduction.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mbg3 scripts/microbench_gram3.cu && ./mbg3
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float max3f(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ unsigned and3(unsigned a, unsigned b, unsigned c) {
    unsigned d;
    asm("lop3.b32 %0, %1, %2, %3, 0x80;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ unsigned long long pk(float a, float b) {
    unsigned long long d;
    asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(a), "f"(b));
    return d;
}
__device__ __forceinline__ unsigned long long ffma2p(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ int imax3(int a, int b, int c) {
    return max(max(a, b), c);  // ptxas may fuse into a 3-input VIMNMX
}

constexpr int W = 256;

// MODE 0: FMNMX3(m, t.x, t.y)          1: two FMNMX            2: LOP3 and3 of the bits
//      3: integer max3 of the bits     4: scalar FFMA x6 + FMNMX3   5: no reduction (sum of t after loop)
template <int R, int MODE>
__global__ void __launch_bounds__(128, 4) k(const float4* __restrict__ cols, float* out, int reps) {
    __shared__ float4 s[W];
    for (int q = threadIdx.x; q < W; q += blockDim.x) s[q] = cols[q];
    __syncthreads();
    float rx[R], ry[R], rz[R], m[R];
    unsigned mb[R];
    float2 acc[R];
    unsigned long long rp[R][3];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        acc[r] = make_float2(0.f, 0.f);
        rx[r] = threadIdx.x * 1e-3f + r;
        ry[r] = rx[r] * 0.5f;
        rz[r] = rx[r] * 0.25f;
        m[r] = -1e30f;
        mb[r] = 0xffffffffu;
        rp[r][0] = pk(rx[r], rx[r]);
        rp[r][1] = pk(ry[r], ry[r]);
        rp[r][2] = pk(rz[r], rz[r]);
    }
    for (int it = 0; it < reps; ++it) {
#pragma unroll 4
        for (int kk = 0; kk < W; kk += 2) {
            const float4 A = s[kk], B = s[kk + 1];
            const float2 X = make_float2(A.x, A.y), Y = make_float2(A.z, A.w), Z = make_float2(B.x, B.y),
                         Wc = make_float2(B.z, B.w);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                float2 t;
                if (MODE == 5) {  // FFMA2 only: per-row chains carried across columns (same op count)
                    acc[r] = __ffma2_rn(make_float2(rx[r], rx[r]), X, acc[r]);
                    acc[r] = __ffma2_rn(make_float2(ry[r], ry[r]), Y, acc[r]);
                    acc[r] = __ffma2_rn(make_float2(rz[r], rz[r]), Z, acc[r]);
                    continue;
                }
                if (MODE == 6) {  // row value held as a full register pair (no scalar broadcast form)
                    unsigned long long tt = ffma2p(rp[r][0], pk(X.x, X.y), pk(Wc.x, Wc.y));
                    tt = ffma2p(rp[r][1], pk(Y.x, Y.y), tt);
                    tt = ffma2p(rp[r][2], pk(Z.x, Z.y), tt);
                    float a, b;
                    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(tt));
                    m[r] = max3f(m[r], a, b);
                    continue;
                }
                if (MODE == 4) {
                    t.x = fmaf(rx[r], X.x, Wc.x);
                    t.y = fmaf(rx[r], X.y, Wc.y);
                    t.x = fmaf(ry[r], Y.x, t.x);
                    t.y = fmaf(ry[r], Y.y, t.y);
                    t.x = fmaf(rz[r], Z.x, t.x);
                    t.y = fmaf(rz[r], Z.y, t.y);
                } else {
                    t = __ffma2_rn(make_float2(rx[r], rx[r]), X, Wc);
                    t = __ffma2_rn(make_float2(ry[r], ry[r]), Y, t);
                    t = __ffma2_rn(make_float2(rz[r], rz[r]), Z, t);
                }
                if (MODE == 0 || MODE == 4) m[r] = max3f(m[r], t.x, t.y);
                if (MODE == 1) m[r] = fmaxf(fmaxf(m[r], t.x), t.y);
                if (MODE == 2) mb[r] = and3(mb[r], __float_as_uint(t.x), __float_as_uint(t.y));
                if (MODE == 3) mb[r] = (unsigned)imax3((int)mb[r], __float_as_int(t.x), __float_as_int(t.y));
            }
        }
    }
    float sum = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r) sum += m[r] + __uint_as_float(mb[r]) + acc[r].x + acc[r].y;
    if (sum == 1234.5f) out[0] = sum;
}

// row-outer order: 4 column pairs in registers, each row runs 4 independent FFMA2 chains
template <int R>
__global__ void __launch_bounds__(128, 4) krow(const float4* __restrict__ cols, float* out, int reps) {
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
        for (int kk = 0; kk < W; kk += 8) {
            float2 X[4], Y[4], Z[4], Wc[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const float4 A = s[kk + 2 * p], B = s[kk + 2 * p + 1];
                X[p] = make_float2(A.x, A.y); Y[p] = make_float2(A.z, A.w);
                Z[p] = make_float2(B.x, B.y); Wc[p] = make_float2(B.z, B.w);
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                float2 t[4];
#pragma unroll
                for (int p = 0; p < 4; ++p) t[p] = __ffma2_rn(make_float2(rx[r], rx[r]), X[p], Wc[p]);
#pragma unroll
                for (int p = 0; p < 4; ++p) t[p] = __ffma2_rn(make_float2(ry[r], ry[r]), Y[p], t[p]);
#pragma unroll
                for (int p = 0; p < 4; ++p) t[p] = __ffma2_rn(make_float2(rz[r], rz[r]), Z[p], t[p]);
#pragma unroll
                for (int p = 0; p < 4; ++p) m[r] = max3f(m[r], t[p].x, t[p].y);
            }
        }
    }
    float sum = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r) sum += m[r];
    if (sum == 1234.5f) out[0] = sum;
}

template <int R>
void runrow(int bps, const char* name) {
    float4* cols;
    float* out;
    cudaMalloc(&cols, W * sizeof(float4));
    cudaMemset(cols, 0, W * sizeof(float4));
    cudaMalloc(&out, 64);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, krow<R>);
    const int blocks = sms * bps, reps = 64;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        krow<R><<<blocks, 128>>>(cols, out, reps);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep && ms < best) best = ms;
    }
    const double pairs = (double)blocks * 128 * reps * W * R;
    printf("%-22s R=%2d regs=%3d b/SM=%d  %.3f Tpair/s  (FMA pipe %.0f%% at 3 lane-FMA/pair)\n", name, R, fa.numRegs,
           bps, pairs / (best * 1e-3) / 1e12, 100.0 * 3.0 * pairs / (best * 1e-3) / 36.3e12);
    cudaFree(cols);
    cudaFree(out);
}

template <int R, int MODE>
void run(int bps, const char* name) {
    float4* cols;
    float* out;
    cudaMalloc(&cols, W * sizeof(float4));
    cudaMemset(cols, 0, W * sizeof(float4));
    cudaMalloc(&out, 64);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k<R, MODE>);
    const int blocks = sms * bps, reps = 64;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        k<R, MODE><<<blocks, 128>>>(cols, out, reps);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep && ms < best) best = ms;
    }
    const double pairs = (double)blocks * 128 * reps * W * R;
    printf("%-22s R=%2d regs=%3d b/SM=%d  %.3f Tpair/s  (FMA pipe %.0f%% at 3 lane-FMA/pair)\n", name, R, fa.numRegs,
           bps, pairs / (best * 1e-3) / 1e12, 100.0 * 3.0 * pairs / (best * 1e-3) / 36.3e12);
    cudaFree(cols);
    cudaFree(out);
}

int main() {
    for (int b : {4}) {
        run<8, 0>(b, "ffma2+fmnmx3");
        run<8, 5>(b, "ffma2 only (chains)");
        run<12, 5>(b, "ffma2 only (chains)");
        run<8, 6>(b, "ffma2 pair-row+fmnmx3");
        run<12, 6>(b, "ffma2 pair-row+fmnmx3");
        runrow<8>(b, "row-outer 4 colpairs");
        runrow<12>(b, "row-outer 4 colpairs");
        runrow<6>(b, "row-outer 4 colpairs");
    }
    return 0;
}
