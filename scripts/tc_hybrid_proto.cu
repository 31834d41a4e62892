// Prototype (not part of libpaircount): tensor-core and FFMA2 Gram filters side
// by side in one CTA.  Warps 0-3 run scripts/tc_gram_proto.cu's path (thread 0
// issues tcgen05.mma into two TMEM accumulators, the 4 warps read them back with
// tcgen05.ld and reduce with FMNMX3); warps 4.. run the count kernel's packed
// loop (3 FFMA2 + 1 FMNMX3 per two pairs, 12 rows per lane, columns from shared
// memory).  Prints each path's pairs/clk/SM alone and together.
//
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tch scripts/tc_hybrid_proto.cu && ./tch
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int M = 128, N = 256, K = 8;

__device__ __forceinline__ float max3f(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    unsigned ok = 0, spins = 0;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
        if (++spins == (1u << 26)) __trap();
    } while (!ok);
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// K-major, no swizzle: core matrix = 8 rows x 16 B; row groups SBO = 128 B apart,
// the two 16-byte K chunks LBO = rows*16 B apart.
__device__ __forceinline__ uint64_t make_desc(unsigned saddr, unsigned rows) {
    const uint64_t lbo = (uint64_t)rows * 16u, sbo = 128u;
    return (uint64_t)(saddr >> 4) | ((lbo >> 4) << 16) | ((sbo >> 4) << 32) | (1ull << 46);
}
__host__ __device__ constexpr uint32_t make_idesc() {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// element (r, k) of a K-major interleaved operand with `rows` rows
__host__ __device__ inline int op_index(int r, int k, int rows) {
    return ((r & 7) * 16 + (r >> 3) * 128 + (k >> 2) * rows * 16 + (k & 3) * 4) / 4;
}


constexpr int W = 256, R = 12;

__device__ __forceinline__ float2 f2_fma(float a, float2 b, float2 c) { return __ffma2_rn(make_float2(a, a), b, c); }

template <int F>
__global__ void __launch_bounds__(128 + 32 * F, 1) hybrid(const float* __restrict__ gA, const float* __restrict__ gB,
                                                          const float4* __restrict__ gC, int tc_iters, int fma_iters,
                                                          float* __restrict__ out) {
    __shared__ __align__(128) float sA[M * K];
    __shared__ __align__(128) float sB[N * K];
    __shared__ __align__(16) float4 sC[W];
    __shared__ __align__(8) unsigned long long bar_full[2], bar_empty[2];
    __shared__ unsigned tmem_base_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int q = threadIdx.x; q < M * K; q += blockDim.x) sA[q] = gA[q];
    for (int q = threadIdx.x; q < N * K; q += blockDim.x) sB[q] = gB[q];
    for (int q = threadIdx.x; q < W; q += blockDim.x) sC[q] = gC[q];
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&bar_full[b]), 1);
            mbar_init(smem_u32(&bar_empty[b]), 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tmem = tmem_base_s;
    float m = -INFINITY;
    if (warp < 4) {
        const uint64_t da = make_desc(smem_u32(sA), M), db = make_desc(smem_u32(sB), N);
        const uint32_t idesc = make_idesc();
        for (int it = 0; it < tc_iters; ++it) {
            const int b = it & 1;
            const unsigned ph = (unsigned)(it >> 1) & 1u;
            if (threadIdx.x == 0) {
                if (it >= 2) mbar_wait(smem_u32(&bar_empty[b]), ph ^ 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                asm volatile(
                    "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
                    ::"r"(tmem + (unsigned)(b * N)), "l"(da), "l"(db), "r"(idesc), "r"(0));
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"(
                    (unsigned long long)smem_u32(&bar_full[b])));
            }
            __syncwarp();
            mbar_wait(smem_u32(&bar_full[b]), ph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
            for (int q = 0; q < N / 32; ++q) {
                unsigned v[32];
                const unsigned taddr = tmem + ((unsigned)(warp * 32) << 16) + (unsigned)(b * N + q * 32);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                      "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                      "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                      "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                      "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int e = 0; e < 32; e += 2) m = max3f(m, __uint_as_float(v[e]), __uint_as_float(v[e + 1]));
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&bar_empty[b]));
        }
    } else {
        float rx[R], ry[R], rz[R], mm[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            rx[r] = threadIdx.x * 1e-3f + r;
            ry[r] = rx[r] * 0.5f;
            rz[r] = rx[r] * 0.25f;
            mm[r] = -1e30f;
        }
        for (int it = 0; it < fma_iters; ++it) {
#pragma unroll 8
            for (int k = 0; k < W; k += 2) {
                const float4 A = sC[k], B = sC[k + 1];
                const float2 cx = make_float2(A.x, A.y), cy = make_float2(A.z, A.w);
                const float2 cz = make_float2(B.x, B.y), cw = make_float2(B.z, B.w);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    float2 t = f2_fma(rx[r], cx, cw);
                    t = f2_fma(ry[r], cy, t);
                    t = f2_fma(rz[r], cz, t);
                    mm[r] = max3f(mm[r], t.x, t.y);
                }
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) m = fmaxf(m, mm[r]);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = m;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int F>
void run(const float* dA, const float* dB, const float4* dC, float* dO, int sms, int tc_iters, int fma_iters) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    hybrid<F><<<sms, 128 + 32 * F>>>(dA, dB, dC, 2, 2, dO);
    cudaEventRecord(e0);
    hybrid<F><<<sms, 128 + 32 * F>>>(dA, dB, dC, tc_iters, fma_iters, dO);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { printf("kernel error: %s\n", cudaGetErrorString(e)); exit(1); }
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double clk = ms * 1e-3 * 1.965e9;
    const double tc = (double)tc_iters * M * N, fm = (double)fma_iters * F * 32 * R * W;
    printf("F=%2d tc_iters=%6d fma_iters=%5d: %8.3f ms  TC %5.1f + FFMA2 %5.1f = %5.1f pairs/clk/SM  (%.2f Tpair/s)\n",
           F, tc_iters, fma_iters, ms, tc / clk, fm / clk, (tc + fm) / clk, (tc + fm) * sms / (ms * 1e-3) / 1e12);
}

int main() {
    std::vector<float> A(M * K, 0.f), B(N * K, 0.f);
    for (int r = 0; r < M; ++r) { for (int k = 0; k < 3; ++k) A[op_index(r, k, M)] = 0.01f * (r + k); A[op_index(r, 3, M)] = 1.f; }
    for (int c = 0; c < N; ++c) for (int k = 0; k < 4; ++k) B[op_index(c, k, N)] = 0.02f * (c - k);
    std::vector<float4> C(W, make_float4(0.1f, 0.2f, 0.3f, -5.f));
    float *dA, *dB, *dO;
    float4* dC;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dC, C.size() * 16);
    cudaMalloc(&dO, (size_t)sms * 1024 * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dC, C.data(), C.size() * 16, cudaMemcpyHostToDevice);
    // each path alone, then together at several work ratios
    run<8>(dA, dB, dC, dO, sms, 8192, 0);
    run<8>(dA, dB, dC, dO, sms, 0, 256);
    run<12>(dA, dB, dC, dO, sms, 0, 256);
    for (int f : {192, 256, 320, 384}) run<8>(dA, dB, dC, dO, sms, 8192, f);
    for (int f : {160, 192, 256}) run<12>(dA, dB, dC, dO, sms, 8192, f);
    return 0;
}
