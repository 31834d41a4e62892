// Prototype (not part of libpaircount): tcgen05 inverse-square sum epilogue with
// the drain pipelined.  scripts/tc_epi_proto.cu drained every accumulator with
// all epilogue warps in lockstep (all load, then all compute), which serialises
// the TMEM read-back and the arithmetic: 22 pairs/clk/SM at best against 42 for
// the loads alone.  Here the epilogue warps form NACC groups, group g drains
// accumulator g (iterations it = g mod NACC), each warp reads its whole slice,
// releases the accumulator, then computes -- so one group's arithmetic overlaps
// another group's loads and the next MMAs.  A separate warp issues the MMAs.
//   MODE 0  count filter (FMNMX3 row max)
//   MODE 2  loads only
//   MODE 5  inverse-square, 8 terms per 2 reciprocals, packed
//   MODE 6  inverse-square, 16 terms per 2 reciprocals, packed
//
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tcs scripts/tc_sum_proto.cu && ./tcs
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int M = 128, K = 8;

__device__ __forceinline__ float max3f(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
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
__device__ __forceinline__ uint64_t make_desc(unsigned saddr, unsigned rows) {
    const uint64_t lbo = (uint64_t)rows * 16u, sbo = 128u;
    return (uint64_t)(saddr >> 4) | ((lbo >> 4) << 16) | ((sbo >> 4) << 32) | (1ull << 46);
}
__host__ __device__ constexpr uint32_t make_idesc(int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__host__ __device__ inline int op_index(int r, int k, int rows) {
    return ((r & 7) * 16 + (r >> 3) * 128 + (k >> 2) * rows * 16 + (k & 3) * 4) / 4;
}

#define LD32(v, base, taddr)                                                                                      \
    asm volatile(                                                                                                 \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"          \
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                \
        : "=r"(v[base + 0]), "=r"(v[base + 1]), "=r"(v[base + 2]), "=r"(v[base + 3]), "=r"(v[base + 4]),          \
          "=r"(v[base + 5]), "=r"(v[base + 6]), "=r"(v[base + 7]), "=r"(v[base + 8]), "=r"(v[base + 9]),          \
          "=r"(v[base + 10]), "=r"(v[base + 11]), "=r"(v[base + 12]), "=r"(v[base + 13]), "=r"(v[base + 14]),     \
          "=r"(v[base + 15]), "=r"(v[base + 16]), "=r"(v[base + 17]), "=r"(v[base + 18]), "=r"(v[base + 19]),     \
          "=r"(v[base + 20]), "=r"(v[base + 21]), "=r"(v[base + 22]), "=r"(v[base + 23]), "=r"(v[base + 24]),     \
          "=r"(v[base + 25]), "=r"(v[base + 26]), "=r"(v[base + 27]), "=r"(v[base + 28]), "=r"(v[base + 29]),     \
          "=r"(v[base + 30]), "=r"(v[base + 31])                                                                  \
        : "r"(taddr))

template <int MODE, int COLS>
__device__ __forceinline__ void epi(const unsigned (&v)[COLS], float& m, float2& acc) {
    if constexpr (MODE == 0) {
#pragma unroll
        for (int e = 0; e < COLS; e += 2) m = max3f(m, __uint_as_float(v[e]), __uint_as_float(v[e + 1]));
    } else if constexpr (MODE == 2) {
        m += __uint_as_float(v[0]) + __uint_as_float(v[COLS - 1]);
    } else if constexpr (MODE == 5) {
#pragma unroll
        for (int e = 0; e < COLS; e += 8) {
            const float2 p1 = make_float2(__uint_as_float(v[e]), __uint_as_float(v[e + 1]));
            const float2 p2 = make_float2(__uint_as_float(v[e + 2]), __uint_as_float(v[e + 3]));
            const float2 p3 = make_float2(__uint_as_float(v[e + 4]), __uint_as_float(v[e + 5]));
            const float2 p4 = make_float2(__uint_as_float(v[e + 6]), __uint_as_float(v[e + 7]));
            const float2 m12 = __fmul2_rn(p1, p2), s12 = __fadd2_rn(p1, p2);
            const float2 m34 = __fmul2_rn(p3, p4), s34 = __fadd2_rn(p3, p4);
            const float2 P = __fmul2_rn(m12, m34);
            const float2 Nn = __ffma2_rn(s34, m12, __fmul2_rn(s12, m34));
            acc = __ffma2_rn(Nn, make_float2(rcp_approx(P.x), rcp_approx(P.y)), acc);
        }
    } else {
#pragma unroll
        for (int e = 0; e < COLS; e += 16) {
            float2 P[2], Nn[2];
#pragma unroll
            for (int g = 0; g < 2; ++g) {
                const int o = e + 8 * g;
                const float2 p1 = make_float2(__uint_as_float(v[o]), __uint_as_float(v[o + 1]));
                const float2 p2 = make_float2(__uint_as_float(v[o + 2]), __uint_as_float(v[o + 3]));
                const float2 p3 = make_float2(__uint_as_float(v[o + 4]), __uint_as_float(v[o + 5]));
                const float2 p4 = make_float2(__uint_as_float(v[o + 6]), __uint_as_float(v[o + 7]));
                const float2 m12 = __fmul2_rn(p1, p2), s12 = __fadd2_rn(p1, p2);
                const float2 m34 = __fmul2_rn(p3, p4), s34 = __fadd2_rn(p3, p4);
                P[g] = __fmul2_rn(m12, m34);
                Nn[g] = __ffma2_rn(s34, m12, __fmul2_rn(s12, m34));
            }
            const float2 PP = __fmul2_rn(P[0], P[1]);
            const float2 NN = __ffma2_rn(Nn[1], P[0], __fmul2_rn(Nn[0], P[1]));
            acc = __ffma2_rn(NN, make_float2(rcp_approx(PP.x), rcp_approx(PP.y)), acc);
        }
    }
}

// EPI epilogue warps in NACC groups (group g: accumulator g); a warp reads TMEM lane quadrant
// w % 4 and column range of its group; warp EPI issues the MMAs.  N columns per accumulator.
template <int EPI, int NACC, int N, int MODE, int KSTEPS>
__global__ void __launch_bounds__(32 * (EPI + 1), 1) sum_proto(const float* __restrict__ gA,
                                                               const float* __restrict__ gB, int iters,
                                                               float* __restrict__ out) {
    static_assert(NACC * N <= 512, "TMEM columns");
    constexpr int WPG = EPI / NACC, RANGES = WPG / 4, COLS = N / RANGES;
    static_assert(WPG % 4 == 0 && COLS <= 128 && COLS % 32 == 0, "epilogue shape");
    __shared__ __align__(128) float sA[M * K];
    __shared__ __align__(128) float sB[N * K];
    __shared__ __align__(8) unsigned long long bar_full[NACC], bar_empty[NACC];
    __shared__ unsigned tmem_base_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int q = threadIdx.x; q < M * K; q += blockDim.x) sA[q] = gA[q];
    for (int q = threadIdx.x; q < N * K; q += blockDim.x) sB[q] = gB[q];
    if (threadIdx.x == 0) {
        for (int b = 0; b < NACC; ++b) {
            mbar_init(smem_u32(&bar_full[b]), 1);
            mbar_init(smem_u32(&bar_empty[b]), WPG);
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
    float2 acc = make_float2(0.f, 0.f);
    double tot = 0.0;
    if (warp == EPI) {
        if (lane == 0) {
            const uint64_t da = make_desc(smem_u32(sA), M), db = make_desc(smem_u32(sB), N);
            for (int it = 0; it < iters; ++it) {
                const int b = it % NACC;
                if (it >= NACC) mbar_wait(smem_u32(&bar_empty[b]), (unsigned)((it / NACC) - 1) & 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                for (int ks = 0; ks < KSTEPS; ++ks)
                    asm volatile(
                        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
                        ::"r"(tmem + (unsigned)(b * N)), "l"(da), "l"(db), "r"(make_idesc(N)), "r"(ks));
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"(
                    (unsigned long long)smem_u32(&bar_full[b])));
            }
        }
    } else {
        const int quad = warp & 3, grp = (warp >> 2) % NACC, range = (warp >> 2) / NACC;
        int k = 0;
        for (int it = grp; it < iters; it += NACC, ++k) {
            mbar_wait(smem_u32(&bar_full[grp]), (unsigned)k & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            unsigned v[COLS];
            const unsigned taddr = tmem + ((unsigned)(quad * 32) << 16) + (unsigned)(grp * N + range * COLS);
#pragma unroll
            for (int q = 0; q < COLS / 32; ++q) LD32(v, 32 * q, taddr + 32u * q);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&bar_empty[grp]));
            epi<MODE, COLS>(v, m, acc);
            if ((k & 7) == 7) {
                tot += acc.x + acc.y;
                acc = make_float2(0.f, 0.f);
            }
        }
    }
    if (warp < EPI) out[blockIdx.x * 32 * EPI + threadIdx.x] = MODE == 0 || MODE == 2 ? m : (float)(tot + acc.x + acc.y);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int EPI, int NACC, int N, int MODE, int KSTEPS>
void run(const float* dA, const float* dB, float* dO, int sms) {
    const int iters = 4096 * 256 / N, grid = sms;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    sum_proto<EPI, NACC, N, MODE, KSTEPS><<<grid, 32 * (EPI + 1)>>>(dA, dB, 64, dO);
    cudaEventRecord(e0);
    sum_proto<EPI, NACC, N, MODE, KSTEPS><<<grid, 32 * (EPI + 1)>>>(dA, dB, iters, dO);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { printf("kernel error: %s\n", cudaGetErrorString(e)); exit(1); }
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double pairs = (double)grid * iters * M * N;
    printf("mode %d epi warps %2d accs %d N %3d K %2d: %.3f ms, %.3f Tpair/s = %.1f pairs/clk/SM\n", MODE, EPI, NACC,
           N, K * KSTEPS, ms, pairs / (ms * 1e-3) / 1e12, pairs / (ms * 1e-3) / sms / 1.965e9);
}

int main() {
    constexpr int NB = 256;
    std::vector<float> A(M * K, 0.f), B(NB * K, 0.f);
    unsigned s = 12345u;
    auto rnd = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 8) & 0xffff) / 8192.0 - 4.0; };
    std::vector<double> qa(M * 3), qb(NB * 3), wb(NB);
    for (int r = 0; r < M; ++r) {
        for (int k = 0; k < 3; ++k) { qa[3 * r + k] = rnd(); A[op_index(r, k, M)] = (float)qa[3 * r + k]; }
        A[op_index(r, 3, M)] = 1.f;
    }
    for (int c = 0; c < NB; ++c) {
        for (int k = 0; k < 3; ++k) { qb[3 * c + k] = rnd(); B[op_index(c, k, NB)] = (float)qb[3 * c + k]; }
        wb[c] = 64.0 + rnd();
        B[op_index(c, 3, NB)] = (float)wb[c];
    }
    float *dA, *dB, *dO;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dO, (size_t)sms * 1024 * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    // N = 128 operands: the first 128 columns, re-laid out for 128 rows
    std::vector<float> B128(128 * K, 0.f);
    for (int c = 0; c < 128; ++c)
        for (int k = 0; k < K; ++k) B128[op_index(c, k, 128)] = B[op_index(c, k, NB)];
    float* dB128;
    cudaMalloc(&dB128, B128.size() * 4);
    cudaMemcpy(dB128, B128.data(), B128.size() * 4, cudaMemcpyHostToDevice);

#define SHAPES(MODE, KS)                           \
    run<8, 2, 128, MODE, KS>(dA, dB128, dO, sms);  \
    run<12, 3, 128, MODE, KS>(dA, dB128, dO, sms); \
    run<16, 4, 128, MODE, KS>(dA, dB128, dO, sms); \
    run<16, 2, 256, MODE, KS>(dA, dB, dO, sms);
    SHAPES(2, 1)
    SHAPES(0, 1)
    SHAPES(5, 1)
    SHAPES(6, 1)
    SHAPES(5, 2)
    SHAPES(6, 2)
    return 0;
}
