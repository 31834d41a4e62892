// Prototype (not part of libpaircount): how fast can the tensor cores feed the
// Gram filter?  Each CTA computes D = A . B^T for A = 128 rows (q_x, q_y, q_z, 1)
// and B = 256 columns (q_x, q_y, q_z, w) with tcgen05.mma kind::tf32 (K = 8,
// zero padded) into TMEM, then 4 epilogue warps read D back with tcgen05.ld
// and reduce it with FMNMX3 into a per-row max -- the count kernel's filter.
// Two TMEM accumulators alternate so the MMA of tile t+1 overlaps the
// read-back of tile t.  Prints the correctness check and pairs/s.
//
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tcp scripts/tc_gram_proto.cu && ./tcp
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

__global__ void __launch_bounds__(128, 1) tc_proto(const float* __restrict__ gA, const float* __restrict__ gB,
                                                   int iters, float* __restrict__ rowmax) {
    __shared__ __align__(128) float sA[M * K];
    __shared__ __align__(128) float sB[N * K];
    __shared__ __align__(8) unsigned long long bar_full[2], bar_empty[2];
    __shared__ unsigned tmem_base_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int q = threadIdx.x; q < M * K; q += blockDim.x) sA[q] = gA[q];
    for (int q = threadIdx.x; q < N * K; q += blockDim.x) sB[q] = gB[q];
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&bar_full[b]), 1);
            mbar_init(smem_u32(&bar_empty[b]), 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // operands written by threads, read by the MMA
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tmem = tmem_base_s;
    const uint64_t da = make_desc(smem_u32(sA), M), db = make_desc(smem_u32(sB), N);
    const uint32_t idesc = make_idesc();
    float m = -INFINITY;
    for (int it = 0; it < iters; ++it) {
        const int b = it & 1;
        const unsigned ph = (unsigned)(it >> 1) & 1u;
        if (threadIdx.x == 0) {
            if (it >= 2) mbar_wait(smem_u32(&bar_empty[b]), ph ^ 1u);  // epilogue of tile it-2 released buffer b
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
    rowmax[blockIdx.x * M + threadIdx.x] = m;  // thread t = TMEM lane t = row t
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    // rows (q, 1) and columns (q, w) in [-4, 4): exactly representable-ish in tf32 is not required for
    // the check -- it compares against a float64 reference with a tf32-sized tolerance
    std::vector<float> A(M * K, 0.f), B(N * K, 0.f);
    std::vector<double> qa(M * 3), qb(N * 3), wb(N);
    unsigned s = 12345u;
    auto rnd = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 8) & 0xffff) / 8192.0 - 4.0; };
    for (int r = 0; r < M; ++r) {
        for (int k = 0; k < 3; ++k) { qa[3 * r + k] = rnd(); A[op_index(r, k, M)] = (float)qa[3 * r + k]; }
        A[op_index(r, 3, M)] = 1.f;
    }
    for (int c = 0; c < N; ++c) {
        for (int k = 0; k < 3; ++k) { qb[3 * c + k] = rnd(); B[op_index(c, k, N)] = (float)qb[3 * c + k]; }
        wb[c] = rnd();
        B[op_index(c, 3, N)] = (float)wb[c];
    }
    float *dA, *dB, *dM;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dM, (size_t)sms * 2 * M * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    // correctness: one CTA, one tile
    tc_proto<<<1, 128>>>(dA, dB, 1, dM);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("kernel error: %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<float> got(M);
    cudaMemcpy(got.data(), dM, M * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int r = 0; r < M; ++r) {
        double best = -1e300;
        for (int c = 0; c < N; ++c) {
            double t = wb[c];
            for (int k = 0; k < 3; ++k) t += qa[3 * r + k] * qb[3 * c + k];
            best = best > t ? best : t;
        }
        maxerr = fmax(maxerr, fabs(best - got[r]));
    }
    printf("check: max |rowmax - float64| = %.3e (tf32 inputs: expect ~1e-2)\n", maxerr);
    for (int bps : {1, 2}) {
        const int iters = 4096, grid = sms * bps;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        tc_proto<<<grid, 128>>>(dA, dB, 64, dM);
        cudaEventRecord(e0);
        tc_proto<<<grid, 128>>>(dA, dB, iters, dM);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        e = cudaGetLastError();
        if (e != cudaSuccess) { printf("kernel error: %s\n", cudaGetErrorString(e)); return 1; }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double pairs = (double)grid * iters * M * N;
        printf("CTAs/SM %d: %.3f ms, %.3f Tpair/s (%.1f pairs/clk/SM at 1.965 GHz)\n", bps, ms,
               pairs / (ms * 1e-3) / 1e12, pairs / (ms * 1e-3) / sms / 1.965e9);
    }
    return 0;
}
