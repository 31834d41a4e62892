// Prototype (not part of libpaircount): how accurate is p = 1 + |a - b|^2 in Gram form,
// A_i + B_j - 2 a_i.b_j, on tcgen05 kind::tf32 with the operands split three ways
// (x = h + m + l, each exactly tf32)?  K = 24:
//   a_h.b_h, a_h.b_m, a_m.b_h, a_h.b_l, a_m.b_m, a_l.b_h   (18, the b side carrying -2)
//   A_h + A_m + A_l, B_h + B_m + B_l                        (6)
// Every product is exact in fp32; what is left is the tensor core's accumulation.  Prints
// max |p_tc - p| / (1 + (|a| + |b|)^2) in units of u = 2^-24 against float64 from the same
// fp32 a, b, A = fl(1 + |a|^2), B = fl(|b|^2), for several row / column geometries; the
// FFMA2 Gram kernel's bound is 8u.
//
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tcp scripts/tc_prec_proto.cu && ./tcp
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

constexpr int M = 128, N = 256, K = 24, KB = 32;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    unsigned ok = 0;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    } while (!ok);
}
__device__ __forceinline__ uint64_t make_desc(unsigned saddr, unsigned rows) {
    const uint64_t lbo = (uint64_t)rows * 16u, sbo = 128u;
    return (uint64_t)(saddr >> 4) | ((lbo >> 4) << 16) | ((sbo >> 4) << 32) | (1ull << 46);
}
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
__host__ __device__ inline int op_index(int r, int k, int rows) {
    return ((r & 7) * 16 + (r >> 3) * 128 + (k >> 2) * rows * 16 + (k & 3) * 4) / 4;
}

__global__ void __launch_bounds__(128, 1) gram_tc(const float* __restrict__ gA, const float* __restrict__ gB,
                                                  float* __restrict__ out) {
    __shared__ __align__(128) float sA[M * K];
    __shared__ __align__(128) float sB[N * K];
    __shared__ __align__(8) unsigned long long bar;
    __shared__ unsigned tmem_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int q = threadIdx.x; q < M * K; q += blockDim.x) sA[q] = gA[q];
    for (int q = threadIdx.x; q < N * K; q += blockDim.x) sB[q] = gB[q];
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tmem = tmem_s;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int ks = 0; ks < K / 8; ++ks) {
            const uint64_t da = make_desc(smem_u32(sA) + ks * 2 * M * 16, M), db = make_desc(smem_u32(sB) + ks * 2 * N * 16, N);
            asm volatile(
                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
                ::"r"(tmem), "l"(da), "l"(db), "r"(kIdesc), "r"(ks));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"((unsigned long long)smem_u32(&bar)));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int c = 0; c < N; ++c) {
        unsigned v;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + ((unsigned)(warp * 32) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        out[(warp * 32 + lane) * N + c] = __uint_as_float(v);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}


// bf16 variant: K = 32 = a_h.b_{h,m,l} + a_m.b_{h,m,l} + a_l.b_{h,m} (8 per coordinate) + A (3) + B (3)
__host__ __device__ inline int op_index_b(int r, int k, int rows) {  // 16-byte K-chunks of 8 bf16
    return ((r & 7) * 16 + (r >> 3) * 128 + (k >> 3) * rows * 16) / 2 + (k & 7);
}
constexpr uint32_t kIdescB = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
__global__ void __launch_bounds__(128, 1) gram_tc_b(const unsigned short* __restrict__ gA, const unsigned short* __restrict__ gB,
                                                    float* __restrict__ out) {
    __shared__ __align__(128) unsigned short sA[M * KB];
    __shared__ __align__(128) unsigned short sB[N * KB];
    __shared__ __align__(8) unsigned long long bar;
    __shared__ unsigned tmem_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int q = threadIdx.x; q < M * KB; q += blockDim.x) sA[q] = gA[q];
    for (int q = threadIdx.x; q < N * KB; q += blockDim.x) sB[q] = gB[q];
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tmem = tmem_s;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int ks = 0; ks < KB / 16; ++ks) {
            const uint64_t da = make_desc(smem_u32(sA) + ks * 2 * M * 16, M), db = make_desc(smem_u32(sB) + ks * 2 * N * 16, N);
            asm volatile(
                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                ::"r"(tmem), "l"(da), "l"(db), "r"(kIdescB), "r"(ks));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"((unsigned long long)smem_u32(&bar)));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int c = 0; c < N; ++c) {
        unsigned v;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + ((unsigned)(warp * 32) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        out[(warp * 32 + lane) * N + c] = __uint_as_float(v);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}
static unsigned short bf16_rn(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    u += 0x7fffu + ((u >> 16) & 1u);
    return (unsigned short)(u >> 16);
}
static float bf16_f(unsigned short b) {
    uint32_t u = (uint32_t)b << 16;
    float r;
    memcpy(&r, &u, 4);
    return r;
}
static void split3b(float x, unsigned short& h, unsigned short& m, unsigned short& l) {
    h = bf16_rn(x);
    const float r = x - bf16_f(h);
    m = bf16_rn(r);
    l = bf16_rn(r - bf16_f(m));
}

static float tf32_rna(float x) {  // round to nearest, ties away, 10 explicit mantissa bits
    uint32_t u;
    memcpy(&u, &x, 4);
    u = (u + 0x1000u) & 0xffffe000u;
    float r;
    memcpy(&r, &u, 4);
    return r;
}
static void split3(float x, float& h, float& m, float& l) {
    h = tf32_rna(x);
    const float r = x - h;  // exact
    m = tf32_rna(r);
    l = r - m;  // exact, fits tf32
}

int main() {
    float *dA, *dB, *dO;
    cudaMalloc(&dA, M * K * 4);
    cudaMalloc(&dB, N * K * 4);
    cudaMalloc(&dO, M * N * 4);
    unsigned s = 987654321u;
    auto uni = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 8) & 0xffffff) / 16777216.0 * 2.0 - 1.0; };
    struct Geo { double ra, rb, dist; };
    const Geo geos[] = {{1, 1, 0}, {1, 1, 2.5}, {2, 2, 3}, {1, 3, 5}, {10, 10, 0}, {10, 10, 30}, {100, 100, 300},
                        {0.3, 0.3, 1}, {1000, 1000, 3000}};
    for (const Geo& g : geos) {
        std::vector<float> A(M * K, 0.f), B(N * K, 0.f), a(M * 3), b(N * 3);
        for (int r = 0; r < M; ++r) for (int k = 0; k < 3; ++k) a[3 * r + k] = (float)(g.ra * uni());
        for (int c = 0; c < N; ++c) for (int k = 0; k < 3; ++k) b[3 * c + k] = (float)(g.rb * uni() + (k == 0 ? g.dist : 0.0));
        for (int r = 0; r < M; ++r) {
            float h[3], m[3], l[3];
            for (int k = 0; k < 3; ++k) split3(a[3 * r + k], h[k], m[k], l[k]);
            const float Ai = 1.f + fmaf(a[3 * r + 2], a[3 * r + 2], fmaf(a[3 * r + 1], a[3 * r + 1], a[3 * r] * a[3 * r]));
            float Ah, Am, Al;
            split3(Ai, Ah, Am, Al);
            const float row[K] = {h[0], h[1], h[2], h[0], h[1], h[2], m[0], m[1], m[2], h[0], h[1], h[2],
                                  m[0], m[1], m[2], l[0], l[1], l[2], Ah, Am, Al, 1.f, 1.f, 1.f};
            for (int k = 0; k < K; ++k) A[op_index(r, k, M)] = row[k];
        }
        std::vector<float> Bj(N);
        for (int c = 0; c < N; ++c) {
            float h[3], m[3], l[3];
            for (int k = 0; k < 3; ++k) split3(-2.f * b[3 * c + k], h[k], m[k], l[k]);
            Bj[c] = fmaf(b[3 * c + 2], b[3 * c + 2], fmaf(b[3 * c + 1], b[3 * c + 1], b[3 * c] * b[3 * c]));
            float Bh, Bm, Bl;
            split3(Bj[c], Bh, Bm, Bl);
            const float col[K] = {h[0], h[1], h[2], m[0], m[1], m[2], h[0], h[1], h[2], l[0], l[1], l[2],
                                  m[0], m[1], m[2], h[0], h[1], h[2], 1.f, 1.f, 1.f, Bh, Bm, Bl};
            for (int k = 0; k < K; ++k) B[op_index(c, k, N)] = col[k];
        }
        std::vector<float> PB(M * N);
        {
            std::vector<unsigned short> Ab(M * KB, 0), Bb(N * KB, 0);
            for (int r = 0; r < M; ++r) {
                unsigned short h[3], m[3], l[3], Ah, Am, Al;
                for (int k = 0; k < 3; ++k) split3b(a[3 * r + k], h[k], m[k], l[k]);
                const float Ai = 1.f + fmaf(a[3 * r + 2], a[3 * r + 2], fmaf(a[3 * r + 1], a[3 * r + 1], a[3 * r] * a[3 * r]));
                split3b(Ai, Ah, Am, Al);
                const unsigned short one = bf16_rn(1.f);
                const unsigned short row[KB] = {h[0], h[1], h[2], h[0], h[1], h[2], h[0], h[1], h[2], m[0], m[1], m[2],
                                                m[0], m[1], m[2], m[0], m[1], m[2], l[0], l[1], l[2], l[0], l[1], l[2],
                                                Ah, Am, Al, one, one, one, 0, 0};
                for (int k = 0; k < KB; ++k) Ab[op_index_b(r, k, M)] = row[k];
            }
            for (int c = 0; c < N; ++c) {
                unsigned short h[3], m[3], l[3], Bh, Bm, Bl;
                for (int k = 0; k < 3; ++k) split3b(-2.f * b[3 * c + k], h[k], m[k], l[k]);
                const float Bjc = fmaf(b[3 * c + 2], b[3 * c + 2], fmaf(b[3 * c + 1], b[3 * c + 1], b[3 * c] * b[3 * c]));
                split3b(Bjc, Bh, Bm, Bl);
                const unsigned short one = bf16_rn(1.f);
                const unsigned short col[KB] = {h[0], h[1], h[2], m[0], m[1], m[2], l[0], l[1], l[2], h[0], h[1], h[2],
                                                m[0], m[1], m[2], l[0], l[1], l[2], h[0], h[1], h[2], m[0], m[1], m[2],
                                                one, one, one, Bh, Bm, Bl, 0, 0};
                for (int k = 0; k < KB; ++k) Bb[op_index_b(c, k, N)] = col[k];
            }
            unsigned short *dAb, *dBb;
            cudaMalloc(&dAb, Ab.size() * 2);
            cudaMalloc(&dBb, Bb.size() * 2);
            cudaMemcpy(dAb, Ab.data(), Ab.size() * 2, cudaMemcpyHostToDevice);
            cudaMemcpy(dBb, Bb.data(), Bb.size() * 2, cudaMemcpyHostToDevice);
            gram_tc_b<<<1, 128>>>(dAb, dBb, dO);
            if (cudaDeviceSynchronize() != cudaSuccess) { printf("kernel error (bf16)\n"); return 1; }
            cudaMemcpy(PB.data(), dO, PB.size() * 4, cudaMemcpyDeviceToHost);
            cudaFree(dAb);
            cudaFree(dBb);
        }
        cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
        gram_tc<<<1, 128>>>(dA, dB, dO);
        if (cudaDeviceSynchronize() != cudaSuccess) { printf("kernel error\n"); return 1; }
        std::vector<float> P(M * N);
        cudaMemcpy(P.data(), dO, P.size() * 4, cudaMemcpyDeviceToHost);
        double worst = 0, worst_rel = 0, worst_ffma = 0, worst_b = 0, worst_b_rel = 0;
        for (int r = 0; r < M; ++r) {
            const double Ai = 1.0 + (double)(1.f + fmaf(a[3 * r + 2], a[3 * r + 2], fmaf(a[3 * r + 1], a[3 * r + 1], a[3 * r] * a[3 * r]))) - 1.0;
            double na = 0;
            for (int k = 0; k < 3; ++k) na += (double)a[3 * r + k] * a[3 * r + k];
            for (int c = 0; c < N; ++c) {
                double nb = 0, d2 = 0, dot = 0;
                for (int k = 0; k < 3; ++k) {
                    nb += (double)b[3 * c + k] * b[3 * c + k];
                    const double d = (double)a[3 * r + k] - (double)b[3 * c + k];
                    d2 += d * d;
                    dot += (double)a[3 * r + k] * b[3 * c + k];
                }
                const double pexact = 1.0 + d2;
                // the Gram form from the rounded A_i, B_j (their own rounding is part of the 8u of the FFMA bound)
                const double pgram = Ai + (double)Bj[c] - 2.0 * dot;
                const double scale = 1.0 + (sqrt(na) + sqrt(nb)) * (sqrt(na) + sqrt(nb));
                worst = fmax(worst, fabs((double)P[r * N + c] - pgram) / scale);
                worst_rel = fmax(worst_rel, fabs((double)P[r * N + c] - pexact) / scale);
                worst_b = fmax(worst_b, fabs((double)PB[r * N + c] - pgram) / scale);
                worst_b_rel = fmax(worst_b_rel, fabs((double)PB[r * N + c] - pexact) / scale);
                // FFMA2 Gram kernel arithmetic on the host (fp32, same association)
                float t = fmaf(-2.f * a[3 * r], b[3 * c], Bj[c]);
                t = fmaf(-2.f * a[3 * r + 1], b[3 * c + 1], t);
                t = fmaf(-2.f * a[3 * r + 2], b[3 * c + 2], t);
                const float pf = t + (1.f + fmaf(a[3 * r + 2], a[3 * r + 2], fmaf(a[3 * r + 1], a[3 * r + 1], a[3 * r] * a[3 * r])));
                worst_ffma = fmax(worst_ffma, fabs((double)pf - pexact) / scale);
            }
        }
        const double u = 5.9604644775390625e-08;
        printf("rows r<=%6g cols r<=%6g at %6g: tf32 vs Gram(A,B rounded) %.2f u, vs exact %.2f u | bf16 %.2f u, %.2f u | ffma vs exact %.2f u\n",
               g.ra, g.rb, g.dist, worst / u, worst_rel / u, worst_b / u, worst_b_rel / u, worst_ffma / u);
    }
    return 0;
}
