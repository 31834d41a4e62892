// Prototype (not part of libpaircount): back-to-back tcgen05.mma throughput on one SM
// per CTA, no epilogue -- kind::tf32 (K = 8) and kind::f16 with bf16 inputs (K = 16),
// M = 128, N = 256, operands in shared memory, K-major, no swizzle vs 128-byte swizzle.
// Answers: how many cycles does one 128 x 256 MMA instruction take here?
//
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tcm scripts/tc_mma_rate.cu && ./tcm
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// no swizzle: LBO = K-chunk stride, SBO = 8-row group stride
__device__ __forceinline__ uint64_t desc_noswz(unsigned saddr, unsigned lbo, unsigned sbo) {
    return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
           (1ull << 46);
}
// 128-byte swizzle (layout type 2 in bits 61-63 for sm100), SBO = 1024 (8 rows x 128 B)
__device__ __forceinline__ uint64_t desc_sw128(unsigned saddr) {
    return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(16u >> 4) << 16) | ((uint64_t)(1024u >> 4) << 32) |
           (1ull << 46) | (2ull << 61);
}

template <int KIND, bool SW>  // KIND 0: tf32, 1: bf16
__global__ void __launch_bounds__(128, 1) mma_rate(int iters, unsigned* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* base = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) unsigned long long bar;
    __shared__ unsigned tmem_s;
    for (int q = threadIdx.x; q < 48 * 1024 / 4; q += blockDim.x) ((unsigned*)base)[q] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tmem = tmem_s;
    // A: 128 rows x 32 B (one K step), B: 256 rows x 32 B
    const unsigned sa = smem_u32(base), sb = smem_u32(base + 16384);
    const uint64_t da = SW ? desc_sw128(sa) : desc_noswz(sa, 128 * 16, 128);
    const uint64_t db = SW ? desc_sw128(sb) : desc_noswz(sb, 256 * 16, 128);
    const uint32_t idesc = KIND == 0 ? ((1u << 4) | (2u << 7) | (2u << 10) | (32u << 17) | (8u << 24))
                                     : ((1u << 4) | (1u << 7) | (1u << 10) | (32u << 17) | (8u << 24));
    long long t0 = clock64();
    if (threadIdx.x == 0) {
        for (int it = 0; it < iters; ++it) {
            if (KIND == 0)
                asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
                             ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(it));
            else
                asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                             ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(it));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"((unsigned long long)smem_u32(&bar)));
        unsigned ok = 0;
        do {
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                         : "=r"(ok) : "r"(smem_u32(&bar)), "r"(0) : "memory");
        } while (!ok);
        out[blockIdx.x] = (unsigned)(clock64() - t0);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

template <int KIND, bool SW>
void run(int sms, unsigned* d) {
    const int iters = 20000, smem = 48 * 1024 + 1024;
    cudaFuncSetAttribute(mma_rate<KIND, SW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    mma_rate<KIND, SW><<<sms, 128, smem>>>(100, d);
    mma_rate<KIND, SW><<<sms, 128, smem>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
    unsigned h[4];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%s %s: %.1f cycles per 128x256 MMA instruction (K = %d)\n", KIND == 0 ? "tf32" : "bf16",
           SW ? "swizzle-128B" : "no-swizzle ", (double)h[0] / iters, KIND == 0 ? 8 : 16);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned* d;
    cudaMalloc(&d, sms * 4);
    run<0, false>(sms, d);
    run<0, true>(sms, d);
    run<1, false>(sms, d);
    run<1, true>(sms, d);
    return 0;
}
