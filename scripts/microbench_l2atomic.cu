// Scattered atomics: L2-resident region vs DRAM-sized region, with and without explicit L2 prefetch.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mbl scripts/microbench_l2atomic.cu && ./mbl
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void gen_keys(unsigned* keys, long long n, unsigned long long cells, unsigned long long seed) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        unsigned long long x = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
        x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 27; x *= 0x94D049BB133111EBull; x ^= x >> 31;
        keys[i] = (unsigned)(x % cells);
    }
}
// keys sorted by slab: slab s = keys in [s*S, (s+1)*S), each slab's keys contiguous (synthetic: key = s*S + rand%S)
__global__ void gen_slab_keys(unsigned* keys, long long n, unsigned long long slab_cells, long long per_slab,
                              unsigned long long seed) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        unsigned long long x = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
        x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 27; x *= 0x94D049BB133111EBull; x ^= x >> 31;
        keys[i] = (unsigned)((i / per_slab) * slab_cells + x % slab_cells);
    }
}

__global__ void atom_ret(const unsigned* __restrict__ keys, long long n, unsigned* grid, unsigned long long* out) {
    unsigned long long c = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        c += atomicAdd(grid + keys[i], 1u);
    if (c == 12345) out[0] = c;
}

// persistent: process slab by slab; before slab s, prefetch slab s+1's grid region into L2 (bulk prefetch)
__global__ void atom_slabs_prefetch(const unsigned* __restrict__ keys, long long per_slab, int nslabs,
                                    unsigned long long slab_cells, unsigned* grid, unsigned long long* out) {
    unsigned long long c = 0;
    const long long slab_bytes = (long long)slab_cells * 4;
    const long long share = ((slab_bytes + gridDim.x - 1) / gridDim.x + 127) & ~127LL;  // 128 B aligned
    for (int s = 0; s < nslabs; ++s) {
        if (s + 1 < nslabs && threadIdx.x == 0) {
            const char* base = (const char*)(grid + (unsigned long long)(s + 1) * slab_cells) + blockIdx.x * share;
            long long len = share;
            const long long lim = slab_bytes - (long long)blockIdx.x * share;
            if (lim < len) len = lim > 0 ? lim : 0;
            for (long long o = 0; o < len; o += 65536) {
                long long sz = len - o < 65536 ? len - o : 65536;
                sz &= ~15LL;
                if (sz > 0)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + o), "r"((unsigned)sz) : "memory");
            }
        }
        const unsigned* k = keys + (long long)s * per_slab;
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < per_slab; i += (long long)gridDim.x * blockDim.x)
            c += atomicAdd(grid + k[i], 1u);
    }
    if (c == 12345) out[0] = c;
}

int main() {
    const long long n = 1LL << 26;
    const unsigned long long cells = 1027ull * 1027 * 1027;
    unsigned *keys, *grid;
    unsigned long long* out;
    cudaMalloc(&keys, n * 4);
    cudaMalloc(&grid, cells * 4 + 1024);
    cudaMalloc(&out, 64);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    auto T = [&](const char* name, auto fn) {
        for (int r = 0; r < 3; ++r) {
            cudaMemset(grid, 0, cells * 4);
            cudaDeviceSynchronize();
            cudaEventRecord(e0);
            fn();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-56s %8.3f ms  %6.1f Gatom/s  %s\n", name, ms, n / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    };
    for (unsigned long long region : {1ull << 20, 1ull << 23, 1ull << 25, cells}) {
        gen_keys<<<sms * 8, 256>>>(keys, n, region, 7);
        char nm[96];
        snprintf(nm, 96, "random atomics in region of %llu MB", region * 4 >> 20);
        T(nm, [&] { atom_ret<<<sms * 16, 256>>>(keys, n, grid, out); });
    }
    for (int shift : {21, 22, 23, 24}) {
        const unsigned long long slab = 1ull << shift;
        const int nslabs = (int)(cells / slab);
        const long long per = n / nslabs;
        gen_slab_keys<<<sms * 8, 256>>>(keys, per * nslabs, slab, per, 9);
        char nm[96];
        snprintf(nm, 96, "slab-ordered keys, slab %llu MB, no prefetch", slab * 4 >> 20);
        T(nm, [&] { atom_ret<<<sms * 16, 256>>>(keys, per * nslabs, grid, out); });
        snprintf(nm, 96, "slab-ordered keys, slab %llu MB, persistent + L2 prefetch", slab * 4 >> 20);
        T(nm, [&] { atom_slabs_prefetch<<<sms * 8, 256>>>(keys, per, nslabs, slab, grid, out); });
    }
    return 0;
}
