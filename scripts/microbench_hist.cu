// Counting-array histogram strategies on B200: 2^26 random keys into a 1027^3 uint32 grid.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mbh scripts/microbench_hist.cu && ./mbh
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

__global__ void atom_ret(const unsigned* __restrict__ keys, long long n, unsigned* grid, unsigned long long* out) {
    unsigned long long c = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        c += atomicAdd(grid + keys[i], 1u);
    if (c == 12345) out[0] = c;
}

__global__ void red_only(const unsigned* __restrict__ keys, long long n, unsigned* grid) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        atomicAdd(grid + keys[i], 1u);  // result unused -> RED
}

// bucket keys by the top bits of the key (slab = key / slab_cells); simple two-pass counting partition
__global__ void bucket_count(const unsigned* __restrict__ keys, long long n, unsigned slab_shift, unsigned* counts) {
    extern __shared__ unsigned h[];
    const int nb = blockDim.x;  // one bucket per thread slot (nb = number of buckets, <= 1024)
    h[threadIdx.x] = 0;
    __syncthreads();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        atomicAdd(&h[keys[i] >> slab_shift], 1u);
    __syncthreads();
    atomicAdd(&counts[threadIdx.x], h[threadIdx.x]);
    (void)nb;
}
__global__ void bucket_scan(unsigned* counts, unsigned* offs, int nb) {
    if (threadIdx.x == 0) { unsigned s = 0; for (int b = 0; b < nb; ++b) { offs[b] = s; s += counts[b]; } }
}
__global__ void bucket_scatter(const unsigned* __restrict__ keys, long long n, unsigned slab_shift, unsigned* offs,
                               unsigned* out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const unsigned k = keys[i];
        const unsigned pos = atomicAdd(&offs[k >> slab_shift], 1u);
        out[pos] = k;
    }
}

__global__ void clear_grid(uint4* g, long long n4) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x)
        g[i] = make_uint4(0, 0, 0, 0);
}

int main() {
    const long long n = 1LL << 26;
    const unsigned long long side = 1027, cells = side * side * side;
    unsigned *keys, *grid, *sorted, *counts, *offs;
    unsigned long long* out;
    cudaMalloc(&keys, n * 4);
    cudaMalloc(&sorted, n * 4);
    cudaMalloc(&grid, cells * 4 + 64);
    cudaMalloc(&counts, 4096 * 4);
    cudaMalloc(&offs, 4096 * 4);
    cudaMalloc(&out, 64);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    gen_keys<<<sms * 8, 256>>>(keys, n, cells, 7);
    cudaMemset(grid, 0, cells * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    auto T = [&](const char* name, auto fn) {
        for (int r = 0; r < 3; ++r) {
            cudaMemset(grid, 0, cells * 4);
            cudaEventRecord(e0);
            fn();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-44s %8.3f ms   err=%s\n", name, ms, cudaGetErrorString(cudaGetLastError()));
    };
    for (int bps : {4, 16, 32}) {
        char nm[64];
        snprintf(nm, 64, "atomic w/ return, random (%d blk/SM)", bps);
        T(nm, [&] { atom_ret<<<sms * bps, 256>>>(keys, n, grid, out); });
        snprintf(nm, 64, "RED, random (%d blk/SM)", bps);
        T(nm, [&] { red_only<<<sms * bps, 256>>>(keys, n, grid); });
    }
    T("memset grid 4.33 GB", [&] { cudaMemsetAsync(grid, 0, cells * 4); });
    T("clear kernel grid 4.33 GB", [&] { clear_grid<<<sms * 16, 256>>>((uint4*)grid, cells / 4); });
    for (int shift : {22, 23, 24, 25}) {  // slab cells = 2^shift (16 MB .. 128 MB)
        const int nb = (int)((cells >> shift) + 1);
        if (nb > 1024) continue;
        char nm[64];
        snprintf(nm, 64, "partition %d slabs of %d MB", nb, (1 << shift) * 4 >> 20);
        T(nm, [&] {
            cudaMemsetAsync(counts, 0, nb * 4);
            bucket_count<<<sms * 8, nb, nb * 4>>>(keys, n, shift, counts);
            bucket_scan<<<1, 32>>>(counts, offs, nb);
            bucket_scatter<<<sms * 8, 256>>>(keys, n, shift, offs, sorted);
        });
        snprintf(nm, 64, "  atomics on partitioned keys");
        T(nm, [&] { atom_ret<<<sms * 16, 256>>>(sorted, n, grid, out); });
    }
    return 0;
}
