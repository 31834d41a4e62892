// Dense-regime counting array (included by paircount.cu inside its anonymous namespace).
//
// Alg. 1 (collisions += space[b]; space[b]++) evaluated
// slab by slab in shared memory instead of with one scattered global atomic
// per bead.  Scattered 4-byte atomics into a 4.3 GB grid run at ~21 G/s on
// B200 (DRAM-resident lines; ~122 G/s when L2-resident, measured in
// scripts/microbench_l2atomic.cu), so 2^26 beads cost ~3 ms that way; this
// path is bound by streaming the finished slabs to HBM instead.
//
//   K1 lat_keys_hist_kernel   validate, write each bead's key (the touched
//                             list), histogram keys by 128K-cell bucket
//   K2 lat_bucket_scan_kernel exclusive scan of the bucket histogram
//   K3 lat_bucket_scatter_kernel  partition keys by bucket (tile-local ranks
//                             + one global reservation per tile and bucket)
//   K4 lat_slab_kernel        persistent, one CTA per SM, buckets round-robin:
//                             stage a bucket's keys on chip, counting-sort them
//                             into 16 slabs of 8K cells, then per slab zero a
//                             32 KB shared-memory
//                             counting array, atomicAdd each bead (old value =
//                             its new collisions; old == 0 marks a touched
//                             cell) and hand the slab to a TMA bulk store
//                             (cp.async.bulk shared->global) while the next
//                             slab accumulates in the other buffer.
//
// Valid only on a clean grid (every cell zero on entry): the slab stores
// overwrite whole cell ranges.  Used when beads outnumber cells/64.

constexpr int kBucketShift = 17;  // 128K cells per bucket
constexpr int kSlabShift = 13;    // 8K cells per shared-memory slab (2 x 32 KB buffers)
constexpr int kSlabCells = 1 << kSlabShift;
constexpr int kSubSlabs = 1 << (kBucketShift - kSlabShift);  // 16
constexpr int kMaxBuckets = 16384;                             // grids below 2^32 cells
constexpr int kKeyCap = 16384;    // keys of one bucket staged on chip (2x the uniform mean)
constexpr int kSlabSmem = (kKeyCap + 8 + kKeyCap + 2 * kSlabCells + 3 * kSubSlabs) * 4;

__global__ void lat_keys_hist_kernel(const void* __restrict__ xyz, int dtype, long long n, long long a,
                                     long long side, unsigned* __restrict__ keys,
                                     unsigned long long* __restrict__ bad, unsigned* __restrict__ ghist,
                                     int nbuckets) {
    extern __shared__ unsigned h_s[];
    for (int b = threadIdx.x; b < nbuckets; b += blockDim.x) h_s[b] = 0u;
    __syncthreads();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long x = coord_i64(xyz, dtype, i, 0), y = coord_i64(xyz, dtype, i, 1),
                        z = coord_i64(xyz, dtype, i, 2);
        if (x < -a || x > a || y < -a || y > a || z < -a || z > a) {  // _validate, lattice_counter.py:98-105
            atomicMin(bad, (unsigned long long)i);
        } else {
            const unsigned key = (unsigned)(((x + a + 1) * side + (y + a + 1)) * side + (z + a + 1));
            keys[i] = key;
            atomicAdd(&h_s[key >> kBucketShift], 1u);
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nbuckets; b += blockDim.x)
        if (h_s[b]) atomicAdd(&ghist[b], h_s[b]);
}

// base[b] = sum of hist[< b]; cursor[b] = base[b]; base[nbuckets] = total.  One CTA of 1024 threads.
__global__ void lat_bucket_scan_kernel(const unsigned* __restrict__ hist, unsigned* __restrict__ base,
                                       unsigned* __restrict__ cursor, int nbuckets) {
    __shared__ unsigned s_part[1024];
    constexpr int kPer = kMaxBuckets / 1024;
    unsigned v[kPer], tot = 0;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const int b = threadIdx.x * kPer + q;
        v[q] = b < nbuckets ? hist[b] : 0u;
        tot += v[q];
    }
    s_part[threadIdx.x] = tot;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {  // Hillis-Steele inclusive scan
        const unsigned add = threadIdx.x >= o ? s_part[threadIdx.x - o] : 0u;
        __syncthreads();
        s_part[threadIdx.x] += add;
        __syncthreads();
    }
    unsigned run = s_part[threadIdx.x] - tot;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const int b = threadIdx.x * kPer + q;
        if (b < nbuckets) {
            base[b] = run;
            cursor[b] = run;
        }
        run += v[q];
    }
    if (threadIdx.x == 1023) base[nbuckets] = s_part[1023];
}

// Partition keys by bucket.  Order inside a bucket is irrelevant (a histogram
// does not care), so ranks come from shared-memory atomics and each tile
// reserves its bucket ranges with one global atomic per (tile, bucket).
// 512 threads x 8 keys (two 16-byte loads) per tile.  (A 32K-key tile with a
// second pass was slower: the scattered 4-byte stores, not the reservations,
// bound this kernel -- ~0.6 ms for 2^26 keys.)
__global__ void __launch_bounds__(512) lat_bucket_scatter_kernel(const unsigned* __restrict__ keys, long long n,
                                                                 unsigned* __restrict__ cursor,
                                                                 unsigned* __restrict__ out, int nbuckets,
                                                                 const unsigned long long* __restrict__ bad) {
    if (*bad != kNoBad) return;
    extern __shared__ unsigned sm[];
    unsigned* h = sm;               // [nbuckets] tile histogram
    unsigned* off = sm + nbuckets;  // [nbuckets] reserved global offsets
    constexpr int kPer = 8;
    const long long tile = (long long)blockDim.x * kPer;
    const bool vec = (reinterpret_cast<uintptr_t>(keys) & 15) == 0;
    for (long long t0 = (long long)blockIdx.x * tile; t0 < n; t0 += (long long)gridDim.x * tile) {
        for (int b = threadIdx.x; b < nbuckets; b += blockDim.x) h[b] = 0u;
        __syncthreads();
        unsigned k[kPer], rank[kPer];
        const long long i0 = t0 + 4LL * threadIdx.x;                 // keys i0..i0+3
        const long long i1 = t0 + 4LL * (threadIdx.x + blockDim.x);  // keys i1..i1+3
        if (vec && i1 + 3 < n) {
            const uint4 a4 = reinterpret_cast<const uint4*>(keys + i0)[0];
            const uint4 b4 = reinterpret_cast<const uint4*>(keys + i1)[0];
            k[0] = a4.x; k[1] = a4.y; k[2] = a4.z; k[3] = a4.w;
            k[4] = b4.x; k[5] = b4.y; k[6] = b4.z; k[7] = b4.w;
        } else {
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
                const long long i = (u < 4 ? i0 : i1) + (u & 3);
                k[u] = i < n ? keys[i] : 0xffffffffu;
            }
        }
#pragma unroll
        for (int u = 0; u < kPer; ++u)
            rank[u] = k[u] != 0xffffffffu ? atomicAdd(&h[k[u] >> kBucketShift], 1u) : 0u;
        __syncthreads();
        for (int b = threadIdx.x; b < nbuckets; b += blockDim.x)
            if (h[b]) off[b] = atomicAdd(&cursor[b], h[b]);
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kPer; ++u)
            if (k[u] != 0xffffffffu) out[off[k[u] >> kBucketShift] + rank[u]] = k[u];
        __syncthreads();
    }
}

__device__ __forceinline__ void bulk_store_s2g(void* gdst, const void* ssrc, unsigned bytes) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(ssrc);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(s), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_le1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Persistent: CTA c walks buckets c, c + gridDim.x, ...  Alg. 1 on shared-memory slabs.
// A bucket's keys (<= kKeyCap) are staged on chip with cp.async -- the next
// bucket's while this one's slabs run -- and counting-sorted by slab in shared
// memory; larger buckets (clustered input) fall back to a global-memory
// sub-partition through `scratch`.
__global__ void __launch_bounds__(1024, 1)
    lat_slab_kernel(const unsigned* __restrict__ sorted, unsigned* __restrict__ scratch,
                    const unsigned* __restrict__ base, int nbuckets, unsigned* __restrict__ grid,
                    unsigned long long cells, const unsigned long long* __restrict__ bad,
                    LatSlot* __restrict__ slots, int* __restrict__ overflow) {
    extern __shared__ __align__(128) unsigned smem[];
    unsigned* keys_in = smem;                           // [kKeyCap + 8] staged keys (16 B aligned window)
    unsigned* keys_s = keys_in + kKeyCap + 8;           // [kKeyCap] keys grouped by slab
    unsigned* cbuf0 = keys_s + kKeyCap;                 // [2][kSlabCells] double-buffered counting arrays
    unsigned* sub_n = cbuf0 + 2 * kSlabCells;           // [kSubSlabs] keys per slab
    unsigned* sub_cur = sub_n + kSubSlabs;              // [kSubSlabs] scatter cursors
    unsigned* sub_start = sub_cur + kSubSlabs;          // [kSubSlabs] slab start offsets
    __shared__ unsigned long long s_a[32], s_b[32];
    unsigned long long acc = 0, first = 0;
    int ovf = 0;
    const bool ok = *bad == kNoBad;
    int flip = 0;

    auto stage = [&](int b) {  // cp.async the bucket's keys (aligned superset) into keys_in
        if (b >= nbuckets) return;
        const unsigned lo = base[b], hi = base[b + 1];
        if (hi - lo > (unsigned)kKeyCap) return;
        const unsigned a0 = lo & ~3u, a1 = (hi + 3u) & ~3u;  // `sorted` is padded by 16 keys
        for (unsigned q = threadIdx.x; q < (a1 - a0) / 4; q += blockDim.x)
            cp_async16(&keys_in[4 * q], &sorted[a0 + 4 * q]);
        cp_async_commit();
    };
    auto slab_pass = [&](int b, const unsigned* keys, bool keys_on_chip) {
        // keys[sub_start[s] .. + sub_n[s]) hold slab s's keys (shared or global memory)
        for (int s = 0; s < kSubSlabs; ++s) {
            const unsigned long long cell0 =
                ((unsigned long long)b << kBucketShift) + ((unsigned long long)s << kSlabShift);
            if (cell0 >= cells) break;
            const unsigned ncell =
                (unsigned)(cells - cell0 < (unsigned long long)kSlabCells ? cells - cell0 : kSlabCells);
            unsigned* cnt = cbuf0 + flip * kSlabCells;
            // the bulk store issued two slabs ago read this buffer: wait for it
            if (threadIdx.x == 0) bulk_wait_read_le1();
            __syncthreads();
            uint4* cnt4 = reinterpret_cast<uint4*>(cnt);
            for (int q = threadIdx.x; q < kSlabCells / 4; q += blockDim.x) cnt4[q] = make_uint4(0u, 0u, 0u, 0u);
            __syncthreads();
            const unsigned s0 = sub_start[s], s1 = s0 + sub_n[s];
            for (unsigned i = s0 + threadIdx.x; i < s1; i += blockDim.x) {
                const unsigned old = atomicAdd(&cnt[keys[i] & (kSlabCells - 1)], 1u);  // Alg. 1
                acc += old;
                first += old == 0u;
                ovf |= old >= 0xfffffffeu;
            }
            (void)keys_on_chip;
            fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the bulk copy
            __syncthreads();
            const unsigned vec_bytes = (ncell * 4u) & ~15u;
            if (threadIdx.x == 0 && vec_bytes) bulk_store_s2g(grid + cell0, cnt, vec_bytes);
            for (unsigned q = vec_bytes / 4 + threadIdx.x; q < ncell; q += blockDim.x) grid[cell0 + q] = cnt[q];
            flip ^= 1;
        }
    };

    if (ok) stage(blockIdx.x);
    for (int b = blockIdx.x; ok && b < nbuckets; b += gridDim.x) {
        const unsigned lo = base[b], hi = base[b + 1];
        const bool on_chip = hi - lo <= (unsigned)kKeyCap;
        if (threadIdx.x < kSubSlabs) sub_n[threadIdx.x] = 0u;
        cp_async_wait<0>();
        __syncthreads();
        if (on_chip) {
            // counting sort by slab, shared memory -> shared memory
            const unsigned* kin = keys_in + (lo & 3u);
            const unsigned cnt_b = hi - lo;
            for (unsigned i = threadIdx.x; i < cnt_b; i += blockDim.x)
                atomicAdd(&sub_n[(kin[i] >> kSlabShift) & (kSubSlabs - 1)], 1u);
            __syncthreads();
            if (threadIdx.x == 0) {
                unsigned run = 0;
                for (int s = 0; s < kSubSlabs; ++s) {
                    sub_start[s] = run;
                    sub_cur[s] = run;
                    run += sub_n[s];
                }
            }
            __syncthreads();
            for (unsigned i = threadIdx.x; i < cnt_b; i += blockDim.x) {
                const unsigned k = kin[i];
                keys_s[atomicAdd(&sub_cur[(k >> kSlabShift) & (kSubSlabs - 1)], 1u)] = k;
            }
            __syncthreads();
            stage(b + gridDim.x);  // keys_in is free again: prefetch the next bucket under this one's slabs
            slab_pass(b, keys_s, true);
        } else {
            // oversized bucket: sub-partition through global scratch
            for (unsigned i = lo + threadIdx.x; i < hi; i += blockDim.x)
                atomicAdd(&sub_n[(sorted[i] >> kSlabShift) & (kSubSlabs - 1)], 1u);
            __syncthreads();
            if (threadIdx.x == 0) {
                unsigned run = lo;
                for (int s = 0; s < kSubSlabs; ++s) {
                    sub_start[s] = run;
                    sub_cur[s] = run;
                    run += sub_n[s];
                }
            }
            __syncthreads();
            for (unsigned i = lo + threadIdx.x; i < hi; i += blockDim.x) {
                const unsigned k = sorted[i];
                scratch[atomicAdd(&sub_cur[(k >> kSlabShift) & (kSubSlabs - 1)], 1u)] = k;
            }
            __syncthreads();
            stage(b + gridDim.x);
            slab_pass(b, scratch, false);
        }
    }
    if (threadIdx.x == 0) bulk_wait_all();
    acc = warp_sum(acc);
    first = warp_sum(first);
    if ((threadIdx.x & 31) == 0) {
        s_a[threadIdx.x >> 5] = acc;
        s_b[threadIdx.x >> 5] = first;
    }
    if (__any_sync(0xffffffffu, ovf) && (threadIdx.x & 31) == 0) atomicOr(overflow, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        LatSlot sl{0, 0};
        for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
            sl.a += s_a[q];
            sl.b += s_b[q];
        }
        slots[blockIdx.x] = sl;
    }
}
