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
//   K3 lat_partition_{coarse,fine}_kernel  two-level partition of the keys
//                             by bucket; tiles sorted on chip, runs written
//                             contiguously
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
constexpr int kMaxBuckets = 16384;                             // grids of up to 2^31 cells
constexpr int kKeyCap = 16384;    // keys of one bucket staged on chip (2x the uniform mean)
#ifndef PC_SLAB_BUFS
#define PC_SLAB_BUFS 3
#endif
constexpr int kSlabBufs = PC_SLAB_BUFS;  // counting-array ring: up to kSlabBufs-1 bulk stores in flight per SM
constexpr int kSlabSmem = (kKeyCap + 8 + kKeyCap + kSlabBufs * kSlabCells + 3 * kSubSlabs) * 4;

__global__ void lat_keys_hist_kernel(const void* __restrict__ xyz, int dtype, long long n, long long a,
                                     long long side, unsigned* __restrict__ keys,
                                     unsigned long long* __restrict__ bad, unsigned* __restrict__ ghist,
                                     int nbuckets) {
    extern __shared__ unsigned h_s[];
    for (int b = threadIdx.x; b < nbuckets; b += blockDim.x) h_s[b] = 0u;
    __syncthreads();
    long long i_scalar = 0;
    if (dtype == PC_I32 && (reinterpret_cast<uintptr_t>(xyz) & 15) == 0 &&
        (reinterpret_cast<uintptr_t>(keys) & 15) == 0) {
        // four beads (48 B of int32 coordinates) per thread: three 16-byte loads, one 16-byte key store
        const int4* src = reinterpret_cast<const int4*>(xyz);
        const long long groups = n / 4;
        for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < groups;
             g += (long long)gridDim.x * blockDim.x) {
            const int4 p0 = src[3 * g], p1 = src[3 * g + 1], p2 = src[3 * g + 2];
            const int c[12] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w, p2.x, p2.y, p2.z, p2.w};
            unsigned kk[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const long long x = c[3 * u], y = c[3 * u + 1], z = c[3 * u + 2];
                if (x < -a || x > a || y < -a || y > a || z < -a || z > a) {
                    atomicMin(bad, (unsigned long long)(4 * g + u));
                    kk[u] = 0u;
                } else {
                    kk[u] = (unsigned)(((x + a + 1) * side + (y + a + 1)) * side + (z + a + 1));
                    atomicAdd(&h_s[kk[u] >> kBucketShift], 1u);
                }
            }
            reinterpret_cast<uint4*>(keys)[g] = make_uint4(kk[0], kk[1], kk[2], kk[3]);
        }
        i_scalar = groups * 4;
    }
    for (long long i = i_scalar + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
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

// ---- two-level partition of the keys by bucket (coarse = key >> 24, then the
// 128 fine buckets inside each coarse one).  Order inside a bucket is
// irrelevant (a histogram does not care), so each tile is sorted locally in
// shared memory with warp-aggregated ranks and then written out as contiguous
// per-bucket runs.  (A one-pass partition into ~8K buckets stored every key
// separately and was bound by L2 store transactions: 0.7 ms for 2^26 keys.)
constexpr int kCoarseShift = 24;
constexpr int kFinePerCoarse = 1 << (kCoarseShift - kBucketShift);  // 128
constexpr int kPartThreads = 512;
constexpr int kPartPer = 8;                          // keys per thread per tile
constexpr int kPartTile = kPartThreads * kPartPer;   // 4096 keys
constexpr int kMaxCoarse = kMaxBuckets / kFinePerCoarse;

// coarse cursors/bases and the per-coarse-bucket tile table for the fine pass
__global__ void lat_coarse_kernel(const unsigned* __restrict__ base, int nbuckets, int ncoarse,
                                  unsigned* __restrict__ ccur, unsigned* __restrict__ cbase,
                                  unsigned* __restrict__ tbase) {
    if (threadIdx.x != 0) return;
    unsigned tiles = 0;
    for (int c = 0; c < ncoarse; ++c) {
        const unsigned lo = base[min(c * kFinePerCoarse, nbuckets)];
        const unsigned hi = base[min((c + 1) * kFinePerCoarse, nbuckets)];
        cbase[c] = lo;
        ccur[c] = lo;
        tbase[c] = tiles;
        tiles += (hi - lo + kPartTile - 1) / kPartTile;
    }
    cbase[ncoarse] = base[nbuckets];
    tbase[ncoarse] = tiles;
}

// Stage keys [t0, t1) of `in` into shared `dst` at index p - (t0 & ~3): a
// 16-byte cp.async per aligned quad, 4-byte ones for the ragged head and
// tail (fine-pass tiles start anywhere; the last tile may end anywhere).
// One commit group per call.
constexpr int kStage = kPartTile + 8;  // staged keys per buffer (tile + alignment slack)
__device__ __forceinline__ void stage_keys(const unsigned* __restrict__ in, long long t0, long long t1,
                                           unsigned* dst) {
    // 32-bit offsets from the aligned base a0 (a tile spans <= kPartTile keys)
    const unsigned* src = in + (t0 & ~3LL);
    const int h0 = (int)(t0 & 3), e = (int)(t1 - (t0 & ~3LL));  // keys live at [h0, e)
    const int b0 = (h0 + 3) & ~3, b1 = e & ~3;                    // 16-byte body [b0, b1)
    const int tid = threadIdx.x;
    if (b0 >= b1) {
        for (int p = h0 + tid; p < e; p += blockDim.x) cp_async4(&dst[p], &src[p]);
    } else {
        if (h0 + tid < b0) cp_async4(&dst[h0 + tid], &src[h0 + tid]);
        for (int q = b0 + 4 * tid; q < b1; q += 4 * blockDim.x) cp_async16(&dst[q], &src[q]);
        if (b1 + tid < e) cp_async4(&dst[b1 + tid], &src[b1 + tid]);
    }
    cp_async_commit();
}

// Sort one staged tile (kin[0 .. cnt)) by digit(key) on chip and append each
// digit's run at cursor[cur_base + digit] of `out`.
template <typename DigitFn>
__device__ void partition_tile(const unsigned* kin, int cnt, unsigned* __restrict__ cursor, int cur_base, int ndig,
                               DigitFn digit, unsigned* __restrict__ out, unsigned* buf, unsigned* h,
                               unsigned* lofs, unsigned* goff) {
    const int lane = threadIdx.x & 31;
    for (int d = threadIdx.x; d < ndig; d += blockDim.x) h[d] = 0u;
    __syncthreads();
    unsigned k[kPartPer], rank[kPartPer];
#pragma unroll
    for (int u = 0; u < kPartPer; ++u) {
        const int p = u * kPartThreads + threadIdx.x;
        k[u] = p < cnt ? kin[p] : 0xffffffffu;
    }
#pragma unroll
    for (int u = 0; u < kPartPer; ++u) rank[u] = k[u] != 0xffffffffu ? atomicAdd(&h[digit(k[u])], 1u) : 0u;
    __syncthreads();
    // block-wide exclusive scan of h (ndig <= kPartThreads) and parallel run reservations
    __shared__ unsigned s_wsum[kPartThreads / 32];
    const int d = threadIdx.x;
    const unsigned v = d < ndig ? h[d] : 0u;
    unsigned x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[threadIdx.x >> 5] = x;
    __syncthreads();
    unsigned before = 0;
    for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) before += s_wsum[w];
    if (d < ndig) {
        const unsigned lo = before + x - v;
        lofs[d] = lo;
        goff[d] = (v ? atomicAdd(&cursor[cur_base + d], v) : 0u) - lo;  // out index = goff[d] + tile position
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kPartPer; ++u)
        if (k[u] != 0xffffffffu) buf[lofs[digit(k[u])] + rank[u]] = k[u];
    __syncthreads();
    for (int p = threadIdx.x; p < cnt; p += blockDim.x) {
        const unsigned key = buf[p];
        out[goff[digit(key)] + p] = key;
    }
    __syncthreads();
}

// Both passes walk their tiles with the next tile's keys in flight (cp.async
// double buffer in dynamic shared memory): the partition itself is a chain of
// barriers, so without the prefetch every tile paid a full DRAM round trip.
constexpr int kPartSmem = 2 * kStage * 4;

__global__ void __launch_bounds__(kPartThreads, 2) lat_partition_coarse_kernel(
    const unsigned* __restrict__ keys, long long n, unsigned* __restrict__ ccur, int ncoarse,
    unsigned* __restrict__ out, const unsigned long long* __restrict__ bad) {
    if (*bad != kNoBad) return;
    extern __shared__ __align__(16) unsigned part_in[];  // [2][kStage]
    __shared__ unsigned buf[kPartTile];
    __shared__ unsigned h[kMaxCoarse], lofs[kMaxCoarse], goff[kMaxCoarse];
    const long long stride = (long long)gridDim.x * kPartTile;
    long long t0 = (long long)blockIdx.x * kPartTile;
    if (t0 < n) stage_keys(keys, t0, min(t0 + kPartTile, n), part_in);
    for (int cur = 0; t0 < n; t0 += stride, cur ^= 1) {
        const long long nx = t0 + stride;
        if (nx < n) {
            stage_keys(keys, nx, min(nx + kPartTile, n), part_in + (cur ^ 1) * kStage);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        partition_tile(part_in + cur * kStage, (int)(min(t0 + kPartTile, n) - t0), ccur, 0, ncoarse,
                       [](unsigned key) { return key >> kCoarseShift; }, out, buf, h, lofs, goff);
    }
}

__global__ void __launch_bounds__(kPartThreads, 2) lat_partition_fine_kernel(
    const unsigned* __restrict__ tmp, const unsigned* __restrict__ cbase, const unsigned* __restrict__ tbase,
    int ncoarse, unsigned* __restrict__ fcur, unsigned* __restrict__ out,
    const unsigned long long* __restrict__ bad) {
    if (*bad != kNoBad) return;
    extern __shared__ __align__(16) unsigned part_in[];  // [2][kStage]
    __shared__ unsigned buf[kPartTile];
    __shared__ unsigned h[kFinePerCoarse], lofs[kFinePerCoarse], goff[kFinePerCoarse];
    __shared__ unsigned s_tb[kMaxCoarse + 1], s_cb[kMaxCoarse + 1];
    for (int q = threadIdx.x; q <= ncoarse; q += blockDim.x) {
        s_tb[q] = tbase[q];
        s_cb[q] = cbase[q];
    }
    __syncthreads();
    const unsigned ntiles = s_tb[ncoarse];
    auto tile_of = [&](unsigned g, int& c, long long& t0, long long& t1) {
        while (s_tb[c + 1] <= g) ++c;  // coarse bucket holding tile g (g only grows; c starts at the last one)
        t0 = (long long)s_cb[c] + (long long)(g - s_tb[c]) * kPartTile;
        t1 = t0 + kPartTile < (long long)s_cb[c + 1] ? t0 + kPartTile : (long long)s_cb[c + 1];
    };
    unsigned g = blockIdx.x;
    int c = 0;
    long long t0 = 0, t1 = 0;
    if (g < ntiles) {
        tile_of(g, c, t0, t1);
        stage_keys(tmp, t0, t1, part_in);
    }
    for (int cur = 0; g < ntiles; g += gridDim.x, cur ^= 1) {
        const unsigned gn = g + gridDim.x;
        int cn = c;
        long long n0 = 0, n1 = 0;
        if (gn < ntiles) {
            tile_of(gn, cn, n0, n1);
            stage_keys(tmp, n0, n1, part_in + (cur ^ 1) * kStage);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        partition_tile(part_in + cur * kStage + (t0 & 3), (int)(t1 - t0), fcur, c * kFinePerCoarse, kFinePerCoarse,
                       [](unsigned key) { return (key >> kBucketShift) & (kFinePerCoarse - 1); }, out, buf, h,
                       lofs, goff);
        c = cn;
        t0 = n0;
        t1 = n1;
    }
}

__device__ __forceinline__ void bulk_store_s2g(void* gdst, const void* ssrc, unsigned bytes) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(ssrc);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(s), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read_le() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
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
    unsigned* cbuf0 = keys_s + kKeyCap;                 // [kSlabBufs][kSlabCells] ring of counting arrays
    unsigned* sub_n = cbuf0 + kSlabBufs * kSlabCells;   // [kSubSlabs] keys per slab
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
            // the bulk store issued kSlabBufs slabs ago read this buffer: wait for it
            if (threadIdx.x == 0) bulk_wait_read_le<kSlabBufs - 1>();
            __syncthreads();
            uint4* cnt4 = reinterpret_cast<uint4*>(cnt);
            for (int q = threadIdx.x; q < kSlabCells / 4; q += blockDim.x) cnt4[q] = make_uint4(0u, 0u, 0u, 0u);
            __syncthreads();
            const unsigned s0 = sub_start[s], s1 = s0 + sub_n[s];
            for (unsigned i = s0 + threadIdx.x; i < s1; i += blockDim.x) {
                PC_CHECK((unsigned long long)keys[i] >> kSlabShift == cell0 >> kSlabShift);  // key in this slab
                const unsigned old = atomicAdd(&cnt[keys[i] & (kSlabCells - 1)], 1u);  // Alg. 1
                acc += old;
                first += old == 0u;
                ovf |= old >= 0xfffffffeu;
            }
            (void)keys_on_chip;
            fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the bulk copy
            __syncthreads();
            const unsigned vec_bytes = (ncell * 4u) & ~15u;
            PC_CHECK(cell0 + vec_bytes / 4 <= cells);
            if (threadIdx.x == 0 && vec_bytes) bulk_store_s2g(grid + cell0, cnt, vec_bytes);
            for (unsigned q = vec_bytes / 4 + threadIdx.x; q < ncell; q += blockDim.x) {
                PC_CHECK(cell0 + q < cells);
                grid[cell0 + q] = cnt[q];
            }
            flip = flip + 1 == kSlabBufs ? 0 : flip + 1;
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
