// Counting array (Alg. 1 / Alg. 2): lattice kernels and the host driver.
// Included by paircount.cu inside its anonymous namespace.

// ------------------------------------------------------------------------
// counting array (Alg. 1 / Alg. 2)
// ------------------------------------------------------------------------
struct LatSlot {
    unsigned long long a, b;
};
constexpr unsigned long long kNoBad = ~0ull;

template <typename KT>
__global__ void lat_keys_kernel(const void* __restrict__ xyz, int dtype, long long n, long long a, long long side,
                                KT* __restrict__ keys, unsigned long long* __restrict__ bad) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long x = coord_i64(xyz, dtype, i, 0), y = coord_i64(xyz, dtype, i, 1),
                        z = coord_i64(xyz, dtype, i, 2);
        if (x < -a || x > a || y < -a || y > a || z < -a || z > a) {  // _validate, lattice_counter.py:98-105
            atomicMin(bad, (unsigned long long)i);
        } else if (keys) {
            keys[i] = (KT)(((x + a + 1) * side + (y + a + 1)) * side + (z + a + 1));  // _flatten, :107-111
        }
    }
}

// Alg. 1 on a clean grid: collisions += space[b]; space[b]++  
template <typename KT>
__global__ void lat_place_clean_kernel(const KT* __restrict__ keys, long long n, unsigned* __restrict__ grid,
                                       const unsigned long long* __restrict__ bad, LatSlot* __restrict__ slots,
                                       int* __restrict__ overflow) {
    __shared__ unsigned long long s_a[8], s_b[8];
    unsigned long long cnt = 0, first = 0;
    int ovf = 0;
    if (*bad == kNoBad) {
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
             i += (long long)gridDim.x * blockDim.x) {
            const unsigned old = atomicAdd(grid + keys[i], 1u);
            cnt += old;
            first += old == 0u;
            ovf |= old >= 0xfffffffeu;
        }
    }
    cnt = warp_sum(cnt);
    first = warp_sum(first);
    if (__any_sync(0xffffffffu, ovf) && (threadIdx.x & 31) == 0) atomicOr(overflow, 1);
    if ((threadIdx.x & 31) == 0) { s_a[threadIdx.x >> 5] = cnt; s_b[threadIdx.x >> 5] = first; }
    __syncthreads();
    if (threadIdx.x == 0) {
        LatSlot sl{0, 0};
        for (int q = 0; q < (int)(blockDim.x >> 5); ++q) { sl.a += s_a[q]; sl.b += s_b[q]; }
        slots[blockIdx.x] = sl;
    }
}

template <typename KT>
__global__ void lat_place_kernel(const KT* __restrict__ keys, long long n, unsigned* __restrict__ grid,
                                 const unsigned long long* __restrict__ bad) {
    if (*bad != kNoBad) return;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        atomicAdd(grid + keys[i], 1u);
}

// sum over beads of (final occupancy - 1) (lattice_counter.py:151-153); b = overflow flag
template <typename KT>
__global__ void lat_gather_kernel(const KT* __restrict__ keys, long long n, const unsigned* __restrict__ grid,
                                  const unsigned long long* __restrict__ bad, LatSlot* __restrict__ slots,
                                  int* __restrict__ overflow) {
    __shared__ unsigned long long s_a[8];
    unsigned long long acc = 0;
    int ovf = 0;
    if (*bad == kNoBad) {
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
             i += (long long)gridDim.x * blockDim.x) {
            const unsigned occ = grid[keys[i]];
            acc += (unsigned long long)occ - 1ull;
            ovf |= occ >= 0xffffffffu;
        }
    }
    acc = warp_sum(acc);
    if (__any_sync(0xffffffffu, ovf) && (threadIdx.x & 31) == 0) atomicOr(overflow, 1);
    if ((threadIdx.x & 31) == 0) s_a[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        LatSlot sl{0, 0};
        for (int q = 0; q < (int)(blockDim.x >> 5); ++q) sl.a += s_a[q];
        slots[blockIdx.x] = sl;
    }
}

// Alg. 2 second loop: six axial neighbour occupancies per bead
template <typename KT>
__global__ void lat_neighbours_kernel(const KT* __restrict__ keys, long long n, long long side,
                                      const unsigned* __restrict__ grid, const unsigned long long* __restrict__ bad,
                                      LatSlot* __restrict__ slots) {
    __shared__ unsigned long long s_a[8];
    unsigned long long acc = 0;
    if (*bad == kNoBad) {
        const long long d2 = side * side;
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
             i += (long long)gridDim.x * blockDim.x) {
            const long long k = (long long)keys[i];
            acc += (unsigned long long)grid[k + d2] + grid[k - d2] + grid[k + side] + grid[k - side] +
                   grid[k + 1] + grid[k - 1];
        }
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) s_a[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        LatSlot sl{0, 0};
        for (int q = 0; q < (int)(blockDim.x >> 5); ++q) sl.a += s_a[q];
        slots[blockIdx.x] = sl;
    }
}

// Distinct-cell count by marking bit 31 of every read cell (own cell, and the
// six neighbours when `with_neighbours`), counting first markers; a second
// call with unmark=1 clears the marks.  Occupancies never reach 2^31 here
// (overflow is reported first).
template <typename KT>
__global__ void lat_mark_kernel(const KT* __restrict__ keys, long long n, long long side, int with_neighbours,
                                int unmark, unsigned* __restrict__ grid, const unsigned long long* __restrict__ bad,
                                LatSlot* __restrict__ slots) {
    __shared__ unsigned long long s_a[8];
    unsigned long long firsts = 0;
    if (*bad == kNoBad) {
        const long long d2 = side * side;
        const long long offs[7] = {0, d2, -d2, side, -side, 1, -1};
        const int m = with_neighbours ? 7 : 1;
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
             i += (long long)gridDim.x * blockDim.x) {
            const long long k = (long long)keys[i];
            for (int q = 0; q < m; ++q) {
                if (unmark) atomicAnd(grid + k + offs[q], 0x7fffffffu);
                else firsts += (atomicOr(grid + k + offs[q], 0x80000000u) & 0x80000000u) ? 0ull : 1ull;
            }
        }
    }
    firsts = warp_sum(firsts);
    if ((threadIdx.x & 31) == 0) s_a[threadIdx.x >> 5] = firsts;
    __syncthreads();
    if (threadIdx.x == 0) {
        LatSlot sl{0, 0};
        for (int q = 0; q < (int)(blockDim.x >> 5); ++q) sl.a += s_a[q];
        slots[blockIdx.x] = sl;
    }
}

template <typename KT>
__global__ void lat_zero_keys_kernel(const KT* __restrict__ keys, long long n, unsigned* __restrict__ grid) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        grid[keys[i]] = 0u;
}

__global__ void lat_zero_beads_kernel(const void* __restrict__ xyz, int dtype, long long n, long long a, long long side,
                                      unsigned* __restrict__ grid, const unsigned long long* __restrict__ bad) {
    if (*bad != kNoBad) return;
    const long long d2 = side * side;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long k = ((coord_i64(xyz, dtype, i, 0) + a + 1) * side + (coord_i64(xyz, dtype, i, 1) + a + 1)) * side +
                            (coord_i64(xyz, dtype, i, 2) + a + 1);
        grid[k] = 0u; grid[k + d2] = 0u; grid[k - d2] = 0u; grid[k + side] = 0u;
        grid[k - side] = 0u; grid[k + 1] = 0u; grid[k - 1] = 0u;
    }
}

__global__ void lat_sum_slots_kernel(const LatSlot* __restrict__ slots, int nslots, unsigned long long* __restrict__ out) {
    __shared__ unsigned long long sa[256], sb[256];
    unsigned long long x = 0, y = 0;
    for (int q = threadIdx.x; q < nslots; q += blockDim.x) { x += slots[q].a; y += slots[q].b; }
    sa[threadIdx.x] = x; sb[threadIdx.x] = y;
    __syncthreads();
    for (int h = blockDim.x / 2; h > 0; h >>= 1) {
        if (threadIdx.x < h) { sa[threadIdx.x] += sa[threadIdx.x + h]; sb[threadIdx.x] += sb[threadIdx.x + h]; }
        __syncthreads();
    }
    if (threadIdx.x == 0) { out[0] = sa[0]; out[1] = sb[0]; }
}

__global__ void count_nonzero_kernel(const uint4* __restrict__ grid4, long long n4, const unsigned* __restrict__ tail,
                                     int ntail, unsigned long long* __restrict__ out) {
    unsigned long long c = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
        const uint4 v = grid4[i];
        c += (v.x != 0u) + (v.y != 0u) + (v.z != 0u) + (v.w != 0u);
    }
    if (blockIdx.x == 0 && (int)threadIdx.x < ntail) c += tail[threadIdx.x] != 0u;
    c = warp_sum(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// Scratch layout for one lattice call: [coords copy][bad u64][overflow int][slots][sums]
#include "lattice_slab.cuh"

// ---- batched small vectors (the paper's 100-1000 vectors per execution) ----
// One CTA per vector; Alg. 1 (collisions += space[b]; space[b]++) on a
// shared-memory counting array addressed by an open-addressing hash of the
// cell key (the dense (2a+3)^3 grid does not fit on chip).  Equivalent to
// count_collisions + reset_sparse per vector on a clean space.
constexpr int kBatchSlots = 8192;  // vectors up to kBatchSlots/2 beads; larger ones go through the grid
constexpr unsigned long long kEmptyKey = ~0ull;
constexpr int kBatchSmem = kBatchSlots * 12;

__global__ void __launch_bounds__(256) lat_batch_kernel(const void* __restrict__ xyz, int dtype,
                                                        const long long* __restrict__ offs, int nvec, long long a,
                                                        long long side, unsigned long long* __restrict__ out) {
    extern __shared__ unsigned long long tkey[];  // [kBatchSlots] keys, then [kBatchSlots] uint32 counts
    unsigned* tcnt = reinterpret_cast<unsigned*>(tkey + kBatchSlots);
    __shared__ unsigned long long s_acc[8], s_first[8];
    __shared__ long long s_bad;
    for (int v = blockIdx.x; v < nvec; v += gridDim.x) {
        const long long lo = offs[v], hi = offs[v + 1];
        for (int q = threadIdx.x; q < kBatchSlots; q += blockDim.x) {
            tkey[q] = kEmptyKey;
            tcnt[q] = 0u;
        }
        if (threadIdx.x == 0) s_bad = -1;
        __syncthreads();
        unsigned long long acc = 0, first = 0;
        if (hi - lo <= kBatchSlots / 2) {
            for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
                const long long x = coord_i64(xyz, dtype, i, 0), y = coord_i64(xyz, dtype, i, 1),
                                z = coord_i64(xyz, dtype, i, 2);
                if (x < -a || x > a || y < -a || y > a || z < -a || z > a) {
                    atomicMin((unsigned long long*)&s_bad, (unsigned long long)(i - lo));
                    continue;
                }
                const unsigned long long key = (unsigned long long)(((x + a + 1) * side + (y + a + 1)) * side + (z + a + 1));
                unsigned h = (unsigned)((key * 0x9E3779B97F4A7C15ull) >> 51) & (kBatchSlots - 1);
                for (;;) {
                    const unsigned long long prev = atomicCAS(&tkey[h], kEmptyKey, key);
                    if (prev == kEmptyKey || prev == key) {
                        const unsigned old = atomicAdd(&tcnt[h], 1u);  // Alg. 1
                        acc += old;
                        first += old == 0u;
                        break;
                    }
                    h = (h + 1) & (kBatchSlots - 1);
                }
            }
        }
        acc = warp_sum(acc);
        first = warp_sum(first);
        if ((threadIdx.x & 31) == 0) {
            s_acc[threadIdx.x >> 5] = acc;
            s_first[threadIdx.x >> 5] = first;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long c = 0, f = 0;
            for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
                c += s_acc[q];
                f += s_first[q];
            }
            const bool big = hi - lo > kBatchSlots / 2;
            out[3 * v] = c;
            out[3 * v + 1] = f;
            // first out-of-range bead (vector-relative), ~0 if none, ~1 if the vector was too long
            out[3 * v + 2] = big ? ~1ull : (unsigned long long)s_bad;
        }
        __syncthreads();
    }
}

// Alg. 2 on a populated grid, dense regime (pc_lattice_contacts after the slab
// histogram): contact_accumulator's doubled sum is sum_b sum_k occ(cell(b) + e_k)
// = sum_c occ(c) * sum_k occ(c + e_k), and count_contacts' cells_touched (own
// cell + six neighbours per bead, lattice_counter.py:189-191) is the number of
// cells c with occ(c) > 0 or an occupied axial neighbour -- one 7-point stencil
// pass over the grid instead of 7N scattered reads and mark/unmark atomics.
// Interior cells never wrap; a padding cell's wrapped "neighbour" is padding
// (zero), so the flat +-1 / +-side / +-side^2 offsets are exact.
__global__ void __launch_bounds__(256) lat_stencil_kernel(const unsigned* __restrict__ grid, long long side,
                                                          unsigned long long cells, LatSlot* __restrict__ slots) {
    // four consecutive cells per thread: one 16-byte load for the cells and
    // their +-1 neighbours, scalar loads for the +-side / +-side^2 ones (measured
    // faster than one cell per lane, 3.5 vs 5.4 ms at 1027^3, and than walking
    // x with a register window, where too few loads were in flight)
    const long long d2 = side * side, nc = (long long)cells;
    unsigned long long doubled = 0, touched = 0;
    const long long groups = (nc + 3) / 4;
    for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < groups;
         g += (long long)gridDim.x * blockDim.x) {
        const long long c0 = 4 * g;
        unsigned o[6];  // cells c0-1 .. c0+4
        if (c0 + 4 <= nc) {
            const uint4 v = *reinterpret_cast<const uint4*>(grid + c0);
            o[1] = v.x; o[2] = v.y; o[3] = v.z; o[4] = v.w;
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) o[1 + u] = c0 + u < nc ? grid[c0 + u] : 0u;
        }
        o[0] = c0 > 0 ? grid[c0 - 1] : 0u;
        o[5] = c0 + 4 < nc ? grid[c0 + 4] : 0u;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const long long c = c0 + u;
            if (c >= nc) break;
            unsigned long long nb = (unsigned long long)o[u] + o[u + 2];
            if (c >= side) nb += grid[c - side];
            if (c + side < nc) nb += grid[c + side];
            if (c >= d2) nb += grid[c - d2];
            if (c + d2 < nc) nb += grid[c + d2];
            doubled += (unsigned long long)o[u + 1] * nb;
            touched += (o[u + 1] != 0u || nb != 0ull) ? 1ull : 0ull;
        }
    }
    __shared__ unsigned long long s_d[8], s_t[8];
    doubled = warp_sum(doubled);
    touched = warp_sum(touched);
    if ((threadIdx.x & 31) == 0) {
        s_d[threadIdx.x >> 5] = doubled;
        s_t[threadIdx.x >> 5] = touched;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        LatSlot sl{0ull, 0ull};
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            sl.a += s_d[w];
            sl.b += s_t[w];
        }
        slots[blockIdx.x] = sl;
    }
}

struct LatScratch {
    const void* xyz;
    int dtype;  // of xyz as staged (host int64 beads arrive narrowed to int32)
    unsigned long long* bad;
    int* overflow;
    LatSlot* slots;
    unsigned long long* sums;  // 8 pairs of (a, b)
    int nslots;
};

int lattice_blocks(long long n) {
    return (int)std::max(1LL, std::min<long long>((n + 255) / 256, (long long)num_sms() * 8));
}

// ---- host int64 beads: narrowed to int32 by host threads into pinned chunks
// that stream to the device while the next chunks are narrowed.  A plain
// pageable copy of the 1.6 GB config-5 vector runs at ~11 GB/s; this moves half
// the bytes from pinned memory.  Every valid coordinate fits int32; one outside
// [-a, a] becomes INT32_MAX, still outside, so the kernels report the same
// first bad bead (its coordinates are read back from the caller's array).
constexpr size_t kStageChunk = 8u << 20;      // int32 bytes per pinned chunk
constexpr int kStageThreads = 16;
constexpr long long kStageMinBeads = 1 << 19;  // below: one plain copy

struct StagePool {
    void* pinned = nullptr;
    cudaEvent_t ev[2 * kStageThreads] = {};
};
StagePool g_stage[64];  // per device, guarded by the arena lock

int stage_narrow_i64(const long long* src, long long n, long long a, int* dst, cudaStream_t s) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    StagePool& sp = g_stage[dev & 63];
    if (!sp.pinned) {
        CK(cudaHostAlloc(&sp.pinned, 2 * kStageThreads * kStageChunk, cudaHostAllocDefault));
        for (auto& e : sp.ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    for (auto& e : sp.ev) CK(cudaEventSynchronize(e));  // a previous call's copies out of the pool are done
    const long long total = 3 * n, per = (long long)(kStageChunk / 4);
    const long long nchunks = (total + per - 1) / per;
    const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
    const int nt = (int)std::min<long long>(std::min(hw, kStageThreads), nchunks);
    std::atomic<long long> next{0};
    std::atomic<int> failed{0};  // first CUDA error of any worker (cudaError_t)
    auto fail = [&](cudaError_t e) {
        int none = 0;
        failed.compare_exchange_strong(none, (int)e);
    };
    auto work = [&](int t) {
        cudaError_t e = cudaSetDevice(dev);
        if (e != cudaSuccess) return fail(e);
        bool used[2] = {false, false};
        for (int k = 0; !failed; ++k) {
            const long long c = next.fetch_add(1);
            if (c >= nchunks) break;
            const int b = k & 1;
            int* buf = (int*)((char*)sp.pinned + (size_t)(2 * t + b) * kStageChunk);
            cudaEvent_t ev = sp.ev[2 * t + b];
            if (used[b] && (e = cudaEventSynchronize(ev)) != cudaSuccess) return fail(e);
            const long long lo = c * per, hi = std::min(total, lo + per);
            const long long* in = src + lo;
            for (long long q = 0; q < hi - lo; ++q) {
                const long long x = in[q];
                buf[q] = (x < -a || x > a) ? INT32_MAX : (int)x;
            }
            if ((e = cudaMemcpyAsync(dst + lo, buf, (size_t)(hi - lo) * 4, cudaMemcpyHostToDevice, s)) != cudaSuccess ||
                (e = cudaEventRecord(ev, s)) != cudaSuccess)
                return fail(e);
            used[b] = true;
        }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t + 1 < nt; ++t) pool.emplace_back(work, t);
    work(nt - 1);
    for (auto& th : pool) th.join();
    if (failed) return cuda_fail("staging host beads to the device", (cudaError_t)failed.load());
    return PC_OK;
}

int lat_prepare(const void* xyz, int dtype, int on_device, long long n, long long a, Arena** ar_out,
                LatScratch* sc, cudaStream_t* s_inout, size_t extra = 0, char** extra_out = nullptr) {
    if (dtype != PC_I32 && dtype != PC_I64) return arg_fail("lattice beads must be int32 or int64");
    const int nb = lattice_blocks(n);
    const bool narrow = !on_device && dtype == PC_I64 && n >= kStageMinBeads;
    const size_t cbytes = on_device ? 0 : align_up((size_t)n * 3 * (narrow ? 4 : dtype_bytes(dtype)), 256);
    const size_t need = cbytes + 256 + align_up((size_t)nb * sizeof(LatSlot), 256) + 256 + align_up(extra, 256);
    Arena* ar = nullptr;
    int rc = arena_get(need, &ar);
    if (rc) return rc;
    char* base = (char*)ar->dev;
    cudaStream_t s = *s_inout;
    sc->dtype = dtype;
    if (narrow) {
        const int rc = stage_narrow_i64((const long long*)xyz, n, a, (int*)base, s);
        if (rc) return rc;
        sc->xyz = base;
        sc->dtype = PC_I32;
    } else if (!on_device) {
        if (n > 0) CK(cudaMemcpyAsync(base, xyz, (size_t)n * 3 * dtype_bytes(dtype), cudaMemcpyHostToDevice, s));
        sc->xyz = base;
    } else {
        sc->xyz = xyz;
    }
    sc->bad = (unsigned long long*)(base + cbytes);
    sc->overflow = (int*)(base + cbytes + 8);
    sc->slots = (LatSlot*)(base + cbytes + 256);
    sc->sums = (unsigned long long*)(base + cbytes + 256 + align_up((size_t)nb * sizeof(LatSlot), 256));
    sc->nslots = nb;
    if (extra_out) *extra_out = (char*)sc->sums + 256;
    CK(cudaMemsetAsync(sc->bad, 0xff, 8, s));
    CK(cudaMemsetAsync(sc->overflow, 0, 4, s));
    *ar_out = ar;
    return PC_OK;
}

// cells_limit: the grid holds only keys [0, cells_limit) (an x-slab of the cube, see
// pc_lattice_collisions_multi); 0 = the whole (2a+3)^3 cube.
template <typename KT>
int lattice_run(const void* xyz_in, int dtype, int on_device, long long n, long long a, unsigned* grid, void* keys_v,
                int clean, int contacts, pc_lattice_result* res, cudaStream_t s,
                unsigned long long cells_limit = 0) {
    g_launches = 0;
    memset(res, 0, sizeof *res);
    res->beads_processed = n;
    if (n == 0) return PC_OK;
    if (!grid || !keys_v) return arg_fail("grid and keys buffers are required");
    KT* keys = (KT*)keys_v;
    const long long side = 2 * a + 3;
    Arena* ar = nullptr;
    LatScratch sc;
    std::unique_lock<std::mutex> lock;
    {
        int dev = 0;
        CK(cudaGetDevice(&dev));
        lock = std::unique_lock<std::mutex>(g_arena[dev & 63].mu);
    }
    const unsigned long long cells = cells_limit ? cells_limit : (unsigned long long)side * side * side;
    // dense regime on a clean grid: shared-memory slab histogram (lattice_slab.cuh)
    // crossover: n scattered atomics at ~21 G/s vs streaming 4 B/cell + ~40 B/bead at HBM rate -> n > cells/67
    // (contacts too: the slab histogram populates the grid, then one stencil pass)
    // the slab path's bucket tables cover kMaxBuckets << kBucketShift = 2^31 cells
    const bool slab = clean && sizeof(KT) == 4 && (unsigned long long)n * 64 > cells && n < (1LL << 32) - 1 &&
                      cells <= ((unsigned long long)kMaxBuckets << kBucketShift);
    const int nbuckets = slab ? (int)((cells + (1ull << kBucketShift) - 1) >> kBucketShift) : 0;
    const size_t kbytes = align_up((size_t)n * 4 + 64, 256);  // +16 keys: aligned staging windows may overrun
    const size_t abytes = align_up((kMaxBuckets + 1) * 4, 256), cbytes4 = align_up((kMaxCoarse + 1) * 4, 256);
    const size_t extra = slab ? 2 * kbytes + 3 * abytes + 3 * cbytes4 + align_up((size_t)nbuckets * sizeof(LatSlot), 256)
                              : 0;
    char* ex = nullptr;
    int rc = lat_prepare(xyz_in, dtype, on_device, n, a, &ar, &sc, &s, extra, &ex);
    if (rc) return rc;
    const int nb = sc.nslots;
    if (slab) {
        unsigned* sorted = (unsigned*)ex;
        unsigned* scratch = (unsigned*)(ex + kbytes);  // coarse-partitioned keys, then the slab kernel's fallback
        unsigned* hist = (unsigned*)(ex + 2 * kbytes);
        unsigned* base = (unsigned*)((char*)hist + abytes);
        unsigned* cursor = (unsigned*)((char*)base + abytes);
        unsigned* ccur = (unsigned*)((char*)cursor + abytes);
        unsigned* cbase = (unsigned*)((char*)ccur + cbytes4);
        unsigned* tbase = (unsigned*)((char*)cbase + cbytes4);
        LatSlot* bslots = (LatSlot*)((char*)tbase + cbytes4);
        const int ncoarse = (int)(((cells - 1) >> kCoarseShift) + 1);
        static thread_local bool attr_set[64] = {false};
        int dev = 0;
        CK(cudaGetDevice(&dev));
        if (!attr_set[dev & 63]) {
            CK(cudaFuncSetAttribute(lat_slab_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSlabSmem));
            CK(cudaFuncSetAttribute(lat_keys_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kMaxBuckets * 4));
            CK(cudaFuncSetAttribute(lat_partition_coarse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kPartSmem));
            CK(cudaFuncSetAttribute(lat_partition_fine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kPartSmem));
            attr_set[dev & 63] = true;
        }
        CK(cudaMemsetAsync(hist, 0, nbuckets * 4, s));
        lat_keys_hist_kernel<<<2 * num_sms(), 1024, nbuckets * 4, s>>>(sc.xyz, sc.dtype, n, a, side, (unsigned*)keys, sc.bad, hist,
                                                           nbuckets);
        CK_LAUNCH("lat_keys_hist_kernel");
        lat_bucket_scan_kernel<<<1, 1024, 0, s>>>(hist, base, cursor, nbuckets);
        CK_LAUNCH("lat_bucket_scan_kernel");
        lat_coarse_kernel<<<1, 32, 0, s>>>(base, nbuckets, ncoarse, ccur, cbase, tbase);
        CK_LAUNCH("lat_coarse_kernel");
        lat_partition_coarse_kernel<<<num_sms() * 2, kPartThreads, kPartSmem, s>>>((const unsigned*)keys, n, ccur, ncoarse,
                                                                          scratch, sc.bad);
        CK_LAUNCH("lat_partition_coarse_kernel");
        lat_partition_fine_kernel<<<num_sms() * 2, kPartThreads, kPartSmem, s>>>(scratch, cbase, tbase, ncoarse, cursor,
                                                                        sorted, sc.bad);
        CK_LAUNCH("lat_partition_fine_kernel");
        const int sgrid = std::min(num_sms(), nbuckets);
        lat_slab_kernel<<<sgrid, 1024, kSlabSmem, s>>>(sorted, scratch, base, nbuckets, grid, cells, sc.bad, bslots,
                                                       sc.overflow);
        CK_LAUNCH("lat_slab_kernel");
        lat_sum_slots_kernel<<<1, 256, 0, s>>>(bslots, sgrid, sc.sums);
        CK_LAUNCH("lat_sum_slots_kernel");
        if (contacts) {
            lat_stencil_kernel<<<nb, 256, 0, s>>>(grid, side, cells, sc.slots);
            CK_LAUNCH("lat_stencil_kernel");
            lat_sum_slots_kernel<<<1, 256, 0, s>>>(sc.slots, nb, sc.sums + 2);  // sums[2] doubled, [3] touched
            CK_LAUNCH("lat_sum_slots_kernel");
        }
    } else {
        lat_keys_kernel<KT><<<nb, 256, 0, s>>>(sc.xyz, sc.dtype, n, a, side, keys, sc.bad);
        CK_LAUNCH("lat_keys_kernel");
    }
    if (slab) {
        // count / cells_touched are in sums[0], sums[1], as for the atomic path
    } else if (clean && !contacts) {
        lat_place_clean_kernel<KT><<<nb, 256, 0, s>>>(keys, n, grid, sc.bad, sc.slots, sc.overflow);
        CK_LAUNCH("lat_place_clean_kernel");
        lat_sum_slots_kernel<<<1, 256, 0, s>>>(sc.slots, nb, sc.sums);
        CK_LAUNCH("lat_sum_slots_kernel");
    } else {
        lat_place_kernel<KT><<<nb, 256, 0, s>>>(keys, n, grid, sc.bad);
        CK_LAUNCH("lat_place_kernel");
        lat_gather_kernel<KT><<<nb, 256, 0, s>>>(keys, n, grid, sc.bad, sc.slots, sc.overflow);
        CK_LAUNCH("lat_gather_kernel");
        lat_sum_slots_kernel<<<1, 256, 0, s>>>(sc.slots, nb, sc.sums);  // sums[0] = sum(occ - 1)
        CK_LAUNCH("lat_sum_slots_kernel");
        if (contacts) {
            lat_neighbours_kernel<KT><<<nb, 256, 0, s>>>(keys, n, side, grid, sc.bad, sc.slots);
            CK_LAUNCH("lat_neighbours_kernel");
            lat_sum_slots_kernel<<<1, 256, 0, s>>>(sc.slots, nb, sc.sums + 2);  // sums[2] = doubled
            CK_LAUNCH("lat_sum_slots_kernel");
        }
        lat_mark_kernel<KT><<<nb, 256, 0, s>>>(keys, n, side, contacts, 0, grid, sc.bad, sc.slots);
        CK_LAUNCH("lat_mark_kernel");
        lat_sum_slots_kernel<<<1, 256, 0, s>>>(sc.slots, nb, sc.sums + 4);  // sums[4] = distinct cells
        CK_LAUNCH("lat_sum_slots_kernel");
        lat_mark_kernel<KT><<<nb, 256, 0, s>>>(keys, n, side, contacts, 1, grid, sc.bad, sc.slots);
        CK_LAUNCH("lat_mark_kernel");
    }
    unsigned long long host[8] = {0};
    unsigned long long bad = 0;
    int ovf = 0;
    CK(cudaMemcpyAsync(host, sc.sums, sizeof host, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&bad, sc.bad, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&ovf, sc.overflow, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (bad != kNoBad) {
        res->error = PC_ERR_RANGE;
        res->detail = (long long)bad;
        return PC_ERR_RANGE;
    }
    if (ovf) {
        res->error = PC_ERR_OVERFLOW;
        return PC_ERR_OVERFLOW;
    }
    if (clean && !contacts) {
        res->count = (long long)host[0];
        res->cells_touched = (long long)host[1];
    } else if (!contacts) {
        res->count = (long long)(host[0] / 2);
        res->cells_touched = (long long)host[4];
    } else {
        res->doubled = (long long)host[2];
        res->count = res->doubled / 2;
        res->cells_touched = (long long)(slab ? host[3] : host[4]);
        if (res->doubled & 1) {
            res->error = PC_ERR_ODD;
            return PC_ERR_ODD;
        }
    }
    return PC_OK;
}


// ---- multi-GPU counting array (x-slab split; pc_lattice_collisions_multi) ----
// Validate every bead (first bad index, as lat_keys_kernel) and append the beads
// with x in [xlo, xhi) to `out` as int32 (x - xlo - a, y, z): in a cube of the
// same half-extent those land on planes 1 .. xhi-xlo, so the keys of the slab's
// (xhi-xlo+2) x side x side grid are the cube formula unchanged.  Order is
// irrelevant to a histogram, so slots come from one warp-aggregated atomic.
__global__ void lat_compact_slab_kernel(const void* __restrict__ xyz, int dtype, long long n, long long a,
                                        long long xlo, long long xhi, int* __restrict__ out,
                                        unsigned long long* __restrict__ count, unsigned long long* __restrict__ bad) {
    const int lane = threadIdx.x & 31;
    for (long long base = (long long)blockIdx.x * blockDim.x; base < n; base += (long long)gridDim.x * blockDim.x) {
        const long long i = base + threadIdx.x;
        bool keep = false;
        long long x = 0, y = 0, z = 0;
        if (i < n) {
            x = coord_i64(xyz, dtype, i, 0);
            y = coord_i64(xyz, dtype, i, 1);
            z = coord_i64(xyz, dtype, i, 2);
            if (x < -a || x > a || y < -a || y > a || z < -a || z > a) atomicMin(bad, (unsigned long long)i);
            else keep = x >= xlo && x < xhi;
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        unsigned long long pos = 0;
        if (lane == 0 && m) pos = atomicAdd(count, (unsigned long long)__popc(m));
        pos = __shfl_sync(0xffffffffu, pos, 0) + __popc(m & ((1u << lane) - 1u));
        if (keep) {
            out[3 * pos] = (int)(x - xlo - a);
            out[3 * pos + 1] = (int)y;
            out[3 * pos + 2] = (int)z;
        }
    }
}

// Per-device state of pc_lattice_collisions_multi: input copy, compacted beads,
// keys and the slab grid (kept all-zero between calls), guarded by its own lock
// (lattice_run takes the arena lock).
struct MultiLat {
    std::mutex mu;
    void* buf = nullptr;
    size_t cap = 0;
    unsigned* grid = nullptr;
    unsigned long long grid_cells = 0;
    cudaStream_t stream = nullptr;
};
MultiLat g_multilat[64];
