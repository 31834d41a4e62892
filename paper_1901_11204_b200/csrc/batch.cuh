// Batched many-small-vector paths (the paper's 100-1000 vectors per execution)
// and their host-side gather helpers.  Included by paircount.cu inside an
// anonymous namespace.

// One lat_batch_kernel launch over device beads + host offsets; fills results.
// Caller holds the device arena lock; `base` is arena memory past the beads.
int lat_batch_run(const void* dxyz, int32_t dtype, const int64_t* offsets, int32_t nvec, int64_t half_extent,
                  char* base, pc_lattice_result* results, cudaStream_t s) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    const size_t obytes = align_up((size_t)(nvec + 1) * 8, 256);
    long long* doffs = (long long*)base;
    unsigned long long* dout = (unsigned long long*)(base + obytes);
    CK(cudaMemcpyAsync(doffs, offsets, (size_t)(nvec + 1) * 8, cudaMemcpyHostToDevice, s));
    static thread_local bool attr_set[64] = {false};
    if (!attr_set[dev & 63]) {
        CK(cudaFuncSetAttribute(lat_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kBatchSmem));
        attr_set[dev & 63] = true;
    }
    const int grid = std::min(nvec, 2 * num_sms());
    lat_batch_kernel<<<grid, 256, kBatchSmem, s>>>(dxyz, dtype, doffs, nvec, half_extent, 2 * half_extent + 3, dout);
    CK_LAUNCH("lat_batch_kernel");
    std::vector<unsigned long long> host((size_t)nvec * 3);
    CK(cudaMemcpyAsync(host.data(), dout, host.size() * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int v = 0; v < nvec; ++v) {
        pc_lattice_result& r = results[v];
        memset(&r, 0, sizeof r);
        r.beads_processed = offsets[v + 1] - offsets[v];
        const unsigned long long st = host[3 * v + 2];
        if (st == ~1ull) {
            r.error = PC_ERR_ARG;  // longer than the on-chip table: caller counts it through a grid
        } else if (st != ~0ull) {
            r.error = PC_ERR_RANGE;
            r.detail = (long long)st;
        } else {
            r.count = (long long)host[3 * v];
            r.cells_touched = (long long)host[3 * v + 1];
        }
    }
    return PC_OK;
}

size_t batch_tail_bytes(int32_t nvec) {
    return align_up((size_t)(nvec + 1) * 8, 256) + align_up((size_t)nvec * 24, 256);
}

// Gather vectors [v0, v1) into dst as int32, mapping any coordinate outside
// [-a, a] to INT32_MAX (itself outside [-a, a], so the kernel still reports
// the first bad bead of that vector -- narrowing can never wrap a bad bead
// into range).
void gather_narrow(const void* const* vecs, const int64_t* offs, int32_t dtype, int64_t a, int v0, int v1,
                   int32_t* dst) {
    for (int v = v0; v < v1; ++v) {
        const long long m = 3 * (offs[v + 1] - offs[v]);
        int32_t* d = dst + 3 * offs[v];
        if (dtype == PC_I32) {
            memcpy(d, vecs[v], (size_t)m * 4);
        } else {
            const long long* src = (const long long*)vecs[v];
            for (long long k = 0; k < m; ++k) {
                const long long x = src[k];
                d[k] = (x < -a || x > a) ? INT32_MAX : (int32_t)x;
            }
        }
    }
}

// Run fn(v0, v1) over contiguous vector groups of ~equal point counts on up
// to 16 host threads (one thread below ~1 MB of data).
template <typename Fn>
void split_vectors(int nvec, const int64_t* offs, size_t total_bytes, Fn fn) {
    const long long n = offs[nvec];
    const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
    const int nt = (int)std::min<long long>(std::min(hw, 16), std::max(1LL, (long long)(total_bytes >> 20)));
    std::vector<std::thread> pool;
    int v0 = 0;
    for (int t = 0; t < nt; ++t) {
        const long long goal = n * (t + 1) / nt;
        int v1 = v0;
        while (v1 < nvec && (t == nt - 1 || offs[v1] < goal)) ++v1;
        if (t == nt - 1) v1 = nvec;
        if (v1 > v0) {
            if (t == nt - 1) fn(v0, v1);
            else pool.emplace_back(fn, v0, v1);
        }
        v0 = v1;
    }
    for (auto& th : pool) th.join();
}

// ---- batched all-pairs over many small vectors (the quadratic side of the
// reference's linear-vs-quadratic harness, bench_cli.py:129-179): one CTA per
// vector, the vector staged in shared memory (int64 or float64), every
// unordered pair once under the balanced ownership (each row ~n/2 partners,
// so the CTA's threads stay balanced), the reference predicate evaluated
// exactly in the reference's arithmetic.
constexpr int kPairsBatchMax = 4096;                   // points per on-chip vector
constexpr int kPairsBatchSmem = kPairsBatchMax * 3 * 8;  // 96 KB

__global__ void __launch_bounds__(256) pairs_batch_kernel(const void* __restrict__ xyz, int dtype,
                                                          const long long* __restrict__ offs, int nvec, int pred,
                                                          int want_sum, unsigned long long* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char pb_smem[];
    long long* si = reinterpret_cast<long long*>(pb_smem);
    double* sd = reinterpret_cast<double*>(pb_smem);
    __shared__ unsigned long long s_cnt[8];
    __shared__ double s_sum[8];
    __shared__ int s_bad;
    const bool is_int = pred != kPredSphere;
    for (int v = blockIdx.x; v < nvec; v += gridDim.x) {
        const long long lo = offs[v];
        const int n = (int)(offs[v + 1] - lo);
        if (n > kPairsBatchMax) {
            if (threadIdx.x == 0) out[3 * v + 2] = ~1ull;  // caller runs it through pc_pairs_host
            continue;
        }
        if (threadIdx.x == 0) s_bad = 0;
        __syncthreads();  // smem free (previous vector done) and s_bad reset
        for (int q = threadIdx.x; q < 3 * n; q += blockDim.x) {
            if (is_int) {
                si[q] = coord_i64(xyz, dtype, lo + q / 3, q % 3);
            } else {
                const double c = coord_f64(xyz, dtype, lo + q / 3, q % 3);
                sd[q] = c;
                if (!isfinite(c)) s_bad = 1;
            }
        }
        __syncthreads();
        unsigned long long cnt = 0;
        double sum = 0.0;
        if (!s_bad) {
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                const int m = n >= 2 ? steps_for_dev(n, i) : 0;
                if (is_int) {
                    const long long ax = si[3 * i], ay = si[3 * i + 1], az = si[3 * i + 2];
                    for (int s = 1, j = i + 1; s <= m; ++s, ++j) {
                        if (j == n) j = 0;
                        // numpy int64 wrap-around differences (lattice_counter.py:238-255)
                        const long long dx = (long long)((unsigned long long)ax - (unsigned long long)si[3 * j]);
                        const long long dy = (long long)((unsigned long long)ay - (unsigned long long)si[3 * j + 1]);
                        const long long dz = (long long)((unsigned long long)az - (unsigned long long)si[3 * j + 2]);
                        if (pred == kPredCoincide) {
                            cnt += (dx == 0 && dy == 0 && dz == 0) ? 1ull : 0ull;
                        } else {
                            const unsigned long long man = (unsigned long long)(dx < 0 ? -dx : dx) +
                                                           (unsigned long long)(dy < 0 ? -dy : dy) +
                                                           (unsigned long long)(dz < 0 ? -dz : dz);
                            cnt += man == 1ull ? 1ull : 0ull;
                        }
                    }
                } else {
                    const double ax = sd[3 * i], ay = sd[3 * i + 1], az = sd[3 * i + 2];
                    for (int s = 1, j = i + 1; s <= m; ++s, ++j) {
                        if (j == n) j = 0;
                        // collision_indicator's float64 arithmetic (spi_engine.py:68-73)
                        const double dx = __dsub_rn(ax, sd[3 * j]), dy = __dsub_rn(ay, sd[3 * j + 1]),
                                     dz = __dsub_rn(az, sd[3 * j + 2]);
                        const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
                        cnt += d2 < 1.0 ? 1ull : 0ull;
                        if (want_sum) sum += 1.0 / (1.0 + d2);
                    }
                }
            }
        }
        cnt = warp_sum(cnt);
        sum = warp_sum(sum);
        if ((threadIdx.x & 31) == 0) {
            s_cnt[threadIdx.x >> 5] = cnt;
            s_sum[threadIdx.x >> 5] = sum;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long c = 0;
            double t = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
                c += s_cnt[w];
                t += s_sum[w];
            }
            out[3 * v] = c;
            out[3 * v + 1] = (unsigned long long)__double_as_longlong(t);
            out[3 * v + 2] = s_bad ? 1ull : 0ull;
        }
    }
}
