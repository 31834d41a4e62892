// The paper's own GPU schemes, literally: one CUDA thread per
// outer row in blocks of 1024 rows, partner columns streamed through shared memory
// tiles shared by the block ("all optimizations applied to both approaches alike").
// With the standard schedule (Alg. 3) block b walks every column after its first row
// -- blocks carry unequal work and, in the block's diagonal tile, threads of a warp
// own different numbers of columns (the two imbalances PAPER.md:417-418 names); with
// the balanced schedule (Alg. 4) every thread owns steps_for(n, i) partners.  Same
// scalar FP32 inner code for both, so naive / balanced measures the schedule, not the
// arithmetic.  A baseline (PC_TILE_THREAD_ROW), not the product path: the warp-tiled
// packed kernels of pairs_kernel.cuh run the same schedules 4-5x faster.
// Included by paircount.cu inside its anonymous namespace; fp32 input only.

constexpr int kRowThreads = 1024;
constexpr int kRowTile = 1024;  // columns per shared-memory tile

__global__ void __launch_bounds__(kRowThreads, 1) pairs_row_kernel(const PairsArgs a, int direct) {
    __shared__ float4 s_col[kRowTile];
    __shared__ unsigned long long s_c[kRowThreads / 32], s_k[kRowThreads / 32];
    __shared__ double s_s[kRowThreads / 32];
    if (direct && f64_takes(*a.st, a.dtype, false)) {  // pairs_f64_kernel takes this call
        if (threadIdx.x == 0) a.slots[blockIdx.x] = Slot{};
        return;
    }
    const float* xyz = (const float*)a.xyz;
    const int n = a.n;
    const bool bal = a.sched == PC_BALANCED;
    const long long i = (long long)a.lo + (long long)blockIdx.x * kRowThreads + threadIdx.x;
    const bool row_ok = i < a.hi;
    const float xi = row_ok ? xyz[3 * i] : 0.f, yi = row_ok ? xyz[3 * i + 1] : 0.f, zi = row_ok ? xyz[3 * i + 2] : 0.f;
    const int lim = row_ok ? (bal ? steps_for_dev(n, (int)i) : n - 1 - (int)i) : 0;  // partners i + 1 .. i + lim
    // the block's column span: offsets s = 1 .. smax from its first row
    const long long i0 = (long long)a.lo + (long long)blockIdx.x * kRowThreads;
    const long long rows = min((long long)kRowThreads, (long long)a.hi - i0);
    const long long smax = bal ? rows - 1 + (n >> 1) : (long long)n - 1 - i0;
    // p = 1 + d^2 against 1 + thr, with a band far wider than the fp32 error of d^2 from exact
    // fp32 inputs: flag conservatively, decide every candidate exactly
    const float thr2 = (float)((1.0 + (double)a.thr) * (1.0 + 1.52587890625e-05));
    unsigned long long cnt = 0, checks = 0;
    double sum = 0.0;
    const int rl = threadIdx.x;
    for (long long t0 = 1; t0 <= smax; t0 += kRowTile) {
        const int tw = (int)min((long long)kRowTile, smax - t0 + 1);
        __syncthreads();
        if (threadIdx.x < tw) {
            long long j = i0 + t0 + threadIdx.x;
            if (j >= n) j -= n;
            s_col[threadIdx.x] = make_float4(xyz[3 * j], xyz[3 * j + 1], xyz[3 * j + 2], 0.f);
        }
        __syncthreads();
        // this thread owns column offset s = t0 + k (from i0) iff 1 <= s - rl <= lim
        const int k_lo = max(0, (int)(rl + 1 - t0)), k_hi = min(tw, (int)(rl + lim - t0 + 1));
        for (int k0 = k_lo; k0 < k_hi; k0 += 64) {  // fp32 partial sums of <= 64 terms, then float64
            float fs = 0.f;
            const int k1 = min(k_hi, k0 + 64);
            for (int k = k0; k < k1; ++k) {
                const float4 c = s_col[k];
                const float dx = xi - c.x, dy = yi - c.y, dz = zi - c.z;
                const float p = fmaf(dz, dz, fmaf(dy, dy, fmaf(dx, dx, 1.0f)));
                if (direct) fs += rcp_approx(p);
                if (p < thr2) {
                    long long j = i0 + t0 + k;
                    if (j >= n) j -= n;
                    ++checks;
                    cnt += exact_pair_call(a.xyz, a.dtype, a.pred, i, j) ? 1ull : 0ull;
                }
            }
            sum += (double)fs;
        }
    }
    cnt = warp_sum(cnt);
    checks = warp_sum(checks);
    sum = warp_sum(sum);
    if ((threadIdx.x & 31) == 0) {
        s_c[threadIdx.x >> 5] = cnt;
        s_k[threadIdx.x >> 5] = checks;
        s_s[threadIdx.x >> 5] = sum;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        Slot sl{};
        for (int w = 0; w < kRowThreads / 32; ++w) {
            sl.count += s_c[w];
            sl.checks += s_k[w];
            sl.sum += s_s[w];
        }
        a.slots[blockIdx.x] = sl;
    }
}
