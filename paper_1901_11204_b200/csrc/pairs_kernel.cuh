// The all-pairs kernel (included by paircount.cu inside its anonymous namespace).
//
// Unit of work: a WARP tile of T = 32*R outer rows (R rows per lane, row
// rl = r*32 + lane, coalesced loads) held in registers, streaming partner
// columns through a warp-private double-buffered shared-memory ring of W
// points (cp.async, 16 B per point).  Warps never wait for each other: the
// only CTA barrier is the final reduction.  (The first version staged
// columns per CTA; ncu showed `barrier` as the top stall at 2.1 warps per
// issue because any warp in the slow path held up the other three.)
//
// Column space: a warp tile starting at row i0 walks offsets s' = 1..L
// (partner j = i0 + s', mod n for the balanced schedule); row rl owns offset
// s' iff 1 <= s' - rl <= lim(i0 + rl) (reference ownership, spi_engine.py:
// 102-106).  FLAT: the tiles * L rectangle is split evenly over all warps of
// a persistent grid.  PER_ROW_TILE: warp g of the grid walks tile g.

template <int WARPS, int R, int W, bool DIRECT, bool FLAT>
__global__ void __launch_bounds__(WARPS * 32, 4) pairs_kernel(const PairsArgs a) {
    constexpr int T = 32 * R;
    static_assert(W % 32 == 0 && W % 2 == 0, "chunk must be a multiple of the warp");
    __shared__ __align__(16) float4 s_pts[WARPS][2][W];
    __shared__ int s_j[WARPS][2][W];
    __shared__ unsigned long long s_red[WARPS][2];
    __shared__ double s_sum[WARPS];

    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const long long gw = (long long)blockIdx.x * WARPS + wid;
    const long long nw = (long long)gridDim.x * WARPS;
    const int n = a.n;
    const bool bal = a.sched == PC_BALANCED;

    // error bands, derived from the prep statistics
    const double M = dec_f64_or0(a.st->mnorm);
    const double X = dec_f64_or0(a.st->maxabs);
    const bool force = !DIRECT && !(M < 1e30);  // fp32 filter unusable: exact path for every pair
    const float half_tb = (float)(0.5 * ((double)a.thr + 3.814697265625e-06 * (M + 4.0)));
    const double bd = 1.52587890625e-05 + (a.dtype == PC_F32 ? 0.0 : 9.5367431640625e-07 * X);
    const float thr2 = (float)(1.0 + (double)a.thr + bd);
    const int steps_min = (n & 1) ? (n - 1) >> 1 : (n >> 1) - 1;

    // this warp's column range
    long long g, g_end;
    int fixed_tile = 0;
    if (FLAT) {
        g = a.total * gw / nw;
        g_end = a.total * (gw + 1) / nw;
    } else {
        fixed_tile = (int)gw;
        g = 0;
        g_end = 0;
        if (gw < a.n_tiles) {
            const int i0 = a.lo + fixed_tile * T;
            g_end = bal ? (long long)(T - 1 + (n >> 1)) : (long long)(n - 1 - i0);
        }
    }
    auto tile_of = [&](long long gg) -> int { return FLAT ? (int)(gg / a.L) : fixed_tile; };
    auto off_of = [&](long long gg) -> int { return FLAT ? (int)(gg % a.L) : (int)gg; };
    auto width_of = [&](long long gg) -> int {
        const long long rem_tile = FLAT ? a.L - gg % a.L : g_end - gg;
        const long long w = rem_tile < (long long)W ? rem_tile : (long long)W;
        return (int)(w < g_end - gg ? w : g_end - gg);
    };

    float4* sp0 = s_pts[wid][0];
    int* sj0 = s_j[wid][0];
    auto stage = [&](int buf, long long gg) {
        const int t = tile_of(gg), off = off_of(gg), wc = width_of(gg);
        const int i0 = a.lo + t * T;
        float4* sp = sp0 + buf * W;
        int* sj = sj0 + buf * W;
#pragma unroll
        for (int q = 0; q < W / 32; ++q) {
            const int k = q * 32 + lane;
            if (k < wc) {
                int j = i0 + off + 1 + k;  // s' = off + 1 + k  (< 2^31: n < 2^31 - 4096)
                if (bal) {
                    if (j >= n) j -= n;
                    if (j >= n) j %= n;
                }
                cp_async16(&sp[k], &a.pts[j]);
                sj[k] = j;
            } else {
                sp[k] = DIRECT ? make_float4(0.f, 0.f, 0.f, 0.f) : make_float4(0.f, 0.f, 0.f, -INFINITY);
                sj[k] = -1;
            }
        }
        cp_async_commit();
    };

    float rx[R], ry[R], rz[R], rc[R];
    int cur_tile = -1;
    unsigned valid_rows = 0;
    unsigned long long cnt = 0, checks = 0;
    double sum = 0.0;

    if (g < g_end) stage(0, g);
    int buf = 0;
    while (g < g_end) {
        const long long g_next = g + width_of(g);
        if (g_next < g_end) {
            stage(buf ^ 1, g_next);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncwarp();

        const int t = tile_of(g), off = off_of(g), wc = width_of(g);
        const int i0 = a.lo + t * T;
        if (t != cur_tile) {
            cur_tile = t;
            valid_rows = 0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int i = i0 + r * 32 + lane;
                const bool ok = i < a.hi;
                const float4 v = ok ? a.pts[i] : make_float4(0.f, 0.f, 0.f, 0.f);
                rx[r] = v.x;
                ry[r] = v.y;
                rz[r] = v.z;
                rc[r] = ok ? (force ? -INFINITY : -v.w - half_tb) : INFINITY;
                valid_rows |= (ok ? 1u : 0u) << r;
            }
        }
        const float4* sp = sp0 + buf * W;
        const int* sj = sj0 + buf * W;
        unsigned fl = 0;

        if (!DIRECT) {
            // ---- Gram filter: 3 FFMA per pair + FMNMX3 per two pairs ----
            float m[R];
#pragma unroll
            for (int r = 0; r < R; ++r) m[r] = -INFINITY;
#pragma unroll 4
            for (int k = 0; k < W; k += 2) {
                const float4 c0 = sp[k], c1 = sp[k + 1];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    float t0 = fmaf(rx[r], c0.x, c0.w);
                    float t1 = fmaf(rx[r], c1.x, c1.w);
                    t0 = fmaf(ry[r], c0.y, t0);
                    t1 = fmaf(ry[r], c1.y, t1);
                    t0 = fmaf(rz[r], c0.z, t0);
                    t1 = fmaf(rz[r], c1.z, t1);
                    m[r] = max3f(m[r], t0, t1);
                }
            }
#pragma unroll
            for (int r = 0; r < R; ++r) fl |= (m[r] > rc[r] ? 1u : 0u) << r;
            if (force) fl = valid_rows;
        } else {
            const bool dense = wc == W && i0 + T <= a.hi && off + 1 >= T && (!bal || off + W <= steps_min);
            float m[R], acc[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                m[r] = INFINITY;
                acc[r] = 0.f;
            }
            if (dense) {
                // ---- direct formula, p = 1 + |dr|^2; two pairs share one reciprocal ----
#pragma unroll 2
                for (int k = 0; k < W; k += 2) {
                    const float4 c0 = sp[k], c1 = sp[k + 1];
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const float dx0 = rx[r] - c0.x, dy0 = ry[r] - c0.y, dz0 = rz[r] - c0.z;
                        const float dx1 = rx[r] - c1.x, dy1 = ry[r] - c1.y, dz1 = rz[r] - c1.z;
                        const float p0 = fmaf(dz0, dz0, fmaf(dy0, dy0, fmaf(dx0, dx0, 1.0f)));
                        const float p1 = fmaf(dz1, dz1, fmaf(dy1, dy1, fmaf(dx1, dx1, 1.0f)));
                        m[r] = min3f(m[r], p0, p1);
                        acc[r] = fmaf(p0 + p1, rcp_approx(p0 * p1), acc[r]);
                    }
                }
            } else {
                // ---- edge chunk: per-pair ownership mask ----
                for (int k = 0; k < W; ++k) {
                    const float4 c0 = sp[k];
                    const int j = sj[k];
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int rl = r * 32 + lane;
                        const int i = i0 + rl;
                        const int lim = i < a.hi ? (bal ? steps_for_dev(n, i) : n - 1 - i) : 0;
                        const bool ok = j >= 0 && (unsigned)(off + k - rl) < (unsigned)lim;
                        const float dx = rx[r] - c0.x, dy = ry[r] - c0.y, dz = rz[r] - c0.z;
                        const float p = fmaf(dz, dz, fmaf(dy, dy, fmaf(dx, dx, 1.0f)));
                        acc[r] += ok ? rcp_approx(p) : 0.0f;
                        m[r] = ok ? fminf(m[r], p) : m[r];
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                sum += (double)acc[r];
                fl |= (m[r] < thr2 ? 1u : 0u) << r;
            }
        }

        // ---- slow path: re-scan flagged rows with the exact reference predicate ----
        if (__any_sync(0xffffffffu, fl != 0)) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (fl & (1u << r)) {
                    const int rl = r * 32 + lane;
                    const int i = i0 + rl;
                    const int lim = bal ? steps_for_dev(n, i) : n - 1 - i;  // flagged rows are valid rows
                    for (int k = 0; k < wc; ++k) {
                        const float4 c0 = sp[k];
                        bool cand;
                        if (DIRECT) {
                            const float dx = rx[r] - c0.x, dy = ry[r] - c0.y, dz = rz[r] - c0.z;
                            cand = fmaf(dz, dz, fmaf(dy, dy, fmaf(dx, dx, 1.0f))) < thr2;
                        } else {
                            float tt = fmaf(rx[r], c0.x, c0.w);
                            tt = fmaf(ry[r], c0.y, tt);
                            tt = fmaf(rz[r], c0.z, tt);
                            cand = force || tt > rc[r];
                        }
                        if (cand && (unsigned)(off + k - rl) < (unsigned)lim) {
                            ++checks;
                            cnt += exact_pair(a.xyz, a.dtype, a.pred, i, sj[k]) ? 1ull : 0ull;
                        }
                    }
                }
            }
        }
        __syncwarp();  // the buffer just read is restaged next iteration
        g = g_next;
        buf ^= 1;
    }

    // ---- CTA reduction (the only CTA barrier): one slot per CTA ----
    cnt = warp_sum(cnt);
    checks = warp_sum(checks);
    sum = warp_sum(sum);
    if (lane == 0) {
        s_red[wid][0] = cnt;
        s_red[wid][1] = checks;
        s_sum[wid] = sum;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        Slot s{0ull, 0ull, 0.0, 0ull};
        for (int q = 0; q < WARPS; ++q) {
            s.count += s_red[q][0];
            s.checks += s_red[q][1];
            s.sum += s_sum[q];
        }
        a.slots[blockIdx.x] = s;
    }
}
