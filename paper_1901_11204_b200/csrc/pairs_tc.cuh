// Tensor-core count kernel (included by paircount.cu after pairs_kernel.cuh).
//
// The count kernel's Gram filter  t = q_i.q_j + w_j > c_i is a
// matrix product: rows A_i = (q_i, 1), columns B_j = (q_j, w_j).  Here it runs
// on the 5th-generation tensor cores: tcgen05.mma kind::tf32 writes a 128 x 256
// tile of t into TMEM, epilogue warps drain it with tcgen05.ld and keep a per-row
// max (FMNMX3); a row whose max beats c_i is re-read and each candidate goes
// through the same exact predicate as every other path (exact_pair_call), so
// counts stay bit-exact.  fp32 precision with tf32 operands: the 3xTF32 split
//   q = qh + ql,  w = wh + wl  (qh, wh rounded to tf32)
//   t ~ qh_i.qh_j + qh_i.ql_j + ql_i.qh_j + wh_j + wl_j          (K = 11 of 16)
// -- tf32 x tf32 products are exact in fp32; the dropped ql.ql and the hardware
// truncation of ql/wl cost <= ~7 * 2^-22 * M, the fp32 accumulation of 11 terms
// <= ~2^-20 * M (M = max |q|^2); the filter can only miss a pair whose error exceeds
// b/2, and the band here is b = 2^-16 * (M + 4) (4x the FFMA kernel's; >= 4x margin
// over that estimate; the cost of a wider band is more exact re-checks: 2^-15 and
// 2^-17 measured within 1.5 % of each other on config 3).
//
// Schedule: the balanced ownership over uniform 128-row tiles (the FLAT tiling
// of pairs_kernel): tile t = rows [128t, 128t+128) scans window columns
// j = (128t + s) mod n, s in [0, 256*C); row rl owns s iff 1 <= s - rl <= lim(i).
// Work items (t, chunk c) are claimed in groups from one counter by a loader
// warp; the window is made contiguous by staging the column operand over an
// extended index range p in [0, n_ext), point p mod n.
//
// Operands live in HBM already in the tcgen05 K-major no-swizzle layout: 8-point
// groups of 512 B, four 128-byte K-chunks each (8 rows x 16 B), so a tile's A
// (8 KB) and a chunk's B (16 KB) are single TMA bulk copies.
//
// CTA = 10 warps, one per SM (the shared-memory request keeps it alone with its
// 512 TMEM columns): warp 0 claims and loads (A on a tile change, B every item)
// into a 7-stage ring; warp 1 allocates TMEM and issues the MMAs (two K=8
// tcgen05.mma per item into one of two 256-column accumulators); warps 2..9
// drain the accumulators (warp w reads TMEM lanes 32*(w%4).., columns
// 128*((w-2)/4)..).
#ifndef PC_TC_DRAIN
#define PC_TC_DRAIN 8  // drain warps: 8 (a 32 x 128 slice each) or 16 (32 x 64)
#endif
constexpr int kTcM = 128, kTcN = 256, kTcStages = 7;
constexpr int kTcDrain = PC_TC_DRAIN, kTcDrainCols = kTcN * 4 / kTcDrain, kTcDrainBlk = kTcDrainCols / 32;
constexpr int kTcWarps = 2 + kTcDrain;
constexpr int kTcABytes = kTcM * 64, kTcBBytes = kTcN * 64;
constexpr int kTcSmem = 2 * kTcABytes + kTcStages * kTcBBytes + 1024;  // > half the SM: one CTA per SM
// PC_TILE_AUTO's range for it: below, the FFMA kernel's small-tile config wins; from
// 2^21 up it stays on the FFMA kernel, whose exact path degrades more gracefully when
// the data are clustered (2^22 clustered spheres: 1.38 s here vs 1.08 s, 214M vs 125M
// candidates through the wider band).
constexpr long long kTcMinN = 1 << 14, kTcMaxN = 1 << 21;

// Candidate queues: (i, j) pairs the filter passed, evaluated by tc_exact_kernel after
// the filter so a flagged row never holds an accumulator through global loads.  Each
// CTA appends to its own slice (shared-memory counter, no global atomics); a full
// slice falls back to the exact check in place.
__host__ __device__ inline long long tc_cand_cap(long long n) {
    const long long c = 8 * n;
    return c < (1 << 16) ? (1 << 16) : c > (1 << 24) ? (1 << 24) : c;
}

// Operands are staged once per call in absolute point order; a row range [lo, hi) runs
// tiles from lo8 = lo rounded down to the 8-point operand group, rows outside [lo, hi)
// masked.  So the row operand covers up to n + 135 rows and the column operand up to
// n + 135 + chunks * 256 points.
struct TcGeom {
    long long chunks, n_rows, n_ext;  // chunks per tile window, staged row / column points
};
__host__ __device__ inline TcGeom tc_geom(long long n) {
    TcGeom g;
    g.chunks = (kTcM + n / 2 + kTcN - 1) / kTcN;  // s up to 127 + n/2
    g.n_rows = ((n + 8 + kTcM - 1) / kTcM + 1) * kTcM;
    g.n_ext = g.n_rows + g.chunks * kTcN;
    return g;
}

struct TcArgs {
    const float4* aop;  // row operand, n_rows points (zeros past n)
    const float4* bop;  // column operand, n_ext points
    const float4* pts_even;  // pairs_kernel staging: w_i for the row thresholds
    const float4* pts_odd;
    const void* xyz;
    const PrepStats* st;
    Slot* slots;
    unsigned long long* work_ctr;
    uint2* cand;            // candidate queues (i, j), cand_per_cta per CTA
    unsigned* cand_counts;  // queue length of each CTA
    long long cand_per_cta;
    int dtype, pred, n;
    int lo, hi, lo8;  // the row range; tiles start at lo8 = lo & ~7
    float thr;
    long long n_tiles, chunks, items;
    int group;  // items per claim
};

__device__ __forceinline__ float tf32_rna(float x) {
    unsigned r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// Byte offset of K-chunk kc of point p in the K-major interleaved operand layout.
__host__ __device__ __forceinline__ size_t tc_off(long long p, int kc) {
    return (size_t)(p >> 3) * 512 + (size_t)kc * 128 + (size_t)(p & 7) * 16;
}

// Row and column operands from the same centred q / w the FFMA count kernel stages.
__global__ void prep_tc_kernel(const void* __restrict__ xyz, int dtype, long long n, const PrepStats* __restrict__ st,
                               long long n_rows, long long n_ext, char* __restrict__ aop, char* __restrict__ bop) {
    double c[3];
    long long ci[3];
    bbox_centre(*st, dtype, c, ci);
    const long long m = n_rows > n_ext ? n_rows : n_ext;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < m; p += (long long)gridDim.x * blockDim.x) {
        const long long i = p % n;
        double nq;
        const float4 v = staged_point<false>(xyz, dtype, i, c, ci, &nq);
        const float q[3] = {v.x, v.y, v.z};
        float h[3], l[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            h[k] = tf32_rna(q[k]);
            l[k] = q[k] - h[k];  // exact
        }
        const float wh = tf32_rna(v.w), wl = v.w - wh;
        if (p < n_rows) {
            const bool real = p < n;
            const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
            *reinterpret_cast<float4*>(aop + tc_off(p, 0)) = real ? make_float4(h[0], h[1], h[2], h[0]) : z;
            *reinterpret_cast<float4*>(aop + tc_off(p, 1)) = real ? make_float4(h[1], h[2], l[0], l[1]) : z;
            *reinterpret_cast<float4*>(aop + tc_off(p, 2)) = real ? make_float4(l[2], 1.f, 1.f, 0.f) : z;
            *reinterpret_cast<float4*>(aop + tc_off(p, 3)) = z;
        }
        if (p < n_ext) {
            *reinterpret_cast<float4*>(bop + tc_off(p, 0)) = make_float4(h[0], h[1], h[2], l[0]);
            *reinterpret_cast<float4*>(bop + tc_off(p, 1)) = make_float4(l[1], l[2], h[0], h[1]);
            *reinterpret_cast<float4*>(bop + tc_off(p, 2)) = make_float4(h[2], wh, wl, 0.f);
            *reinterpret_cast<float4*>(bop + tc_off(p, 3)) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
}

// smem matrix descriptor, K-major no swizzle: K-chunks 128 B apart (LBO), 8-row groups 512 B apart (SBO)
__device__ __forceinline__ uint64_t tc_desc(unsigned saddr) {
    return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(512u >> 4) << 32) |
           (1ull << 46);
}
// instruction descriptor: D f32, A/B tf32, both K-major, N = 256, M = 128
constexpr uint32_t kTcIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kTcN >> 3) << 17) |
                              ((uint32_t)(kTcM >> 4) << 24);

__device__ __forceinline__ void tc_commit(unsigned bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"((unsigned long long)bar)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_plain(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

#define PC_TC_LD32(v, taddr)                                                                                 \
    asm volatile(                                                                                            \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"     \
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                           \
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),    \
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),           \
          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),         \
          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),         \
          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])                                                              \
        : "r"(taddr))

__global__ void __launch_bounds__(kTcWarps * 32, 1) pairs_tc_kernel(const TcArgs a) {
    extern __shared__ __align__(1024) unsigned char tc_smem[];
    // 1024-aligned operand buffers: A[2], then B[kTcStages]
    unsigned char* base = (unsigned char*)(((uintptr_t)tc_smem + 1023) & ~(uintptr_t)1023);
    unsigned char* sA = base;
    unsigned char* sB = base + 2 * kTcABytes;
    __shared__ __align__(8) unsigned long long bar_bfull[kTcStages], bar_bempty[kTcStages];
    __shared__ __align__(8) unsigned long long bar_afull[2], bar_aempty[2];
    __shared__ __align__(8) unsigned long long bar_accfull[2], bar_accempty[2];
    // loader -> MMA: tag = t << 24 | c (-1: done), bit 61 first item of a tile, bit 62 its A buffer
    __shared__ long long s_item[kTcStages];
    __shared__ long long s_acc_item[2];  // MMA -> epilogue: t << 24 | c
    __shared__ unsigned s_tmem;
    __shared__ unsigned s_ncand;
    __shared__ unsigned long long s_red[kTcWarps][2];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned b_full = (unsigned)__cvta_generic_to_shared(bar_bfull);
    const unsigned b_empty = (unsigned)__cvta_generic_to_shared(bar_bempty);
    const unsigned a_full = (unsigned)__cvta_generic_to_shared(bar_afull);
    const unsigned a_empty = (unsigned)__cvta_generic_to_shared(bar_aempty);
    const unsigned acc_full = (unsigned)__cvta_generic_to_shared(bar_accfull);
    const unsigned acc_empty = (unsigned)__cvta_generic_to_shared(bar_accempty);
    if (threadIdx.x == 0) {
        for (int k = 0; k < kTcStages; ++k) {
            mbar_init(b_full + 8 * k, 1);
            mbar_init(b_empty + 8 * k, 1);
        }
        for (int k = 0; k < 2; ++k) {
            mbar_init(a_full + 8 * k, 1);
            mbar_init(a_empty + 8 * k, 1);
            mbar_init(acc_full + 8 * k, 2);  // the MMA thread's item hand-off + the MMAs' commit
            mbar_init(acc_empty + 8 * k, kTcDrain);
        }
        mbar_init_fence();
        s_ncand = 0;
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (unsigned)__cvta_generic_to_shared(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tmem = s_tmem;
    const long long C = a.chunks;
    unsigned long long cnt = 0, checks = 0;

    if (warp == 0) {
        // ---------------- loader: claim groups of items, stage A (tile change) and B
        if (lane == 0) {
            long long it = 0, next = 0, end = 0, cur_tile = -1, t = 0, c = 0;
            int abuf = 1, sg = 0;
            unsigned ph_empty = 0;  // bit s: parity of stage s's next b_empty completion
            long long aloads[2] = {0, 0};
            for (;; ++it, sg = sg + 1 == kTcStages ? 0 : sg + 1) {
                if (next == end) {
                    next = (long long)atomicAdd(a.work_ctr, (unsigned long long)a.group);
                    end = next + a.group < a.items ? next + a.group : a.items;
                    if (next >= a.items) next = end = a.items;
                    t = next / C;  // one division per claim; items then advance (t, c) incrementally
                    c = next - t * C;
                }
                if (it >= kTcStages) {
                    mbar_wait(b_empty + 8 * sg, (ph_empty >> sg) & 1u);
                    ph_empty ^= 1u << sg;
                }
                if (next >= a.items) {
                    s_item[sg] = -1;
                    mbar_arrive_plain(b_full + 8 * sg);
                    break;
                }
                ++next;
                long long flag = 0;
                if (t != cur_tile) {
                    abuf ^= 1;
                    if (aloads[abuf] > 0) mbar_wait(a_empty + 8 * abuf, (unsigned)((aloads[abuf] - 1) & 1));
                    mbar_expect_tx(a_full + 8 * abuf, kTcABytes);
                    bulk_g2s(sA + abuf * kTcABytes, (const char*)a.aop + tc_off(a.lo8 + t * kTcM, 0), kTcABytes,
                             a_full + 8 * abuf);
                    ++aloads[abuf];
                    cur_tile = t;
                    flag = 1ll << 61;
                }
                s_item[sg] = (t << 24) | c | ((long long)abuf << 62) | flag;
                mbar_expect_tx(b_full + 8 * sg, kTcBBytes);
                bulk_g2s(sB + sg * kTcBBytes, (const char*)a.bop + tc_off(a.lo8 + t * kTcM + c * kTcN, 0), kTcBBytes,
                         b_full + 8 * sg);
                if (++c == C) {
                    c = 0;
                    ++t;
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        if (lane == 0) {
            long long it = 0;
            long long aloads[2] = {0, 0};
            int cur_abuf = -1, sg = 0;
            unsigned ph_full = 0;  // bit s: parity of stage s's next b_full completion
            for (;; ++it, sg = sg + 1 == kTcStages ? 0 : sg + 1) {
                mbar_wait(b_full + 8 * sg, (ph_full >> sg) & 1u);
                ph_full ^= 1u << sg;
                const long long tag = s_item[sg];
                const int acc = (int)(it & 1);
                if (it >= 2) mbar_wait(acc_empty + 8 * acc, (unsigned)((it >> 1) - 1) & 1u);
                if (tag < 0) {
                    s_acc_item[acc] = -1;
                    mbar_arrive_plain(acc_full + 8 * acc);
                    mbar_arrive_plain(acc_full + 8 * acc);
                    break;
                }
                const int ab = (int)((tag >> 62) & 1);
                if ((tag >> 61) & 1) {  // first item of a tile: its A buffer landed; the previous A is free after the MMAs so far
                    if (cur_abuf >= 0) tc_commit(a_empty + 8 * cur_abuf);
                    mbar_wait(a_full + 8 * ab, (unsigned)(aloads[ab] & 1));
                    ++aloads[ab];
                    cur_abuf = ab;
                }
                s_acc_item[acc] = tag & ((1ll << 61) - 1);
                mbar_arrive_plain(acc_full + 8 * acc);  // release: the epilogue reads the item after its wait
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const unsigned sa = (unsigned)__cvta_generic_to_shared(sA + ab * kTcABytes);
                const unsigned sb = (unsigned)__cvta_generic_to_shared(sB + sg * kTcBBytes);
#pragma unroll
                for (int kh = 0; kh < 2; ++kh) {  // K = 16 as two K = 8 steps (K-chunks 2kh, 2kh+1)
                    const uint64_t da = tc_desc(sa + 256u * kh), db = tc_desc(sb + 256u * kh);
                    asm volatile(
                        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem + (unsigned)(acc * kTcN)),
                        "l"(da), "l"(db), "r"(kTcIdesc), "r"(kh));
                }
                tc_commit(b_empty + 8 * sg);
                tc_commit(acc_full + 8 * acc);
            }
        }
    } else {
        // ---------------- epilogue: 8 warps, lane quadrant warp%4, column half (warp-2)/4
        const int quad = warp & 3, half = (warp - 2) >> 2;  // half: this warp's column slice
        const double M = dec_f64_or0(a.st->mnorm);
        const bool force = !(M < 1e30);
        const float half_tb = (float)(0.5 * ((double)a.thr + 1.52587890625e-05 * (M + 4.0)));  // b = 2^-16 (M + 4)
        const int n = a.n;
        long long cur_tile = -1;
        float rc = INFINITY;
        int lim = 0;
        for (long long it = 0;; ++it) {
            const int acc = (int)(it & 1);
            mbar_wait(acc_full + 8 * acc, (unsigned)(it >> 1) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const long long item = s_acc_item[acc];
            if (item < 0) break;
            const long long t = item >> 24, c = item & ((1ll << 24) - 1);
            const int rl = quad * 32 + lane;
            const long long i = a.lo8 + t * kTcM + rl;
            const bool valid = i >= a.lo && i < a.hi;
            if (t != cur_tile) {
                cur_tile = t;
                if (valid) {
                    const float4 e = ((i & 1) ? a.pts_odd : a.pts_even)[2 * (i >> 1) + 1];
                    rc = force ? -INFINITY : -e.z - half_tb;  // e = (z_i, z_i1, w_i, w_i1)
                    lim = steps_for_dev(n, (int)i);
                } else {
                    rc = INFINITY;
                    lim = 0;
                }
            }
            const unsigned taddr = tmem + ((unsigned)(quad * 32) << 16) + (unsigned)(acc * kTcN + half * kTcDrainCols);
            // the whole 32 x 128 slice into registers, then the accumulator goes straight back to
            // the MMA warp: the reduction and any candidate handling overlap the next MMAs
            unsigned v[kTcDrainBlk][32];
#pragma unroll
            for (int q = 0; q < kTcDrainBlk; ++q) PC_TC_LD32(v[q], taddr + 32u * q);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive_plain(acc_empty + 8 * acc);
            float bm[kTcDrainBlk], bmax = -INFINITY;
#pragma unroll
            for (int q = 0; q < kTcDrainBlk; ++q) {
                bm[q] = -INFINITY;
#pragma unroll
                for (int e = 0; e < 32; e += 2) bm[q] = max3f(bm[q], __uint_as_float(v[q][e]), __uint_as_float(v[q][e + 1]));
                bmax = fmaxf(bmax, bm[q]);
            }
            // s of this lane's first column; rows own 1 <= s - rl <= lim
            const long long s0 = c * kTcN + half * kTcDrainCols;
            const bool any_owned = valid && s0 + (kTcDrainCols - 1) - rl >= 1 && s0 - rl <= lim;
            const bool flag = any_owned && (force || bmax > rc);
            if (flag) {
                // queue this row's owned candidates for the exact pass
#pragma unroll
                for (int q = 0; q < kTcDrainBlk; ++q) {
                    if (!(force || bm[q] > rc)) continue;
                    const unsigned* vq = v[q];
                    unsigned m = 0xffffffffu;
                    if (!force) {
                        m = 0;
#pragma unroll
                        for (int e = 0; e < 32; ++e) m |= (__uint_as_float(vq[e]) > rc ? 1u : 0u) << e;
                    }
                    while (m) {
                        const int e = __ffs(m) - 1;
                        m &= m - 1;
                        const long long d = s0 + 32 * q + e - rl;
                        if (d >= 1 && d <= lim) {
                            long long j = i + d;
                            if (j >= n) j -= n;
                            const unsigned k = atomicAdd(&s_ncand, 1u);
                            if ((long long)k < a.cand_per_cta) {
                                a.cand[blockIdx.x * a.cand_per_cta + k] = make_uint2((unsigned)i, (unsigned)j);
                            } else {
                                ++checks;
                                cnt += exact_pair_call(a.xyz, a.dtype, a.pred, i, j) ? 1ull : 0ull;
                            }
                        }
                    }
                }
            }
        }
    }
    cnt = warp_sum(cnt);
    checks = warp_sum(checks);
    if (lane == 0) {
        s_red[warp][0] = cnt;
        s_red[warp][1] = checks;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        Slot sl{};
        for (int w = 0; w < kTcWarps; ++w) {
            sl.count += s_red[w][0];
            sl.checks += s_red[w][1];
        }
        a.slots[blockIdx.x] = sl;
        a.cand_counts[blockIdx.x] = (unsigned)min((long long)s_ncand, a.cand_per_cta);
    }
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

// The exact predicate over the queued candidates: block b takes filter CTA b's queue.
__global__ void __launch_bounds__(256) tc_exact_kernel(const TcArgs a, Slot* __restrict__ slots) {
    __shared__ unsigned long long s_c[8], s_k[8];
    const long long m = a.cand_counts[blockIdx.x];
    const uint2* q = a.cand + blockIdx.x * a.cand_per_cta;
    unsigned long long cnt = 0, checks = 0;
    for (long long k = threadIdx.x; k < m; k += blockDim.x) {
        const uint2 p = q[k];
        PC_CHECK((int)p.x < a.n && (int)p.y < a.n && p.x != p.y);
        ++checks;
        cnt += exact_pair(a.xyz, a.dtype, a.pred, (long long)p.x, (long long)p.y) ? 1ull : 0ull;
    }
    cnt = warp_sum(cnt);
    checks = warp_sum(checks);
    if ((threadIdx.x & 31) == 0) {
        s_c[threadIdx.x >> 5] = cnt;
        s_k[threadIdx.x >> 5] = checks;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        Slot sl{};
        for (int w = 0; w < 8; ++w) {
            sl.count += s_c[w];
            sl.checks += s_k[w];
        }
        slots[blockIdx.x] = sl;
    }
}
