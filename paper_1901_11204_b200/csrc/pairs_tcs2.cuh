// The tensor-core sum on SM pairs (included by paircount.cu after pairs_tcsum.cuh).
//
// pairs_tcs_kernel (one SM per item) keeps both row halves of an item in its TMEM -- all
// 512 columns -- so each drain group has one accumulator and waits for its refill after
// every release.  Here a cluster of two CTAs on one TPC shares every item through
// tcgen05.mma.cta_group::2 (M = 256): CTA r stages rows 128r.. of the tile (its half of A)
// and columns 128r.. of the chunk (its half of B), and receives rows 128r.. x all 256
// columns in its own TMEM.  Per SM an item is then one 256-column accumulator, so two
// items are in flight: all eight drain warps read item k (one round of 128 columns each),
// release it, and fold it while the MMA fills the other accumulator with item k+1.
// The operand build per SM halves too (128 columns and 128 rows).
//
// Measured (2^20, B200): 110.6 ms against 66.2 for pairs_tcs_kernel, so it is off by default
// (PAIRCOUNT_TCS2=1 selects it).  Per SM an item is half as much work, but the column-operand
// build's per-item latency (two producer warps, 128 columns) barely shrinks, and the producers
// starve the MMA (ncu: the drain waits on acc_full 32 % of its samples, the MMA thread on
// b_full).  Cross-CTA arrivals with release.cluster semantics (MEMBAR.ALL.GPU + ERRBAR in
// SASS) and cluster-scope acquire polls (CCTL.IVALL per poll) cost 167.8 -> 142 ms; the
// peer's operand arrivals are relaxed after its proxy fence, the drain's after wait::ld.
//
// Same items, same chunk bitmap, same arithmetic and bound as pairs_tcs_kernel (fp32
// points, bitmap present); claims are dealt to clusters round-robin (cluster k takes
// claims k, k + clusters, ...), so both CTAs walk the same items without talking.
// Barriers: the leader (cluster rank 0) owns b_full / a_full / acc_empty, which count
// arrivals from both CTAs (the peer's remotely); the MMA commits b_empty / a_empty /
// acc_full to both CTAs (multicast); the drain warps walk the same item sequence
// themselves, so no per-item message crosses the pair.

#ifndef PC_TC2_PROD
#define PC_TC2_PROD 2  // producer warps per CTA (2: 11 warps, 168 registers; 4: 13 warps, 128 registers)
#endif
constexpr int kTc2Prod = PC_TC2_PROD, kTc2Epi = 8, kTc2Warps = 1 + kTc2Prod + kTc2Epi;
constexpr int kTc2PT = kTc2Prod * 32, kTc2PR = 128 / kTc2PT;  // producer threads, points per thread
#ifndef PC_TC2_ROUND
#define PC_TC2_ROUND 128  // drain columns per round (64 when the register budget is 128)
#endif
constexpr int kTc2Round = PC_TC2_ROUND;
constexpr int kTc2Half = kTcsHalf;  // bytes of a 128-point operand half (8 KB)
#ifndef PC_TC2_STAGES
#define PC_TC2_STAGES 6
#endif
constexpr int kTc2Stages = PC_TC2_STAGES;
constexpr int kTc2Smem = 2 * kTc2Half + kTc2Stages * kTc2Half + 1024;
constexpr long long kTc2Parts = 2 * kTc2Epi;  // float64 partials per claim (both CTAs' drain warps)
// instruction descriptor: D f32, A/B bf16, K-major, N = 256, M = 256 (cta_group::2)
constexpr uint32_t kTc2Idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) |
                               ((uint32_t)(256 >> 4) << 24);

__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned mapa_shared(unsigned addr, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(unsigned cluster_addr) {  // any CTA's barrier
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(unsigned cluster_addr) {  // no ordering of prior memory ops
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_cluster() { asm volatile("fence.acq_rel.cluster;" ::: "memory"); }
__device__ __forceinline__ bool mbar_try_wait_cl(unsigned bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cl(unsigned bar, unsigned parity) {
    unsigned spins = 0;
    while (!mbar_try_wait_cl(bar, parity))
        if (++spins == (1u << 28)) __trap();
}
__device__ __forceinline__ void tc2_commit_both(unsigned bar) {  // arrives on bar in both CTAs of the pair
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(bar), "h"((unsigned short)3) : "memory");
}
__device__ __forceinline__ void st_cluster_s64(unsigned cluster_addr, long long v) {
    asm volatile("st.shared::cluster.b64 [%0], %1;" ::"r"(cluster_addr), "l"(v) : "memory");
}

// The cluster's items in order -- claims cid, cid + clusters, ...; the chunk bitmap selects --
// walked by a whole warp, 32 items' bits per round (one load per lane, a ballot), so no lane
// ever waits on a bitmap load per item.
struct Tc2Walker {
    const TcsArgs* a;
    long long nclusters, c, nu, nu1, wbase;
    unsigned wmask;
    __device__ Tc2Walker(const TcsArgs* a_, long long cid, long long ncl) : a(a_), nclusters(ncl), c(cid), wmask(0u) {
        nu = c * a->S;
        nu1 = min(nu + a->S, a->items);
        wbase = nu;
    }
    // next item (claim, item index); false at the end.  Call with the whole warp converged.
    __device__ bool next(long long& claim, long long& u) {
        const int lane = threadIdx.x & 31;
        while (wmask == 0u) {
            if (c >= a->nclaims) return false;
            if (nu >= nu1) {
                c += nclusters;
                nu = c * a->S;
                nu1 = min(nu + a->S, a->items);
                continue;
            }
            const long long uu = nu + lane;
            bool take = false;
            if (uu < nu1) {
                const long long t = uu / a->cpw, b = t * a->cpw_pad + (uu - t * a->cpw);
                take = (__ldg(a->bits + (b >> 5)) >> (b & 31)) & 1u;
            }
            wmask = __ballot_sync(0xffffffffu, take);
            wbase = nu;
            nu = min(nu + 32, nu1);
        }
        const int e = __ffs(wmask) - 1;
        wmask &= wmask - 1;
        claim = c;
        u = wbase + e;
        return true;
    }
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kTc2Warps * 32, 1) pairs_tcs2_kernel(const TcsArgs a) {
    extern __shared__ __align__(1024) unsigned char tc2_smem[];
    unsigned char* base = (unsigned char*)(((uintptr_t)tc2_smem + 1023) & ~(uintptr_t)1023);
    unsigned char* sA = base;                  // [2][kTc2Half]: this CTA's 128 rows
    unsigned char* sB = base + 2 * kTc2Half;   // [kTc2Stages][kTc2Half]: this CTA's 128 columns
    __shared__ __align__(8) unsigned long long bar_bfull[kTc2Stages], bar_bempty[kTc2Stages];
    __shared__ __align__(8) unsigned long long bar_afull[2], bar_aempty[2];
    __shared__ __align__(8) unsigned long long bar_accfull[2], bar_accempty[2];
    __shared__ long long s_item[kTc2Stages];  // leader: claim << 2 | abuf << 1 | new tile; -1 = done
    __shared__ unsigned s_tmem;
    __shared__ unsigned s_items;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned rank = cluster_rank();
    const bool leader = rank == 0;
    // every block of the launch takes the same decision, so the pair stays together
    const bool skip = f64_takes(*a.st, a.dtype, false) || a.n_tiles == 0 || !a.bits;
    if (skip) {
        if (threadIdx.x == 0) a.slots[blockIdx.x] = Slot{};
        return;
    }
    const unsigned b_full = (unsigned)__cvta_generic_to_shared(bar_bfull);
    const unsigned b_empty = (unsigned)__cvta_generic_to_shared(bar_bempty);
    const unsigned a_full = (unsigned)__cvta_generic_to_shared(bar_afull);
    const unsigned a_empty = (unsigned)__cvta_generic_to_shared(bar_aempty);
    const unsigned acc_full = (unsigned)__cvta_generic_to_shared(bar_accfull);
    const unsigned acc_empty = (unsigned)__cvta_generic_to_shared(bar_accempty);
    if (threadIdx.x == 0) {
        for (int k = 0; k < kTc2Stages; ++k) {
            mbar_init(b_full + 8 * k, 2 * kTc2Prod);  // leader's: both CTAs' producer warps
            mbar_init(b_empty + 8 * k, 1);
        }
        for (int k = 0; k < 2; ++k) {
            mbar_init(a_full + 8 * k, 2 * kTc2Prod);
            mbar_init(a_empty + 8 * k, 1);
            mbar_init(acc_full + 8 * k, 1);           // the MMAs' commit
            mbar_init(acc_empty + 8 * k, 2 * kTc2Epi);  // leader's: both CTAs' drain warps
        }
        mbar_init_fence();
        s_items = 0;
    }
    cluster_sync_all();  // the peer's barriers exist before anyone arrives on them
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (unsigned)__cvta_generic_to_shared(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tmem = s_tmem;
    const int n = a.n;
    const long long nclusters = (long long)(gridDim.x >> 1), cid = (long long)(blockIdx.x >> 1);
    // the leader's barriers as seen from this CTA (its own when this is the leader)
    const unsigned L_bfull = mapa_shared(b_full, 0), L_afull = mapa_shared(a_full, 0),
                   L_accempty = mapa_shared(acc_empty, 0);
    double sum = 0.0;

    if (warp == 0) {
        // ---------------- MMA issuer (the leader's elected thread)
        if (leader && lane == 0) {
            const uint64_t dA0 = tcs_desc((unsigned)__cvta_generic_to_shared(sA));
            const uint64_t dB0 = tcs_desc((unsigned)__cvta_generic_to_shared(sB));
            long long it = 0, aloads[2] = {0, 0};
            int cur_abuf = -1, sg = 0;
            unsigned items = 0;
            for (;; ++it, sg = sg + 1 == kTc2Stages ? 0 : sg + 1) {
                // the peer's operand writes were released at cluster scope by its arrival (after its proxy
                // fence); the MMA is ordered after this observation by tcgen05.fence::after_thread_sync
                mbar_wait(b_full + 8 * sg, (unsigned)((it / kTc2Stages) & 1));
                const long long tag = s_item[sg];
                if (tag < 0) break;  // the drains count their own items and stop by themselves
                const int acc = (int)(it & 1);
                if (it >= 2) mbar_wait(acc_empty + 8 * acc, (unsigned)(((it >> 1) - 1) & 1));
                ++items;
                const int ab = (int)((tag >> 1) & 1);
                if (tag & 1) {
                    if (cur_abuf >= 0) tc2_commit_both(a_empty + 8 * cur_abuf);
                    mbar_wait(a_full + 8 * ab, (unsigned)(aloads[ab] & 1));
                    ++aloads[ab];
                    cur_abuf = ab;
                }
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint64_t da = dA0 + (uint64_t)((ab * kTc2Half) >> 4), db = dB0 + (uint64_t)((sg * kTc2Half) >> 4);
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    asm volatile(
                        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                        " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem + (unsigned)(acc * 256)),
                        "l"(da + (uint64_t)(16 * ks)), "l"(db + (uint64_t)(16 * ks)), "r"(kTc2Idesc), "r"(ks));
                }
                tc2_commit_both(acc_full + 8 * acc);
                tc2_commit_both(b_empty + 8 * sg);
            }
            s_items = items;
        }
    } else if (warp <= kTc2Prod) {
        // ---------------- producers (both CTAs): this CTA's half of every operand
        const int tid = (warp - 1) * 32 + lane;  // points tid, tid + kTc2PT, ... of the half
        long long it = 0;
        int sg = 0, abuf = 1;
        long long aloads[2] = {0, 0};
        int a_tile = -1, o_tile = -1;
        float o[3] = {0.f, 0.f, 0.f};
        const long long C = a.cpw;
        const float* xyz = (const float*)a.xyz;
        auto row0t = [&](int tt) -> int { return a.lo + tile_abs(tt, a.tstride, a.toff) * kTcsT; };
        Tc2Walker walk(&a, cid, nclusters);
        auto advance = [&](long long& c_out, long long& u_out) -> bool { return walk.next(c_out, u_out); };
        auto col0 = [&](long long u) -> int {  // this CTA's first column of item u's chunk
            const long long t = u / C;
            int jw = row0t((int)t) + (int)((u - t * C) * kTcsW) + 1 + 128 * (int)rank;
            while (jw >= n) jw -= n;
            return jw;
        };
        auto load2 = [&](int j0, float (&q)[3 * kTc2PR]) {
#pragma unroll
            for (int h = 0; h < kTc2PR; ++h) {
                int j = j0 + tid + kTc2PT * h;
                if (j >= n) j -= n;
                PC_CHECK(j >= 0 && j < n);
                const float* src = xyz + 3ll * j;
                q[3 * h] = __ldg(src);
                q[3 * h + 1] = __ldg(src + 1);
                q[3 * h + 2] = __ldg(src + 2);
            }
        };
        long long c = 0, u = 0, c2 = 0, u2 = 0;
        float cur[3 * kTc2PR], nxt[3 * kTc2PR];
        bool have = advance(c, u);
        if (have) load2(col0(u), cur);
        while (have) {
            const bool have2 = advance(c2, u2);
            if (have2) load2(col0(u2), nxt);
            const long long t = u / C;
            const int tt = (int)t, i0 = row0t(tt);
            if (tt != o_tile) {  // the origin: the centre of the tile's origin group's box (chunk_geom_g's o)
                o_tile = tt;
                float gmn[3], gmx[3];
                tcs_group_box(a.blk_box, a.lo, a.hi, tile_abs(tt, a.tstride, a.toff), lane, gmn, gmx);
#pragma unroll
                for (int k = 0; k < 3; ++k) o[k] = __fmul_rn(0.5f, __fadd_rn(gmn[k], gmx[k]));
            }
            long long flag = 0;
            if (tt != a_tile) {  // this CTA's 128 rows of the new tile
                abuf ^= 1;
                if (aloads[abuf] > 0) mbar_wait(a_empty + 8 * abuf, (unsigned)((aloads[abuf] - 1) & 1));
                unsigned char* dA = sA + abuf * kTc2Half;
#pragma unroll
                for (int h = 0; h < kTc2PR; ++h) {
                    const int p = tid + kTc2PT * h;
                    const int i = i0 + 128 * (int)rank + p;
                    PC_CHECK(i >= a.lo && i < a.hi);
                    const float* q = xyz + 3ll * i;
                    tcs_write_row(dA, p, __fsub_rn(__ldg(q), o[0]), __fsub_rn(__ldg(q + 1), o[1]),
                                  __fsub_rn(__ldg(q + 2), o[2]));
                }
                fence_proxy_async_shared();
                __syncwarp();
                if (lane == 0) {  // the leader's own: a CTA-scope release; the peer's: after its proxy fence
                    if (leader) mbar_arrive_plain(a_full + 8 * abuf);
                    else mbar_arrive_cluster_relaxed(L_afull + 8 * abuf);
                }
                ++aloads[abuf];
                a_tile = tt;
                flag = 1;
            }
            // this CTA's 128 columns of the chunk (coordinates already loaded)
            if (it >= kTc2Stages) mbar_wait(b_empty + 8 * sg, (unsigned)(((it / kTc2Stages) - 1) & 1));
            unsigned char* dB = sB + sg * kTc2Half;
#pragma unroll
            for (int h = 0; h < kTc2PR; ++h) {
                const int p = tid + kTc2PT * h;
                tcs_write_col(dB, p, __fsub_rn(cur[3 * h], o[0]), __fsub_rn(cur[3 * h + 1], o[1]),
                              __fsub_rn(cur[3 * h + 2], o[2]));
            }
            fence_proxy_async_shared();
            __syncwarp();
            if (leader && tid == 0) s_item[sg] = (c << 2) | ((long long)abuf << 1) | flag;
            if (lane == 0) {
                if (leader) mbar_arrive_plain(b_full + 8 * sg);
                else mbar_arrive_cluster_relaxed(L_bfull + 8 * sg);
            }
            ++it;
            sg = sg + 1 == kTc2Stages ? 0 : sg + 1;
            have = have2;
            c = c2;
            u = u2;
#pragma unroll
            for (int k = 0; k < 3 * kTc2PR; ++k) cur[k] = nxt[k];
        }
        if (it >= kTc2Stages) mbar_wait(b_empty + 8 * sg, (unsigned)(((it / kTc2Stages) - 1) & 1));
        if (leader && tid == 0) s_item[sg] = -1;
        if (lane == 0) {
            if (leader) mbar_arrive_plain(b_full + 8 * sg);
            else mbar_arrive_cluster_relaxed(L_bfull + 8 * sg);
        }
    } else {
        // ---------------- drain (both CTAs): 8 warps on one accumulator, 32 rows x 128 columns each
        const int ew = warp - 1 - kTc2Prod, quad = warp & 3, chalf = ew >> 2;
        const long long C = a.cpw;
        long long it = 0, cur = -1, c = 0, u = 0;
        Tc2Walker walk(&a, cid, nclusters);
        for (;;) {
            const bool more = walk.next(c, u);
            if (!more || c != cur) {  // the finished claim's float64 partial
                if (cur >= 0) {
                    const double cs = warp_sum(sum);
                    PC_CHECK(cur < a.nclaims);
                    if (lane == 0) a.claim_sums[cur * kTc2Parts + rank * kTc2Epi + ew] = cs;
                    sum = 0.0;
                }
                cur = c;
            }
            if (!more) break;
            {
                const int acc = (int)(it & 1);
                mbar_wait(acc_full + 8 * acc, (unsigned)((it >> 1) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const unsigned taddr = tmem + ((unsigned)(quad * 32) << 16) + (unsigned)(acc * 256 + chalf * 128);
                float2 facc = make_float2(0.f, 0.f), facc2 = make_float2(0.f, 0.f);
#pragma unroll 1
                for (int rd = 0; rd < 128 / kTc2Round; ++rd) {
                unsigned v[kTc2Round / 32][32];
#pragma unroll
                for (int w = 0; w < kTc2Round / 32; ++w) PC_TC_LD32(v[w], taddr + (unsigned)(kTc2Round * rd) + 32u * w);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (rd == 128 / kTc2Round - 1) {
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    __syncwarp();
                    // the loads have completed (wait::ld): a relaxed arrival suffices to free the accumulator
                    if (lane == 0) mbar_arrive_cluster_relaxed(L_accempty + 8 * acc);
                }
#pragma unroll
                for (int w = 0; w < kTc2Round / 32; ++w) {
#pragma unroll
                    for (int e = 0; e < 32; e += 8) {
                        const float2 p1 = make_float2(__uint_as_float(v[w][e]), __uint_as_float(v[w][e + 1]));
                        const float2 p2 = make_float2(__uint_as_float(v[w][e + 2]), __uint_as_float(v[w][e + 3]));
                        const float2 p3 = make_float2(__uint_as_float(v[w][e + 4]), __uint_as_float(v[w][e + 5]));
                        const float2 p4 = make_float2(__uint_as_float(v[w][e + 6]), __uint_as_float(v[w][e + 7]));
                        const float2 m12 = __fmul2_rn(p1, p2), s12 = __fadd2_rn(p1, p2);
                        const float2 m34 = __fmul2_rn(p3, p4), s34 = __fadd2_rn(p3, p4);
                        const float2 P = __fmul2_rn(m12, m34);
                        const float2 Nn = __ffma2_rn(s34, m12, __fmul2_rn(s12, m34));
                        if (e & 8) facc2 = __ffma2_rn(Nn, make_float2(rcp_approx(P.x), rcp_approx(P.y)), facc2);
                        else facc = __ffma2_rn(Nn, make_float2(rcp_approx(P.x), rcp_approx(P.y)), facc);
                    }
                }
                }
                ++it;
                facc = __fadd2_rn(facc, facc2);
                sum += (double)(facc.x + facc.y) * (double)kTcsS;  // (the column operand's scale)
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        Slot sl{};
        sl.pad[0] = s_items;  // the leader counts the items (chunks) once
        a.slots[blockIdx.x] = sl;
    }
    cluster_sync_all();  // both CTAs done with TMEM and with each other's barriers
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}
