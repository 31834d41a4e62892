// The all-pairs kernel (included by paircount.cu inside its anonymous namespace).
//
// Unit of work: a WARP tile of T = 32*R outer rows (R rows per lane, row
// rl = r*32 + lane) held in registers, streaming partner columns through a
// warp-private double-buffered shared-memory ring of W columns.  Warps never
// wait for each other; the only CTA barrier is the final reduction.  (A
// first version staged columns per CTA; ncu showed `barrier` as the top
// stall, 2.1 warps per issue, because one warp in the slow path held up the
// other three.)
//
// Packed FP32: columns are staged as interleaved PAIRS (x_j, x_j+1, y_j,
// y_j+1)(z_j, z_j+1, w_j, w_j+1), so one FFMA2/FADD2 (sm_100 f32x2) with the
// row value broadcast evaluates two pairs.  The prep kernel writes the pair
// arrays E (pairs starting at even j) and O (odd j), each pair holding point
// j and point (j+1) mod n, so any window position is two 16-byte copies and a
// window of consecutive columns is one contiguous run.  The sum kernel moves
// full chunks and whole row tiles with one TMA bulk copy each (lane 0, per-warp
// mbarrier per buffer); the count kernel and ragged chunks use per-lane
// cp.async.  A tile's rows are staged into a warp-private row buffer with the
// chunk that first needs them, so a tile switch never stalls on a global load.
//
// Column space: a warp tile starting at row i0 walks offsets s' = 1..L
// (partner j = i0 + s', mod n for the balanced schedule); row rl owns offset
// s' iff 1 <= s' - rl <= lim(i0 + rl) (reference ownership, spi_engine.py:
// 102-106).  Dense chunks (every cell owned) run unmasked; the few edge
// chunks of each tile mask per pair.  FLAT: the tiles * L rectangle is one
// uniform work space; the warps of a persistent grid (SMs x occupancy CTAs)
// claim super-chunks (1..16 chunks, ~8 per warp) from an atomic counter (a
// static split left a ~30% occupancy tail in ncu).  PER_ROW_TILE: warp g
// walks tile g.

__device__ __forceinline__ float min3f(float a, float b, float c) {
    float d;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ float warp_min_f(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_max_f(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float2 f2_fma(float a, float2 b, float2 c) {  // a*b + c, a broadcast
    return __ffma2_rn(make_float2(a, a), b, c);
}
__device__ __forceinline__ float2 f2_rsub(float a, float2 b) {  // a - b, a broadcast
    unsigned long long bb = *reinterpret_cast<unsigned long long*>(&b), dd;
    asm("{.reg .b64 t; mov.b64 t, {%1, %1}; sub.rn.f32x2 %0, t, %2;}" : "=l"(dd) : "f"(a), "l"(bb));
    return *reinterpret_cast<float2*>(&dd);
}

// The sorted sum's per-chunk geometry: tile centre o, squared box gap, |a|max + |b|max.
// Shared by the FFMA kernel and the producers here, with explicit round-to-nearest
// operations so both compile to the same arithmetic and agree on every chunk.
struct ChunkGeom {
    float o[3];
    float gap2, ab;
};
__device__ __forceinline__ ChunkGeom chunk_geom(const float tmin[3], const float tmax[3], const float cl[3],
                                                const float ch[3]) {
    ChunkGeom g;
    float gap2 = 0.f, rt2 = 0.f, bm2 = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        g.o[k] = __fmul_rn(0.5f, __fadd_rn(tmin[k], tmax[k]));
        const float d = fmaxf(0.f, fmaxf(__fsub_rn(cl[k], tmax[k]), __fsub_rn(tmin[k], ch[k])));
        gap2 = __fadd_rn(gap2, __fmul_rn(d, d));
        const float ht = __fmul_rn(0.5f, __fsub_rn(tmax[k], tmin[k]));
        rt2 = __fadd_rn(rt2, __fmul_rn(ht, ht));
        const float bb = fmaxf(fabsf(__fsub_rn(cl[k], g.o[k])), fabsf(__fsub_rn(ch[k], g.o[k])));
        bm2 = __fadd_rn(bm2, __fmul_rn(bb, bb));
    }
    g.gap2 = gap2;
    g.ab = __fadd_rn(__fsqrt_rn(rt2), __fsqrt_rn(bm2));
    return g;
}
// The tensor-core sum (pairs_tcsum.cuh) centres a and b on the box of an origin GROUP of kTcsOrgG
// consecutive 256-row tiles (absolute tile index / kTcsOrgG), so one column operand serves the items
// (t + k, c - k) of the group's tiles along its diagonal.  Its chunk test: the tile's box (for |a|)
// and the chunk's box (for |b|, the gap) about the group's centre o.
#ifndef PC_TCS_G
#define PC_TCS_G 4  // (pipelined drain, 2^20 step: 3 / 4 tiles 62.0 / 61.4 ms, each at its best ring depth)
#endif
constexpr int kTcsOrgG = PC_TCS_G;
static_assert(kTcsOrgG >= 1 && kTcsOrgG <= 4, "an origin group's per-32 boxes: one per lane");
// Tile parts (pc_pairs_part_async): blocks of kTcsOrgG consecutive row tiles dealt round-robin, part
// toff of tstride holding blocks toff, toff + tstride, ...  The call's i-th tile is absolute tile
// tile_abs(i) -- whole origin groups per part, so a part's tensor-core sum keeps the column reuse.
__host__ __device__ __forceinline__ int tile_abs(int i, int tstride, int toff) {
    if (tstride == 1) return i + toff;
    return (i / kTcsOrgG) * (kTcsOrgG * tstride) + toff * kTcsOrgG + i % kTcsOrgG;
}
// the origin group's box: the union of the per-32 boxes of its full tiles (rows lo + 256 t ..
// + 255 < hi), lo a multiple of 32; warp-collective, min / max exact (every caller gets the same box)
__device__ __forceinline__ void tcs_group_box(const float4* __restrict__ blk_box, int lo, int hi, int tabs, int lane,
                                              float gmin[3], float gmax[3]) {
    const int tq = tabs / kTcsOrgG * kTcsOrgG + (lane >> 3);
    float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    if ((lane >> 3) < kTcsOrgG && (long long)lo + 256ll * (tq + 1) <= hi) {
        const int b = (lo >> 5) + 8 * tq + (lane & 7);
        const float4 lo4 = __ldg(blk_box + 2 * b), hi4 = __ldg(blk_box + 2 * b + 1);
        mn[0] = lo4.x; mn[1] = lo4.y; mn[2] = lo4.z;
        mx[0] = hi4.x; mx[1] = hi4.y; mx[2] = hi4.z;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        gmin[k] = warp_min_f(mn[k]);
        gmax[k] = warp_max_f(mx[k]);
    }
}
__device__ __forceinline__ ChunkGeom chunk_geom_g(const float tmin[3], const float tmax[3], const float gmin[3],
                                                  const float gmax[3], const float cl[3], const float ch[3]) {
    ChunkGeom g;
    float gap2 = 0.f, ra2 = 0.f, bm2 = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        g.o[k] = __fmul_rn(0.5f, __fadd_rn(gmin[k], gmax[k]));
        const float d = fmaxf(0.f, fmaxf(__fsub_rn(cl[k], tmax[k]), __fsub_rn(tmin[k], ch[k])));
        gap2 = __fadd_rn(gap2, __fmul_rn(d, d));
        const float aa = fmaxf(fabsf(__fsub_rn(tmin[k], g.o[k])), fabsf(__fsub_rn(tmax[k], g.o[k])));
        ra2 = __fadd_rn(ra2, __fmul_rn(aa, aa));
        const float bb = fmaxf(fabsf(__fsub_rn(cl[k], g.o[k])), fabsf(__fsub_rn(ch[k], g.o[k])));
        bm2 = __fadd_rn(bm2, __fmul_rn(bb, bb));
    }
    g.gap2 = gap2;
    g.ab = __fadd_rn(__fsqrt_rn(ra2), __fsqrt_rn(bm2));
    return g;
}
// a dense chunk the tensor-core sum kernel takes (pairs_tcsum.cuh): the Gram test below, 8u (|a|+|b|)^2
// <= 5e-6 (1 + dmin^2) written as 5u (..)^2 <= 3.125e-6 (..), dmin^2 > 4.5, and |a|+|b| <= 3e4 (the
// epilogue's four-term products stay finite)
__device__ __forceinline__ bool tcs_takes(const ChunkGeom& g) {
    return g.gap2 > 4.5f && g.ab <= 3e4f &&
           __fmul_rn(2.98023223876953125e-07f, __fmul_rn(g.ab, g.ab)) <= __fmul_rn(3.125e-6f, __fadd_rn(1.f, g.gap2));
}

// Pair-buffer layouts (one entry per column pair k, k+1):
//   PS = 2 float4: (x, x', y, y')(z, z', w, w')                       Gram / direct
//   PS = 3 float4: (x, x', y, y')(z, z', xl, xl')(yl, yl', zl, zl')   compensated direct:
//   the centred coordinate is the unevaluated fp32 sum hi + lo (non-f32 inputs)
template <bool COMP>
__device__ __forceinline__ float4 col_hi(const float4* sp, int k) {  // (x, y, z, w) of element k
    constexpr int PS = COMP ? 3 : 2;
    const float4* b = sp + PS * (k >> 1);
    const float4 A = b[0], B = b[1];
    if (COMP) return (k & 1) ? make_float4(A.y, A.w, B.y, 0.f) : make_float4(A.x, A.z, B.x, 0.f);
    return (k & 1) ? make_float4(A.y, A.w, B.y, B.w) : make_float4(A.x, A.z, B.x, B.z);
}
__device__ __forceinline__ float4 col_lo(const float4* sp, int k) {  // (xl, yl, zl, 0), PS = 3 only
    const float4* b = sp + 3 * (k >> 1);
    const float4 B = b[1], C = b[2];
    return (k & 1) ? make_float4(B.w, C.y, C.w, 0.f) : make_float4(B.z, C.x, C.z, 0.f);
}

// ---- TMA bulk staging (cp.async.bulk global -> shared, completion on an mbarrier)
#ifndef PC_TMA_GRAM
#define PC_TMA_GRAM 0
#endif
#ifndef PC_TMA_STAGE
#define PC_TMA_STAGE 1
#endif
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    unsigned spins = 0;
    while (!mbar_try_wait(bar, parity))
        if (++spins == (1u << 28)) __trap();  // a lost transaction must fail loudly, never hang the GPU
}
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, unsigned bytes, unsigned bar) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(d), "l"(gsrc), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_shared() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

#ifndef PC_MINB
#define PC_MINB 4
#endif
#ifndef PC_GRAM_UNROLL
#define PC_GRAM_UNROLL 12
#endif
#ifndef PC_DIRECT_UNROLL
#define PC_DIRECT_UNROLL 1
#endif
constexpr int kDirectUnroll = PC_DIRECT_UNROLL;
constexpr int kGramUnroll = PC_GRAM_UNROLL;


// dynamic shared memory per warp: 2 column buffers of W + one row buffer of T (PS/2 float4 per element)
template <int R, int W, bool COMP = false>
constexpr int pairs_smem_per_warp() {
    return (2 * W + 32 * R) / 2 * (COMP ? 3 : 2) * (int)sizeof(float4);
}

// SORTED (sum kernel, whole-range calls on spatially sorted fp32 points): a chunk whose
// columns are far from the tile's rows (per-32-point bounding boxes) is
// evaluated in Gram form against tile-local origins, p = A_i + (B_j - 2 a_i.b_j), with
// a_i = q_i - o, b_j = q_j - o, A_i = 1 + |a_i|^2, B_j = |b_j|^2: 4 packed ops per two
// pairs instead of 6.  Taken only where the bound on the form's rounding error,
// 8u (|a|max + |b|max)^2 (the subtractions a = q - o, b = q - o, the |b|^2 chain, three
// FFMA2 and the FADD2), is below 5e-6 (1 + dmin^2) -- every such term within 5e-6
// relative; the chunk is accumulated in two fp32 halves (gamma_32 = 1.9e-6), so the total
// stays below 1e-5 (DESIGN.md §3 "Error budget") -- and dmin > 2.12, so the chunk holds
// no contact.
// The boxes also decide the contact test: more than 1.5 apart, none; closer, each row's
// smallest p flags its candidates (the chunk-sum test would flag every row there).
template <int WARPS, int R, int W, bool DIRECT, bool FLAT, bool COMP = false, bool SORTED = false>
__global__ void __launch_bounds__(WARPS * 32, PC_MINB) pairs_kernel(const PairsArgs a) {
    constexpr int T = 32 * R;
    constexpr int PS = COMP ? 3 : 2;  // float4 per column pair
    static_assert(DIRECT || !COMP, "compensated staging is for the direct (sum) formula");
    static_assert(W % 64 == 0 && T % 64 == 0, "buffers must hold whole pairs for every lane");
    extern __shared__ __align__(16) float4 s_dyn[];
    __shared__ unsigned long long s_red[WARPS][2];
    // per-warp bookkeeping kept out of the register file (the loops run at 126-128 registers):
    // chunks per inner loop (kPath*) + rescanned rows, and the claim ids of the current / next chunk
    __shared__ unsigned s_path[WARPS][kNumPaths + 1];
    __shared__ long long s_claim[WARPS][2];
    __shared__ float s_tbox[WARPS][6];  // SORTED count: the claimed tile's box (min xyz, max xyz), raw coordinates
    __shared__ __align__(8) unsigned long long s_bar[WARPS][2];  // per-warp TMA completion, one per column buffer
    __shared__ double s_sum[WARPS];

    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const long long gw = (long long)blockIdx.x * WARPS + wid;
#ifdef PC_TIMELINE  // debug: per-warp start / end (globaltimer ns) into the claim-sum area's tail
    unsigned long long t_start = 0;
    if (DIRECT && FLAT) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
#endif
#ifndef PC_NO_F64EXIT
    if (DIRECT && f64_takes(*a.st, a.dtype, COMP)) {  // pairs_f64_kernel takes this call
        if (threadIdx.x == 0) a.slots[blockIdx.x] = Slot{};
        return;
    }
#endif
    const int n = a.n;
    const bool bal = a.sched == PC_BALANCED;

    // error bands, derived from the prep statistics
    const double M = dec_f64_or0(a.st->mnorm);
    const double X = dec_f64_or0(a.st->maxabs);
    const bool force = !DIRECT && !(M < 1e30);  // fp32 filter unusable: exact path for every pair
    const float half_tb = (float)(0.5 * ((double)a.thr + 3.814697265625e-06 * (M + 4.0)));
    const double bd = 1.52587890625e-05 + (a.dtype == PC_F32 ? 0.0 : 9.5367431640625e-07 * X);
    const float thr2 = (float)(1.0 + (double)a.thr + bd);
    // a contact's term 1/p exceeds 1/thr2; chunk sums of positive terms keep that (fp32 slack 2^-16)
    const float sum_flag = (float)((1.0 / (double)thr2) * (1.0 - 1.52587890625e-05));
    const int steps_min = (n & 1) ? (n - 1) >> 1 : (n >> 1) - 1;

    // this warp's walk: `left` columns starting at (tile, off); L = window length
    int tile, off, L;
    long long left = 0;
    // FLAT: warps claim work from one global counter in guided stages (kMaxStages), so
    // SM-to-SM speed differences and slow-path rescans cannot leave a tail.
    // Claims index a block-transposed order of the (tile, window column) space: block b of blk_cols
    // columns is window block b / n_tiles of tile b % n_tiles (window blocks ordered 0, last, 1, 2,
    // ...), so every tile's leading block (the masked self chunk and, on sorted points, the near
    // chunks with their rescans) and its trailing block (the ragged masked end of the window) are
    // handed out before any far block, and the tail is uniform far work.  A claim never crosses a block
    // (stage sizes are powers of two dividing the block); one that falls past a window's end is
    // empty and skipped.
    auto count_path = [&](int k, unsigned v) {
#ifndef PC_NO_PATHS
        if (lane == 0) s_path[wid][k] += v;
#endif
    };
    // SORTED count (pruning, PAPER.md:443 -- the all-pairs count composed with a box test): the
    // union box of sorted points [j, j + cnt) (mod n) from the per-32 (lvl 1) or per-1024 (lvl 2)
    // boxes against the claimed tile's box; a gap beyond the contact distance decides every pair
    // of the range (no contact) without evaluating it -- counted apart (kPathFar), never as
    // evaluated pairs.
    const float cull_gap2 = a.thr * 1.0001f;
    auto union_far = [&](long long j, long long cnt, const float4* box, int shift) -> bool {
        long long ja = j >= n ? j - n : j;
        const long long je = ja + cnt - 1;  // last column before wrapping
        const int b0 = (int)(ja >> shift), b1 = (int)(min(je, (long long)n - 1) >> shift);
        const int nb1 = b1 - b0 + 1, nb2 = je >= n ? (int)((je - n) >> shift) + 1 : 0;
        float g2 = 0.f;
        for (int base = 0; base < nb1 + nb2; base += 32) {  // chunks: <= 8 boxes; claims: a few dozen
            float cmn[3] = {INFINITY, INFINITY, INFINITY}, cmx[3] = {-INFINITY, -INFINITY, -INFINITY};
            const int q = base + lane;
            if (q < nb1 + nb2) {
                const int b = q < nb1 ? b0 + q : q - nb1;
                const float4 lo4 = box[2 * b], hi4 = box[2 * b + 1];
                cmn[0] = lo4.x; cmn[1] = lo4.y; cmn[2] = lo4.z;
                cmx[0] = hi4.x; cmx[1] = hi4.y; cmx[2] = hi4.z;
            }
            float gg = 0.f;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const float cl = warp_min_f(cmn[k]), ch = warp_max_f(cmx[k]);
                const float gk = fmaxf(0.f, fmaxf(cl - s_tbox[wid][3 + k], s_tbox[wid][k] - ch));
                gg += gk * gk;
            }
            if (base == 0) g2 = gg;
            else g2 = fminf(g2, gg);  // a union over several passes: the nearest part decides
        }
        return g2 > cull_gap2;
    };
    auto tile_box = [&](int tt) {  // the rows of tile tt from the per-32 boxes
        const int i0t = a.lo + tile_abs(tt, a.tstride, a.toff) * T;
        const int i1t = min(i0t + T, a.hi) - 1;
        const int b0 = i0t >> 5, nb = (i1t >> 5) - b0 + 1;
        float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
        if (lane < nb) {
            const float4 lo4 = a.blk_box[2 * (b0 + lane)], hi4 = a.blk_box[2 * (b0 + lane) + 1];
            mn[0] = lo4.x; mn[1] = lo4.y; mn[2] = lo4.z;
            mx[0] = hi4.x; mx[1] = hi4.y; mx[2] = hi4.z;
        }
        float v[6];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            v[k] = warp_min_f(mn[k]);
            v[3 + k] = warp_max_f(mx[k]);
        }
        __syncwarp();
        if (lane == 0) {
#pragma unroll
            for (int k = 0; k < 6; ++k) s_tbox[wid][k] = v[k];
        }
        __syncwarp();
    };
    auto claim = [&](int& t, int& o, long long& lft) {
        for (;;) {
            unsigned long long c = 0;
            if (lane == 0) c = atomicAdd(a.work_ctr, 1ull);
            c = __shfl_sync(0xffffffffu, c, 0);
            int k = 0;
            while (k < a.nstage && (long long)c >= a.st_c0[k + 1]) ++k;
            if (k == a.nstage) {
                lft = 0;
                return;
            }
            const long long v = a.st_b0[k] + ((long long)c - a.st_c0[k]) * a.st_s[k];
            const long long blk = v / a.blk_cols;
            const int tt = (int)(blk % a.n_tiles);
            long long ob = blk / a.n_tiles;  // window blocks in the order 0, last, 1, 2, ...: both ragged ends early
            ob = ob == 0 ? 0 : ob == 1 ? a.win_blks - 1 : ob - 1;
            const long long oo = ob * a.blk_cols + (v - blk * a.blk_cols);
            const long long len = min(a.st_s[k], (long long)L - oo);
            if (len <= 0) continue;  // past the end of the window
            if (SORTED && !DIRECT) {
                tile_box(tt);
                const long long jc = (long long)a.lo + (long long)tile_abs(tt, a.tstride, a.toff) * T + oo + 1;
                if (union_far(jc, len, a.blk2_box, 10)) {
                    count_path(kPathFar, (unsigned)((len + W - 1) / W));
                    continue;  // every pair of the claim decided by its boxes
                }
            }
            if (lane == 0) s_claim[wid][1] = (long long)c;  // the next chunk's claim
            t = tt;
            o = (int)oo;
            lft = len;
            return;
        }
    };
    // first row of tile t of this call (tiles toff, toff + tstride, ... of [lo, hi))
    auto row0 = [&](int t) -> int { return a.lo + tile_abs(t, a.tstride, a.toff) * T; };
    if (lane < kNumPaths + 1) s_path[wid][lane] = 0u;
    __syncwarp();
    if (FLAT) {
        L = (int)a.L;
        tile = 0;
        off = 0;
        claim(tile, off, left);
    } else {
        tile = (int)gw;
        off = 0;
        L = 0;
        if (gw < a.n_tiles) {
            const int i0 = row0(tile);
            L = bal ? T - 1 + (n >> 1) : n - 1 - i0;
        }
        left = L;
    }
    auto width = [&](int o, long long lft) -> int {
        const int w = min(W, L - o);
        return (int)(w < lft ? w : lft);
    };
    // SORTED sum with the tensor-core split and its chunk bitmap (tcs_classify_kernel): step over the
    // chunks pairs_tcs_kernel evaluates before staging them, claiming on as claims run out
    auto skip_tc = [&](int& t, int& o, long long& lft) {
        if (!(SORTED && DIRECT && FLAT) || !a.tc_bits) return;
        while (lft > 0) {
            const long long b = (long long)t * a.tc_cpw_pad + o / W;
            if (!((__ldg(a.tc_bits + (b >> 5)) >> (b & 31)) & 1u)) return;
            const int w_ = width(o, lft);
            o += w_;
            if (o == L) {
                ++t;
                o = 0;
            }
            lft -= w_;
            if (lft == 0) claim(t, o, lft);
        }
    };
    if (FLAT) {
        skip_tc(tile, off, left);
        if (lane == 0) s_claim[wid][0] = s_claim[wid][1];
    }
    auto wrap = [&](int j) -> int {
        if (j >= n) j -= n;
        if (j >= n) j %= n;
        return j;
    };
    auto pair_src = [&](int j) -> const float4* {  // pair (j, (j+1) mod n)
        PC_CHECK(j >= 0 && j < n);
        return (j & 1 ? a.pts_odd : a.pts_even) + PS * (j >> 1);
    };

    float4* sp0 = s_dyn + (size_t)wid * ((2 * W + T) / 2 * PS);  // column buffers [2][W elements]
    float4* rowbuf = sp0 + W * PS;                                // row buffer [T elements]
    // a far column (0, 0, 0, fw): its Gram value is -inf, never a candidate
    const float fw = DIRECT ? 0.f : -INFINITY;
    auto stage_cols = [&](int buf, int t, int o, int wc) {
        const int j0 = row0(t) + o + 1;  // column k sits at j0 + k (mod n when balanced)
        float4* sp = sp0 + buf * (W / 2 * PS);
#pragma unroll
        for (int q = 0; q < W / 64; ++q) {
            const int k = 2 * (q * 32 + lane);  // columns k, k+1
            float4* d = sp + PS * (k >> 1);
            if (k + 1 < wc) {
                const float4* src = pair_src(bal ? wrap(j0 + k) : j0 + k);
#pragma unroll
                for (int p = 0; p < PS; ++p) cp_async16(&d[p], src + p);
            } else if (k < wc) {  // last column of an odd-width chunk: second half is a far point
                const float4* src = pair_src(bal ? wrap(j0 + k) : j0 + k);
                const float4 A = src[0], B = src[1];
                d[0] = make_float4(A.x, 0.f, A.z, 0.f);
                d[1] = make_float4(B.x, 0.f, B.z, COMP ? 0.f : fw);
                if (COMP) {
                    const float4 C = src[2];
                    d[PS - 1] = make_float4(C.x, 0.f, C.z, 0.f);
                }
            } else {
                d[0] = make_float4(0.f, 0.f, 0.f, 0.f);
                d[1] = make_float4(0.f, 0.f, COMP ? 0.f : fw, COMP ? 0.f : fw);
                if (COMP) d[PS - 1] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
    };
    auto stage_rows = [&](int t) {  // rows i0 .. i0+T-1 (only those < n are read)
        const int i0 = row0(t);
#pragma unroll
        for (int q = 0; q < T / 64; ++q) {
            const int rl = 2 * (q * 32 + lane);  // rows rl, rl+1
            if (i0 + rl < n) {
                const float4* src = pair_src(i0 + rl);
#pragma unroll
                for (int p = 0; p < PS; ++p) cp_async16(&rowbuf[PS * (rl >> 1) + p], src + p);
            }
        }
    };

    float rx[R], ry[R], rz[R], rc[R];
    float tmin[3] = {0.f, 0.f, 0.f}, tmax[3] = {0.f, 0.f, 0.f};  // SORTED: the tile's bounding box
    float rxl[R], ryl[R], rzl[R];  // COMP: low parts of the row coordinates
    int cur_tile = -1;
    unsigned valid_rows = 0;
    unsigned long long cnt = 0, checks = 0;
    double sum = 0.0;

    // Staging of chunk (t, o, wcn) into column buffer b, with the tile's rows when asked.  A full
    // chunk whose window does not wrap is ONE contiguous run of pair entries, and a whole row tile
    // is one too: lane 0 hands each to a TMA bulk copy that completes on the buffer's mbarrier.
    // Ragged chunks (partial, wrapping, odd width) and the last row tile take per-lane cp.async.
    // TMA staging is on for the sum kernel (+1.0 %); the count kernel keeps per-lane cp.async, where
    // the extra live state cost 1.5 % (it runs at 128 registers).
    constexpr bool kTma = PC_TMA_STAGE && (DIRECT || PC_TMA_GRAM);
    const unsigned bar_base = (unsigned)__cvta_generic_to_shared(&s_bar[wid][0]);
    if (kTma) {
        if (lane == 0) {
            mbar_init(bar_base, 1);
            mbar_init(bar_base + 8, 1);
            mbar_init_fence();
        }
        __syncwarp();
    }
    unsigned pend = 0;  // bit b: TMA in flight into buffer b; bit 2: a cp.async group in flight
    unsigned phase = 0; // bit b: parity of buffer b's next mbarrier phase
    auto stage = [&](int b, int t, int o, int wcn, bool rows) {
        const int i0n = row0(t);
        int jw = i0n + o + 1;
        if (bal) jw = wrap(jw);
        const bool cols_tma = kTma && wcn == W && jw + W - 1 < n;
        const bool rows_tma = kTma && rows && i0n + T <= n;
        if (cols_tma || rows_tma) {
            if (lane == 0) {
                fence_proxy_async_shared();  // this warp's earlier generic reads of the buffers come first
                const unsigned cb = cols_tma ? W / 2 * PS * 16 : 0u, rb = rows_tma ? T / 2 * PS * 16 : 0u;
                const unsigned bar = bar_base + 8u * b;
                mbar_expect_tx(bar, cb + rb);
                PC_CHECK(!cols_tma || (jw >= 0 && jw + W <= n));
                PC_CHECK(!rows_tma || (i0n >= 0 && i0n + T <= n));
                if (cols_tma) bulk_g2s(sp0 + b * (W / 2 * PS), pair_src(jw), cb, bar);
                if (rows_tma) bulk_g2s(rowbuf, pair_src(i0n), rb, bar);
            }
            pend |= 1u << b;
        }
        if (!cols_tma || (rows && !rows_tma)) {
            if (!cols_tma) stage_cols(b, t, o, wcn);
            if (rows && !rows_tma) stage_rows(t);
            cp_async_commit();
            pend |= 4u;
        }
    };

    int wc = left > 0 ? width(off, left) : 0;
    if (left > 0) {
        if (kTma) {
            stage(0, tile, off, wc, true);
        } else {
            stage_rows(tile);
            stage_cols(0, tile, off, wc);
            cp_async_commit();
        }
    }
    int buf = 0;
    int staged_tile = tile;  // tile whose rows the row buffer receives / holds
    while (left > 0) {
        // chunk `buf` (and, on a switch, its tile's rows) landed
        if (kTma) {
            if (pend & 4u) {
                cp_async_wait<0>();
                pend &= ~4u;
            }
            if (pend & (1u << buf)) {
                mbar_wait(bar_base + 8u * buf, (phase >> buf) & 1u);
                phase ^= 1u << buf;
                pend &= ~(1u << buf);
            }
        } else {
            cp_async_wait<0>();
        }
        __syncwarp();
        const int i0 = row0(tile);
        if (tile != cur_tile) {
            cur_tile = tile;
            valid_rows = 0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int rl = r * 32 + lane;
                const bool ok = i0 + rl < a.hi;
                const float4 v = col_hi<COMP>(rowbuf, rl);
                rx[r] = ok ? v.x : 0.f;
                ry[r] = ok ? v.y : 0.f;
                rz[r] = ok ? v.z : 0.f;
                if (COMP) {
                    const float4 vl = col_lo(rowbuf, rl);
                    rxl[r] = ok ? vl.x : 0.f;
                    ryl[r] = ok ? vl.y : 0.f;
                    rzl[r] = ok ? vl.z : 0.f;
                }
                rc[r] = ok ? (force ? -INFINITY : -v.w - half_tb) : INFINITY;
                valid_rows |= (ok ? 1u : 0u) << r;
            }
            if (SORTED && DIRECT) {
                float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if ((valid_rows >> r) & 1u) {
                        mn[0] = fminf(mn[0], rx[r]); mx[0] = fmaxf(mx[0], rx[r]);
                        mn[1] = fminf(mn[1], ry[r]); mx[1] = fmaxf(mx[1], ry[r]);
                        mn[2] = fminf(mn[2], rz[r]); mx[2] = fmaxf(mx[2], rz[r]);
                    }
                }
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    tmin[k] = warp_min_f(mn[k]);
                    tmax[k] = warp_max_f(mx[k]);
                }
            }
            __syncwarp();  // the row buffer may be restaged below
        }

        // SORTED count: is this chunk beyond contact distance of its tile?  (decided before the next
        // claim, which may load the next tile's box)
        bool chunk_far = false;
        if (SORTED && !DIRECT) chunk_far = union_far((long long)i0 + off + 1, wc, a.blk_box, 5);
        // next chunk's coordinates (incremental: no divisions in the loop); stage it now
        int ntile = tile, noff = off + wc;
        if (noff == L) {
            ++ntile;
            noff = 0;
        }
        long long nleft = left - wc;
        if (FLAT && nleft == 0) claim(ntile, noff, nleft);
        if (FLAT) skip_tc(ntile, noff, nleft);
        const int nwc = nleft > 0 ? width(noff, nleft) : 0;
        if (nleft > 0) {
            if (kTma) {
                const bool new_rows = ntile != staged_tile;
                staged_tile = ntile;
                stage(buf ^ 1, ntile, noff, nwc, new_rows);
            } else {
                if (ntile != staged_tile) {
                    stage_rows(ntile);
                    staged_tile = ntile;
                }
                stage_cols(buf ^ 1, ntile, noff, nwc);
                cp_async_commit();
            }
        }

        const float4* sp = sp0 + buf * (W / 2 * PS);
        const int j0 = i0 + off + 1;
        // every cell of the chunk owned by its row?  (see header comment)
        const bool dense = wc == W && i0 + T <= a.hi && off + 1 >= T && (!bal || off + W <= steps_min);
        unsigned fl = 0;

        if (!DIRECT) {
            float m[R];
#pragma unroll
            for (int r = 0; r < R; ++r) m[r] = -INFINITY;
            count_path(chunk_far ? kPathFar : off + 1 >= T ? kPathMain : kPathEdge, 1u);
            if (chunk_far) {
                // no pair of this chunk can be in contact: nothing to evaluate
            } else if (off + 1 >= T) {
                // ---- Gram filter, packed: 3 FFMA2 + 1 FMNMX3 per two pairs.  Unowned
                // cells past a row's window only cost a rescan if they are contacts.
#pragma unroll kGramUnroll
                for (int k = 0; k < W; k += 2) {
                    const float4 A = sp[k], B = sp[k + 1];
                    const float2 cx = make_float2(A.x, A.y), cy = make_float2(A.z, A.w);
                    const float2 cz = make_float2(B.x, B.y), cw = make_float2(B.z, B.w);
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        float2 t = f2_fma(rx[r], cx, cw);
                        t = f2_fma(ry[r], cy, t);
                        t = f2_fma(rz[r], cz, t);
                        m[r] = max3f(m[r], t.x, t.y);
                    }
                }
            } else {
                // ---- leading chunk: mask cells at or before the row (incl. the self pair)
                for (int k = 0; k < W; k += 2) {
                    const float4 A = sp[k], B = sp[k + 1];
                    const float2 cx = make_float2(A.x, A.y), cy = make_float2(A.z, A.w);
                    const float2 cz = make_float2(B.x, B.y), cw = make_float2(B.z, B.w);
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int d = off + k - (r * 32 + lane);  // s' - rl - 1 for column k
                        float2 t = f2_fma(rz[r], cz, f2_fma(ry[r], cy, f2_fma(rx[r], cx, cw)));
                        m[r] = max3f(m[r], d >= 0 ? t.x : -INFINITY, d + 1 >= 0 ? t.y : -INFINITY);
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < R; ++r) fl |= (m[r] > rc[r] ? 1u : 0u) << r;
            if (force) fl = valid_rows;
        } else {
            float2 acc[R];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = make_float2(0.f, 0.f);
            bool gram = false, no_contact = false, tc_skip = false;
            unsigned near_fl = 0;  // SORTED near chunks: rows with some p < thr2
            float o[3] = {0.f, 0.f, 0.f};
            if (SORTED && dense) {
                // the chunk's bounding box from the per-32-point boxes it covers; columns are
                // j0 .. j0+W-1 mod n: one run of blocks, or two when the window wraps
                const int jw = j0 >= n ? j0 - n : j0;
                const int jend = jw + W - 1;  // last column, before wrapping
                const int nb1 = (min(jend, n - 1) >> 5) - (jw >> 5) + 1;
                const int nb2 = jend >= n ? ((jend - n) >> 5) + 1 : 0;
                float cmn[3] = {INFINITY, INFINITY, INFINITY}, cmx[3] = {-INFINITY, -INFINITY, -INFINITY};
                if (lane < nb1 + nb2) {
                    const int b = lane < nb1 ? (jw >> 5) + lane : lane - nb1;
                    const float4 lo4 = a.blk_box[2 * b], hi4 = a.blk_box[2 * b + 1];
                    cmn[0] = lo4.x; cmn[1] = lo4.y; cmn[2] = lo4.z;
                    cmx[0] = hi4.x; cmx[1] = hi4.y; cmx[2] = hi4.z;
                }
                float cl[3], ch[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    cl[k] = warp_min_f(cmn[k]);
                    ch[k] = warp_max_f(cmx[k]);
                }
                const ChunkGeom cg = chunk_geom(tmin, tmax, cl, ch);
#pragma unroll
                for (int k = 0; k < 3; ++k) o[k] = cg.o[k];
                const float gap2 = cg.gap2, ab = cg.ab;
                // a chunk the tensor-core kernel evaluates (pairs_tcsum.cuh): nothing to do here
                // (with the bitmap: skipped above; in-loop, the same test about the origin group's centre)
                if (a.tc_split && !a.tc_bits) {
                    PC_CHECK(T == 256 && W == 256);
                    float gmn[3], gmx[3];
                    tcs_group_box(a.blk_box, a.lo, a.hi, tile_abs(tile, a.tstride, a.toff), lane, gmn, gmx);
                    tc_skip = tcs_takes(chunk_geom_g(tmin, tmax, gmn, gmx, cl, ch));
                }
#ifdef PC_DBG_SKIPALL  // debug (timing only): every dense chunk skipped -- the walk's own cost
                tc_skip = true;
#endif
                // 8u (|a| + |b|)^2 <= 5e-6 (1 + dmin^2), u = 2^-24 -- written as the same
                // inequality 5u (..)^2 <= 3.125e-6 (..): eight roundings of terms of at most
                // (|a| + |b|)^2 against p >= 1 + dmin^2
#ifndef PC_GRAM_HALVES
#define PC_GRAM_HALVES 1
#endif
#ifndef PC_GRAM_BUDGET
#define PC_GRAM_BUDGET (PC_GRAM_HALVES ? 3.125e-6f : 2e-6f)
#endif
#ifndef PC_GRAM_GAP2
#define PC_GRAM_GAP2 4.5f
#endif
                // compensated (float64) points: a = (hi - o) + lo rounds once more: 10u instead of 8u
                constexpr float kGramU = COMP ? 3.725290298461914e-07f : 2.98023223876953125e-07f;
                gram = !tc_skip && gap2 > PC_GRAM_GAP2 && kGramU * ab * ab <= PC_GRAM_BUDGET * (1.f + gap2);
                // boxes more than 1.5 apart: no contact, so no rescan however large the chunk's
                // sums (on sorted points the chunks next to a tile have many near terms)
                no_contact = gap2 > 2.25f;
            }
            if (SORTED && tc_skip) {
                // evaluated on the tensor cores (no contact: gap > 2.12)
            } else if (SORTED && gram) {
                // columns to tile-local form in place: (bx, by, bz, B = |b|^2) per point
                // (compensated entries: b = (hi - o) + lo, written over the entry's first two float4)
                float4* spw = const_cast<float4*>(sp);
#pragma unroll
                for (int q = 0; q < W / 64; ++q) {
                    const int e = q * 32 + lane;  // pair entry: points 2e, 2e+1 of the chunk
                    const float4 A = spw[PS * e], B = spw[PS * e + 1];
                    float bx0 = A.x - o[0], bx1 = A.y - o[0], by0 = A.z - o[1], by1 = A.w - o[1];
                    float bz0 = B.x - o[2], bz1 = B.y - o[2];
                    if (COMP) {
                        const float4 C = spw[PS * e + 2];
                        bx0 += B.z; bx1 += B.w; by0 += C.x; by1 += C.y; bz0 += C.z; bz1 += C.w;
                    }
                    spw[PS * e] = make_float4(bx0, bx1, by0, by1);
                    spw[PS * e + 1] = make_float4(bz0, bz1, fmaf(bz0, bz0, fmaf(by0, by0, bx0 * bx0)),
                                                  fmaf(bz1, bz1, fmaf(by1, by1, bx1 * bx1)));
                }
                __syncwarp();
                // rows in Gram form in the row registers themselves (restored from the row
                // buffer after the chunk): -2 a_i and A_i = 1 + |a_i|^2
                float ga[R];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    float ax = rx[r] - o[0], ay = ry[r] - o[1], az = rz[r] - o[2];
                    if (COMP) {
                        ax += rxl[r];
                        ay += ryl[r];
                        az += rzl[r];
                    }
                    rx[r] = -2.f * ax;
                    ry[r] = -2.f * ay;
                    rz[r] = -2.f * az;
                    ga[r] = 1.f + fmaf(az, az, fmaf(ay, ay, ax * ax));
                }
                float* gx = rx;
                float* gy = ry;
                float* gz = rz;
#if PC_GRAM_HALVES
                // two halves of W/2 columns, each row's fp32 partial flushed to float64 in between:
                // the in-chunk accumulation error of a Gram chunk is gamma_32, not gamma_64, which
                // pays for the wider Gram error budget (DESIGN.md §3 "Error budget")
#pragma unroll 1
                for (int half = 0; half < 2; ++half) {
                if (half) {
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        sum += (double)(acc[r].x + acc[r].y);
                        acc[r] = make_float2(0.f, 0.f);
                    }
                }
#pragma unroll kDirectUnroll
                for (int k = half * (W / 2); k < (half + 1) * (W / 2); k += 4) {
#else
#pragma unroll kDirectUnroll
                for (int k = 0; k < W; k += 4) {
#endif
                    const float4* E = sp + PS * (k >> 1);  // entries of columns k, k+1 and k+2, k+3
                    const float4 A0 = E[0], B0 = E[1], A1 = E[PS], B1 = E[PS + 1];
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        float2 t0 = f2_fma(gx[r], make_float2(A0.x, A0.y), make_float2(B0.z, B0.w));
                        t0 = f2_fma(gy[r], make_float2(A0.z, A0.w), t0);
                        t0 = f2_fma(gz[r], make_float2(B0.x, B0.y), t0);
                        float2 t1 = f2_fma(gx[r], make_float2(A1.x, A1.y), make_float2(B1.z, B1.w));
                        t1 = f2_fma(gy[r], make_float2(A1.z, A1.w), t1);
                        t1 = f2_fma(gz[r], make_float2(B1.x, B1.y), t1);
                        const float2 p0 = __fadd2_rn(t0, make_float2(ga[r], ga[r]));
                        const float2 p1 = __fadd2_rn(t1, make_float2(ga[r], ga[r]));
                        const float2 pr = __fmul2_rn(p0, p1), sm = __fadd2_rn(p0, p1);
                        acc[r] = __ffma2_rn(sm, make_float2(rcp_approx(pr.x), rcp_approx(pr.y)), acc[r]);
                    }
                }
#if PC_GRAM_HALVES
                }
#endif
            } else if (COMP && dense) {
                // ---- compensated direct formula: dr = (hi_i - hi_j) + (lo_i - lo_j) keeps the
                // separation to ~2u relative however far the points sit from the centre
                const float2 one = make_float2(1.0f, 1.0f);
#pragma unroll 1
                for (int k = 0; k < W; k += 4) {
                    const float4* P = sp + 3 * (k >> 1);
                    const float4 A0 = P[0], B0 = P[1], C0 = P[2], A1 = P[3], B1 = P[4], C1 = P[5];
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        float2 dx = __fadd2_rn(f2_rsub(rx[r], make_float2(A0.x, A0.y)), f2_rsub(rxl[r], make_float2(B0.z, B0.w)));
                        float2 dy = __fadd2_rn(f2_rsub(ry[r], make_float2(A0.z, A0.w)), f2_rsub(ryl[r], make_float2(C0.x, C0.y)));
                        float2 dz = __fadd2_rn(f2_rsub(rz[r], make_float2(B0.x, B0.y)), f2_rsub(rzl[r], make_float2(C0.z, C0.w)));
                        const float2 p0 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __ffma2_rn(dx, dx, one)));
                        dx = __fadd2_rn(f2_rsub(rx[r], make_float2(A1.x, A1.y)), f2_rsub(rxl[r], make_float2(B1.z, B1.w)));
                        dy = __fadd2_rn(f2_rsub(ry[r], make_float2(A1.z, A1.w)), f2_rsub(ryl[r], make_float2(C1.x, C1.y)));
                        dz = __fadd2_rn(f2_rsub(rz[r], make_float2(B1.x, B1.y)), f2_rsub(rzl[r], make_float2(C1.z, C1.w)));
                        const float2 p1 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __ffma2_rn(dx, dx, one)));
                        const float2 pr = __fmul2_rn(p0, p1), sm = __fadd2_rn(p0, p1);
                        acc[r] = __ffma2_rn(sm, make_float2(rcp_approx(pr.x), rcp_approx(pr.y)), acc[r]);
                    }
                }
            } else if (SORTED && dense && !no_contact) {
                // ---- a chunk next to the tile on sorted points: many moderately near terms, so
                // the chunk-sum test would flag nearly every row; track each row's smallest p
                // instead (two FMNMX3 per four pairs) and flag the rows with a candidate
                const float2 one = make_float2(1.0f, 1.0f);
                float pm[R];
#pragma unroll
                for (int r = 0; r < R; ++r) pm[r] = INFINITY;
#pragma unroll 1
                for (int k = 0; k < W; k += 4) {
                    const float4 A0 = sp[k], B0 = sp[k + 1], A1 = sp[k + 2], B1 = sp[k + 3];
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        float2 dx = f2_rsub(rx[r], make_float2(A0.x, A0.y));
                        float2 dy = f2_rsub(ry[r], make_float2(A0.z, A0.w));
                        float2 dz = f2_rsub(rz[r], make_float2(B0.x, B0.y));
                        const float2 p0 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __ffma2_rn(dx, dx, one)));
                        dx = f2_rsub(rx[r], make_float2(A1.x, A1.y));
                        dy = f2_rsub(ry[r], make_float2(A1.z, A1.w));
                        dz = f2_rsub(rz[r], make_float2(B1.x, B1.y));
                        const float2 p1 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __ffma2_rn(dx, dx, one)));
                        pm[r] = fminf(min3f(pm[r], p0.x, p0.y), fminf(p1.x, p1.y));
                        const float2 pr = __fmul2_rn(p0, p1), sm = __fadd2_rn(p0, p1);
                        acc[r] = __ffma2_rn(sm, make_float2(rcp_approx(pr.x), rcp_approx(pr.y)), acc[r]);
                    }
                }
#pragma unroll
                for (int r = 0; r < R; ++r) near_fl |= (pm[r] < thr2 ? 1u : 0u) << r;
            } else if (dense) {
                // ---- direct formula, packed: p = 1 + |dr|^2 for two columns per FADD2/FFMA2;
                // two column pairs share one FMUL2/FADD2/FFMA2 for 1/pa + 1/pc = (pa+pc)/(pa*pc)
                const float2 one = make_float2(1.0f, 1.0f);
#pragma unroll kDirectUnroll
                for (int k = 0; k < W; k += 4) {
                    const float4 A0 = sp[k], B0 = sp[k + 1], A1 = sp[k + 2], B1 = sp[k + 3];
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        float2 dx = f2_rsub(rx[r], make_float2(A0.x, A0.y));
                        float2 dy = f2_rsub(ry[r], make_float2(A0.z, A0.w));
                        float2 dz = f2_rsub(rz[r], make_float2(B0.x, B0.y));
                        const float2 p0 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __ffma2_rn(dx, dx, one)));
                        dx = f2_rsub(rx[r], make_float2(A1.x, A1.y));
                        dy = f2_rsub(ry[r], make_float2(A1.z, A1.w));
                        dz = f2_rsub(rz[r], make_float2(B1.x, B1.y));
                        const float2 p1 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __ffma2_rn(dx, dx, one)));
                        const float2 pr = __fmul2_rn(p0, p1), sm = __fadd2_rn(p0, p1);
                        acc[r] = __ffma2_rn(sm, make_float2(rcp_approx(pr.x), rcp_approx(pr.y)), acc[r]);
                    }
                }
            } else {
                // ---- edge chunk: per-pair ownership mask ----
                for (int k = 0; k < W; ++k) {
                    const float4 c0 = col_hi<COMP>(sp, k);
                    const float4 l0 = COMP ? col_lo(sp, k) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int rl = r * 32 + lane;
                        const int i = i0 + rl;
                        const int lim = i < a.hi ? (bal ? steps_for_dev(n, i) : n - 1 - i) : 0;
                        const bool ok = k < wc && (unsigned)(off + k - rl) < (unsigned)lim;
                        float dx = rx[r] - c0.x, dy = ry[r] - c0.y, dz = rz[r] - c0.z;
                        if (COMP) {
                            dx += rxl[r] - l0.x;
                            dy += ryl[r] - l0.y;
                            dz += rzl[r] - l0.z;
                        }
                        const float p = fmaf(dz, dz, fmaf(dy, dy, fmaf(dx, dx, 1.0f)));
                        acc[r].x += ok ? rcp_approx(p) : 0.0f;
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const float cs = acc[r].x + acc[r].y;
                sum += (double)cs;
                fl |= (cs > sum_flag ? 1u : 0u) << r;  // conservative: a contact's term alone exceeds it
            }
            if (!(SORTED && tc_skip)) {
                count_path((SORTED && gram) ? kPathGram
                           : !dense ? kPathEdge
                           : (SORTED && !COMP && !no_contact) ? kPathNear
                           : (SORTED && COMP) ? (no_contact ? kPathFar : kPathMain)
                           : SORTED ? kPathFar : kPathMain, 1u);
            }
            if (SORTED && no_contact) fl = 0;  // also covers the Gram chunks, whose columns were rewritten
            if (SORTED && !COMP && dense && !no_contact) fl = near_fl;  // exact candidates, not chunk sums
            if (SORTED && gram && staged_tile == tile) {
                // back to the raw rows for the tile's next chunks (a new tile reloads them anyway)
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const float4 v = col_hi<COMP>(rowbuf, r * 32 + lane);
                    const bool ok = (valid_rows >> r) & 1u;
                    rx[r] = ok ? v.x : 0.f;
                    ry[r] = ok ? v.y : 0.f;
                    rz[r] = ok ? v.z : 0.f;
                }
            }
        }

        // ---- slow path (warp-cooperative): each flagged row is broadcast and all
        // 32 lanes re-test its W columns in parallel; every owned candidate is
        // re-evaluated with the exact reference predicate by the lane that found it.
        // (A lane-serial rescan cost ~800 instructions per flagged row and, 8x
        // unrolled, thrashed the I-cache at N = 65,536 where ~1 chunk in 1 flags.)
        if (__any_sync(0xffffffffu, fl != 0)) {
            auto rescan = [&](float vx, float vy, float vz, float vc, int r, unsigned owners) {
                while (owners) {
                    const int src = __ffs(owners) - 1;
                    owners &= owners - 1;
                    const float qx = __shfl_sync(0xffffffffu, vx, src);
                    const float qy = __shfl_sync(0xffffffffu, vy, src);
                    const float qz = __shfl_sync(0xffffffffu, vz, src);
                    const float qc = __shfl_sync(0xffffffffu, vc, src);
                    const int rl = r * 32 + src;
                    const int i = i0 + rl;
                    const int lim = bal ? steps_for_dev(n, i) : n - 1 - i;  // flagged rows are valid rows
#pragma unroll 2
                    for (int q = 0; q < W / 32; ++q) {
                        const int k = q * 32 + lane;
                        const float4 c0 = col_hi<COMP>(sp, k);
                        bool cand;
                        if (DIRECT) {
                            const float dx = qx - c0.x, dy = qy - c0.y, dz = qz - c0.z;
                            cand = fmaf(dz, dz, fmaf(dy, dy, fmaf(dx, dx, 1.0f))) < thr2;
                        } else {
                            const float tt = fmaf(qz, c0.z, fmaf(qy, c0.y, fmaf(qx, c0.x, c0.w)));
                            cand = force || tt > qc;
                        }
                        if (cand && k < wc && (unsigned)(off + k - rl) < (unsigned)lim) {
                            ++checks;
                            const int j = bal ? wrap(j0 + k) : j0 + k;
                            PC_CHECK(i >= a.lo && i < a.hi && j >= 0 && j < n && j != i);
                            cnt += exact_pair_call(a.xyz, a.dtype, a.pred, i, j) ? 1ull : 0ull;
                        }
                    }
                }
            };
            // One out-of-line copy of the rescan and the exact re-check for all R
            // rows, the row's registers picked by an unrolled select (no dynamic
            // register indexing).  Inlined once per row the kernel was 178 KB of
            // SASS; slim it is 1.4% faster for the sum, 8% for the count at
            // N = 65,536 and 7% on the clustered 2^22 set (most chunks flag a row).
            // rows flagged by any lane, one REDUX; visit only those
            unsigned rows_any = __reduce_or_sync(0xffffffffu, fl);
            while (rows_any) {
                const int r = __ffs(rows_any) - 1;
                rows_any &= rows_any - 1;
                const unsigned owners = __ballot_sync(0xffffffffu, (fl >> r) & 1u);
                count_path(kNumPaths, __popc(owners));
                float vx = 0.f, vy = 0.f, vz = 0.f, vc = 0.f;
#pragma unroll
                for (int rr = 0; rr < R; ++rr)
                    if (rr == r) {
                        vx = rx[rr];
                        vy = ry[rr];
                        vz = rz[rr];
                        vc = rc[rr];
                    }
                rescan(vx, vy, vz, vc, r, owners);
            }
        }
        __syncwarp();  // the buffer just read is restaged next iteration (and s_claim is visible)
        if (FLAT) {
            // end of a claim (a new one was taken for the next chunk, or the work ran out): its
            // float64 partial goes to its own slot, a fixed association (DESIGN.md §3 "Slots").
            // Decided from shared memory so no flag stays live across the inner loops.
            const long long c0 = s_claim[wid][0], c1 = s_claim[wid][1];
            if (c0 != c1 || nleft == 0) {
                if (DIRECT) {
                    const double cs = warp_sum(sum);
                    PC_CHECK(c0 >= 0 && c0 < a.st_c0[a.nstage]);
                    if (lane == 0) a.claim_sums[c0] = cs;
                    sum = 0.0;
                }
                __syncwarp();
                if (lane == 0) s_claim[wid][0] = c1;
            }
        }
        tile = ntile;
        off = noff;
        left = nleft;
        wc = nwc;
        buf ^= 1;
    }

#ifdef PC_TIMELINE
    if (DIRECT && FLAT && lane == 0) {
        unsigned long long t_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        unsigned long long* tl = reinterpret_cast<unsigned long long*>(a.claim_sums + (kClaimsCap - 2 * 8192));
        if (gw < 4096) {
            tl[2 * gw] = t_start;
            tl[2 * gw + 1] = t_end;
        }
    }
#endif
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
        Slot s{};
        for (int q = 0; q < WARPS; ++q) {
            s.count += s_red[q][0];
            s.checks += s_red[q][1];
            s.sum += s_sum[q];
            for (int k = 0; k < kNumPaths; ++k) s.path[k] += s_path[q][k];
            s.rescans += s_path[q][kNumPaths];
        }
        a.slots[blockIdx.x] = s;
    }
}
