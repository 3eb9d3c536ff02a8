// K2 v3 — "tiled phases": gather-sum-select with 4 users per lane
// (Eq. 5; Algorithm 1).
//
// The binding resource of Eq. 5 is the shared-memory lookup rate
// (148 SMs x 32 four-byte words per clock).  K2 v2 reached it only halfway
// because every lookup cost three issue slots (address op, LDS.32, FADD) and
// the TMEM-resident splits cost more.  Here a lane serves FOUR users of one item:
//
//   * Table layout (as v2): a CTA owns 16 users; row (k, c') of split k is 16
//     fp32 words (64 B = half the banks), word w = user w.  pq_create has
//     2-coloured the sub-ids (stored code c' parity = colour) and paired items
//     whose colours are complementary at every split.
//   * Lane l: pair (l >> 3) of the warp's slot, item h = (l >> 2) & 1 of the
//     pair, user quad q = l & 3 (users 4q .. 4q+3).  One LDS.128 per lane per
//     split returns the item's 4 users' sub-scores.  A 128-bit shared load is
//     served per quarter-warp: lanes 0-3 read item A's row, lanes 4-7 item B's
//     row, the two rows lie in opposite bank halves -> one conflict-free
//     wavefront per quarter, 128 lookups per 4 wavefronts (the peak rate).
//   * The 4 users' sums are two FADD2 (packed fp32x2 add, IEEE RN per lane,
//     the same rounding as the scalar add), so a split costs 1 address op +
//     1 LDS.128 + 2 FADD2 for 4 lookups (v2: 12 issue slots).
//
// Capacity.  16 users x m x b x 4 B must fit in shared memory for the whole
// table (m*b <= 2048 with double buffering off: C2/C3 m = 8, 128 KB).  For
// m = 16 (256 KB, C4) the splits are processed in NP phases of PS = 4 splits:
// phase tables (64 KB) are double-buffered in shared memory and loaded by the
// TMA bulk engine (cp.async.bulk + mbarrier) from a pre-tiled copy of S; the
// running partial sums of a tile of 4096 items x 16 users live in TENSOR
// MEMORY between phases (tcgen05.st / tcgen05.ld 32x32b.x4: lane = TMEM row,
// 4 columns per slot; each warp owns 512/(W/4) columns of its lane quadrant).
// The fp32 order is unchanged: acc = S[0], then + S[1], ..., + S[m-1] split by
// split (a phase boundary is a store/load of the exact fp32 value), and +0.0f
// is added when a candidate is keyed (x + 0 = x except -0 -> +0: R1/R2).
//
// Codes.  pq_create stores 16-bit pre-shifted codes (c' * 64 = byte offset of
// the row in its split table) PHASE-BLOCKED: for every tile of TR rows the PS
// codes of phase ph of all rows are contiguous ([tile][ph][row][PS]), so a
// warp's code load for one slot is 8 rows x PS x 2 B contiguous bytes and
// every code byte crosses HBM / L2 once per user group.
//
// Selection.  Per (warp, user) candidate buffers of `cap` keys in global
// memory (L2-resident, touched only by inserts), per-CTA user thresholds
// tau_sh[u] (the best proved K-th key), per-lane score filters for the lane's
// 4 users.  A buffer about to overflow is shrunk by a warp-cooperative radix
// select to its K best keys, which proves the new threshold.  At the end of a
// work unit one warp per user merges the W warp buffers into the unit's exact
// top-K list for K3 (same candidate format as v1/v2).
#include "k2_common.cuh"

namespace pq {

struct K2TArgs {
    const uint16_t* codes;     // phase-blocked pre-shifted codes (see above)
    const int32_t* perm;       // [tiles * TR] row -> local id (-1 = padding)
    const float* St;           // [n_groups][m][b][16] tiled sub-score tables
    int64_t n_tiles;           // tiles in the catalogue
    int B, K;
    uint32_t id_base;
    int n_groups, chunks;
    int64_t chunk_tiles;       // tiles per item chunk
    uint64_t* lanebuf;         // [grid][W][16][cap] candidate buffers
    int cap;
    uint64_t* cand;            // [B][chunks][K]
    uint64_t* mscr;            // [grid][16][W * cap] merge scratch
    unsigned long long* gtau;  // [B] per-user proved thresholds shared by all units (zeroed per call)
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}"
        :: "r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        :: "r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tm_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tm_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tm_st4(uint32_t taddr, float4 v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};"
                 :: "r"(taddr), "r"(__float_as_uint(v.x)), "r"(__float_as_uint(v.y)),
                    "r"(__float_as_uint(v.z)), "r"(__float_as_uint(v.w)));
}
// Asynchronous TMEM load: the registers are valid only after tm_ld_wait(r),
// which names them as in/out operands so no use can be scheduled before it.
__device__ __forceinline__ void tm_ld_issue(uint32_t taddr, uint32_t (&r)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(taddr));
}
__device__ __forceinline__ void tm_ld_wait(uint32_t (&r)[4]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]));
}
__device__ __forceinline__ float4 tm_ld4(uint32_t taddr) {
    uint32_t a, b, c, d;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(taddr) : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    return make_float4(__uint_as_float(a), __uint_as_float(b), __uint_as_float(c), __uint_as_float(d));
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float4 lds128(const char* p) {
    return *reinterpret_cast<const float4*>(p);
}
// 4 users' running sums += 4 sub-scores (two packed fp32x2 adds, RN, no FTZ)
__device__ __forceinline__ void add4(float4& acc, const float4 v) {
    float2 lo = __fadd2_rn(make_float2(acc.x, acc.y), make_float2(v.x, v.y));
    float2 hi = __fadd2_rn(make_float2(acc.z, acc.w), make_float2(v.z, v.w));
    acc = make_float4(lo.x, lo.y, hi.x, hi.y);
}
__device__ __forceinline__ float tau_to_filter(uint64_t t) {
    return t ? key_score(t) : -INFINITY;
}

// Code word(s) of one row for one phase: PS 16-bit codes.
template <int PS> struct CodeW;
template <> struct CodeW<4> {
    uint32_t w[2];
    __device__ __forceinline__ void load(const char* p) {
        const uint2 t = __ldg(reinterpret_cast<const uint2*>(p)); w[0] = t.x; w[1] = t.y;
    }
};
template <> struct CodeW<8> {
    uint32_t w[4];
    __device__ __forceinline__ void load(const char* p) {
        const uint4 t = __ldg(reinterpret_cast<const uint4*>(p));
        w[0] = t.x; w[1] = t.y; w[2] = t.z; w[3] = t.w;
    }
};
__device__ __forceinline__ uint32_t hi16_add(uint32_t w, uint32_t add) {
    uint32_t r;
    asm("mad.hi.u32 %0, %1, 65536, %2;" : "=r"(r) : "r"(w), "r"(add));
    return r;                                   // (w >> 16) + add
}

__device__ __forceinline__ void refresh(float (&tf)[4], const unsigned long long* tau_sh, int q) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (tf[j] != INFINITY)
            tf[j] = fmaxf(tf[j], tau_to_filter(*reinterpret_cast<const volatile unsigned long long*>(&tau_sh[4 * q + j])));
}

// Candidate entries.  The hot loop appends RAW entries (order-preserving score
// bits << 32 | layout row) without touching the row -> item permutation, so the
// slow path has no dependent global load; a buffer's raw tail [nconv, n) is
// converted to ranking keys (score bits << 32 | ~global id, R3) in one batched
// pass when the buffer is flushed or merged.  Padding rows (perm = -1) become
// key 0 ("empty") and are dropped.
__device__ __forceinline__ uint64_t make_raw(float s, uint32_t row) {
    const uint32_t u = __float_as_uint(s);
    const uint32_t o = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    return ((uint64_t)o << 32) | row;
}
__device__ __forceinline__ uint64_t raw_to_key(uint64_t r, const int32_t* perm, uint32_t id_base) {
    const int32_t lid = perm[(uint32_t)r];
    return lid < 0 ? 0ull : ((r & 0xFFFFFFFF00000000ull) | (uint64_t)(0xFFFFFFFFu - (id_base + (uint32_t)lid)));
}
// Whole warp: convert ub[nc, n) in place.
__device__ __forceinline__ void convert_tail(uint64_t* ub, int nc, int n, const int32_t* perm, uint32_t id_base) {
    for (int i = nc + (int)(threadIdx.x & 31); i < n; i += 32) ub[i] = raw_to_key(ub[i], perm, id_base);
    __syncwarp();
}

// Whole warp: keep the K best keys of ub[0, n) (n >= K; zero keys dropped),
// return the K-th key (0 if fewer than K non-zero keys) and the new count.
__device__ __noinline__ uint64_t shrink_to_k(uint64_t* ub, int n, int K, uint32_t* hist, int& n_out) {
    const int lane = threadIdx.x & 31;
    const uint64_t kth = warp_kth(ub, n, (uint32_t)K, hist);
    int pos = 0;
    for (int i0 = 0; i0 < n; i0 += 32) {
        const int i = i0 + lane;
        const uint64_t v = i < n ? ub[i] : 0ull;
        const bool keep = (i < n) && (v >= kth) && v != 0ull;
        const unsigned bm = __ballot_sync(FULL, keep);
        __syncwarp();
        if (keep) ub[pos + __popc(bm & lanemask_lt())] = v;
        pos += __popc(bm);
        __syncwarp();
    }
    n_out = pos;
    return kth;
}

// After a slot with candidates: shrink every (warp, user) buffer that could
// overflow on the next slot (> cap - 8 entries; a slot adds <= 8 per user) to
// its K best keys; the K-th key is a proved threshold for the user.
__device__ __noinline__ void flush_full(uint64_t* wbuf, int cap, int K, int* cnt_w, int* nconv_w,
                                        unsigned long long* tau_sh, uint32_t* hist,
                                        const int32_t* perm, uint32_t id_base,
                                        unsigned long long* gtau_g, int n_valid) {
    __syncwarp();
    const int lane = threadIdx.x & 31;
    const int cu = lane < 16 ? *reinterpret_cast<volatile int*>(&cnt_w[lane]) : 0;
    unsigned need = __ballot_sync(FULL, cu > cap - 8);
    while (need) {
        const int u = __ffs(need) - 1;
        need &= need - 1;
        const int n = __shfl_sync(FULL, cu, u);
        uint64_t* ub = wbuf + (int64_t)u * cap;
        convert_tail(ub, nconv_w[u], n, perm, id_base);
        int nn;
        const uint64_t kth = shrink_to_k(ub, n, K, hist, nn);
        if (lane == 0) {
            cnt_w[u] = nn;
            nconv_w[u] = nn;
            if (kth) {
                atomicMax(&tau_sh[u], (unsigned long long)kth);
                if (u < n_valid) atomicMax(&gtau_g[u], (unsigned long long)kth);
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------- the kernel
// M splits, PS per phase (NP = M / PS phases), BT sub-ids, W warps, D slots of
// code prefetch.
template <int M, int PS, int BT, int W, int D>
__global__ void __launch_bounds__(W * 32, 1) k2_tiled(const K2TArgs a) {
    constexpr int NP = M / PS;
    constexpr int NB = NP > 1 ? 3 : 1;                 // table buffers (ring)
    constexpr int SL = 512 / W;                        // slots per warp per tile
    constexpr int TR = W * SL * 8;                     // rows per tile (4096)
    constexpr uint32_t TBLB = (uint32_t)PS * BT * 64;  // bytes per table buffer
    constexpr uint32_t SPLITB = (uint32_t)BT * 64;     // bytes per split table
    constexpr int CB = PS * 2;                         // code bytes per row per phase
    static_assert(M % PS == 0, "phases");
    static_assert(SL % D == 0, "prefetch depth");

    extern __shared__ __align__(1024) unsigned char sm_raw[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    // smem carve: [tables NB x TBLB][hist W x 1 KB][tau 16 x u64][cnt W x 16][nconv W x 16]
    //             [mbar NB x u64][done NB][tmem slot]
    uint32_t* hist_all = reinterpret_cast<uint32_t*>(sm_raw + NB * TBLB);
    uint32_t* hist = hist_all + warp * 256;
    unsigned long long* tau_sh = reinterpret_cast<unsigned long long*>(hist_all + W * 256);
    int* cnt_all = reinterpret_cast<int*>(tau_sh + 16);
    int* cnt_w = cnt_all + warp * 16;
    int* nconv_all = cnt_all + W * 16;
    int* nconv_w = nconv_all + warp * 16;
    unsigned long long* mbar = reinterpret_cast<unsigned long long*>(nconv_all + W * 16);
    int* done = reinterpret_cast<int*>(mbar + NB);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + NB);
    const uint32_t tbl0 = smem_u32(sm_raw);
    const uint32_t bar0 = smem_u32(mbar);

    const int64_t units = (int64_t)a.n_groups * a.chunks;
    auto unit_tiles = [&](int64_t u) -> int64_t {
        const int64_t ch = u / a.n_groups;
        const int64_t t0 = ch * a.chunk_tiles;
        return min(a.n_tiles, t0 + a.chunk_tiles) - t0;
    };
    // TMA bulk copy: tables of (unit, phase) -> ring buffer `buf`
    auto issue_load = [&](int64_t u, int ph, int buf) {
        const int grp = (int)(u % a.n_groups);
        const char* src = reinterpret_cast<const char*>(a.St) +
                          ((int64_t)grp * M + (int64_t)ph * PS) * SPLITB;
        const uint32_t bar = bar0 + 8u * buf;
        fence_proxy_async();
        mbar_expect_tx(bar, TBLB);
        constexpr uint32_t PIECE = 16384;
#pragma unroll 1
        for (uint32_t off = 0; off < TBLB; off += PIECE)
            bulk_g2s(tbl0 + buf * TBLB + off, src + off, PIECE < TBLB - off ? PIECE : TBLB - off, bar);
    };
    // (unit, tile, phase) sequence position advanced by one
    auto advance = [&](int64_t& u, int64_t& t, int& ph) {
        if (++ph == NP) {
            ph = 0;
            if (++t == unit_tiles(u)) { t = 0; u += gridDim.x; }
        }
    };

    // ---- one-time setup -------------------------------------------------
    if (threadIdx.x == 0) {
        for (int i = 0; i < NB; ++i) { mbar_init(bar0 + 8u * i, 1); done[i] = 0; }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = threadIdx.x; i < W * 32; i += blockDim.x) cnt_all[i] = 0;   // cnt + nconv
    if (threadIdx.x < 16) tau_sh[threadIdx.x] = 0ull;
    uint32_t tmem_base = 0;
    if constexpr (NP > 1) {
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                         :: "r"(smem_u32(tmem_slot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        tm_fence_before();
    }
    __syncthreads();
    if constexpr (NP > 1) {
        tm_fence_after();
        tmem_base = *reinterpret_cast<volatile uint32_t*>(tmem_slot);
    }
    // first loads: sequence positions 0 .. NB-1
    if (threadIdx.x == 0 && (int64_t)blockIdx.x < units) {
        int64_t u = blockIdx.x, t = 0;
        int ph = 0;
        for (int i = 0; i < NB && u < units; ++i) {
            issue_load(u, ph, i);
            advance(u, t, ph);
        }
    }

    // TMEM: this warp's lane quadrant and column range
    constexpr int WPQ = W / 4;                         // warps per lane quadrant
    const uint32_t tcol0 = tmem_base + ((uint32_t)((warp & 3) * 32) << 16) +
                           (uint32_t)((warp >> 2) * (512 / WPQ));

    const int q = lane & 3;
    const uint32_t q16 = (uint32_t)q * 16u;
    uint64_t* wbuf = a.lanebuf + ((int64_t)blockIdx.x * W + warp) * 16 * a.cap;
    int64_t gseq = 0;                                  // table uses so far (NP > 1)
    int64_t useq = 0;                                  // units done by this CTA (NP == 1)

    for (int64_t unit = blockIdx.x; unit < units; unit += gridDim.x) {
        const int chunk = (int)(unit / a.n_groups);
        const int grp = (int)(unit - (int64_t)chunk * a.n_groups);
        const int64_t tile0 = (int64_t)chunk * a.chunk_tiles;
        const int64_t ntl = unit_tiles(unit);

        unsigned long long* gtau_g = a.gtau + grp * 16;          // this group's users
        const int n_valid = min(16, a.B - grp * 16);
        if (threadIdx.x < n_valid)                                // K keys >= gtau exist elsewhere
            atomicMax(&tau_sh[threadIdx.x], *reinterpret_cast<volatile unsigned long long*>(&gtau_g[threadIdx.x]));
        __syncthreads();
        float tf[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) tf[j] = (4 * q + j < n_valid) ? -INFINITY : INFINITY;
        refresh(tf, tau_sh, q);

        for (int64_t t = 0; t < ntl; ++t) {
            const int64_t tile = tile0 + t;
#pragma unroll
            for (int ph = 0; ph < NP; ++ph) {
                const int buf = NP > 1 ? (int)(gseq % NB) : 0;
                const uint32_t par = NP > 1 ? (uint32_t)((gseq / NB) & 1) : (uint32_t)(useq & 1);
                mbar_wait(bar0 + 8u * buf, par);
                const char* tb = reinterpret_cast<const char*>(sm_raw) + buf * TBLB;
                const uint32_t row0 = (uint32_t)(tile * TR) + (uint32_t)(warp * SL * 8) + (uint32_t)(lane >> 2);
                const char* cp = reinterpret_cast<const char*>(a.codes) + ((tile * NP + ph) * TR +
                                 (int64_t)warp * SL * 8 + (lane >> 2)) * CB;
                constexpr int64_t SSTR = 8 * CB;       // bytes per slot
                CodeW<PS> cw[D];
#pragma unroll
                for (int d = 0; d < D; ++d) cw[d].load(cp + d * SSTR);
                cp += D * SSTR;
                uint32_t tcur[4] = {0u, 0u, 0u, 0u};          // partial sums of slot s (ph > 0)
                if (ph > 0) {
                    tm_ld_issue(tcol0, tcur);
                    tm_ld_wait(tcur);
                }
#pragma unroll 1
                for (int s0 = 0; s0 < SL; s0 += D) {
#pragma unroll
                    for (int d = 0; d < D; ++d) {
                        const int s = s0 + d;
                        uint32_t off[PS];              // row offsets | user-quad offset
#pragma unroll
                        for (int kk = 0; kk < PS; ++kk) {
                            const uint32_t w = cw[d].w[kk >> 1];
                            off[kk] = (kk & 1) ? hi16_add(w, q16) : ((w & 0xFFFFu) | q16);
                        }
                        cw[d].load(cp);                // D slots ahead (buffer is padded)
                        cp += SSTR;
                        float4 v[PS];
#pragma unroll
                        for (int kk = 0; kk < PS; ++kk) v[kk] = lds128(tb + kk * SPLITB + off[kk]);
                        uint32_t tnxt[4];
                        if (ph > 0)                    // next slot's partials (the last slot re-reads its own)
                            tm_ld_issue(tcol0 + (uint32_t)min(s + 1, SL - 1) * 4u, tnxt);
                        float4 acc;
                        if (ph == 0) {
                            acc = v[0];
                        } else {
                            acc = make_float4(__uint_as_float(tcur[0]), __uint_as_float(tcur[1]),
                                              __uint_as_float(tcur[2]), __uint_as_float(tcur[3]));
                            add4(acc, v[0]);
                        }
#pragma unroll
                        for (int kk = 1; kk < PS; ++kk) add4(acc, v[kk]);
                        if (ph > 0) {
                            tm_ld_wait(tnxt);
#pragma unroll
                            for (int x = 0; x < 4; ++x) tcur[x] = tnxt[x];
                        }
                        if (ph < NP - 1) {
                            tm_st4(tcol0 + (uint32_t)s * 4u, acc);
                            continue;
                        }
                        // ---- last phase: candidate filter (rare slow path, no loads)
                        const bool c0 = acc.x >= tf[0], c1 = acc.y >= tf[1];
                        const bool c2 = acc.z >= tf[2], c3 = acc.w >= tf[3];
                        const bool any = c0 | c1 | c2 | c3;
                        if (any) {
                            const uint32_t row = row0 + (uint32_t)s * 8u;
                            const float v[4] = {acc.x, acc.y, acc.z, acc.w};
                            const bool cc[4] = {c0, c1, c2, c3};
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                if (!cc[j]) continue;
                                const int u = 4 * q + j;
                                const int p = atomicAdd(&cnt_w[u], 1);
                                wbuf[(int64_t)u * a.cap + p] = make_raw(v[j] + 0.0f, row);
                            }
                        }
                        if (__any_sync(FULL, any)) {
                            flush_full(wbuf, a.cap, a.K, cnt_w, nconv_w, tau_sh, hist, a.perm, a.id_base,
                                       gtau_g, n_valid);
                            refresh(tf, tau_sh, q);
                        }
                    }
                }
                if constexpr (NP > 1) {
                    if (ph < NP - 1) tm_wait_st();
                    // release the buffer: the last warp to finish with it loads
                    // the table this ring slot serves next (position + NB)
                    __syncwarp();
                    if (lane == 0) {
                        const int old = atomicAdd(&done[buf], 1);
                        if (old == W - 1) {
                            done[buf] = 0;
                            int64_t u2 = unit, t2 = t;
                            int ph2 = ph;
                            for (int st = 0; st < NB; ++st) advance(u2, t2, ph2);
                            if (u2 < units) issue_load(u2, ph2, buf);
                        }
                    }
                    ++gseq;
                }
            }
            if (warp == (int)(t % W) && lane < n_valid)
                atomicMax(&tau_sh[lane], *reinterpret_cast<volatile unsigned long long*>(&gtau_g[lane]));
            refresh(tf, tau_sh, q);
        }

        // ---- end of unit: convert raw tails, then merge the W warp buffers
        // of each user into the unit's top-K list -----------------------------
#pragma unroll 1
        for (int u = 0; u < 16; ++u)
            convert_tail(wbuf + (int64_t)u * a.cap, nconv_w[u], cnt_w[u], a.perm, a.id_base);
        __syncthreads();
        if constexpr (NP == 1) {
            // every warp is done with the table: prefetch the next unit's
            if (threadIdx.x == 0 && unit + gridDim.x < units) issue_load(unit + gridDim.x, 0, 0);
        }
        for (int uu = warp; uu < 16; uu += W) {
            const int gu = grp * 16 + uu;
            if (gu >= a.B) continue;
            const uint64_t th = tau_sh[uu] ? tau_sh[uu] : 1ull;     // key 0 = padding
            uint64_t* out = a.cand + ((int64_t)gu * a.chunks + chunk) * a.K;
            int tot = 0;
            for (int w2 = 0; w2 < W; ++w2) {
                const int n = cnt_all[w2 * 16 + uu];
                const uint64_t* src = a.lanebuf + (((int64_t)blockIdx.x * W + w2) * 16 + uu) * a.cap;
                for (int i = lane; i < n; i += 32) tot += src[i] >= th ? 1 : 0;
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(FULL, tot, o);
            uint64_t* dst = tot <= a.K ? out : a.mscr + ((int64_t)blockIdx.x * 16 + uu) * W * a.cap;
            int pos = 0;
            for (int w2 = 0; w2 < W; ++w2) {
                const int n = cnt_all[w2 * 16 + uu];
                const uint64_t* src = a.lanebuf + (((int64_t)blockIdx.x * W + w2) * 16 + uu) * a.cap;
                for (int i0 = 0; i0 < n; i0 += 32) {
                    const int i = i0 + lane;
                    const uint64_t v = i < n ? src[i] : 0ull;
                    const bool keep = (i < n) && (v >= th);
                    const unsigned bm = __ballot_sync(FULL, keep);
                    if (keep) dst[pos + __popc(bm & lanemask_lt())] = v;
                    pos += __popc(bm);
                }
            }
            if (tot <= a.K) {
                for (int j = tot + lane; j < a.K; j += 32) out[j] = 0ull;
            } else {
                __syncwarp();
                const uint64_t kth = warp_kth(dst, tot, (uint32_t)a.K, hist);
                if (lane == 0) atomicMax(&a.gtau[gu], (unsigned long long)kth);
                int p2 = 0;
                for (int i0 = 0; i0 < tot; i0 += 32) {
                    const int i = i0 + lane;
                    const uint64_t v = i < tot ? dst[i] : 0ull;
                    const bool keep = (i < tot) && (v >= kth);
                    const unsigned bm = __ballot_sync(FULL, keep);
                    if (keep) out[p2 + __popc(bm & lanemask_lt())] = v;
                    p2 += __popc(bm);
                }
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < W * 32; i += blockDim.x) cnt_all[i] = 0;
        if (threadIdx.x < 16) tau_sh[threadIdx.x] = 0ull;
        __syncthreads();
        ++useq;
    }

    if constexpr (NP > 1) {
        tm_fence_before();
        __syncthreads();
        tm_fence_after();
        if (warp == 0)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem_base));
    }
}

// ---------------------------------------------------------------- K2a: tiled S
// St[g][k][c'][w] = S[16 g + w][k][cmap[k][c']] (0 for padding users): the
// 16-user interleaved, colour-renumbered table layout, so K2 can stage a
// phase's tables with one contiguous bulk copy.
__global__ void k2_tile_S(const float* __restrict__ S, const uint8_t* __restrict__ cmap, int B, int m,
                          int b, int n_groups, float* __restrict__ St) {
    const int64_t total = (int64_t)n_groups * m * b * 16;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int w = (int)(x & 15);
        const int64_t r = x >> 4;                      // (g, k, c')
        const int c = (int)(r % b);
        const int64_t gk = r / b;
        const int k = (int)(gk % m);
        const int g = (int)(gk / m);
        const int user = g * 16 + w;
        St[x] = user < B ? S[((int64_t)user * m + k) * b + cmap[k * b + c]] : 0.0f;
    }
}

// ---------------------------------------------------------------- host side
typedef void (*K2TFn)(const K2TArgs);

template <int M, int PS>
static K2TFn tiled_fn_w(int W) {
    if (W == 16) return k2_tiled<M, PS, 256, 16, 4>;
    return k2_tiled<M, PS, 256, 8, 4>;
}
static K2TFn tiled_fn(int m, int W) {
    switch (m) {
        case 4: return tiled_fn_w<4, 4>(W);
        case 8: return tiled_fn_w<8, 8>(W);
        case 16: return tiled_fn_w<16, 4>(W);
        default: return nullptr;
    }
}
int k2_tiled_ps(int m) { return m == 16 ? 4 : m; }
bool k2_tiled_supported(int m, int b) { return b == 256 && (m == 4 || m == 8 || m == 16); }
int k2_tiled_rows_per_tile(int W) { return W * (512 / W) * 8; }

size_t k2_tiled_smem(int m, int b, int W) {
    const int ps = k2_tiled_ps(m);
    const int nb = (m / ps) > 1 ? 3 : 1;
    return (size_t)nb * ps * b * 64 + (size_t)W * 1024 + 16 * 8 + (size_t)W * 32 * 4 +
           3 * 8 + 3 * 4 + 16;
}

static int choose_chunks_tiles(int64_t n_tiles, int n_groups, int grid_full) {
    const int64_t max_c = std::max<int64_t>(1, std::min<int64_t>(4096, n_tiles));
    int best = 1;
    double best_eff = -1.0;
    for (int64_t c = 1; c <= max_c; ++c) {
        const int64_t ct = ceil_div(n_tiles, c);
        const int64_t cc = ceil_div(n_tiles, ct);        // chunks actually formed
        // work is proportional to tiles; the last chunk may be short
        const int64_t units = (int64_t)n_groups * cc;
        const int64_t per_cta = ceil_div(units, grid_full);
        const double eff = (double)n_groups * n_tiles / ((double)per_cta * grid_full * ct);
        if (eff > best_eff + 1e-9) { best_eff = eff; best = (int)cc; }
        if (eff >= 0.97) break;
    }
    return best;
}

void plan_k2_tiled(const pq_index_s* idx, int B, int K, K2Plan& p) {
    p.variant = 3;
    const pq_tuning& t = idx->tuning;
    p.W = (t.warps == 8 || t.warps == 16) ? t.warps : 16;
    p.G = 16; p.Ug = 16; p.J = 1;
    p.tm = (idx->m / k2_tiled_ps(idx->m)) > 1 ? idx->m - k2_tiled_ps(idx->m) : 0;
    p.n_groups = (int)ceil_div(B, 16);
    p.cap = (int)align_up((size_t)std::max(2 * K, K + 32), 32);
    p.smem = k2_tiled_smem(idx->m, idx->b, p.W);
    K2TFn fn = tiled_fn(idx->m, p.W);
    if (!fn) fail(PQ_ERR_UNSUPPORTED, "tiled scoring kernel: unsupported m");
    PQ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
    int occ = 0;
    PQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, p.W * 32, p.smem));
    if (occ < 1) fail(PQ_ERR_UNSUPPORTED, "tiled scoring kernel cannot be resident");
    occ = 1;                                           // one TMEM allocation / table set per SM
    const int grid_full = idx->num_sms * occ;
    const int64_t n_tiles = idx->v3_tiles;
    p.chunks = t.chunks > 0 ? (int)std::min<int64_t>(t.chunks, n_tiles)
                            : choose_chunks_tiles(n_tiles, p.n_groups, grid_full);
    const int64_t ct = ceil_div(n_tiles, p.chunks);
    p.chunk_items = ct;                                // tiles per chunk
    p.chunks = (int)ceil_div(n_tiles, ct);
    const int64_t units = (int64_t)p.n_groups * p.chunks;
    p.grid = (int)std::min<int64_t>(units, t.ctas > 0 ? t.ctas : grid_full);
    p.lanebuf_bytes = (size_t)p.grid * p.W * 16 * p.cap * 8;
    p.cand_bytes = (size_t)B * p.chunks * K * 8;
    p.ghist_bytes = 0;
    p.mscr_bytes = (size_t)p.grid * 16 * p.W * p.cap * 8;
    p.st_bytes = align_up((size_t)p.n_groups * idx->m * idx->b * 16 * 4, 256) + (size_t)p.n_groups * 16 * 8;
}

static unsigned long long* gtau_of(const pq_index_s* idx, const K2Plan& p, const float* St) {
    return reinterpret_cast<unsigned long long*>(const_cast<char*>(reinterpret_cast<const char*>(St)) +
                                                 align_up((size_t)p.n_groups * idx->m * idx->b * 16 * 4, 256));
}

void launch_k2_tiled_prep(const pq_index_s* idx, const K2Plan& p, const float* S, int B, float* St,
                          cudaStream_t st) {
    PQ_CUDA(cudaMemsetAsync(gtau_of(idx, p, St), 0, (size_t)p.n_groups * 16 * 8, st));
    {
        const int64_t total = (int64_t)p.n_groups * idx->m * idx->b * 16;
        const int threads = 256;
        const int blocks = (int)std::min<int64_t>(ceil_div(total, threads), (int64_t)idx->num_sms * 16);
        k2_tile_S<<<blocks, threads, 0, st>>>(S, idx->d_cmap3, B, idx->m, idx->b, p.n_groups, St);
        count_launch();
        check_launch("k2_tile_S");
    }
}

void launch_k2_tiled(const pq_index_s* idx, const K2Plan& p, int B, int K,
                     uint64_t* lanebuf, uint64_t* mscr, const float* St, uint64_t* cand, cudaStream_t st) {
    K2TArgs a{};
    a.codes = idx->d_codes3;
    a.perm = idx->d_perm3;
    a.St = St;
    a.n_tiles = idx->v3_tiles;
    a.B = B; a.K = K;
    a.id_base = (uint32_t)idx->id_base;
    a.n_groups = p.n_groups; a.chunks = p.chunks; a.chunk_tiles = p.chunk_items;
    a.lanebuf = lanebuf; a.cap = p.cap; a.cand = cand; a.mscr = mscr;
    a.gtau = gtau_of(idx, p, St);
    K2TFn fn = tiled_fn(idx->m, p.W);
    fn<<<p.grid, p.W * 32, p.smem, st>>>(a);
    count_launch();
    check_launch("k2_tiled");
}

}  // namespace pq
