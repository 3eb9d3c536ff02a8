// K2 v3 — "tiled phases": gather-sum-select with 4 users per lane
// (Eq. 5; Algorithm 1).
//
// The binding resource of Eq. 5 is the shared-memory lookup rate
// (148 SMs x 32 four-byte words per clock).  K2 v2 reached it only halfway
// because every lookup cost three issue slots (address op, LDS.32, FADD) and
// its TMEM-resident splits cost more.  Here a lane serves FOUR users of one
// item, so a split costs 1 address op + 1 LDS.128 + 2 FADD2 per 4 lookups.
//
// Table layout.  A CTA owns a group of R users (R = 16 or 32).  Row (k, c) of
// split k's table holds the R users' sub-scores S[u][k][c] (R*4 bytes).  Lane
// l serves user quad q = l % (R/4) (users 4q..4q+3) of row l / (R/4) of the
// warp's slot; one LDS.128 per lane per split returns 4 users' sub-scores.
// A 128-bit shared load is served per quarter-warp (8 lanes = 128 bytes):
//   * R = 32: a quarter-warp reads one whole 128-byte row: conflict free for
//     any codes (the catalogue stays in item order);
//   * R = 16: a quarter-warp reads the rows of two items.  pq_create has
//     2-coloured every split's sub-ids (stored code parity = colour) and
//     paired items whose colours are complementary at every split (rows 2p,
//     2p+1), so the two 64-byte rows lie in opposite bank halves: conflict free
//     for every matched pair.
// R = 32 is used when 32 users' whole table fits in shared memory (e.g. C5:
// m = 4, b = 16); R = 16 otherwise (C2/C3: m*b = 2048; C4: 4096).
//
// Phases.  When the R users' tables exceed shared memory (C4: 16 users x 16
// splits x 256 x 64 B = 256 KB) the splits are processed in NP phases of PS
// splits: phase tables are loaded by the TMA bulk engine (cp.async.bulk +
// mbarrier) from a pre-tiled copy of S into a 2-slot shared-memory ring, and
// the running partial sums of a tile (TR items x R users) stay in TENSOR
// MEMORY between phases (tcgen05.st / tcgen05.ld 32x32b.x4: lane = TMEM row,
// 4 columns per slot; each warp owns 512/(W/4) columns of its lane quadrant).
// The fp32 order is unchanged: acc = S[0], then + S[1], ..., + S[m-1] split by
// split (a phase boundary is an exact store/load of the fp32 value), and +0.0f
// is added when a candidate is keyed (x + 0 = x except -0 -> +0: R1/R2).
//
// Codes.  pq_create stores 16-bit pre-shifted codes (c * R * 4 = byte offset of
// the row in its split table) PHASE-BLOCKED: for every tile of TR rows, the PS
// codes of phase ph of all rows are contiguous ([tile][ph][row][PS]), so a
// warp's code load for one slot is contiguous and every code byte crosses
// HBM / L2 once per user group.
//
// Selection.  Per-user candidate buffers shared by the CTA (global memory,
// L2-resident, touched only by inserts) and per-user thresholds tau_sh[u] (a
// proved K-th key).  The hot loop only filters (acc >= threshold score) and
// appends RAW entries (score bits, layout row) with one shared atomic.  At the
// end of a tile, if some buffer could overflow during the next tile, the whole
// CTA stops and one warp per user shrinks that user's buffer to its exact K
// best keys (radix select), which raises the user's threshold to the CTA-wide
// K-th best.  Thresholds are also shared across CTAs through gtau[user]
// (a unit may drop an item whenever K better items are known anywhere: the
// global top-K still survives in the union of the unit lists that K3 merges).
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "k2_common.cuh"
#include "ptx_dev.cuh"

namespace pq {

// Stored code width: 1 = the (colour-renumbered) sub-id byte, the kernel forms
// the row offset (code * R * 4 | quad offset) with two integer ops; 2 = 16-bit
// pre-shifted row offsets (one op, twice the code bytes).
// Tiles of warp skew the tile-end protocol allows (S, 1..3; -DK2_SLACK=S for
// A/B: S = 2 / 3 measured within +-2% of S = 1 on C2-C5, r02 slack A/B).
#ifndef K2_SLACK
#define K2_SLACK 1
#endif
#ifndef K2_CODE_BYTES
#define K2_CODE_BYTES 1
#endif
int k2_tiled_code_bytes() { return K2_CODE_BYTES; }

// Union floors (large K): a finished unit publishes, per user, the keys of rank
// ceil(K / c) of its list for c = 2, 4, 8, 16 (K2_NQ levels).  If c finished
// units of a user each published a level-c key >= v, then c * ceil(K / c) >= K
// distinct items (the chunks are disjoint) have keys >= v, so v is a proved
// floor for that user's top-K (like gtau, which is the c = 1 level).  A unit
// starting later takes the largest such v over the levels: after j finished
// chunks it admits ~K / j items per user instead of ~K (C5: K = 1000).
constexpr int K2_NQ = 4;
struct K2TArgs {
    const void* codes;         // phase-blocked codes (see above), K2_CODE_BYTES each
    int64_t codes_bytes;       // allocated bytes of `codes` (checked builds bound every load)
    const int32_t* perm;       // [tiles * TR] row -> local id (-1 = padding)
    const float* St;           // [n_groups][m][b][R] tiled sub-score tables
    int64_t n_tiles;           // tiles in the catalogue
    int B, K;
    uint32_t id_base;
    int n_groups, chunks;
    int64_t chunk_tiles;       // tiles per item chunk
    uint64_t* ubuf;            // [grid][R][cap] per-user candidate buffers
    int cap;                   // >= 2K + (2 slack + 1) TR + 96 (see the shrink protocol)
    int wm;                    // shrink watermark (<= cap - (2 slack + 1) TR - 32)
    uint64_t* cand;            // [B][chunks][K]
    unsigned long long* gtau;  // [n_groups * R] per-user proved thresholds (zeroed per call)
    unsigned long long* qk;    // [n_groups * R][chunks][K2_NQ] union-floor keys (zeroed per call), or null
    int32_t* lcnt;             // [n_groups * R][chunks] entries of each unit's list in cand (no padding)
    long long* trace;          // diagnostics (PQTOPK_K2_TRACE): CTA 0 phase timeline, or null
    int trace_stride;          // trace every trace_stride-th tile (PQTOPK_K2_TRACE_STRIDE)
    int trace_from;            // first traced tile of CTA 0 (PQTOPK_K2_TRACE_FROM)
    int* dbg;                  // diagnostics (PQTOPK_K2_DEBUG): bounded spins record state here
    // Balanced partition (single-phase tables): CTA x scores positions [cut[x], cut[x + 1])
    // of the group-major (group, tile) sequence g * n_tiles + t -- one unit per group it
    // touches; n_cut = 0: legacy units (chunk x group, round-robin)
    int n_cut;
    int32_t cut[K2_MAX_CUT + 1];
};
// Phase traces are compiled in only for diagnostics builds (PQTOPK_NVCC_EXTRA=-DK2_TRACE);
// otherwise every trace branch folds away.
#ifdef K2_TRACE
constexpr bool kTrace = true;
#else
constexpr bool kTrace = false;
#endif
constexpr int TRACE_PH = 256;  // traced table uses (CTA 0): [W][TRACE_PH][3]; then CTA 0 units [TRACE_PH/2][2];
constexpr int TRACE_CTAS = 1024;  // then per-CTA [TRACE_CTAS][3] = (start ns, end ns, tiles)

// ---------------------------------------------------------------- PTX helpers
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
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float4 lds128(const char* p) {
    return *reinterpret_cast<const float4*>(p);
}
// the same load from a 32-bit shared address plus a compile-time offset
__device__ __forceinline__ float4 lds128_s(uint32_t addr, uint32_t imm) {
    float4 v;
    asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr + imm));
    return v;
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

// Code words of one row for one phase and TWO consecutive slots: pq_create
// interleaves slot pairs ([slot pair][row][2][PS] inside a phase block), so a
// lane fetches both slots' PS codes with one or two vector loads.
template <int PS> struct CodePair {
    static constexpr int BYTES = 2 * PS * K2_CODE_BYTES;     // per lane per slot pair
    static constexpr int NW = BYTES / 4;
    uint32_t w[NW];
#ifdef PQTOPK_CHECKED
    static __device__ __forceinline__ void check(const char* p, const char* base, int64_t nbytes) {
        PQ_DCHECK(p >= base && p + BYTES <= base + nbytes);
    }
#else
    static __device__ __forceinline__ void check(const char*, const char*, int64_t) {}
#endif
    __device__ __forceinline__ void load(const char* p) {
        if constexpr (NW == 1) {
            w[0] = __ldg(reinterpret_cast<const uint32_t*>(p));
        } else if constexpr (NW == 2) {
            const uint2 t = __ldg(reinterpret_cast<const uint2*>(p));
            w[0] = t.x; w[1] = t.y;
        } else {
#pragma unroll
            for (int x = 0; x < NW; x += 4) {
                const uint4 t = __ldg(reinterpret_cast<const uint4*>(p) + x / 4);
                w[x] = t.x; w[x + 1] = t.y; w[x + 2] = t.z; w[x + 3] = t.w;
            }
        }
    }
    // byte offset of split kk's row for slot parity e, OR-ed with the quad offset
    template <int RB>
    __device__ __forceinline__ uint32_t off(int e, int kk, uint32_t q16) const {
        if constexpr (K2_CODE_BYTES == 1) {
            const uint32_t wd = w[(e * PS + kk) >> 2];     // PS here = stored codes per row
#ifndef K2_NO_ASM_LDS
            if constexpr (true)                            // PRMT + one IMAD (code * RB + base) per gather
#else
            if constexpr (PS == 4)                         // byte extract by PRMT (C4: -0.6%)
#endif
                return __byte_perm(wd, 0u, 0x4440u | (uint32_t)((e * PS + kk) & 3)) * RB + q16;
            else
                return ((wd >> (8 * ((e * PS + kk) & 3))) & 0xFFu) * RB + q16;
        } else {
            const uint32_t wd = w[(e * PS + kk) >> 1];
            return ((e * PS + kk) & 1) ? ((wd >> 16) + q16) : ((wd & 0xFFFFu) | q16);
        }
    }
};

// Candidate entries.  The hot loop appends RAW entries (order-preserving score
// bits << 32 | layout row) without touching the row -> item permutation, so the
// slow path has no dependent global load; a buffer's raw tail [nconv, n) is
// converted to ranking keys (score bits << 32 | ~global id, R3) in one batched
// pass (shrink_user) when the buffer is shrunk or merged.  Padding rows (perm = -1) become
// key 0 ("empty") and are dropped.
__device__ __forceinline__ uint64_t make_raw(float s, uint32_t row) {
    const uint32_t u = __float_as_uint(s);
    const uint32_t o = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    return ((uint64_t)o << 32) | row;
}

// The K-th largest of up to 32 * SR keys held in registers (key index
// u * 32 + lane in v[u]; 0 = empty), n >= K >= 1: MSD radix select, 8 bits per
// pass, with the early exit of warp_kth (select_dev.cuh) -- the keys are read
// from registers, not re-read from memory on every pass.
template <int SR>
__device__ __forceinline__ uint64_t warp_kth_regs(const uint64_t (&v)[SR], int n, uint32_t K, uint32_t* hist) {
    uint64_t prefix = 0;
    uint32_t krem = K;
    const int lane = threadIdx.x & 31;
    for (int shift = 56; shift >= 0; shift -= 8) {
        const uint64_t hmask = (shift == 56) ? 0ull : (~0ull << (shift + 8));
#pragma unroll
        for (int i = lane; i < 256; i += 32) hist[i] = 0;
        __syncwarp();
#pragma unroll
        for (int u = 0; u < SR; ++u) {
            const bool ok = (u * 32 + lane < n) && ((v[u] & hmask) == prefix);
            hist_add(hist, ok, (uint32_t)(v[u] >> shift) & 255u);
        }
        __syncwarp();
        uint32_t dg, ab;
        warp_find_digit(hist, krem, dg, ab);
        const uint32_t inbin = hist[dg];
        prefix |= (uint64_t)dg << shift;
        krem -= ab;
        __syncwarp();
        if (shift > 0 && inbin == krem) {              // the K-th key = the smallest key carrying prefix
            const uint64_t pmask = ~0ull << shift;
            uint64_t mn = ~0ull;
#pragma unroll
            for (int u = 0; u < SR; ++u)
                if (u * 32 + lane < n && (v[u] & pmask) == prefix && v[u] < mn) mn = v[u];
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const uint64_t t = __shfl_xor_sync(FULL, mn, o);
                mn = t < mn ? t : mn;
            }
            return mn;
        }
    }
    return prefix;
}

// shrink_user for a buffer of at most 32 * SR entries, selected in registers: one read
// of the buffer instead of one per radix pass.
template <int SR>
__device__ __forceinline__ uint64_t shrink_user_regs(uint64_t* ub, int nc, int n, int K, uint64_t floor,
                                                     uint64_t* dst, uint32_t* hist, const int32_t* perm,
                                                     uint32_t id_base, int& n_out) {
    const int lane = threadIdx.x & 31;
    uint64_t v[SR];
#pragma unroll
    for (int u = 0; u < SR; ++u) {
        const int i = u * 32 + lane;
        v[u] = i < n ? ub[i] : 0ull;
    }
    int32_t lid[SR];
#pragma unroll
    for (int u = 0; u < SR; ++u) {
        const int i = u * 32 + lane;
        lid[u] = (i >= nc && i < n) ? __ldg(&perm[(uint32_t)v[u]]) : 0;
    }
#pragma unroll
    for (int u = 0; u < SR; ++u) {
        const int i = u * 32 + lane;
        if (i >= nc && i < n)
            v[u] = lid[u] < 0 ? 0ull
                              : ((v[u] & 0xFFFFFFFF00000000ull) | (uint64_t)(0xFFFFFFFFu - (id_base + (uint32_t)lid[u])));
    }
    const uint64_t kth = n > K ? warp_kth_regs<SR>(v, n, (uint32_t)K, hist) : 0ull;
    uint64_t th = kth > floor ? kth : floor;
    if (th == 0ull) th = 1ull;                               // key 0 = padding: never kept
    int pos = 0;
#pragma unroll
    for (int u = 0; u < SR; ++u) {
        const bool keep = u * 32 + lane < n && v[u] >= th;
        const unsigned bm = __ballot_sync(FULL, keep);
        if (keep) dst[pos + __popc(bm & lanemask_lt())] = v[u];
        pos += __popc(bm);
    }
    n_out = pos;
    return kth;
}

// Whole warp, one user: convert the raw tail, then keep only keys >= the K-th
// best (and >= `floor`), writing them to `dst` (may alias ub).  Returns the
// K-th key (0 if the buffer has fewer than K non-zero keys) and the count.
// Buffers of up to 256 entries (a shrink at the watermark 2K + 64 for K <= 96,
// e.g. C2's K = 10) are selected in registers, 2, 4 or 8 entries per lane (C2's
// first-tile shrink holds ~40 entries, its end-of-unit list ~140; a larger
// register window spills in the caller).
// BIG: register windows of 12 and 16 entries per lane too (K = 100 shrinks at 264+
// entries: C3 -0.25%, C2 -0.85%).  Not for the first-pair-table kernels (C5, K = 1000:
// buffers far beyond 512 entries), whose allocation around the call came out 2.5% slower
// with the larger callee.
template <bool BIG>
__device__ __noinline__ uint64_t shrink_user(uint64_t* ub, int nc, int n, int K, uint64_t floor,
                                             uint64_t* dst, uint32_t* hist, const int32_t* perm,
                                             uint32_t id_base, int& n_out) {
    const int lane = threadIdx.x & 31;
    auto to_key = [&](uint64_t raw, int32_t lid) -> uint64_t {
        return lid < 0 ? 0ull
                       : ((raw & 0xFFFFFFFF00000000ull) | (uint64_t)(0xFFFFFFFFu - (id_base + (uint32_t)lid)));
    };
    if (n <= 64) return shrink_user_regs<2>(ub, nc, n, K, floor, dst, hist, perm, id_base, n_out);
    if (n <= 128) return shrink_user_regs<4>(ub, nc, n, K, floor, dst, hist, perm, id_base, n_out);
    if (n <= 256) return shrink_user_regs<8>(ub, nc, n, K, floor, dst, hist, perm, id_base, n_out);
    if constexpr (BIG) {
        if (n <= 384) return shrink_user_regs<12>(ub, nc, n, K, floor, dst, hist, perm, id_base, n_out);
        if (n <= 512) return shrink_user_regs<16>(ub, nc, n, K, floor, dst, hist, perm, id_base, n_out);
    }
    constexpr int U = 8;                               // independent loads in flight per lane
    for (int i0 = nc; i0 < n; i0 += 32 * U) {
        uint64_t r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * 32 + lane;
            r[u] = i < n ? ub[i] : 0ull;
        }
        int32_t lid[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * 32 + lane;
            lid[u] = i < n ? __ldg(&perm[(uint32_t)r[u]]) : -1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * 32 + lane;
            if (i < n) ub[i] = to_key(r[u], lid[u]);
        }
    }
    __syncwarp();
    const uint64_t kth = n > K ? warp_kth(ub, n, (uint32_t)K, hist) : 0ull;
    uint64_t th = kth > floor ? kth : floor;
    if (th == 0ull) th = 1ull;                                   // key 0 = padding: never kept
    int pos = 0;
    constexpr int UC = 4;
    for (int i0 = 0; i0 < n; i0 += 32 * UC) {
        // in-place safe: writes land at indices <= the chunk being read
        uint64_t v[UC];
#pragma unroll
        for (int u = 0; u < UC; ++u) {
            const int i = i0 + u * 32 + lane;
            v[u] = i < n ? ub[i] : 0ull;
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < UC; ++u) {
            const bool keep = v[u] >= th;                         // (0 for i >= n)
            const unsigned bm = __ballot_sync(FULL, keep);
            if (keep) dst[pos + __popc(bm & lanemask_lt())] = v[u];
            pos += __popc(bm);
        }
        __syncwarp();
    }
    n_out = pos;
    return kth;
}

// Union floors at a unit's start (see K2_NQ): warp w takes users w, w + W, ...;
// lane l holds chunks l and l + 32 of the user's published keys.  Out of line so
// that its registers do not shape the scoring loop's allocation.
template <int W>
__device__ __noinline__ void union_floors(const volatile unsigned long long* qg, int chunks, int n_valid,
                                          unsigned long long* tau_sh, unsigned long long* gtau_g) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int u = warp; u < n_valid; u += W) {
        const volatile unsigned long long* qu = qg + (int64_t)u * chunks * K2_NQ;
        uint64_t v[2][K2_NQ];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int ch = lane + 32 * i;
#pragma unroll
            for (int l = 0; l < K2_NQ; ++l) v[i][l] = ch < chunks ? qu[ch * K2_NQ + l] : 0ull;
        }
        int c_ge[2][K2_NQ] = {};                          // published keys >= mine, per level
#pragma unroll 4
        for (int j = 0; j < 32; ++j) {
#pragma unroll
            for (int i2 = 0; i2 < 2; ++i2)
#pragma unroll
                for (int l = 0; l < K2_NQ; ++l) {
                    const uint64_t w = __shfl_sync(FULL, v[i2][l], j);
#pragma unroll
                    for (int i = 0; i < 2; ++i) c_ge[i][l] += w >= v[i][l];
                }
        }
        uint64_t fl = 0ull;
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int l = 0; l < K2_NQ; ++l)
                if (v[i][l] != 0ull && c_ge[i][l] >= (2 << l) && v[i][l] > fl) fl = v[i][l];
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const uint64_t t = __shfl_xor_sync(FULL, fl, o);
            fl = t > fl ? t : fl;
        }
        if (lane == 0 && fl != 0ull) {
            atomicMax(&tau_sh[u], (unsigned long long)fl);
            atomicMax(&gtau_g[u], (unsigned long long)fl);
        }
    }
}

// A finished unit's list -> its K2_NQ union-floor keys (one warp; out of line).
__device__ __noinline__ void union_publish(volatile unsigned long long* qo, const uint64_t* out, int nn, int K,
                                           uint32_t* hist) {
    const int lane = threadIdx.x & 31;
    __syncwarp();                                      // the list written by every lane
#pragma unroll 1
    for (int l = 0; l < K2_NQ; ++l) {
        const int r = (K + (2 << l) - 1) / (2 << l);
        const uint64_t key = nn >= r ? warp_kth(out, nn, (uint32_t)r, hist) : 0ull;
        if (lane == 0) qo[l] = key;
        __syncwarp();
    }
}

// ---------------------------------------------------------------- the kernel
// M splits, PS per phase (NP = M / PS phases), BT sub-ids, R users per table
// row, W warps, D slots of code prefetch, BT0 rows in split 0's table (BT0 !=
// BT: the exact first-pair table, single-phase only — see below).
// UQ: union floors (K2_NQ) compiled in -- a separate instantiation, selected by the
// planner for large K, so the other configurations' kernels do not carry its code.
// BAL: the balanced partition (K2TArgs::cut) instead of chunk x group units -- also
// its own instantiation (compiled into the common kernel it cost C5 2.5%).
template <int M, int PS, int BT, int R, int W, int D, int BT0 = BT, bool UQ = false, bool BAL = false>
__global__ void __launch_bounds__(W * 32, 1) k2_tiled(const K2TArgs a) {
    constexpr int NP = M / PS;
    // table buffers: NP == 1: one; NP > 1: a 2-slot ring (buffers 0, 1) for phases
    // 1 .. NP-1 plus buffer 2 holding phase 0's table for the whole unit (it is
    // the same for every tile of the unit), so a tile refills NP - 1 tables
    constexpr int NB = NP > 1 ? 3 : 1;
    constexpr int RES = 2;                             // resident phase-0 buffer (NP > 1)
    constexpr int LPR = R / 4;                         // lanes per row
    constexpr int RPS = 32 / LPR;                      // rows per warp slot
    constexpr int SL = 512 / W;                        // slots per warp per tile
    constexpr int TR = W * SL * RPS;                   // rows per tile
    constexpr uint32_t RB = R * 4;                     // bytes per table row
    constexpr uint32_t SPLITB = (uint32_t)BT * RB;     // bytes per split table (splits >= 1)
    constexpr uint32_t TBLB = (uint32_t)(BT0 + (PS - 1) * BT) * RB;   // bytes per table buffer
    constexpr int PSS = (PS == 3 || PS == 7) ? PS + 1 : PS;           // stored codes per row per phase
    constexpr int CB = PSS * K2_CODE_BYTES;            // code bytes per row per phase
    static_assert(M % PS == 0, "phases");
    static_assert(BT0 == BT || M == PS, "a first-pair table needs a single-phase table");
    // byte offset of split kk's table inside a buffer
    auto split_off = [](int kk) -> uint32_t { return kk == 0 ? 0u : (uint32_t)(BT0 + (kk - 1) * BT) * RB; };
    static_assert(SL % D == 0 && D % 2 == 0, "prefetch depth");
    static_assert(R == 16 || R == 32, "users per row");

    extern __shared__ __align__(1024) unsigned char sm_raw[];
    const long long t_kstart = kTrace ? clock64() : 0;  // diagnostics builds (-DK2_TRACE) only
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    // smem: [tables NB x TBLB][hist W x 1 KB][tau R x u64][cnt R][nconv R][mbar NB][done NB][tmem]
    uint32_t* hist_all = reinterpret_cast<uint32_t*>(sm_raw + NB * TBLB);
    uint32_t* hist = hist_all + warp * 256;
    unsigned long long* tau_sh = reinterpret_cast<unsigned long long*>(hist_all + W * 256);
    int* cnt_u = reinterpret_cast<int*>(tau_sh + R);
    int* nconv_u = cnt_u + R;
    unsigned long long* mbar = reinterpret_cast<unsigned long long*>(nconv_u + R);
    int* done = reinterpret_cast<int*>(mbar + NB);
    int* tiles_done = done + NB;                       // [W] tiles finished by each warp
    int* sflag = tiles_done + W;                       // [4] shrink requests (ring of slack + 1)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sflag + 4);
    constexpr int LM = RPS * W;                        // lanes per user in the CTA
    uint64_t* lmk = reinterpret_cast<uint64_t*>(sm_raw + align_up((size_t)(reinterpret_cast<char*>(tmem_slot + 4) -
                                                                  reinterpret_cast<char*>(sm_raw)), 16));
    const uint32_t tbl0 = smem_u32(sm_raw);
    const uint32_t bar0 = smem_u32(mbar);

    // Unit, tile and sequence counters are 32-bit (the planner bounds units and tiles by
    // 2^31; the sequence counters are only compared modulo small powers of two or over
    // short distances): 64-bit ones hold ~8 more registers live across the tile loop
    // (same-box A/B: C4 0.8782 -> 0.880, C3 +0.2%, C2 +0.5%).  The first-pair-table
    // kernels (C5) keep the 64-bit ones: their allocation came out 2.2% slower with 32.
    constexpr bool WIDE = BT0 != BT;
    using ctr_t = std::conditional_t<WIDE, int64_t, int>;
    using uctr_t = std::conditional_t<WIDE, int64_t, uint32_t>;
    const ctr_t n_tiles = (ctr_t)a.n_tiles, chunk_tiles = (ctr_t)a.chunk_tiles;
    const uctr_t units = (uctr_t)a.n_groups * (uctr_t)a.chunks;
    auto unit_tiles = [&](uctr_t u) -> ctr_t {
        const ctr_t t0 = (ctr_t)((uint32_t)u / (uint32_t)a.n_groups) * chunk_tiles;
        return min(n_tiles, t0 + chunk_tiles) - t0;
    };
    // TMA bulk copy: tables of (unit, phase) -> ring buffer `buf`
    auto issue_load_g = [&](int grp, int ph, int buf) {
        const char* src = reinterpret_cast<const char*>(a.St) +
                          (int64_t)grp * (BT0 + (M - 1) * BT) * RB + (int64_t)ph * PS * SPLITB;
        const uint32_t bar = bar0 + 8u * buf;
        fence_proxy_async();
        mbar_expect_tx(bar, TBLB);
        constexpr uint32_t PIECE = 16384;
#pragma unroll 1
        for (uint32_t off = 0; off < TBLB; off += PIECE)
            bulk_g2s(tbl0 + buf * TBLB + off, src + off, PIECE < TBLB - off ? PIECE : TBLB - off, bar);
    };
    auto issue_load = [&](uctr_t u, int ph, int buf) {
        issue_load_g((int)((uint32_t)u % (uint32_t)a.n_groups), ph, buf);
    };
    // balanced partition: this CTA's range of the (group, tile) sequence
    constexpr bool bal = BAL && NP == 1;
    ctr_t blin = bal ? a.cut[blockIdx.x] : 0;
    const ctr_t bend = bal ? a.cut[blockIdx.x + 1] : 0;
    // ring sequence (phases 1 .. NP-1 of every tile, unit by unit) advanced by one
    auto advance = [&](uctr_t& u, ctr_t& t, int& ph) {
        if (++ph == NP) {
            ph = 1;
            if (++t == unit_tiles(u)) { t = 0; u += gridDim.x; }
        }
    };

    // ---- one-time setup -------------------------------------------------
    if (threadIdx.x == 0) {
        for (int i = 0; i < NB; ++i) { mbar_init(bar0 + 8u * i, 1); done[i] = 0; }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < R) { tau_sh[threadIdx.x] = 0ull; cnt_u[threadIdx.x] = 0; nconv_u[threadIdx.x] = 0; }
    if (threadIdx.x < W) tiles_done[threadIdx.x] = 0;
    if (threadIdx.x < 4) sflag[threadIdx.x] = 0;
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
    // everything above overlapped the predecessor (PDL); the tables, thresholds
    // and buffers below are written by it or by earlier calls
    pdl_wait();
    pdl_trigger();                                     // K3 may be scheduled (it waits for this grid)
    // first loads: the unit's phase-0 table and ring positions 0, 1
    if (threadIdx.x == 0 && (bal ? blin < bend : (uctr_t)blockIdx.x < units)) {
        if constexpr (NP == 1) {
            if (bal) issue_load_g((int)((uint32_t)blin / (uint32_t)n_tiles), 0, 0);
            else issue_load(blockIdx.x, 0, 0);
        } else {
            issue_load(blockIdx.x, 0, RES);
            uctr_t u = blockIdx.x;
            ctr_t t = 0;
            int ph = 1;
            for (int i = 0; i < 2 && u < units; ++i) {
                issue_load(u, ph, i);
                advance(u, t, ph);
            }
        }
    }

    // TMEM: this warp's lane quadrant and column range
    constexpr int WPQ = W / 4;                         // warps per lane quadrant
    const uint32_t tcol0 = tmem_base + ((uint32_t)((warp & 3) * 32) << 16) +
                           (uint32_t)((warp >> 2) * (512 / WPQ));

    const int q = lane % LPR;                          // user quad
    const uint32_t q16 = (uint32_t)q * 16u;
    uint64_t* ubuf = a.ubuf + (int64_t)blockIdx.x * R * a.cap;
    uctr_t gseq = 0;                                   // table uses so far (NP > 1)
    uctr_t useq = 0;                                   // units done by this CTA (NP == 1)
    // Shrink protocol (no per-tile barrier), with a skew allowance of S = slack
    // tiles: the insert that takes a user's buffer to `wm` entries during tile
    // T records T + S in sflag[T % (S + 1)]; at the end of tile T + S every warp
    // (having waited until all warps finished tile T) sees the same flag and the
    // CTA shrinks (a warp passes the end of tile X once all warps finished X - S).
    // Uniformity: a warp reads the slot only after every warp finished tile T,
    // so the flag is final; a request forces a CTA barrier before anyone can
    // start tile T + S + 1, whose requests reuse the slot.  Capacity: when a warp
    // in tile T makes the request, slower warps may still be in tile T - S; with
    // tiles up to T + S that is at most (2S + 1) * TR entries per user before
    // the shrink: cap >= wm + (2S + 1) * TR.
    const int wm = a.wm;
    ctr_t tseq = 0;                                    // tiles done by this CTA

    constexpr int64_t PSTR = 2 * RPS * CB;             // code bytes per slot pair
    constexpr int DP = D / 2;                          // slot pairs per group
    __shared__ unsigned long long t_start_ns;
    if (kTrace && a.trace && threadIdx.x == 0) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start_ns));
    }
    for (uctr_t unit = blockIdx.x; bal ? blin < bend : unit < units; unit += gridDim.x) {
        if (kTrace && a.trace && blockIdx.x == 0 && threadIdx.x == 0 && useq < TRACE_PH / 2)
            a.trace[(int64_t)W * TRACE_PH * 3 + 2 * useq] = clock64();
#define K2_STAMP(i) do { if (kTrace && a.dbg && blockIdx.x == 0 && threadIdx.x == 0 && useq == 0) \
        a.dbg[32 + (i)] = (int)(clock64() - t_kstart); } while (0)
        K2_STAMP(0);
        int chunk, grp;
        ctr_t tile0, ntl;
        if constexpr (bal) {
            grp = (int)((uint32_t)blin / (uint32_t)n_tiles);
            const ctr_t g0 = (ctr_t)grp * n_tiles;
            tile0 = blin - g0;
            ntl = min(bend - blin, n_tiles - tile0);
            int p0 = blockIdx.x;                       // the CTA whose range holds the group's first tile
            while (p0 > 0 && a.cut[p0] > g0) --p0;
            chunk = (int)blockIdx.x - p0;
            blin += ntl;                               // (now the next unit's first position)
        } else {
            chunk = (int)((uint32_t)unit / (uint32_t)a.n_groups);
            grp = (int)(unit - (uctr_t)chunk * (uctr_t)a.n_groups);
            tile0 = (ctr_t)chunk * chunk_tiles;
            ntl = unit_tiles(unit);
        }
        unsigned long long* gtau_g = a.gtau + (int64_t)grp * R;  // this group's users
        const int n_valid = min(R, a.B - grp * R);
        if (threadIdx.x < n_valid)                                // K keys >= gtau exist elsewhere
            tau_sh[threadIdx.x] = *reinterpret_cast<volatile unsigned long long*>(&gtau_g[threadIdx.x]);
        __syncthreads();
        if constexpr (UQ) {                                       // union floors (chunks <= 64)
            union_floors<W>(a.qk + (int64_t)grp * R * a.chunks * K2_NQ, a.chunks, n_valid, tau_sh, gtau_g);
            __syncthreads();
        }
        float tf[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            tf[j] = (4 * q + j < n_valid) ? tau_to_filter(tau_sh[4 * q + j]) : INFINITY;

        // Threshold seeding (single-phase tables, no threshold known yet): one
        // extra pass over the unit's first tile computes, per user, each lane's
        // best score; the K-th largest of those LM lane maxima (distinct items)
        // proves a score floor, so the real first pass inserts ~K candidates
        // per user instead of the whole tile (which would then need a costly
        // shrink).
        K2_STAMP(1);
        if constexpr (NP == 1) {
            bool any_unset = false;
            for (int u = 0; u < n_valid; ++u) any_unset |= tau_sh[u] == 0ull;
            if (any_unset && a.K <= LM) {
                const char* tb = reinterpret_cast<const char*>(sm_raw);
                const int64_t tile = tile0;
                const char* cp = reinterpret_cast<const char*>(a.codes) +
                                 (tile * TR + ((int64_t)warp * SL * RPS + (lane / LPR) * 2)) * CB;
                const uint32_t row0 = (uint32_t)(tile * TR) + (uint32_t)(warp * SL * RPS) + (uint32_t)(lane / LPR);
                float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
                bool got = false;
                // a quarter of the tile suffices; every code word and padding flag is
                // requested before the wait for the table, so the pass itself is SEEDP
                // slot pairs of shared-memory gathers (it was a chain of dependent global
                // loads; C2 K2 -1% on the same box)
                constexpr int SEEDP = SL / 8;
                CodePair<PSS> cps[SEEDP];
                int32_t pad[SEEDP][2];
#pragma unroll
                for (int i = 0; i < SEEDP; ++i) {
                    CodePair<PSS>::check(cp + (int64_t)i * 2 * RPS * CB,
                                         reinterpret_cast<const char*>(a.codes), a.codes_bytes);
                    cps[i].load(cp + (int64_t)i * 2 * RPS * CB);
                }
#pragma unroll
                for (int i = 0; i < SEEDP; ++i)
#pragma unroll
                    for (int e = 0; e < 2; ++e) pad[i][e] = __ldg(&a.perm[row0 + (uint32_t)(2 * i + e) * RPS]);
                mbar_wait(bar0, (uint32_t)(useq & 1));
#pragma unroll
                for (int i = 0; i < SEEDP; ++i) {
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                        for (int kk = 0; kk < PS; ++kk) {
                            const uint32_t off = cps[i].template off<RB>(e, kk, q16);
                            const float4 v = lds128(tb + split_off(kk) + off);
                            if (kk == 0) acc = v; else add4(acc, v);
                        }
                        if (pad[i][e] >= 0) {
                            got = true;
                            mx[0] = fmaxf(mx[0], acc.x); mx[1] = fmaxf(mx[1], acc.y);
                            mx[2] = fmaxf(mx[2], acc.z); mx[3] = fmaxf(mx[3], acc.w);
                        }
                    }
                }
                const int li = warp * RPS + lane / LPR;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float v = mx[j] + 0.0f;
                    const uint32_t ub = __float_as_uint(v);
                    const uint32_t o = (ub & 0x80000000u) ? ~ub : (ub | 0x80000000u);
                    lmk[(4 * q + j) * LM + li] = got ? (((uint64_t)o << 32) | (uint32_t)(li + 1)) : 0ull;
                }
                __syncthreads();
                for (int u = warp; u < n_valid; u += W) {
                    if (tau_sh[u] != 0ull) continue;
                    const uint64_t kth = warp_kth(lmk + u * LM, LM, (uint32_t)a.K, hist);
                    // K distinct items score >= kth's score: floor = that score, any id
                    if (lane == 0 && kth != 0ull) tau_sh[u] = kth & 0xFFFFFFFF00000000ull;
                }
                __syncthreads();
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (tf[j] != INFINITY) tf[j] = fmaxf(tf[j], tau_to_filter(tau_sh[4 * q + j]));
            }
        }

        K2_STAMP(2);
        for (ctr_t t = 0; t < ntl; ++t) {
            const int64_t tile = tile0 + t;
#pragma unroll
            for (int ph = 0; ph < NP; ++ph) {
                const int buf = NP == 1 ? 0 : (ph == 0 ? RES : (int)(gseq & 1));
                const uint32_t par = (NP == 1 || ph == 0) ? (uint32_t)(useq & 1) : (uint32_t)((gseq >> 1) & 1);
                int64_t tix = TRACE_PH;
                bool trc = false;
                if constexpr (kTrace) {
                    const int64_t tq = tseq - a.trace_from;
                    tix = (tq >= 0 && tq % a.trace_stride == 0) ? (tq / a.trace_stride) * NP + ph : TRACE_PH;
                    trc = a.trace && blockIdx.x == 0 && lane == 0 && tix < TRACE_PH;
                }
                if (trc) a.trace[((int64_t)warp * TRACE_PH + tix) * 3 + 0] = clock64();
                mbar_wait(bar0 + 8u * buf, par);
                if (trc) a.trace[((int64_t)warp * TRACE_PH + tix) * 3 + 1] = clock64();
                const char* tb = reinterpret_cast<const char*>(sm_raw) + buf * TBLB;
#ifndef K2_NO_ASM_LDS
                uint32_t tbq32 = tbl0 + (uint32_t)buf * TBLB + q16;
                asm volatile("" : "+r"(tbq32) :: "memory");   // defined after the wait: no gather moves above it
#endif
                const uint32_t row0 = (uint32_t)(tile * TR) + (uint32_t)(warp * SL * RPS) + (uint32_t)(lane / LPR);
                // codes of this warp's slot pairs: [pair][row][2 slots][PS]
                const char* cp = reinterpret_cast<const char*>(a.codes) + ((tile * NP + ph) * TR +
                                 ((int64_t)warp * SL * RPS + (lane / LPR) * 2)) * CB;
                CodePair<PSS> cw[DP];
#pragma unroll
                for (int d = 0; d < DP; ++d) {
                    CodePair<PSS>::check(cp + d * PSTR, reinterpret_cast<const char*>(a.codes), a.codes_bytes);
                    cw[d].load(cp + d * PSTR);
                }
                cp += DP * PSTR;
                uint32_t tcur[4] = {0u, 0u, 0u, 0u};   // partial sums of slot s (ph > 0)
                if (ph > 0) {
                    tm_ld_issue(tcol0, tcur);
                    tm_ld_wait(tcur);
                }
#pragma unroll 1
                for (int s0 = 0; s0 < SL; s0 += D) {
                    float4 accs[D];                    // last phase: candidate sums of the group
                    unsigned cmask = 0u;               // last phase: bits 4d..4d+3 = slot d's users may qualify
                    // software pipeline (single-phase tables): the gathers of slot
                    // d + 1 are issued before the adds of slot d (two slots of loads
                    // in flight); with TMEM phases the register budget favours one
                    constexpr bool PIPE = (NP == 1);
                    float4 vb[2][PS];
                    auto gather = [&](int d, float4 (&dst)[PS]) {
#pragma unroll
                        for (int kk = 0; kk < PS; ++kk) {
                            PQ_DCHECK(split_off(kk) + cw[d >> 1].template off<RB>(d & 1, kk, q16) + 16 <= TBLB);
#ifndef K2_NO_ASM_LDS
                            // 32-bit shared address = code * RB + (buffer + quad offset): ONE IMAD per
                            // gather (with a generic pointer the compiler adds base and quad separately)
                            dst[kk] = lds128_s(cw[d >> 1].template off<RB>(d & 1, kk, tbq32), split_off(kk));
#else
                            dst[kk] = lds128(tb + split_off(kk) + cw[d >> 1].template off<RB>(d & 1, kk, q16));
#endif
                        }
                        if (d & 1) {                   // both slots of the pair addressed: refill
                            CodePair<PSS>::check(cp, reinterpret_cast<const char*>(a.codes), a.codes_bytes);
                            cw[d >> 1].load(cp);       // DP pairs ahead (buffer is padded)
                            cp += PSTR;
                        }
                    };
                    if constexpr (PIPE) gather(0, vb[0]);
#pragma unroll
                    for (int d = 0; d < D; ++d) {
                        const int s = s0 + d;
                        if constexpr (PIPE) {
                            if (d + 1 < D) gather(d + 1, vb[(d + 1) & 1]);
                        } else {
                            gather(d, vb[d & 1]);
                        }
                        float4 (&v)[PS] = vb[d & 1];
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
                        } else {
                            // last phase: branch-free candidate filter for the group
                            accs[d] = acc;
                            if constexpr (NP == 1) {
                                // acc + (-tf) >= 0 <=> acc >= tf exactly (IEEE subtraction keeps
                                // the sign and is 0 only for equal operands; -inf / +inf
                                // thresholds give +inf / -inf): a packed subtract pair and a
                                // max tree per slot (measured faster for single-phase tables)
                                const float2 dlo = __fadd2_rn(make_float2(acc.x, acc.y), make_float2(-tf[0], -tf[1]));
                                const float2 dhi = __fadd2_rn(make_float2(acc.z, acc.w), make_float2(-tf[2], -tf[3]));
                                const float mx = fmaxf(fmaxf(dlo.x, dlo.y), fmaxf(dhi.x, dhi.y));
                                cmask |= (mx >= 0.0f ? 0xFu : 0u) << (4 * d);
                            } else {
                                cmask |= ((acc.x >= tf[0]) ? 1u : 0u) << (4 * d);
                                cmask |= ((acc.y >= tf[1]) ? 2u : 0u) << (4 * d);
                                cmask |= ((acc.z >= tf[2]) ? 4u : 0u) << (4 * d);
                                cmask |= ((acc.w >= tf[3]) ? 8u : 0u) << (4 * d);
                            }
                        }
                    }
                    if (ph == NP - 1 && cmask) {       // rare slow path: shared atomic + store
#pragma unroll
                        for (int d = 0; d < D; ++d) {
                            const uint32_t row = row0 + (uint32_t)(s0 + d) * RPS;
                            const float vv[4] = {accs[d].x, accs[d].y, accs[d].z, accs[d].w};
#pragma unroll
                            if (!(cmask >> (4 * d) & 0xFu)) continue;
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                if (!(cmask >> (4 * d + j) & 1u) || !(vv[j] >= tf[j])) continue;
                                const int u = 4 * q + j;
                                const int p = atomicAdd(&cnt_u[u], 1);
#ifdef K2_TRACE_INSERTS                                         // (global atomics: distorts the timeline)
                                if (kTrace && a.dbg) {
                                    atomicAdd(reinterpret_cast<unsigned long long*>(a.dbg + 16), 1ull);   // inserts
                                    if (t == 0) atomicAdd(reinterpret_cast<unsigned long long*>(a.dbg + 28), 1ull);
                                }
#endif
                                if (p >= a.cap) __trap();      // protocol invariant: cap >= wm + (2S + 1) TR
                                ubuf[(int64_t)u * a.cap + p] = make_raw(vv[j] + 0.0f, row);
                                if (p == wm) {
                                    *reinterpret_cast<volatile int*>(&sflag[(uint32_t)tseq % (uint32_t)(K2_SLACK + 1)]) =
                                        (int)(tseq + K2_SLACK);
                                    __threadfence_block();
                                }
                            }
                        }
                    }
                }
                if (NP == 1 && trc) a.trace[((int64_t)warp * TRACE_PH + tix) * 3 + 2] = clock64();
                if constexpr (NP > 1) {
                    if (ph < NP - 1) tm_wait_st();
                    // release the buffer: the last warp to finish with it loads
                    // the table this ring slot serves next (position + NB)
                    __syncwarp();
                    if (lane == 0) {
                        const int old = atomicAdd(&done[buf], 1);
                        if (trc) a.trace[((int64_t)warp * TRACE_PH + tix) * 3 + 2] = clock64();
                        if (old == W - 1) {
                            done[buf] = 0;
                            if (ph == 0) {             // resident table: reload after the unit's last tile
                                if (t + 1 == ntl && unit + gridDim.x < units) issue_load(unit + gridDim.x, 0, RES);
                            } else {                   // ring: load the position this slot serves next
                                uctr_t u2 = unit;
                                ctr_t t2 = t;
                                int ph2 = ph;
                                for (int st = 0; st < 2; ++st) advance(u2, t2, ph2);
                                if (u2 < units) issue_load(u2, ph2, buf);
                            }
                        }
                    }
                    if (ph > 0) ++gseq;
                }
            }

            // ---- end of tile T = tseq: shrink if requested during tile T - 1
            // (no memory fence here: a fence would also wait for this warp's
            // outstanding global loads; the only cross-warp data read without a
            // barrier is sflag, fenced by its writer, and __syncwarp orders the
            // writer lane before lane 0's tiles_done store)
            const long long t_eot = kTrace ? clock64() : 0;   // diagnostics builds only
            if (t == 0) K2_STAMP(3);
            __syncwarp();
            if (lane == 0) *reinterpret_cast<volatile int*>(&tiles_done[warp]) = (int)(tseq + 1);
            // wait until every warp has finished tile T - S (bounds the skew to S tiles)
            for (long long spins = 0;; ++spins) {
                if (kTrace && a.dbg && spins == 1 && lane == 0)
                    atomicAdd(reinterpret_cast<unsigned long long*>(a.dbg + 24), 1ull);   // waits
                const int td = lane < W ? *reinterpret_cast<volatile int*>(&tiles_done[lane]) : INT_MAX;
                if (__all_sync(FULL, td >= (int)tseq - K2_SLACK + 1)) break;
                PQ_DCHECK(spins < PQ_SPIN_LIMIT);      // checked builds: a lost warp traps
                __nanosleep(64);                       // back off: spinning would steal smem cycles
                if (a.dbg && spins > (1ll << 26)) {
                    if (lane == 0 && atomicAdd(&a.dbg[0], 1) == 0) {
                        a.dbg[1] = blockIdx.x; a.dbg[2] = warp; a.dbg[3] = (int)tseq;
                        a.dbg[4] = 0; a.dbg[5] = (int)unit; a.dbg[6] = (int)t; a.dbg[7] = (int)ntl;
                        a.dbg[8] = sflag[0]; a.dbg[9] = sflag[1];
                    }
                    break;
                }
            }
            // (always after a unit's first tile: it ran with the unit's initial,
            // usually weak or only seeded, thresholds -- an early exact K-th keeps
            // the next tiles' candidate lists short; measured: C3 -1.1%)
            const bool need = (t == 0) || (tseq >= K2_SLACK &&
                *reinterpret_cast<volatile int*>(&sflag[(uint32_t)(tseq - K2_SLACK) % (uint32_t)(K2_SLACK + 1)]) ==
                    (int)tseq);
            const long long t_shr = kTrace ? clock64() : 0;
            if (need) {                                // uniform across the CTA
                __syncthreads();                       // every insert so far is visible
                if (kTrace && a.dbg && threadIdx.x == 0) atomicAdd(a.dbg + 18, 1);   // shrinks
                for (int u = warp; u < n_valid; u += W) {
                    const int n = cnt_u[u];
                    if (n <= a.K) continue;
                    uint64_t* ub = ubuf + (int64_t)u * a.cap;
                    int nn;
                    const uint64_t kth = shrink_user<BT0 == BT>(ub, nconv_u[u], n, a.K, tau_sh[u], ub, hist,
                                                     a.perm, a.id_base, nn);
                    if (lane == 0) {
                        cnt_u[u] = nn;
                        nconv_u[u] = nn;
                        if (kth) {
                            atomicMax(&tau_sh[u], (unsigned long long)kth);
                            atomicMax(&gtau_g[u], (unsigned long long)kth);
                        }
                    }
                }
                // adopt thresholds proved by other CTAs on other chunks of these users (loading
                // them before the selections measured 2% slower on C2)
                if (threadIdx.x < n_valid)
                    atomicMax(&tau_sh[threadIdx.x], *reinterpret_cast<volatile unsigned long long*>(&gtau_g[threadIdx.x]));
                __syncthreads();
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (tf[j] != INFINITY) tf[j] = fmaxf(tf[j], tau_to_filter(tau_sh[4 * q + j]));
            }
            if (kTrace && a.dbg && lane == 0) {
                const long long t_end = clock64();
                atomicAdd(reinterpret_cast<unsigned long long*>(a.dbg + 20), (unsigned long long)(t_end - t_eot));
                atomicAdd(reinterpret_cast<unsigned long long*>(a.dbg + 22), (unsigned long long)(t_end - t_shr));
            }
            if (t == 0) K2_STAMP(4);
            ++tseq;
        }
        K2_STAMP(5);

        // ---- end of unit: each user's buffer -> the unit's top-K list -------
        __syncthreads();
        if constexpr (NP == 1) {
            // every warp is done with the table: prefetch the next unit's
            // (nothing about the next unit is kept live across the tile loop: two more
            // registers there cost C5 2.5%)
            if constexpr (bal) {
                if (threadIdx.x == 0 && blin < bend) issue_load_g(grp + 1, 0, 0);
            } else {
                if (threadIdx.x == 0 && unit + gridDim.x < units) issue_load(unit + gridDim.x, 0, 0);
            }
        }
        for (int u = warp; u < n_valid; u += W) {
            const int gu = grp * R + u;
            PQ_DCHECK(gu < a.B && chunk < a.chunks && cnt_u[u] <= a.cap);
            uint64_t* out = a.cand + ((int64_t)gu * a.chunks + chunk) * a.K;
            uint64_t* ub = ubuf + (int64_t)u * a.cap;
            int nn;
            const uint64_t kth = shrink_user<BT0 == BT>(ub, nconv_u[u], cnt_u[u], a.K, tau_sh[u], out, hist,
                                             a.perm, a.id_base, nn);
            if (lane == 0 && kth) atomicMax(&gtau_g[u], (unsigned long long)kth);
            if (a.lcnt) {                                  // K3 reads nn entries: no padding
                if (lane == 0) a.lcnt[(int64_t)gu * a.chunks + chunk] = nn;
            } else {
                for (int j = nn + lane; j < a.K; j += 32) out[j] = 0ull;
            }
            if constexpr (UQ)                              // publish this chunk's union-floor keys
                union_publish(a.qk + ((int64_t)gu * a.chunks + chunk) * K2_NQ, out, nn, a.K, hist);
        }
        __syncthreads();
        K2_STAMP(6);
        if (threadIdx.x < R) { tau_sh[threadIdx.x] = 0ull; cnt_u[threadIdx.x] = 0; nconv_u[threadIdx.x] = 0; }
        if (kTrace && a.trace && blockIdx.x == 0 && threadIdx.x == 0 && useq < TRACE_PH / 2)
            a.trace[(int64_t)W * TRACE_PH * 3 + 2 * useq + 1] = clock64();
        ++useq;
    }
    if (kTrace && a.trace && threadIdx.x == 0 && blockIdx.x < TRACE_CTAS) {
        unsigned long long t_end_ns;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end_ns));
        long long* c = a.trace + (int64_t)W * TRACE_PH * 3 + TRACE_PH + 3 * blockIdx.x;
        c[0] = (long long)t_start_ns; c[1] = (long long)t_end_ns; c[2] = tseq;
    }

    if (kTrace && a.dbg && lane == 0) {                // diagnostics: warp lifetime
        long long t_now = clock64();
        atomicAdd(reinterpret_cast<unsigned long long*>(a.dbg + 26), (unsigned long long)(t_now - t_kstart));
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
// St[g][k][c][w] = S[R g + w][k][cmap[k][c]] (0 for padding users): the R-user
// interleaved table layout (colour-renumbered for R = 16), so K2 can stage a
// phase's tables with one contiguous bulk copy.
__global__ void k2_tile_S(const float* __restrict__ S, const uint8_t* __restrict__ cmap, int B, int m,
                          int b, int R, int n_groups, float* __restrict__ St, unsigned long long* gtau, int64_t nz) {
    pdl_wait();                                        // S comes from K1
    pdl_trigger();
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < nz; x += (int64_t)gridDim.x * blockDim.x)
        gtau[x] = 0ull;                                // the call's shared thresholds (+ union floors) start unset
    const int64_t total = (int64_t)n_groups * m * b * R;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        // (g, k, c, w) of x; the table has < 2^32 entries: 32-bit unsigned arithmetic
        const uint32_t xx = (uint32_t)x;
        const int w = (int)(xx % (uint32_t)R);
        const uint32_t r = xx / (uint32_t)R;
        const int c = (int)(r % (uint32_t)b);
        const uint32_t gk = r / (uint32_t)b;
        const int k = (int)(gk % (uint32_t)m);
        const int g = (int)(gk / (uint32_t)m);
        const int user = g * R + w;
        St[x] = user < B ? S[((int64_t)user * m + k) * b + cmap[k * b + c]] : 0.0f;
    }
}

// First-pair tables: St[g][row][w], rows 0..255 = fl(S[u][0][c % 16] + S[u][1][c / 16])
// (the first partial sum of Eq. 5 in the sequential order), then 16 rows per
// remaining split k = 2 .. m-1.
__global__ void k2_tile_S_pair(const float* __restrict__ S, int B, int m, int R, int n_groups,
                               float* __restrict__ St, unsigned long long* gtau, int64_t nz) {
    pdl_wait();                                        // S comes from K1
    pdl_trigger();
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < nz; x += (int64_t)gridDim.x * blockDim.x)
        gtau[x] = 0ull;                                // the call's shared thresholds (+ union floors) start unset
    const int rows = 256 + (m - 2) * 16;
    const int64_t total = (int64_t)n_groups * rows * R;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t xx = (uint32_t)x;               // < 2^32 entries
        const int w = (int)(xx % (uint32_t)R);
        const uint32_t r = xx / (uint32_t)R;
        const int row = (int)(r % (uint32_t)rows);
        const int g = (int)(r / (uint32_t)rows);
        const int user = g * R + w;
        float v = 0.0f;
        if (user < B) {
            const float* Su = S + (int64_t)user * m * 16;
            if (row < 256) v = Su[row % 16] + Su[16 + row / 16];          // fp32 RN, split 0 then 1
            else v = Su[(2 + (row - 256) / 16) * 16 + (row - 256) % 16];
        }
        St[x] = v;
    }
}

// ---------------------------------------------------------------- host side
typedef void (*K2TFn)(const K2TArgs);

template <int M, int PS, int BT, int R, int BT0 = BT>
static K2TFn tiled_fn_w(int W, bool uq, bool bal) {
    // deeper code prefetch for m = 16 (C4: -1.7 %; m = 8 and m = 64 prefer 4)
    if constexpr (M == PS) {                           // single-phase tables: balanced / union-floor variants
        if (bal) {
            if (W == 16) return k2_tiled<M, PS, BT, R, 16, 4, BT0, false, true>;
            return k2_tiled<M, PS, BT, R, 8, 4, BT0, false, true>;
        }
        if (uq) {
            if (W == 16) return k2_tiled<M, PS, BT, R, 16, 4, BT0, true>;
            return k2_tiled<M, PS, BT, R, 8, 4, BT0, true>;
        }
    }
    if (W == 16) return k2_tiled<M, PS, BT, R, 16, (M == 16 ? 8 : 4), BT0>;
    return k2_tiled<M, PS, BT, R, 8, 4, BT0>;
}
// Exact first-pair tables (b = 16, m in {4, 8}): splits 0 and 1 become one
// 256-row "split" whose row c = g0 + 16 g1 holds fl(S[0][g0] + S[1][g1]) -- the
// first partial sum of Eq. 5 exactly as the sequential order computes it -- so
// an item costs m - 1 lookups.
static K2TFn tiled_pair_fn(int m_v, int W, bool uq = false, bool bal = false) {
    if (m_v == 3) return tiled_fn_w<3, 3, 16, 32, 256>(W, uq, bal);
    if (m_v == 7) return tiled_fn_w<7, 7, 16, 32, 256>(W, uq, bal);
    return nullptr;
}
// Instantiated shapes: R = 16 (paired layout) for b = 256, m in {8, 16, 32, 64};
// R = 32 (item order) when the 32-user table fits: (m, b) in {(4, 16), (8, 16), (4, 256)}.
static K2TFn tiled_fn(int m, int b, int R, int W, bool uq = false, bool bal = false) {
    if (R == 16 && b == 256) {
        if (m == 16) return tiled_fn_w<16, 4, 256, 16>(W, uq, bal);
        if (m == 8) return tiled_fn_w<8, 8, 256, 16>(W, uq, bal);
    }
    if (R == 32 && b == 16) {
        if (m == 4) return tiled_fn_w<4, 4, 16, 32>(W, uq, bal);
        if (m == 8) return tiled_fn_w<8, 8, 16, 32>(W, uq, bal);
    }
    if (R == 32 && b == 256 && m == 4) return tiled_fn_w<4, 4, 256, 32>(W, uq, bal);
    // many splits (Fig. 2b's m = 64): 16 users, phases of 4 splits; pq_create pairs
    // items on complementary colours over the first 20 splits (64-split signatures
    // have no complements), so those splits' gathers are conflict-free
    if (R == 16 && b == 256 && m == 32) return tiled_fn_w<32, 4, 256, 16>(W, uq, bal);
    if (R == 16 && b == 256 && m == 64) return tiled_fn_w<64, 4, 256, 16>(W, uq, bal);
    return nullptr;
}
int k2_tiled_ps(int m) { return m >= 16 ? 4 : m; }

TiledShape k2_tiled_shape(int m, int b) {
    TiledShape t{};
    if (b == 16 && (m == 4 || m == 8) && tiled_pair_fn(m - 1, 16)) {
        t.R = 32; t.pair = 1; t.m_v = m - 1; t.ps = m - 1; t.bt = 16; t.bt0 = 256;
    } else if (tiled_fn(m, b, 32, 16)) {
        t.R = 32; t.m_v = m; t.ps = k2_tiled_ps(m); t.bt = b; t.bt0 = b;
    } else if (tiled_fn(m, b, 16, 16)) {
        t.R = 16; t.m_v = m; t.ps = k2_tiled_ps(m); t.bt = b; t.bt0 = b;
    } else {
        return t;                                      // R = 0: unsupported
    }
    t.pss = (t.ps == 3 || t.ps == 7) ? t.ps + 1 : t.ps;
    return t;
}
static K2TFn tiled_fn_shape(const TiledShape& t, int W, bool uq = false, bool bal = false) {
    return t.pair ? tiled_pair_fn(t.m_v, W, uq, bal) : tiled_fn(t.m_v, t.bt, t.R, W, uq, bal);
}
int k2_tiled_users(int m, int b) { return k2_tiled_shape(m, b).R; }
bool k2_tiled_supported(int m, int b) { return k2_tiled_users(m, b) > 0; }
int k2_tiled_rows_per_tile(int R) { return R == 32 ? 2048 : 4096; }

size_t k2_tiled_smem(const TiledShape& t, int W) {
    const int R = t.R;
    const int nb = (t.m_v / t.ps) > 1 ? 3 : 1;
    const size_t tbl = (size_t)(t.bt0 + (t.ps - 1) * t.bt) * R * 4;
    const size_t base = (size_t)nb * tbl + (size_t)W * 1024 + (size_t)R * 8 + (size_t)R * 8 +
                        3 * 8 + 3 * 4 + (size_t)(W + 4) * 4 + 16;
    const size_t lm = nb == 1 ? (size_t)R * (32 / (R / 4)) * W * 8 : 0;   // threshold seeding keys
    return align_up(base, 16) + lm + 16;
}
static int k2_slack() { return K2_SLACK; }
static int64_t qk_words(const K2Plan& p) { return p.qk ? (int64_t)p.n_groups * p.G * p.chunks * K2_NQ : 0; }
static size_t st_table_bytes(const TiledShape& t, int n_groups) {
    return (size_t)n_groups * (t.bt0 + (t.m_v - 1) * t.bt) * t.R * 4;
}

// Item chunks per user group.  Units (group x chunk) are dealt round-robin to
// the persistent CTAs; a unit costs its tiles plus a fixed overhead (first-tile
// shrink, end-of-unit merge and, for single-phase tables, the table load), in
// tile units `ovh`.  Pick the chunk count with the best modelled efficiency.
static int choose_chunks_tiles(int64_t n_tiles, int n_groups, int grid_full, double ovh) {
    const int64_t max_c = std::max<int64_t>(1, std::min<int64_t>(4096, n_tiles));
    int best = 1;
    double best_eff = -1.0;
    for (int64_t c = 1; c <= max_c; ++c) {
        const int64_t ct = ceil_div(n_tiles, c);
        const int64_t cc = ceil_div(n_tiles, ct);        // chunks actually formed
        const int64_t units = (int64_t)n_groups * cc;
        const int64_t per_cta = ceil_div(units, grid_full);
        const double eff = (double)n_groups * n_tiles / ((double)per_cta * grid_full * (ct + ovh));
        if (eff > best_eff + 1e-9) { best_eff = eff; best = (int)cc; }
    }
    return best;
}

// Balanced partition for single-phase tables.  The (group, tile) pairs in group-major
// order are cut into at most P contiguous ranges, one per CTA; a range costs its tiles
// plus `ovh4` quarter-tiles for every group it touches (table load, seeding, first-tile
// shrink, end-of-unit list: a unit each).  The smallest feasible bound on a range's
// cost is found by bisection over a greedy fill.  Returns that bound (quarter-tiles)
// and fills cut[0 .. n_cut]; 0 if no partition into <= P ranges exists.
static int64_t balanced_cuts(int64_t T, int G, int P, int64_t ovh4, std::vector<int64_t>& cut) {
    const int64_t total = (int64_t)G * T;
    auto fill = [&](int64_t M4, std::vector<int64_t>* out) -> int {
        int64_t lin = 0;
        int np = 0;
        if (out) { out->clear(); out->push_back(0); }
        while (lin < total) {
            int64_t budget = M4;
            const int64_t lin0 = lin;
            while (lin < total) {
                const int64_t left = (lin / T + 1) * T - lin;
                const int64_t avail = (budget - ovh4) / 4;
                if (avail < 1) break;
                const int64_t take = std::min(left, avail);
                lin += take;
                budget -= ovh4 + 4 * take;
                if (take < left) break;
            }
            if (lin == lin0) return INT_MAX;            // not even one tile fits
            if (out) out->push_back(lin);
            if (++np > P) return np;
        }
        return np;
    };
    int64_t lo = ovh4 + 4, hi = 4 * total + (int64_t)G * ovh4 + 4;
    if (fill(hi, nullptr) > P) return 0;
    while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (fill(mid, nullptr) <= P) hi = mid; else lo = mid + 1;
    }
    fill(lo, &cut);
    return lo;
}

void plan_k2_tiled(const pq_index_s* idx, int B, int K, K2Plan& p) {
    p.variant = 3;
    const pq_tuning& t = idx->tuning;
    const TiledShape sh = k2_tiled_shape(idx->m, idx->b);
    const int R = sh.R;
    p.W = (t.warps == 8 || t.warps == 16) ? t.warps : 16;
    p.G = R; p.Ug = R; p.J = 1;
    p.tm = (sh.m_v / sh.ps) > 1 ? sh.m_v - sh.ps : 0;
    p.n_groups = (int)ceil_div(B, R);
    const int TR = k2_tiled_rows_per_tile(R);
    // shrink watermark: 2K + 64, but >= 2048 for K <= 16 -- with a small K the early,
    // weak-threshold tiles would otherwise shrink (a CTA barrier that absorbs the
    // warps' skew) again and again: C2 K2 0.2117 -> 0.2067 ms; larger watermarks cost
    // C3 (K = 100) time in the end-of-unit selection (r03 A/B, PQTOPK_K2_WMIN)
    static const int wmin = getenv("PQTOPK_K2_WMIN") ? atoi(getenv("PQTOPK_K2_WMIN")) : 0;
    const int wm_auto = std::max(std::max(2 * K + 64, K <= 16 ? 2048 : 0), wmin);
    p.cap = (int)align_up((size_t)(wm_auto + (2 * k2_slack() + 1) * TR + 32), 32);
    p.smem = k2_tiled_smem(sh, p.W);
    K2TFn fn = tiled_fn_shape(sh, p.W);
    if (!fn) fail(PQ_ERR_UNSUPPORTED, "tiled scoring kernel: unsupported shape");
    ensure_max_smem(reinterpret_cast<const void*>(fn), (int)p.smem);
    int occ = 0;
    PQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, p.W * 32, p.smem));
    if (occ < 1) fail(PQ_ERR_UNSUPPORTED, "tiled scoring kernel cannot be resident");
    occ = 1;                                           // one TMEM allocation / table set per SM
    const int grid_full = idx->num_sms * occ;
    const int64_t n_tiles = idx->v3_tiles;
    p.chunks = t.chunks > 0 ? (int)std::min<int64_t>(t.chunks, n_tiles)
                            : choose_chunks_tiles(n_tiles, p.n_groups, grid_full,
                                                  (sh.m_v / sh.ps) > 1 ? 0.3 : 0.6);
    const int64_t ct = ceil_div(n_tiles, p.chunks);
    p.chunk_items = ct;                                // tiles per chunk
    p.chunks = (int)ceil_div(n_tiles, ct);
    const int64_t units = (int64_t)p.n_groups * p.chunks;
    if (units >= ((int64_t)1 << 31)) fail(PQ_ERR_UNSUPPORTED, "tiled scoring kernel: too many work units");
    p.grid = (int)std::min<int64_t>(units, t.ctas > 0 ? t.ctas : grid_full);
    p.n_cut = 0;
    {
        // balanced partition (single-phase tables, no forced chunk count): taken when its
        // modelled makespan beats the legacy units' (A/B: PQTOPK_K2_BAL=0 turns it off;
        // PQTOPK_K2_UNIT_OVH = a unit's fixed cost in quarter-tiles)
        static const char* be = getenv("PQTOPK_K2_BAL");
        static const char* oe = getenv("PQTOPK_K2_UNIT_OVH");
        const int P = t.ctas > 0 ? t.ctas : grid_full;
        const int64_t ovh4 = oe ? std::max(0, atoi(oe)) : 8 + K / 12;
        // Only for short jobs (< 128 tiles per CTA), where one more tile on the longest CTA
        // and the units' fixed costs are several percent (C2: 18 -> 17 tiles, K2 208.5 ->
        // 199.4 us).  Long jobs keep the chunk-major legacy order, in which the CTAs of all
        // groups stream the same chunk of the codes together (one DRAM read, L2 hits for the
        // rest) and late units start from thresholds proved by earlier ones: measured on the
        // same box, C3 2.607 -> 2.608 ms and C5 316.2 -> 328.1 ms with this partition.
        const bool short_job = (int64_t)p.n_groups * n_tiles < 128 * (int64_t)P || (be && *be == '2');
        if ((sh.m_v / sh.ps) == 1 && t.chunks <= 0 && !(be && *be == '0') && P <= K2_MAX_CUT && short_job &&
            (int64_t)p.n_groups * n_tiles < ((int64_t)1 << 31) && (int64_t)p.n_groups * n_tiles >= 2 * (int64_t)P) {
            std::vector<int64_t> cut;
            const int64_t m4 = balanced_cuts(n_tiles, p.n_groups, P, ovh4, cut);
            const int64_t legacy4 = ceil_div(units, (int64_t)p.grid) * (4 * ct + ovh4);
            if (m4 > 0 && m4 < legacy4) {
                p.n_cut = (int)cut.size() - 1;
                for (int i = 0; i <= p.n_cut; ++i) p.cut[i] = (int32_t)cut[i];
                int cmax = 1;                          // lists per user = CTAs touching its group
                for (int g = 0, lo = 0; g < p.n_groups; ++g) {
                    while (lo + 1 < p.n_cut && cut[lo + 1] <= (int64_t)g * n_tiles) ++lo;
                    int hi = lo;
                    while (hi + 1 < p.n_cut && cut[hi + 1] < (int64_t)(g + 1) * n_tiles) ++hi;
                    cmax = std::max(cmax, hi - lo + 1);
                }
                p.chunks = cmax;
                p.grid = p.n_cut;
            }
        }
    }
    p.lanebuf_bytes = (size_t)p.grid * R * p.cap * 8;
    p.cand_bytes = (size_t)B * p.chunks * K * 8;
    p.mscr_bytes = 0;
    // union floors (K2_NQ levels per finished unit) for large K on single-phase tables:
    // each unit otherwise admits ~K items per user (C5: K = 1000, 37 chunks; K2 DRAM
    // bytes 8.2 -> 4.3 GB, time -0.5%).  Not for K = 100 (C3: the unit-end level
    // selections cost 1.4% and save 10% of a small traffic)
    static const char* qe = getenv("PQTOPK_K2_UNION");   // A/B: 0 = off
    p.qk = (sh.m_v / sh.ps) == 1 && K >= 256 && p.chunks >= 3 && p.chunks <= 64 && p.n_cut == 0 &&
           !(qe && *qe == '0');
    if (p.qk) ensure_max_smem(reinterpret_cast<const void*>(tiled_fn_shape(sh, p.W, true)), (int)p.smem);
    if (p.n_cut > 0) ensure_max_smem(reinterpret_cast<const void*>(tiled_fn_shape(sh, p.W, false, true)), (int)p.smem);
    p.st_bytes = align_up(st_table_bytes(sh, p.n_groups), 256) + (size_t)p.n_groups * R * 8 +
                 (size_t)qk_words(p) * 8 + (size_t)p.n_groups * R * p.chunks * 4;
}

// St workspace: [tables][gtau: n_groups R u64][qk: n_groups R chunks K2_NQ u64 when p.qk][lcnt: n_groups R chunks i32]
static unsigned long long* gtau_of(const pq_index_s* idx, const K2Plan& p, const float* St) {
    return reinterpret_cast<unsigned long long*>(const_cast<char*>(reinterpret_cast<const char*>(St)) +
                                                 align_up(st_table_bytes(k2_tiled_shape(idx->m, idx->b), p.n_groups), 256));
}
static unsigned long long* qk_of(const pq_index_s* idx, const K2Plan& p, const float* St) {
    return p.qk ? gtau_of(idx, p, St) + (int64_t)p.n_groups * p.G : nullptr;
}
const int32_t* k2_tiled_list_counts(const pq_index_s* idx, const K2Plan& p, const float* St) {
    return reinterpret_cast<const int32_t*>(gtau_of(idx, p, St) + (int64_t)p.n_groups * p.G + qk_words(p));
}

void launch_k2_tiled_prep(const pq_index_s* idx, const K2Plan& p, const float* S, int B, float* St,
                          cudaStream_t st) {
    const TiledShape sh = k2_tiled_shape(idx->m, idx->b);
    const int64_t total = (int64_t)(st_table_bytes(sh, p.n_groups) / 4);
    if (total >= ((int64_t)1 << 32)) fail(PQ_ERR_UNSUPPORTED, "tiled tables exceed 2^32 entries (batch too large)");
    const int threads = 256;
    const int blocks = (int)std::min<int64_t>(ceil_div(total, threads), (int64_t)idx->num_sms * 16);
    unsigned long long* gtau = gtau_of(idx, p, St);
    // zeroed per call: thresholds, union floors and -- balanced partition: a group may be
    // touched by fewer CTAs than `chunks` -- the list counts
    const int64_t nz = (int64_t)p.n_groups * p.G + qk_words(p) +
                       (p.n_cut > 0 ? ceil_div((int64_t)p.n_groups * p.G * p.chunks, (int64_t)2) : 0);
    if (sh.pair) launch_pdl(k2_tile_S_pair, dim3(blocks), dim3(threads), 0, st, S, B, idx->m, p.G, p.n_groups, St, gtau, nz);
    else launch_pdl(k2_tile_S, dim3(blocks), dim3(threads), 0, st, S, (const uint8_t*)idx->d_cmap3, B, idx->m, idx->b, p.G,
                    p.n_groups, St, gtau, nz);
    count_launch();
    check_launch("k2_tile_S");
}

void launch_k2_tiled(const pq_index_s* idx, const K2Plan& p, int B, int K,
                     uint64_t* lanebuf, uint64_t* mscr, const float* St, uint64_t* cand, cudaStream_t st) {
    (void)mscr;
    K2TArgs a{};
    a.codes = idx->d_codes3;
    a.codes_bytes = idx->v3_code_bytes;
    a.perm = idx->d_perm3;
    a.St = St;
    a.n_tiles = idx->v3_tiles;
    a.B = B; a.K = K;
    a.id_base = (uint32_t)idx->id_base;
    a.n_groups = p.n_groups; a.chunks = p.chunks; a.chunk_tiles = p.chunk_items;
    a.ubuf = lanebuf; a.cap = p.cap; a.cand = cand;
    {
        const int TR = k2_tiled_rows_per_tile(p.G);
        const int wmax = p.cap - (2 * k2_slack() + 1) * TR - 32;
        const int tw = idx->tuning.shrink_watermark;
        a.wm = tw > 0 ? std::min(std::max(tw, K + 1), wmax) : wmax;
    }
    a.n_cut = p.n_cut;
    for (int i = 0; i <= p.n_cut; ++i) a.cut[i] = p.cut[i];
    a.gtau = gtau_of(idx, p, St);
    a.qk = qk_of(idx, p, St);
    a.lcnt = const_cast<int32_t*>(k2_tiled_list_counts(idx, p, St));
    const char* dbe = getenv("PQTOPK_K2_DEBUG");
    if (dbe && *dbe) {
        PQ_CUDA(cudaMalloc(&a.dbg, 64 * 4));
        PQ_CUDA(cudaMemsetAsync(a.dbg, 0, 64 * 4, st));
    }
    const char* tf = getenv("PQTOPK_K2_TRACE");
    const char* tsd = getenv("PQTOPK_K2_TRACE_STRIDE");
    a.trace_stride = tsd ? std::max(1, atoi(tsd)) : 1;
    const char* tfr = getenv("PQTOPK_K2_TRACE_FROM");
    a.trace_from = tfr ? std::max(0, atoi(tfr)) : 0;
    const size_t tn = (size_t)p.W * TRACE_PH * 3 + TRACE_PH + 3 * TRACE_CTAS;
    if (tf && *tf) {
        if (!kTrace) fprintf(stderr, "PQTOPK_K2_TRACE: rebuild with PQTOPK_NVCC_EXTRA=-DK2_TRACE to record traces\n");
        PQ_CUDA(cudaMalloc(&a.trace, tn * 8));
        PQ_CUDA(cudaMemsetAsync(a.trace, 0, tn * 8, st));
    }
    K2TFn fn = tiled_fn_shape(k2_tiled_shape(idx->m, idx->b), p.W, p.qk != 0, p.n_cut > 0);
    launch_pdl(fn, dim3(p.grid), dim3(p.W * 32), p.smem, st, a);   // after k2_tile_S (PDL)
    count_launch();
    check_launch("k2_tiled");
    if (a.dbg) {
        int h[64];
        PQ_CUDA(cudaMemcpyAsync(h, a.dbg, sizeof h, cudaMemcpyDeviceToHost, st));
        PQ_CUDA(cudaStreamSynchronize(st));
        cudaFree(a.dbg);
        unsigned long long ins = 0, eot = 0, shr = 0, waits = 0, life = 0;
        memcpy(&ins, h + 16, 8);
        memcpy(&eot, h + 20, 8);
        memcpy(&shr, h + 22, 8);
        memcpy(&waits, h + 24, 8);
        memcpy(&life, h + 26, 8);
        fprintf(stderr, "k2_tiled debug: warp-cycles end-of-tile %.4f of warp lifetime (shrink part %.4f), "
                "tile-end waits %llu\n", (double)eot / (double)(life ? life : 1), (double)shr / (double)(life ? life : 1),
                waits);
        fprintf(stderr, "k2_tiled debug: stuck=%d cta=%d warp=%d tseq=%d arrivals=%d unit=%d t=%d ntl=%d sflag=%d,%d "
                "inserts=%llu (%.1f per user) shrinks=%d units=%lld\n",
                h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8], h[9], ins, (double)ins / B, h[18],
                (long long)p.n_groups * p.chunks);
        unsigned long long ins0 = 0;
        memcpy(&ins0, h + 28, 8);
        fprintf(stderr, "k2_tiled debug: first-tile inserts %llu (%.1f per user per unit); CTA 0 unit 0 cycles: start %d "
                "seed %d..%d tile0 scored %d tile0 done %d last tile %d merged %d\n", ins0,
                (double)ins0 / ((double)p.n_groups * p.G * p.chunks), h[32], h[33], h[34], h[35], h[36], h[37], h[38]);
    }
    if (a.trace) {                       // diagnostics only: dump CTA 0's phase timeline
        std::vector<long long> h(tn);
        PQ_CUDA(cudaMemcpyAsync(h.data(), a.trace, tn * 8, cudaMemcpyDeviceToHost, st));
        PQ_CUDA(cudaStreamSynchronize(st));
        cudaFree(a.trace);
        if (FILE* f = fopen(tf, "wb")) {
            const int hdr[2] = {p.W, TRACE_PH};
            fwrite(hdr, sizeof hdr, 1, f);
            fwrite(h.data(), 8, tn, f);
            fclose(f);
        }
    }
}

}  // namespace pq
