// K7 — the whole hot path of one small batch (B <= 4: the paper's serving case,
// one user per query; mRT below ~1e6 items) in ONE launch, for
// catalogues whose per-CTA share of the code matrix fits in shared memory
// (m = 8: up to ~1.8M items on 148 SMs; C1, C2a).  Latency-first design:
//
//   (0) each CTA issues ONE bulk TMA copy of its whole item chunk's code rows
//       (no ring, no refills) before anything else, so the HBM stream of the
//       codes overlaps the sub-id score phase;
//   (1) S (Eq. 4): the grid splits the B*m*b entries evenly, four
//       threads per entry, one fp64 fma chain each over t = j (mod 4), combined
//       as (c0 + c1) + (c2 + c3) and rounded to fp32 once — K1's order (R5b),
//       so S is bit-identical to pq_subscores.  Each entry is published as ONE
//       64-bit word (1 << 32 | fp32 bits): the word is its own ready flag, so a
//       reader polls exactly the entries it needs and no grid barrier, fence or
//       counter round trip sits between the producer and the consumers
//       (cooperative launch: every CTA is resident);
//   (2) each CTA polls its user's E = m*b words and writes G copies of the
//       table into shared memory (lane l reads copy l mod G);
//   (3) r_ui (Eq. 5, Alg. 1): thread t scores items t + 512 j of the
//       resident chunk, split-major over its J items (J independent fp32 add
//       chains in the sequential order j = 0..m-1, R1), scores kept in
//       registers;
//   (4) the chunk's exact top-K (R3 key: score desc, id asc): a proved floor
//       (the K-th largest of the per-warp top-min(K,32) thread maxima — K
//       distinct items reach it), keys only for the items that reach it,
//       ranked all-pairs (or radix-selected when many);
//   (5) each chunk writes its sorted list and K-th key to fixed slots; the last
//       CTA of the user (one ticket atomic) takes floor = max chunk K-th key
//       (that chunk alone holds K keys >= it), keeps the keys >= floor, ranks
//       them and writes ids / scores.
//
// The tagged S words and the tickets live in the call's workspace and are
// zeroed by the one-CTA k7_reset kernel launched before K7 as its programmatic
// dependent (griddepcontrol.wait precedes the first access to them).
#include "k2_common.cuh"
#include "ptx_dev.cuh"
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace pq {

struct K7Args {
    const uint8_t* codes;          // [N][mp] item-order rows (K0 layout, >= 16 bytes of tail pad)
    const float* phi;              // [B][d]
    const float* psi;              // [m][b][L], L = d / m
    float* S_out;                  // optional [B][m][b] copy of the sub-id scores
    unsigned long long* Sx;        // [B][E] tagged sub-id scores (zeroed by k7_reset)
    unsigned int* done;            // [B] finished-chunk tickets (zeroed by k7_reset)
    uint64_t* cand;                // [B][chunks][K] per-chunk sorted lists
    int32_t* ids;                  // [B][K]
    float* scores;                 // [B][K]
    long long* trace;              // diagnostics (-DK6_TRACE + PQTOPK_K6_TRACE): [grid][32] stamps
    int64_t N;
    int mp, b, B, K, d, L;
    uint32_t id_base;
    int chunks;                    // per user
    int chunk_items;               // multiple of 16, <= K7_THREADS * K7_JMAX
    int cl;                        // > 0: CLUSTER mode -- one thread-block cluster of cl CTAs per user
                                   // (chunks == cl, d/m = 4 or 8): the CTAs split the user's S, exchange
                                   // it through distributed shared memory, score their chunks and merge
                                   // in rank 0 -- no global exchange, reset kernel or ticket; 0 = grid mode
};

constexpr int K7_THREADS = 512;
constexpr int K7_NWARP = K7_THREADS / 32;
constexpr int K7_JMAX = 24;        // items per thread
constexpr int K7_MAXK = 512;

// (Warp-collective helpers stay inline: out of line, every shuffle becomes a
// divergence-safe WARPSYNC.COLLECTIVE sequence.)

// one key per lane, bitonic across the warp, descending (lane 0 = largest)
__device__ __forceinline__ uint64_t k7_warp_sort_desc(uint64_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const uint64_t o = __shfl_xor_sync(FULL, v, j);
            const bool desc = (lane & k) == 0, lower = (lane & j) == 0;
            v = (lower == desc) ? (o > v ? o : v) : (o < v ? o : v);
        }
    return v;
}

__device__ __noinline__ uint64_t k7_block_kth(const uint64_t* buf, int n, uint32_t K, uint32_t* hist,
                                              unsigned long long* sc) {
    return block_kth(buf, n, K, hist, sc);
}

// Rank of `mine` among buf[0..n) (keys unique; 0 = empty never outranks):
// the number of keys above it.  Eight independent 128-bit broadcast loads in
// flight (the loop is load-latency bound otherwise).  buf 16-byte aligned.
__device__ __forceinline__ int k7_rank(const uint64_t* buf, int n, uint64_t mine) {
    int r0 = 0, r1 = 0;
    int j = 0;
    for (; j + 16 <= n; j += 16) {
        ulonglong2 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = *reinterpret_cast<const ulonglong2*>(buf + j + 2 * q);
#pragma unroll
        for (int q = 0; q < 8; ++q) { r0 += v[q].x > mine ? 1 : 0; r1 += v[q].y > mine ? 1 : 0; }
    }
    for (; j < n; ++j) r0 += buf[j] > mine ? 1 : 0;
    return r0 + r1;
}

__device__ __forceinline__ uint64_t k7_warp_max(uint64_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const uint64_t t = __shfl_xor_sync(FULL, v, o);
        v = t > v ? t : v;
    }
    return v;
}

// Warp-aggregated append of `key` (if keep) to buf at the shared counter.
__device__ __forceinline__ void k7_append(bool keep, uint64_t key, uint64_t* buf, int* count) {
    const unsigned bm = __ballot_sync(FULL, keep);
    if (bm) {
        const int lane = threadIdx.x & 31;
        int base = 0;
        if (lane == 0) base = atomicAdd(count, __popc(bm));
        base = __shfl_sync(FULL, base, 0);
        if (keep) buf[base + __popc(bm & lanemask_lt())] = key;
    }
}

// The exact top-K (sorted) of n unique nonzero keys in smem buf -> out[rank]
// (global memory) for rank < min(K, n).  n <= 32: warp 0 sorts them; n <= 256:
// ranked all-pairs; larger: radix-select the K-th key, keep the K keys >= it
// (into tmp, >= K slots) and rank those.  All threads call it.
__device__ __forceinline__ void k7_topk(const uint64_t* buf, int n, int K, uint64_t* tmp, int* count,
                                     uint32_t* hist, unsigned long long* sc, uint64_t* out) {
    const int tid = threadIdx.x;
    if (n <= 32) {
        if (tid < 32) {
            const uint64_t srt = k7_warp_sort_desc(tid < n ? buf[tid] : 0ull);
            if (tid < n && tid < K) out[tid] = srt;
        }
        return;
    }
    if (n > 256) {
        const uint64_t kk = k7_block_kth(buf, n, (uint32_t)K, hist, sc);
        if (tid == 0) *count = 0;
        __syncthreads();
        for (int c0 = 0; c0 < n; c0 += K7_THREADS) {
            const int i = c0 + tid;
            const uint64_t v = i < n ? buf[i] : 0ull;
            k7_append(i < n && v >= kk, v, tmp, count);
        }
        __syncthreads();
        n = *count;                                    // == K (keys are unique)
        buf = tmp;
    }
    for (int i = tid; i < n; i += K7_THREADS) {
        const uint64_t mine = buf[i];
        const int rk = k7_rank(buf, n, mine);
        if (rk < K) out[rk] = mine;
    }
}

__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
// this CTA's shared address `local` in cluster CTA `rank`
__device__ __forceinline__ uint32_t dsmem_addr(uint32_t local, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}

// Shared memory: [T: M*b*G fp32 | R: codes of the chunk (each row's first 4
// bytes then hold the item's score), then candidate keys] (dynamic) + fk[1024]
// keys, hist[256], small scalars (static).  The last CTA of a user reuses T + R
// as merge scratch (chunks * K keys, checked by the plan).
template <int M, int G>
__global__ void __launch_bounds__(K7_THREADS, 1) k7_resident(const K7Args a) {
    constexpr int MP = (M + 3) / 4 * 4;
    constexpr int NW = MP / 4;
    constexpr int JB = 8;                              // items per thread in flight while scoring
    extern __shared__ __align__(128) unsigned char sm_raw[];
    __shared__ __align__(16) uint64_t fk[2 * K7_THREADS];
    __shared__ uint32_t hist[256];
    __shared__ unsigned long long sc[4];
    __shared__ unsigned long long floor_key;
    __shared__ int count;
    __shared__ int is_last;
    __shared__ __align__(8) unsigned long long mbar[K7_JMAX / 8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int bq = a.b;
    const int E = M * bq;
    const int K = a.K;
    const size_t tb0 = align_up((size_t)E * G * 4, 128), tb1 = (size_t)a.chunk_items * 8;
    const size_t tbytes = tb0 > tb1 ? tb0 : tb1;
    float* T = reinterpret_cast<float*>(sm_raw);
    unsigned char* Rg = sm_raw + tbytes;
    uint64_t* cbuf = reinterpret_cast<uint64_t*>(sm_raw);   // candidates: over T once scored
    const int u = blockIdx.x / a.chunks;
    const int chunk = blockIdx.x - u * a.chunks;
    const int64_t i0 = (int64_t)chunk * a.chunk_items;
    const int nit = (int)max((int64_t)0, min((int64_t)a.chunk_items, a.N - i0));
    const uint32_t cbytes = (uint32_t)align_up((size_t)nit * MP, 16);
    const uint32_t bar0 = smem_u32(mbar);
    constexpr uint32_t PIECE = 8u * K7_THREADS * MP;   // code bytes of one scoring batch (JB items per thread)
    auto stamp = [&](int i) {                          // diagnostics builds only (-DK6_TRACE)
#ifdef K6_TRACE
        if (a.trace && tid == 0) {
            long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            a.trace[(int64_t)blockIdx.x * 32 + i] = t;
        }
#else
        (void)i;
#endif
    };
    stamp(0);
    // the chunk's code rows -> R in bulk TMA copies (no ring: the whole chunk is
    // resident), one mbarrier per scoring batch so scoring starts on the first
    // piece.  Issued by thread 0 right after its own sub-id score loads, so the
    // sub-id score requests are not queued behind the codes.
    auto issue_codes = [&]() {
        for (uint32_t o = 0, p = 0; o < cbytes; o += PIECE, ++p) {
            const uint32_t nb = min(PIECE, cbytes - o);
            mbar_expect_tx(bar0 + 8u * p, nb);
            bulk_g2s(smem_u32(Rg) + o, a.codes + i0 * MP + o, nb, bar0 + 8u * p);
        }
    };
    if (tid == 0) {
        for (int p = 0; p < K7_JMAX / 8; ++p) mbar_init(bar0 + 8u * p, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        count = 0;
        floor_key = 0ull;
    }
    bool issued = false;

    // cluster mode: the staging of the user's E sub-id scores (then rank 0's merge area)
    float* Sst = reinterpret_cast<float*>(Rg + align_up((size_t)a.chunk_items * MP, 128));
    if (a.cl) {
        // ---- cluster mode: rank r computes entries [r E / cl, (r + 1) E / cl) of its user,
        // four per thread with all their Psi / phi loads in flight (one thread per
        // entry, K1's four fp64 chains, R5b), and stores each into the staging of
        // every CTA of the cluster (distributed shared memory)
        pdl_wait();                                    // phi may come from the stream predecessor
        const int q4 = a.L / 4;                        // <= 2
        const float* phu = a.phi + (int64_t)u * a.d;
        const int per = E / a.cl, e_lo = chunk * per, e_hi = e_lo + per;
        const uint32_t sst = smem_u32(Sst);
        for (int eb = e_lo; eb < e_hi; eb += 4 * K7_THREADS) {
            float4 pv[4][2], fv[4][2];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int e = eb + r * K7_THREADS + tid;
                const bool ok = e < e_hi;
                const float4* pr = reinterpret_cast<const float4*>(a.psi + (int64_t)(ok ? e : e_lo) * a.L);
                const float4* fr = reinterpret_cast<const float4*>(phu + (int64_t)((ok ? e : e_lo) / bq) * a.L);
#pragma unroll
                for (int i = 0; i < 2; ++i)
                    if (i < q4) { pv[r][i] = __ldg(pr + i); fv[r][i] = __ldg(fr + i); }
            }
            if (tid == 0 && !issued) { issue_codes(); issued = true; }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int e = eb + r * K7_THREADS + tid;
                double x0 = 0.0, x1 = 0.0, x2 = 0.0, x3 = 0.0;
#pragma unroll
                for (int i = 0; i < 2; ++i)
                    if (i < q4) {
                        x0 = fma((double)pv[r][i].x, (double)fv[r][i].x, x0);
                        x1 = fma((double)pv[r][i].y, (double)fv[r][i].y, x1);
                        x2 = fma((double)pv[r][i].z, (double)fv[r][i].z, x2);
                        x3 = fma((double)pv[r][i].w, (double)fv[r][i].w, x3);
                    }
                if (e < e_hi) {
                    const float v = (float)((x0 + x1) + (x2 + x3));
                    if (a.S_out) a.S_out[(int64_t)u * E + e] = v;
                    for (int q = 0; q < a.cl; ++q)
                        asm volatile("st.shared::cluster.f32 [%0], %1;" :: "r"(dsmem_addr(sst + 4u * (uint32_t)e, q)),
                                     "f"(v) : "memory");
                }
            }
        }
        if (tid == 0 && !issued) issue_codes();
        cluster_arrive();                              // this CTA's share is in every staging
        cluster_wait();                                // ... and every share is in this CTA's
        // G copies of each entry into the local table (bank-rotated stores)
        const int rot = lane * G / 32;
        for (int e = tid; e < E; e += K7_THREADS) {
            const float v = Sst[e];
            if constexpr (G >= 4) {
                constexpr int NQ = G / 4;
                const float4 v4 = make_float4(v, v, v, v);
                float4* dst = reinterpret_cast<float4*>(T + (size_t)e * G);
#pragma unroll
                for (int c = 0; c < NQ; ++c) dst[(c + rot) % NQ] = v4;
            } else {
#pragma unroll
                for (int c = 0; c < G; ++c) T[(size_t)e * G + c] = v;
            }
        }
        cluster_arrive();                              // staging read: rank 0 may reuse its own (merge)
    } else
    // ---- (1) this CTA's share of the B*E sub-id scores, K1's fp64 order (R5b)
    {
        const int EB = a.B * E;
        const int per = (EB + (int)gridDim.x - 1) / (int)gridDim.x;
        const int e0 = (int)blockIdx.x * per, e1 = min(EB, e0 + per);
        const int j = tid & 3;
        for (int base = e0; base < e1; base += K7_THREADS / 4) {
            const int ent = base + (tid >> 2);
            const bool ok = ent < e1;
            const int uu = ok ? ent / E : 0, ee = ok ? ent - uu * E : 0;
            const float* pr = a.psi + (int64_t)ee * a.L;
            const float* fr = a.phi + (int64_t)uu * a.d + (int64_t)(ee / bq) * a.L;
            double x = 0.0;
            for (int t0 = j; t0 < a.L; t0 += 64) {     // 16 terms of the chain per pass
                float pv[16], fv[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const int t = t0 + 4 * q;
                    const bool in = ok && t < a.L;
                    pv[q] = in ? __ldg(pr + t) : 0.0f;
                    fv[q] = in ? __ldg(fr + t) : 0.0f;
                }
                if (tid == 0 && !issued) { issue_codes(); issued = true; }
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    if (t0 + 4 * q < a.L) x = fma((double)pv[q], (double)fv[q], x);
            }
            // (c0 + c1) + (c2 + c3): lanes 4e .. 4e + 3 hold c0 .. c3
            const double x1 = __shfl_down_sync(FULL, x, 1);
            const double s01 = x + x1;                 // valid in lanes j = 0, 2
            const double s23 = __shfl_down_sync(FULL, s01, 2);
            if (base == e0) stamp(1);
            // the tagged words are zeroed by k7_reset: no access before it completed
            asm volatile("griddepcontrol.wait;" ::: "memory");
            if (j == 0 && ok) {
                const float v = (float)(s01 + s23);
                st_relaxed_u64(a.Sx + ent, (1ull << 32) | (unsigned long long)__float_as_uint(v));
                if (a.S_out) a.S_out[ent] = v;
            }
        }
    }
    if (!a.cl) {
    if (tid == 0 && !issued) issue_codes();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    stamp(2);

    // ---- (2) poll this user's E words, replicate G times (bank-rotated stores)
    {
        const unsigned long long* Su = a.Sx + (int64_t)u * E;
        const int rot = lane * G / 32;
#pragma unroll 1
        for (int e0 = 0; e0 < E; e0 += 4 * K7_THREADS) {
            unsigned long long w[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int e = e0 + q * K7_THREADS + tid;
                w[q] = e < E ? ld_relaxed_u64(Su + e) : (1ull << 32);
            }
#pragma unroll 1
            for (int q = 0; q < 4; ++q) {
                const int e = e0 + q * K7_THREADS + tid;
                unsigned long long wq = w[0];
                if (q == 1) wq = w[1];
                if (q == 2) wq = w[2];
                if (q == 3) wq = w[3];
                long long spins = 0;
                (void)spins;
                while ((wq >> 32) == 0ull) {
                    __nanosleep(32);
                    wq = ld_relaxed_u64(Su + e);
                    PQ_SPIN_CHECK(spins);
                }
                if (e < E) {
                    const float v = __uint_as_float((uint32_t)wq);
                    if constexpr (G >= 4) {
                        constexpr int NQ = G / 4;
                        const float4 v4 = make_float4(v, v, v, v);
                        float4* dst = reinterpret_cast<float4*>(T + (size_t)e * G);
#pragma unroll
                        for (int c = 0; c < NQ; ++c) dst[(c + rot) % NQ] = v4;
                    } else {
#pragma unroll
                        for (int c = 0; c < G; ++c) T[(size_t)e * G + c] = v;
                    }
                }
            }
        }
    }
    }
    stamp(3);
    __syncthreads();                                   // table ready
    stamp(4);

    // ---- (3) gather-sum: thread t scores items t + 512 j, JB at a time, split-major;
    // each item's fp32 score replaces the first 4 code bytes of its row.  (Colour-
    // paired rows, K6's layout for long streams, were slower here: each CTA's best
    // key and every candidate then need a row -> id load from cold HBM.)
    const uint32_t gid0 = a.id_base + (uint32_t)i0;
    auto gid = [&](int li) { return gid0 + (uint32_t)li; };
    const int lrow = tid;
    uint64_t km = 0ull;                                // this thread's best key (0: no items)
    {
        const char* Tb = reinterpret_cast<const char*>(T + lane % G);
        auto look = [&](int k, uint32_t w, int s) {
            const uint32_t g = __byte_perm(w, 0u, 0x4440u | (uint32_t)s);
            return *reinterpret_cast<const float*>(Tb + (size_t)k * bq * G * 4 + (size_t)g * (G * 4));
        };
        int jbst = -1;
        float best = 0.0f;
#pragma unroll 1
        for (int jb = 0; jb * K7_THREADS < nit; jb += JB) {
            mbar_wait(bar0 + 8u * (uint32_t)(jb / JB), 0);   // this batch's code rows resident
            uint32_t cw[JB][NW];
#pragma unroll
            for (int q = 0; q < JB; ++q) {
                const int li = (jb + q) * K7_THREADS + lrow;
                const unsigned char* row = Rg + (size_t)(li < nit ? li : 0) * MP;
                if constexpr (NW == 1) {
                    cw[q][0] = *reinterpret_cast<const uint32_t*>(row);
                } else if constexpr (NW == 2) {
                    const uint2 t = *reinterpret_cast<const uint2*>(row);
                    cw[q][0] = t.x; cw[q][1] = t.y;
                } else {
                    const uint4 t = *reinterpret_cast<const uint4*>(row);
                    cw[q][0] = t.x; cw[q][1] = t.y; cw[q][2] = t.z; cw[q][3] = t.w;
                }
            }
            // two items per packed fp32x2 add (FADD2, RN: the same IEEE adds as scalar FADDs)
            float2 acc2[JB / 2];
#pragma unroll
            for (int q = 0; q < JB / 2; ++q)
                acc2[q] = make_float2(look(0, cw[2 * q][0], 0), look(0, cw[2 * q + 1][0], 0));
#pragma unroll
            for (int k = 1; k < M; ++k)
#pragma unroll
                for (int q = 0; q < JB / 2; ++q)
                    acc2[q] = __fadd2_rn(acc2[q], make_float2(look(k, cw[2 * q][k >> 2], k & 3),
                                                              look(k, cw[2 * q + 1][k >> 2], k & 3)));
            float acc[JB];
#pragma unroll
            for (int q = 0; q < JB / 2; ++q) { acc[2 * q] = acc2[q].x; acc[2 * q + 1] = acc2[q].y; }
#pragma unroll
            for (int q = 0; q < JB; ++q) {
                const int li = (jb + q) * K7_THREADS + lrow;
                if (li < nit) {
                    const float sc0 = acc[q] + 0.0f;   // R1-R3: +0 canonical
                    *reinterpret_cast<float*>(Rg + (size_t)li * MP) = sc0;
                    if (jbst < 0 || sc0 > best) { jbst = li; best = sc0; }   // first max = smallest id
                }
            }
        }
        if (jbst >= 0) km = make_key(best, gid(jbst));
    }

    // ---- (4) proved floor, candidates, the chunk's sorted top K
    uint64_t fl;
    if (K <= K7_NWARP) {
        // floor = the K-th largest warp maximum (K distinct items reach it); every
        // warp sorts the NWARP maxima itself -- one barrier
        const uint64_t wm = k7_warp_max(km);
        if (lane == 0) fk[warp] = wm;
        __syncthreads();                               // also: every warp is done with the codes
        stamp(5);
        const uint64_t srt = k7_warp_sort_desc(lane < K7_NWARP ? fk[lane] : 0ull);
        fl = __shfl_sync(FULL, srt, K - 1);
        stamp(12);
    } else {
        // K > NWARP: the K-th largest of the per-warp top-min(K, 32) thread maxima
        const int KW = K < 32 ? K : 32;
        const uint64_t srt = k7_warp_sort_desc(km);
        if (lane < KW) fk[warp * KW + lane] = srt;
        __syncthreads();
        stamp(5);
        fl = k7_block_kth(fk, K7_NWARP * KW, (uint32_t)K, hist, sc);   // >= K keys (K <= 512)
    }
    {
        // candidates = keys >= fl: count per thread (four loads in flight), one
        // atomic per warp, write
        const float fs = fl ? key_score(fl) : -INFINITY;
        auto cand = [&](int li, float s, uint64_t& key) {
            if (!(s >= fs)) return false;
            key = make_key(s, gid(li));
            return key >= fl;
        };
        auto score = [&](int li) { return *reinterpret_cast<const float*>(Rg + (size_t)li * MP); };
        int nc = 0;
        int li = tid;
#pragma unroll 1
        for (; li + 3 * K7_THREADS < nit; li += 4 * K7_THREADS) {
            float s4[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) s4[q] = score(li + q * K7_THREADS);
#pragma unroll
            for (int q = 0; q < 4; ++q) { uint64_t key; nc += cand(li + q * K7_THREADS, s4[q], key) ? 1 : 0; }
        }
#pragma unroll 1
        for (; li < nit; li += K7_THREADS) { uint64_t key; nc += cand(li, score(li), key) ? 1 : 0; }
        int incl = nc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += t;
        }
        const int tot = __shfl_sync(FULL, incl, 31);
        int base = 0;
        if (lane == 31 && tot) base = atomicAdd(&count, tot);
        base = __shfl_sync(FULL, base, 31) + incl - nc;
        if (nc) {
#pragma unroll 1
            for (int l2 = tid; l2 < nit; l2 += K7_THREADS) {
                uint64_t key;
                if (cand(l2, score(l2), key)) cbuf[base++] = key;
            }
        }
    }
    __syncthreads();
    stamp(6);
    if (a.cl) {
        // cluster mode: this chunk's sorted top K -> rank 0's merge area (its staging,
        // read by rank 0 only before the second cluster arrive); rank 0 merges the
        // cl * K keys (0 = empty ranks last) and writes the user's ids / scores
        const int n = count;
        uint64_t* res = fk + K7_THREADS;
        k7_topk(cbuf, n, K, fk, &count, hist, sc, res);
        __syncthreads();
        cluster_wait();                                // every CTA is past its staging reads
        uint64_t* mrg = reinterpret_cast<uint64_t*>(Sst);
        const uint32_t m0 = smem_u32(mrg);
        for (int j = tid; j < K; j += K7_THREADS) {
            const uint64_t key = j < n ? res[j] : 0ull;
            asm volatile("st.shared::cluster.u64 [%0], %1;" :: "r"(dsmem_addr(m0 + 8u * (uint32_t)(chunk * K + j), 0)),
                         "l"(key) : "memory");
        }
        cluster_arrive();
        cluster_wait();                                // rank 0's merge area complete
        if (chunk != 0) return;
        uint64_t* out = fk + K7_THREADS;
        for (int j = tid; j < K; j += K7_THREADS) out[j] = 0ull;   // slots past the real keys stay empty
        __syncthreads();
        k7_topk(mrg, a.cl * K, K, fk, &count, hist, sc, out);
        __syncthreads();
        for (int j = tid; j < K; j += K7_THREADS) {
            const uint64_t key = out[j];
            a.ids[(int64_t)u * K + j] = key ? key_id(key) : -1;
            a.scores[(int64_t)u * K + j] = key ? key_score(key) : -INFINITY;
        }
        return;
    }
    {
        const int n = count;
        uint64_t* out = a.cand + ((int64_t)u * a.chunks + chunk) * K;
        k7_topk(cbuf, n, K, fk, &count, hist, sc, out);
        for (int j = n + tid; j < K; j += K7_THREADS) out[j] = 0ull;   // pad: K-th key 0 = fewer than K
    }
    stamp(7);

    // ---- (5) ticket; the last CTA of the user merges.  Every thread's list
    // writes precede the barrier; thread 0's acq_rel ticket releases them at gpu
    // scope (and, in the last CTA, acquires the other CTAs' lists).
    __syncthreads();
    if (tid == 0) {
        unsigned int old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(a.done + u) : "memory");
        is_last = old == (unsigned)(a.chunks - 1);
    }
    __syncthreads();
    if (!is_last) return;
    stamp(8);
    // Every chunk list is sorted and 0-padded, so list c's first key is the
    // chunk maximum and its K-th key the chunk K-th (0: fewer than K).  The
    // user's top K are among the keys >= floor = max(largest chunk K-th key,
    // largest per-32-chunk K-th chunk maximum): either proves K keys >= floor.
    uint64_t* mk = reinterpret_cast<uint64_t*>(sm_raw);   // T + R: merge scratch
    uint64_t* mx = fk;                                    // chunk maxima [chunks] (<= 2 * threads)
    const int n2 = a.chunks * K;
    const uint64_t* cu = a.cand + (int64_t)u * n2;
    constexpr int PQ = 4;
    uint64_t v[PQ];
    if (tid == 0) { count = 0; floor_key = 0ull; }
#pragma unroll
    for (int q = 0; q < PQ; ++q) {
        const int i = q * K7_THREADS + tid;
        v[q] = i < n2 ? __ldcg(cu + i) : 0ull;
    }
    {
        uint64_t f = 0ull;
#pragma unroll 1
        for (int c = tid; c < a.chunks; c += K7_THREADS) {
            const int ik = c * K + K - 1;
            if (ik >= PQ * K7_THREADS) {                // else in registers (below)
                const uint64_t t = __ldcg(cu + ik);
                f = t > f ? t : f;
            }
            if (c * K >= PQ * K7_THREADS) mx[c] = __ldcg(cu + (int64_t)c * K);
        }
#pragma unroll
        for (int q = 0; q < PQ; ++q) {
            const int i = q * K7_THREADS + tid;
            if (i < n2) {
                const int r = i % K;
                if (r == K - 1) f = v[q] > f ? v[q] : f;
                if (r == 0) mx[i / K] = v[q];
            }
        }
        f = k7_warp_max(f);
        __syncthreads();                               // count / floor_key reset seen; mx complete
        stamp(13);
        if (lane == 0 && f) atomicMax(&floor_key, (unsigned long long)f);
        // a floor from the chunk maxima: each warp's K-th largest of its 32 chunk
        // maxima (K chunks hold a key >= it); the largest over the warps
        if (K <= 32) {
            for (int w0 = warp * 32; w0 < a.chunks; w0 += K7_THREADS) {
                const int c = w0 + lane;
                const uint64_t srt = k7_warp_sort_desc(c < a.chunks ? mx[c] : 0ull);
                const uint64_t kk = __shfl_sync(FULL, srt, K - 1);
                if (lane == 0 && kk) atomicMax(&floor_key, (unsigned long long)kk);
            }
        } else if (a.chunks >= K) {
            const uint64_t t = k7_block_kth(mx, a.chunks, (uint32_t)K, hist, sc);
            if (tid == 0 && t) atomicMax(&floor_key, (unsigned long long)t);
        }
        __syncthreads();
    }
    stamp(9);
    {
        const uint64_t fl2 = floor_key;
#pragma unroll
        for (int q = 0; q < PQ; ++q) k7_append(v[q] != 0ull && v[q] >= fl2, v[q], mk, &count);
#pragma unroll 1
        for (int i0m = PQ * K7_THREADS; i0m < n2; i0m += K7_THREADS) {
            const int i = i0m + tid;
            const uint64_t t = i < n2 ? __ldcg(cu + i) : 0ull;
            k7_append(t != 0ull && t >= fl2, t, mk, &count);
        }
    }
    __syncthreads();
    stamp(10);
    {
        // the sorted top K keys -> fk[K7_THREADS ..] (free now), then ids / scores
        const int n3 = count;
        uint64_t* res = fk + K7_THREADS;
        k7_topk(mk, n3, K, fk, &count, hist, sc, res);
        __syncthreads();
        for (int j = tid; j < K; j += K7_THREADS) {
            const uint64_t key = j < n3 ? res[j] : 0ull;
            a.ids[(int64_t)u * K + j] = key ? key_id(key) : -1;
            a.scores[(int64_t)u * K + j] = key ? key_score(key) : -INFINITY;
        }
    }
    stamp(11);
}


// Zeroes the call's tickets and tagged S words ([bytes] at p, 16-byte multiple);
// K7 is its programmatic dependent and starts at once.
__global__ void k7_reset(uint4* p, int n16) {
    asm volatile("griddepcontrol.launch_dependents;");
    for (int i = threadIdx.x; i < n16; i += blockDim.x) p[i] = make_uint4(0u, 0u, 0u, 0u);
}

// ---------------------------------------------------------------- host side
typedef void (*K7Fn)(const K7Args);

static K7Fn k7_fn(int m, int G) {
    switch (m) {
        case 4: return G == 16 ? k7_resident<4, 16> : nullptr;
        case 8: return G == 16 ? k7_resident<8, 16> : nullptr;
        case 16: return G == 16 ? k7_resident<16, 16> : (G == 8 ? k7_resident<16, 8> : nullptr);
        default: return nullptr;
    }
}
static int k7_mp(int m) { return (m + 3) / 4 * 4; }
static size_t k7_rbytes(int m, int64_t ci) { return align_up((size_t)ci * (size_t)k7_mp(m), 128); }
// the table region, also the candidate buffer once the chunk is scored (>= 1 key per item)
static size_t k7_tbytes(int m, int b, int G, int64_t ci) {
    return std::max(align_up((size_t)m * b * G * 4, 128), (size_t)ci * 8);
}
static size_t k7_static_bytes() { return 2 * K7_THREADS * 8 + 256 * 4 + 256; }

// Workspace: [done B u32 | pad to 256][Sx B*E u64][cand B*chunks*K u64]
static size_t k7_reset_bytes(int B, int E) { return 256 + align_up((size_t)B * E * 8, 256); }

bool k7_resident_plan(const pq_index_s* idx, int B, int d, int K, K6Plan& p) {
    const int m = idx->m, b = idx->b;
    const pq_tuning& t = idx->tuning;
    if (t.cluster > 0) return false;                   // cluster modes are K6's
    if (B < 1 || B > 4 || K < 1 || K > K7_MAXK || d % m) return false;
    if (m != 4 && m != 8 && m != 16) return false;
    int G = (size_t)m * b * 16 * 4 <= 128 * 1024 ? 16 : 8;
    if (t.users_per_row > 0) G = std::min(G, pow2_ceil(t.users_per_row));
    K7Fn fn = k7_fn(m, G);
    if (!fn) return false;
    const int64_t N = idx->N;
    const int cap = idx->num_sms / B;                  // one CTA per SM, one wave
    if (cap < 1) return false;
    int64_t ch = std::max<int64_t>(1, std::min<int64_t>(cap, ceil_div(N, 512)));   // >= 512 items per CTA
    const size_t budget = idx->smem_optin - k7_static_bytes();
    // cluster mode (one cluster of cl CTAs per user, no global exchange) when a user's
    // catalogue fits cl chunks: small catalogues (C1); cl = 8 unless the catalogue is tiny
    int cl = 0;
    {
        const int L = d / m;
        const int want = (int)std::min<int64_t>(8, std::max<int64_t>(1, N / 1024));
        for (int c = 8; c >= 1 && !cl; c >>= 1) {
            if (c > want || (m * b) % c || (int64_t)B * c > idx->num_sms || c * K > 256) continue;
            const int64_t cc = (int64_t)align_up((size_t)ceil_div(N, c), 16);
            const size_t sc1 = k7_tbytes(m, b, G, cc) + k7_rbytes(m, cc) + align_up((size_t)m * b * 4, 128);
            if (L % 4 == 0 && L <= 8 && cc <= (int64_t)K7_THREADS * K7_JMAX && sc1 <= budget) cl = c;
        }
        if (t.chunks > 0 || t.variant == 5) cl = 0;
    }
    if (cl) ch = cl;
    if (t.chunks > 0) ch = std::min<int64_t>(t.chunks, cap);
    int64_t ci = 0;
    size_t smem = 0;
    for (;; --ch) {                                    // fewer chunks while the merge scratch does not fit
        ci = (int64_t)align_up((size_t)ceil_div(N, ch), 16);
        const int64_t che = ceil_div(N, ci);
        const size_t tr = k7_tbytes(m, b, G, ci) + k7_rbytes(m, ci);
        smem = std::max(tr, align_up((size_t)che * K * 8, 128));   // T + R: merge scratch
        if (smem <= budget || ch == 1 || (size_t)che * K * 8 <= tr) break;
    }
    ch = ceil_div(N, ci);
    if (ci > (int64_t)K7_THREADS * K7_JMAX || smem > budget) return false;
    if (cl) {                                          // the staging / merge area after R
        smem = k7_tbytes(m, b, G, ci) + k7_rbytes(m, ci) + align_up((size_t)m * b * 4, 128);
        if (smem > budget || ceil_div(N, ci) > cl) return false;
        ch = cl;                                       // whole clusters (a trailing CTA may hold no items)
    }
    // auto: grid-mode catalogues too small for >= 2048 items per CTA go to K6
    if (t.variant != 7 && !cl && ci < 2048) return false;
    ensure_max_smem(reinterpret_cast<const void*>(fn), (int)smem);
    int per_sm = 0;
    PQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, K7_THREADS, smem));
    if (per_sm < 1 || (int64_t)per_sm * idx->num_sms < (int64_t)B * ch) return false;
    p = K6Plan{};
    p.resident = 1;
    p.cl = cl;
    p.G = G;
    p.gridsync = 1;
    p.chunks = (int)ch;
    p.chunk_items = ci;
    p.grid = B * (int)ch;
    p.smem = smem;
    p.cand_bytes = (size_t)B * ch * K * 8;
    return true;
}

size_t k7_resident_ws_bytes(const K6Plan& p, int B, int E) {
    return k7_reset_bytes(B, E) + align_up(p.cand_bytes, 256);
}

void launch_k7_resident(const pq_index_s* idx, const K6Plan& p, const float* phi, const float* psi, int B,
                        int d, int K, void* ws, float* S_out, int32_t* ids, float* scores, cudaStream_t st) {
    const int E = idx->m * idx->b;
    K7Args a{};
    a.codes = idx->d_codes;
    a.phi = phi; a.psi = psi; a.S_out = S_out;
    char* w = static_cast<char*>(ws);
    a.done = reinterpret_cast<unsigned int*>(w);
    a.Sx = reinterpret_cast<unsigned long long*>(w + 256);
    const size_t rb = k7_reset_bytes(B, E);
    a.cand = reinterpret_cast<uint64_t*>(w + rb);
    a.ids = ids; a.scores = scores;
    a.N = idx->N;
    a.mp = idx->lay.mp; a.b = idx->b; a.B = B; a.K = K; a.d = d; a.L = d / idx->m;
    a.id_base = (uint32_t)idx->id_base;
    a.chunks = p.chunks;
    a.chunk_items = (int)p.chunk_items;
    a.cl = p.cl;
    if (!p.cl) {
        k7_reset<<<1, 256, 0, st>>>(reinterpret_cast<uint4*>(w), (int)(rb / 16));
        count_launch();
        check_launch("k7_reset");
    }
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[2];
    cfg.gridDim = dim3((unsigned)p.grid);
    cfg.blockDim = dim3(K7_THREADS);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = st;
    // grid mode: CTAs that poll each other's sub-id scores must be co-resident (a
    // cooperative launch); cluster mode: a cluster of cl CTAs per user
    cudaLaunchAttribute at3[3];
    (void)at;
    int na = 0;
    if (!p.cl) {
        at3[na].id = cudaLaunchAttributeCooperative;
        at3[na].val.cooperative = 1;
        ++na;
    } else if (p.cl > 1) {
        at3[na].id = cudaLaunchAttributeClusterDimension;
        at3[na].val.clusterDim.x = (unsigned)p.cl;
        at3[na].val.clusterDim.y = 1;
        at3[na].val.clusterDim.z = 1;
        ++na;
    }
    at3[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // after k7_reset / the producer of phi
    at3[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
    cfg.attrs = at3;
    cfg.numAttrs = na;
    const char* tf = getenv("PQTOPK_K6_TRACE");
    if (tf && *tf) {
        PQ_CUDA(cudaMalloc(&a.trace, (size_t)p.grid * 32 * 8));
        PQ_CUDA(cudaMemsetAsync(a.trace, 0, (size_t)p.grid * 32 * 8, st));
    }
    PQ_CUDA(cudaLaunchKernelEx(&cfg, k7_fn(idx->m, p.G), a));
    count_launch();
    check_launch("k7_resident");
    if (a.trace) {                                     // diagnostics only: per-CTA phase stamps
        std::vector<long long> h((size_t)p.grid * 32);
        PQ_CUDA(cudaMemcpyAsync(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost, st));
        PQ_CUDA(cudaStreamSynchronize(st));
        cudaFree(a.trace);
        if (FILE* f = fopen(tf, "wb")) {
            const int hdr[2] = {p.grid, 32};
            fwrite(hdr, sizeof hdr, 1, f);
            fwrite(h.data(), 8, h.size(), f);
            fclose(f);
        }
    }
}

}  // namespace pq
