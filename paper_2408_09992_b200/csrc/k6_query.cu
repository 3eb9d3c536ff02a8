// K6 — the whole hot path of one small batch (B <= 4, the paper's serving
// case: one user per query, mRT; elbow below 1e5 items) in ONE
// kernel launch ("fuse K1 into K2's prologue").
//
// One thread-block cluster of CL CTAs serves one user and CL consecutive item
// chunks; every CTA needs the user's whole table S_u (Eq. 4):
//   (1) S_u: CTA rank r of the cluster computes its 1/CL share of the m*b
//       entries, each one exactly as K1 does (four fp64 fma chains over
//       t = j (mod 4), combined as (c0 + c1) + (c2 + c3), rounded to fp32 once
//       — bit-identical to pq_subscores, R5/R5b), and stores it into
//       the S staging of EVERY CTA of the cluster (distributed shared memory),
//       so Psi is read once per cluster instead of once per CTA; after a
//       cluster barrier each CTA replicates the table G times locally;
//   (2) r_ui (Eq. 5, Alg. 1): lane = item over the chunk's code
//       rows, streamed by a TMA/mbarrier ring — the K2 v4 loop (k2_latency.cu);
//   (3) the chunk's exact top-K under the (score desc, id asc) key (R3);
//   (4) the last CTA of the user to finish (a device-scope counter, zeroed
//       by the caller before the launch) merges the chunks' lists (K3) and
//       writes ids / scores: no second launch.
// The code stream's TMA loads are issued before (1), so the HBM latency of the
// first rounds overlaps the sub-id score computation.
#include "k2_common.cuh"
#include "ptx_dev.cuh"
#include <cooperative_groups.h>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace cg = cooperative_groups;

namespace pq {

struct K6Args {
    const uint8_t* codes;      // [N][mp] item-order uint8 rows (K0 layout)
    const int32_t* perm;       // row -> local item id, or null (identity)
    const uint8_t* cmap;       // colour-paired rows (idx->d_codes_p): [m][b] stored sub-id -> sub-id, else null
    const float* phi;          // [B][d]
    const float* psi;          // [m][b][L], L = d / m
    float* S_out;              // optional [B][m][b] copy of the sub-id scores
    int64_t N;
    int mp, b, B, K, d, L;
    uint32_t id_base;
    int chunks;                // per user, a multiple of the cluster size
    int64_t chunk_items;       // multiple of 16
    uint64_t* cand;            // [B][chunks][K] per-chunk lists
    uint64_t* kth;             // [B][chunks] each list's K-th key (0: fewer than K keys)
    uint64_t* kmax;            // [B][chunks] each list's largest key (0: empty)
    unsigned int* done;        // [B] finished-chunk counters, then the grid barrier (zero at launch)
    float* Sg;                 // grid mode: [B][m][b] sub-id scores in global memory (S_out or workspace)
    int gridsync;              // 1: cooperative grid, S computed once per user and shared through L2
    int32_t* ids;              // [B][K]
    float* scores;             // [B][K]
    int nst;                   // code stages in flight
    long long* trace;          // diagnostics (PQTOPK_K6_TRACE): [grid][32] globaltimer stamps, or null
};

#ifndef K6_THREADS_N
#define K6_THREADS_N 256
#endif
constexpr int K6_THREADS = K6_THREADS_N;
// Round size: 24 KB of codes (3072 items at m = 8, 12 per thread) -- twice the
// independent add chains of the 16 KB rounds and a third fewer rounds: c7
// 2.38 -> 2.05 ms (32 KB rounds leave room for only two stages and measured
// 3.37 ms).  A multiple of 8 KB, so every m in {4, 8, 16} gets an even J.
#ifndef K6_STAGE_BYTES
#define K6_STAGE_BYTES 24576
#endif
#ifndef K6_CAP_SLACK
#define K6_CAP_SLACK 512                               // 0: candidate buffer of 2 rounds of items
#endif
constexpr int K6_STAGE = K6_STAGE_BYTES;               // code bytes per round (one TMA stage)
// candidate buffer: one round of items + room for the K kept ones (K <= 512)
__host__ __device__ constexpr int k6_cap(int ipr) { return K6_CAP_SLACK ? ipr + K6_CAP_SLACK : 2 * ipr; }

// Bitonic sort of one key per lane across a warp, descending (lane 0 = largest).
__device__ __forceinline__ uint64_t warp_sort32_desc(uint64_t v) {
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

// Rank of each of up to blockDim keys among buf[0..n) (n <= blockDim; keys
// unique, 0 = empty): thread i holds key i and counts the keys above it — n
// broadcast reads per thread, no sorting network and one barrier.  Used for
// the short candidate lists of the small-batch path (K6).
__device__ __forceinline__ int block_rank(const uint64_t* buf, int n, uint64_t& mine) {
    mine = (int)threadIdx.x < n ? buf[threadIdx.x] : 0ull;
    int rk = 0;
#pragma unroll 4
    for (int j = 0; j < n; ++j) rk += buf[j] > mine ? 1 : 0;
    return rk;
}

// Out-of-line copies of the block-wide selection helpers: they run a few times
// per work unit, so they should not bloat the kernel's instruction footprint.
__device__ __noinline__ uint64_t k6_block_kth(const uint64_t* buf, int n, uint32_t K, uint32_t* hist,
                                              unsigned long long* sc) {
    return block_kth(buf, n, K, hist, sc);
}
__device__ __noinline__ void k6_block_sort(uint64_t* s, int n) { block_bitonic_desc(s, n); }

// Shared-memory bytes of the prologue region: phi_u + the cluster's S staging
// (then reused as the candidate buffer).
__host__ __device__ __forceinline__ size_t k6_pro_bytes(int cap_keys, int d, int E, int B) {
    const size_t pro = ((size_t)d * 8 + 15) / 16 * 16 + (size_t)E * 4;   // phi_u as fp64 | S staging
    const size_t prog = (size_t)B * d * 8;                                 // grid mode: phi of all users
    size_t r = (size_t)cap_keys * 8;
    r = pro > r ? pro : r;
    r = prog > r ? prog : r;
    return (r + 127) / 128 * 128;
}

// M splits, G table copies, BB = b when known at compile time (256), else 0.
template <int M, int G, int BB>
__global__ void __launch_bounds__(K6_THREADS) k6_query(const K6Args a) {
    constexpr int MP = (M + 3) / 4 * 4;
    constexpr int NW = MP / 4;
    constexpr int IPR = K6_STAGE / MP;                // items per round
    constexpr int J = IPR / K6_THREADS;
    constexpr int CAP = k6_cap(IPR);
    constexpr int NWARP = K6_THREADS / 32;
    extern __shared__ __align__(128) unsigned char sm_raw[];
    const int bq = BB > 0 ? BB : a.b;                 // sub-ids per split
    const int E = M * bq;                             // entries of S_u
    const size_t tbytes = align_up((size_t)M * bq * G * 4, 128);
    float* T = reinterpret_cast<float*>(sm_raw);                                  // [M][b][G]
    unsigned char* ring = sm_raw + tbytes;                                        // [nst][STAGE]
    unsigned char* pro = ring + (size_t)a.nst * K6_STAGE;                         // phi_u | S staging; then cbuf
    const size_t pbytes = k6_pro_bytes(CAP, a.d, E, a.B);
    uint32_t* hist = reinterpret_cast<uint32_t*>(pro + pbytes);                   // [256]
    uint64_t* cbuf = reinterpret_cast<uint64_t*>(pro);
    double* phd = reinterpret_cast<double*>(pro);
    float* Sst = reinterpret_cast<float*>(pro + ((size_t)a.d * 8 + 15) / 16 * 16);
    __shared__ int count;
    __shared__ unsigned long long tau, seed, floor_key;
    __shared__ unsigned long long sc[4];
    __shared__ int wsum[NWARP];
    __shared__ int is_last;
    __shared__ __align__(8) unsigned long long mbar[8];
    cg::cluster_group cluster = cg::this_cluster();
    const int crank = (int)cluster.block_rank(), CL = (int)cluster.num_blocks();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // lanes 2i and 2i + 1 share table copy i (G = 16; copy = lane * G / 32 in
    // general): on colour-paired rows they hold the complementary rows 2p, 2p + 1
    // (opposite parity at every split -> opposite bank halves of the copy), and the
    // code words of a warp stay one contiguous 256-byte block
    const int lrow = (int)threadIdx.x;
    auto src = [&](int e) { return a.cmap ? e - e % (BB > 0 ? BB : a.b) + (int)__ldg(a.cmap + e) : e; };
    const int u = blockIdx.x / a.chunks;
    const int chunk = blockIdx.x % a.chunks;
    const int64_t i0 = (int64_t)chunk * a.chunk_items;
    const int64_t i1 = min(a.N, i0 + a.chunk_items);
    const int64_t rounds = i1 > i0 ? (i1 - i0 + IPR - 1) / IPR : 0;
    const uint32_t bar0 = smem_u32(mbar), ring0 = smem_u32(ring);
    auto stamp = [&](int i) {                         // diagnostics builds only (-DK6_TRACE)
#ifdef K6_TRACE
        if (a.trace && threadIdx.x == 0) {
            long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            a.trace[(int64_t)blockIdx.x * 32 + i] = t;
        }
#else
        (void)i;
#endif
    };
    stamp(0);

    auto issue = [&](int64_t r) {
        const int slot = (int)((uint32_t)r % (uint32_t)a.nst);   // rounds < 2^32 per chunk
        const int64_t s0 = i0 + r * IPR;
        const uint32_t bytes = (uint32_t)align_up((size_t)(min((int64_t)IPR, i1 - s0) * MP), 16);
        const uint32_t bar = bar0 + 8u * slot;
        fence_proxy_async();
        mbar_expect_tx(bar, bytes);
        bulk_g2s(ring0 + (uint32_t)slot * K6_STAGE, a.codes + s0 * MP, bytes, bar);
    };
    if (threadIdx.x == 0) {
        for (int i = 0; i < a.nst; ++i) mbar_init(bar0 + 8u * i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int64_t r = 0; r < min((int64_t)a.nst, rounds); ++r) issue(r);
        count = 0; tau = 0ull; seed = ~0ull; floor_key = 0ull;
    }

    // ---- (1a) grid mode: the whole grid computes every user's S once (each CTA
    // a 1/grid share of the B * m * b entries, K1's fp64 order), publishes it in
    // global memory and meets at a grid barrier; each CTA then replicates its
    // user's table from L2.  Co-residency is guaranteed by a cooperative launch.
    if (a.gridsync) {
        const int EB = a.B * E;
        const int per = (EB + (int)gridDim.x - 1) / (int)gridDim.x;
        const int e0 = (int)blockIdx.x * per, e1 = min(EB, e0 + per);
        const int q4 = a.L / 4;
        // the usual case, at most one entry per thread: its Psi row is requested
        // before phi is staged, so the two memory latencies overlap
        const bool one = per <= K6_THREADS && (a.L & 3) == 0 && a.L <= 64;
        const int em = e0 + (int)threadIdx.x;
        const bool has = one && em < e1;
        float4 ra[16];
        if (has) {
            const float4* pr4 = reinterpret_cast<const float4*>(a.psi + (int64_t)(em % E) * a.L);
#pragma unroll
            for (int i = 0; i < 16; ++i)
                if (i < q4) ra[i] = __ldg(pr4 + i);
        }
        for (int i = threadIdx.x; i < a.B * a.d; i += K6_THREADS) phd[i] = (double)a.phi[i];
        __syncthreads();
        if (one) {
            if (has) {
                const int uu = em / E, ee = em - uu * E;
                const double* fd = phd + (int64_t)uu * a.d + (ee / bq) * a.L;
                double x0 = 0.0, x1 = 0.0, x2 = 0.0, x3 = 0.0;   // K1's order (R5b)
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    if (i < q4) {
                        x0 = fma((double)ra[i].x, fd[4 * i], x0);
                        x1 = fma((double)ra[i].y, fd[4 * i + 1], x1);
                        x2 = fma((double)ra[i].z, fd[4 * i + 2], x2);
                        x3 = fma((double)ra[i].w, fd[4 * i + 3], x3);
                    }
                a.Sg[em] = (float)((x0 + x1) + (x2 + x3));
            }
        } else
        for (int e = e0 + (int)threadIdx.x; e < e1; e += K6_THREADS) {
            const int uu = e / E, ee = e - uu * E;
            const float* pr = a.psi + (int64_t)ee * a.L;
            const double* fd = phd + (int64_t)uu * a.d + (ee / bq) * a.L;
            double x0 = 0.0, x1 = 0.0, x2 = 0.0, x3 = 0.0;   // K1's order (R5b)
            int t = 0;
            for (; t + 4 <= a.L; t += 4) {
                x0 = fma((double)__ldg(pr + t), fd[t], x0);
                x1 = fma((double)__ldg(pr + t + 1), fd[t + 1], x1);
                x2 = fma((double)__ldg(pr + t + 2), fd[t + 2], x2);
                x3 = fma((double)__ldg(pr + t + 3), fd[t + 3], x3);
            }
            if (t < a.L) x0 = fma((double)__ldg(pr + t), fd[t], x0);
            if (t + 1 < a.L) x1 = fma((double)__ldg(pr + t + 1), fd[t + 1], x1);
            if (t + 2 < a.L) x2 = fma((double)__ldg(pr + t + 2), fd[t + 2], x2);
            a.Sg[e] = (float)((x0 + x1) + (x2 + x3));
        }
        stamp(2);
        // grid barrier (all CTAs resident: cooperative launch)
        __syncthreads();
        if (threadIdx.x == 0) {
            // the counters are zeroed by the preceding k6_reset launch (programmatic
            // dependent launch: everything above overlapped it)
            asm volatile("griddepcontrol.wait;" ::: "memory");
            unsigned int* gb = a.done + a.B;
            __threadfence();
            atomicAdd(gb, 1u);
            unsigned int seen;
            long long spins = 0;
            (void)spins;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(gb) : "memory");
                if (seen < gridDim.x) __nanosleep(64);
                PQ_SPIN_CHECK(spins);                  // checked builds: a missing CTA traps
            } while (seen < gridDim.x);
        }
        __syncthreads();
        stamp(3);
        const int rot = lane * G / 32;
        const float* Su = a.Sg + (int64_t)u * E;
        constexpr int RB = 16;                         // entries per thread loaded before any store
        for (int e0r = 0; e0r < E; e0r += RB * K6_THREADS) {
            float vv[RB];
#pragma unroll
            for (int q = 0; q < RB; ++q) {
                const int e = e0r + q * K6_THREADS + (int)threadIdx.x;
                vv[q] = e < E ? __ldcg(Su + src(e)) : 0.0f;
            }
#pragma unroll
            for (int q = 0; q < RB; ++q) {
            const int e = e0r + q * K6_THREADS + (int)threadIdx.x;
            if (e >= E) break;
            const float v = vv[q];
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
        __syncthreads();
    } else
    // ---- (1b) cluster mode: this CTA's share of user u -> every CTA's S staging
    {
        const int per = (E + CL - 1) / CL;
        const int e0 = crank * per, e1 = min(E, e0 + per);
        const int LS = a.L + 4;                        // padded smem row (floats): conflict-free LDS.128
        const int rows_pp = (int)(tbytes / ((size_t)LS * 4));
        const int q4 = a.L / 4;
        const bool staged = (a.L & 3) == 0 && a.L > 16 && a.L <= 64 && rows_pp >= 1;
        // Psi rows of a pass -> the (not yet used) table region, coalesced 16-byte
        // cp.async into padded rows; issued first so the HBM latency overlaps phi
        auto stage = [&](int p0) {
            const int np = min(rows_pp, e1 - p0);
            const float* src = a.psi + (int64_t)p0 * a.L;
            for (int c = threadIdx.x; c < np * q4; c += K6_THREADS) {
                const int row = c / q4, col = c - row * q4;
                const uint32_t dst = smem_u32(T + (size_t)row * LS + 4 * col);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src + 4 * (size_t)c) : "memory");
            }
        };
        if (staged && e0 < e1) stage(e0);
        const float* ph = a.phi + (int64_t)u * a.d;
        for (int i = threadIdx.x; i < a.d; i += K6_THREADS) phd[i] = (double)ph[i];
        const uint32_t sst = smem_u32(Sst);
        auto put = [&](int e, float v) {               // v -> S staging of every CTA of the cluster
            if (a.S_out) a.S_out[(int64_t)u * E + e] = v;
#pragma unroll 1
            for (int q = 0; q < CL; ++q) {
                uint32_t ra;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(sst + 4u * (uint32_t)e), "r"(q));
                asm volatile("st.shared::cluster.f32 [%0], %1;" :: "r"(ra), "f"(v) : "memory");
            }
        };
        // K1's order (R5b): chain j sums t = j, j+4, ... (ascending) in fp64 with exact
        // products; S = fl32((c0 + c1) + (c2 + c3)).  Four chains per entry in flight.
        auto fin = [](double x0, double x1, double x2, double x3) { return (float)((x0 + x1) + (x2 + x3)); };
        if ((a.L & 3) == 0 && a.L <= 16) {
            // short rows: straight from global, a whole row's loads in flight
            __syncthreads();
            for (int e = e0 + (int)threadIdx.x; e < e1; e += K6_THREADS) {
                const float4* pr = reinterpret_cast<const float4*>(a.psi + (int64_t)e * a.L);
                float4 ra[4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (i < q4) ra[i] = __ldg(pr + i);
                const double* fd = phd + (e / bq) * a.L;
                double x0 = 0.0, x1 = 0.0, x2 = 0.0, x3 = 0.0;
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (i < q4) {
                        x0 = fma((double)ra[i].x, fd[4 * i], x0);
                        x1 = fma((double)ra[i].y, fd[4 * i + 1], x1);
                        x2 = fma((double)ra[i].z, fd[4 * i + 2], x2);
                        x3 = fma((double)ra[i].w, fd[4 * i + 3], x3);
                    }
                put(e, fin(x0, x1, x2, x3));
            }
        } else if (staged) {
            for (int p0 = e0; p0 < e1; p0 += rows_pp) {
                const int np = min(rows_pp, e1 - p0);
                if (p0 != e0) stage(p0);
                asm volatile("cp.async.wait_all;" ::: "memory");
                __syncthreads();
                if (p0 - e0 < 2 * rows_pp) stamp(25 + 2 * ((p0 - e0) / rows_pp));
                for (int r = threadIdx.x; r < np; r += K6_THREADS) {
                    const float4* pr = reinterpret_cast<const float4*>(T + (size_t)r * LS);
                    const double* fd = phd + ((p0 + r) / bq) * a.L;
                    double x0 = 0.0, x1 = 0.0, x2 = 0.0, x3 = 0.0;
#pragma unroll 4
                    for (int i = 0; i < q4; ++i) {
                        const float4 p = pr[i];
                        x0 = fma((double)p.x, fd[4 * i], x0);
                        x1 = fma((double)p.y, fd[4 * i + 1], x1);
                        x2 = fma((double)p.z, fd[4 * i + 2], x2);
                        x3 = fma((double)p.w, fd[4 * i + 3], x3);
                    }
                    put(p0 + r, fin(x0, x1, x2, x3));
                }
                __syncthreads();                       // the staging rows are reused by the next pass
                if (p0 - e0 < 2 * rows_pp) stamp(26 + 2 * ((p0 - e0) / rows_pp));
            }
        } else {
            __syncthreads();
            for (int e = e0 + (int)threadIdx.x; e < e1; e += K6_THREADS) {
                const float* pr = a.psi + (int64_t)e * a.L;
                const double* fd = phd + (e / bq) * a.L;
                double x[4] = {0.0, 0.0, 0.0, 0.0};
                int t = 0;
                for (; t + 4 <= a.L; t += 4) {
                    x[0] = fma((double)__ldg(pr + t), fd[t], x[0]);
                    x[1] = fma((double)__ldg(pr + t + 1), fd[t + 1], x[1]);
                    x[2] = fma((double)__ldg(pr + t + 2), fd[t + 2], x[2]);
                    x[3] = fma((double)__ldg(pr + t + 3), fd[t + 3], x[3]);
                }
                if (t < a.L) x[0] = fma((double)__ldg(pr + t), fd[t], x[0]);
                if (t + 1 < a.L) x[1] = fma((double)__ldg(pr + t + 1), fd[t + 1], x[1]);
                if (t + 2 < a.L) x[2] = fma((double)__ldg(pr + t + 2), fd[t + 2], x[2]);
                put(e, fin(x[0], x[1], x[2], x[3]));
            }
        }
        stamp(2);
        cluster.sync();                                // every CTA's S staging is complete
        stamp(3);
        // G copies of each entry into the local table (bank-rotated stores)
        const int rot = lane * G / 32;
        for (int e = threadIdx.x; e < E; e += K6_THREADS) {
            const float v = Sst[src(e)];
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
        __syncthreads();                               // table ready; the staging becomes cbuf
    }

    // ---- (2)+(3) gather-sum over the chunk (lane = item), CTA-wide exact selection
    float tf = -INFINITY;
    const float* Tl = T + ((lane * G) >> 5);
    int slot = 0;
    uint32_t phase = 0;
    for (int64_t r = 0; r < rounds; ++r) {
        mbar_wait(bar0 + 8u * slot, phase);
        if (r < 4) stamp(7 + 3 * (int)r);
        const unsigned char* cs = ring + (size_t)slot * K6_STAGE;
        const int64_t r0 = i0 + r * IPR;
        const int64_t nvalid = i1 - r0;                // items of this round (< IPR only in the last)
        // split-major over the thread's J items: J independent add chains in flight;
        // each lookup = byte extract (PRMT) + scaled add (LEA) + LDS + FADD
        uint32_t cw[J][NW];
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int li = j * K6_THREADS + lrow;
            if constexpr (NW == 1) {
                cw[j][0] = *reinterpret_cast<const uint32_t*>(cs + (size_t)li * MP);
            } else if constexpr (NW == 2) {
                const uint2 t = *reinterpret_cast<const uint2*>(cs + (size_t)li * MP);
                cw[j][0] = t.x; cw[j][1] = t.y;
            } else {
                const uint4 t = *reinterpret_cast<const uint4*>(cs + (size_t)li * MP);
                cw[j][0] = t.x; cw[j][1] = t.y; cw[j][2] = t.z; cw[j][3] = t.w;
            }
        }
        const char* Tb = reinterpret_cast<const char*>(Tl);
        auto look = [&](int k, uint32_t w, int s) {
            const uint32_t g = __byte_perm(w, 0u, 0x4440u | (uint32_t)s);
            return *reinterpret_cast<const float*>(Tb + (size_t)k * bq * G * 4 + (size_t)g * (G * 4));
        };
        // two items' running sums per packed fp32x2 add (FADD2, RN: each lane of the
        // pair is the same IEEE add as a scalar FADD, so the sums are unchanged)
        static_assert(J % 2 == 0, "items in pairs");
        float2 acc2[J / 2];
#pragma unroll
        for (int j = 0; j < J / 2; ++j) acc2[j] = make_float2(look(0, cw[2 * j][0], 0), look(0, cw[2 * j + 1][0], 0));
#pragma unroll
        for (int k = 1; k < M; ++k)
#pragma unroll
            for (int j = 0; j < J / 2; ++j)
                acc2[j] = __fadd2_rn(acc2[j], make_float2(look(k, cw[2 * j][k >> 2], k & 3),
                                                          look(k, cw[2 * j + 1][k >> 2], k & 3)));
        float accs[J];
#pragma unroll
        for (int j = 0; j < J / 2; ++j) { accs[2 * j] = acc2[j].x; accs[2 * j + 1] = acc2[j].y; }
        auto item_key = [&](float acc, int j) {        // R1-R3: +0 canonical score, global id
            const int64_t item = r0 + j * K6_THREADS + lrow;
            const uint32_t lid = a.perm ? (uint32_t)a.perm[item] : (uint32_t)item;
            return make_key(acc + 0.0f, a.id_base + lid);
        };
        // items past the chunk's end (last round only) score NaN: no comparison
        // passes and fmaxf skips them, so the hot path needs no per-item range checks
        if (nvalid < IPR) {
#pragma unroll
            for (int j = 0; j < J; ++j)
                if (j * K6_THREADS + lrow >= (int)nvalid) accs[j] = __int_as_float(0x7fffffff);
        }
        float tfr = tf;
        if (r == 0 && a.K <= NWARP * 32) {
            // threshold seeding: warp w's jk-th largest lane maximum (jk = ceil(K / NWARP))
            // proves jk items of the warp reach it; the minimum over the warps proves
            // NWARP * jk >= K items, so it is a floor for the chunk's K-th key
            int jb = -1;
            float bv = 0.0f;
#pragma unroll
            for (int j = 0; j < J; ++j)
                if (accs[j] == accs[j] && (jb < 0 || accs[j] > bv)) { jb = j; bv = accs[j]; }   // (NaN: no item)
            const uint64_t mx = jb >= 0 ? item_key(bv, jb) : 0ull;
            const uint64_t srt = warp_sort32_desc(mx);
            const int jk = (a.K + NWARP - 1) / NWARP;
            const uint64_t wk = __shfl_sync(FULL, srt, jk - 1);
            if (lane == 0) atomicMin(&seed, (unsigned long long)wk);
            __syncthreads();
            if (threadIdx.x == 0 && seed != ~0ull && seed > 1ull) tau = seed - 1ull;   // keys >= seed pass
            __syncthreads();
            if (tau) tfr = key_score(tau);
        }
        // candidates: score >= the proved threshold score (keys only for those);
        // once the threshold is strong a whole warp usually has none
        float amx = accs[0];
#pragma unroll
        for (int j = 1; j < J; ++j) amx = fmaxf(amx, accs[j]);
        if (__any_sync(FULL, amx >= tfr))
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const bool c = accs[j] >= tfr;
            const unsigned bm = __ballot_sync(FULL, c);
            if (bm) {
                int base = 0;
                if (lane == 0) base = atomicAdd(&count, __popc(bm));
                base = __shfl_sync(FULL, base, 0);
                if (base + __popc(bm) > CAP) __trap();
                if (c) cbuf[base + __popc(bm & lanemask_lt())] = item_key(accs[j], j);
            }
        }
        __syncthreads();
        if (r < 4) stamp(8 + 3 * (int)r);
        const int n_now = count;
        if (n_now <= K6_THREADS && n_now > a.K && (r == 0 || n_now > 2 * a.K + 32)) {
            // few candidates: rank them, keep the K best and raise the threshold to
            // the K-th (exact from the first round on)
            uint64_t mine;
            const int rk = block_rank(cbuf, n_now, mine);
            __syncthreads();
            if ((int)threadIdx.x < n_now && rk < a.K) cbuf[rk] = mine;
            if ((int)threadIdx.x < n_now && rk == a.K - 1) tau = mine;
            if (threadIdx.x == 0) count = a.K;
        } else if (n_now > CAP - IPR && n_now > a.K) { // the next round could overflow: shrink to K
            const uint64_t kth = k6_block_kth(cbuf, n_now, (uint32_t)a.K, hist, sc);
            int base = 0;
            for (int c0 = 0; c0 < n_now; c0 += K6_THREADS) {
                const int i = c0 + threadIdx.x;
                const uint64_t v = i < n_now ? cbuf[i] : 0ull;
                const bool keep = i < n_now && v >= kth;
                const int nk = __syncthreads_count(keep);
                const unsigned bm = __ballot_sync(FULL, keep);
                if (lane == 0) wsum[warp] = __popc(bm);
                __syncthreads();
                int off = 0;
                for (int w = 0; w < warp; ++w) off += wsum[w];
                if (keep) cbuf[base + off + __popc(bm & lanemask_lt())] = v;
                base += nk;
                __syncthreads();
            }
            if (threadIdx.x == 0) { count = base; tau = kth; }
        }
        __syncthreads();
        if (r < 4) stamp(9 + 3 * (int)r);
        tf = tau ? key_score(tau) : -INFINITY;
        // every thread is past this round's reads of the slot: refill it (off the
        // barrier's critical path -- only warp 0 waits for the proxy fence)
        if (threadIdx.x == 0 && r + a.nst < rounds) issue(r + a.nst);
        if (++slot == a.nst) { slot = 0; phase ^= 1u; }
    }

    // ---- the chunk's exact top-K list -> cand[u][chunk][0..K), its K-th key -> kth[u][chunk]
    stamp(4);
    {
        const int n = count;
        uint64_t* out = a.cand + ((int64_t)u * a.chunks + chunk) * a.K;
        if (threadIdx.x == 0 && a.trace) a.trace[(int64_t)blockIdx.x * 32 + 29] = n;
        if (n <= K6_THREADS) {                         // rank the candidates: sorted top K straight out
            uint64_t mine;
            const int rk = block_rank(cbuf, n, mine);
            if ((int)threadIdx.x < n && rk < a.K) out[rk] = mine;
            if ((int)threadIdx.x < n && rk == a.K - 1) a.kth[(int64_t)u * a.chunks + chunk] = mine;
            if ((int)threadIdx.x < n && rk == 0) a.kmax[(int64_t)u * a.chunks + chunk] = mine;
            if (threadIdx.x == 0 && n == 0) a.kmax[(int64_t)u * a.chunks + chunk] = 0ull;
            for (int j = n + (int)threadIdx.x; j < a.K; j += K6_THREADS) out[j] = 0ull;
            if (threadIdx.x == 0 && n < a.K) a.kth[(int64_t)u * a.chunks + chunk] = 0ull;
        } else {
            uint64_t kth = 0ull;                       // 0: fewer than K keys, all are kept
            if (n > a.K) kth = k6_block_kth(cbuf, n, (uint32_t)a.K, hist, sc);
            const uint64_t mx = k6_block_kth(cbuf, n, 1u, hist, sc);
            if (threadIdx.x == 0) a.kmax[(int64_t)u * a.chunks + chunk] = mx;
            if (warp == 0) {
                int pos = 0;
                for (int c0 = 0; c0 < n; c0 += 32) {
                    const int i = c0 + lane;
                    const uint64_t v = i < n ? cbuf[i] : 0ull;
                    const bool keep = i < n && v >= kth;
                    const unsigned bm = __ballot_sync(FULL, keep);
                    if (keep) out[pos + __popc(bm & lanemask_lt())] = v;
                    pos += __popc(bm);
                }
                for (int j = pos + lane; j < a.K; j += 32) out[j] = 0ull;
                if (lane == 0) a.kth[(int64_t)u * a.chunks + chunk] = kth;
            }
        }
        stamp(19);
    }
    stamp(20);
    __threadfence();                                   // publish this chunk's list (device scope)
    __syncthreads();
    stamp(5);
    if (threadIdx.x == 0) {
        asm volatile("griddepcontrol.wait;" ::: "memory");   // (no-op once waited)
        is_last = atomicAdd(&a.done[u], 1u) == (unsigned)(a.chunks - 1);
    }
    __syncthreads();
    if (!is_last) return;

    // ---- (4) last CTA of user u: merge the chunks' lists (K3) and write the answer.
    // floor = the largest chunk K-th key (that chunk alone holds K keys >= it), or
    // the K-th largest chunk maximum (K chunks hold a key >= it), whichever is
    // larger: the user's top K are among the keys >= floor of all lists.
    __threadfence();
    const int n2 = a.chunks * a.K;
    uint64_t* mk = reinterpret_cast<uint64_t*>(ring) + K6_THREADS;   // ring + prologue region: merge scratch
    const uint64_t* cu = a.cand + (int64_t)u * a.chunks * a.K;
    {
        // one pass: each thread loads its chunks' K-th and largest keys together
        uint64_t* cm = reinterpret_cast<uint64_t*>(ring);
        uint64_t f = 0ull;
        for (int c = threadIdx.x; c < a.chunks; c += K6_THREADS) {
            const uint64_t v = __ldcg(a.kth + (int64_t)u * a.chunks + c);
            const uint64_t mx = __ldcg(a.kmax + (int64_t)u * a.chunks + c);
            f = v > f ? v : f;
            cm[c] = mx;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const uint64_t t = __shfl_xor_sync(FULL, f, o);
            f = t > f ? t : f;
        }
        if (lane == 0) atomicMax(&floor_key, (unsigned long long)f);
        if (threadIdx.x == 0) count = 0;
        __syncthreads();
        if (a.chunks >= a.K && a.chunks <= K6_THREADS) {
            uint64_t mine;
            const int rk = block_rank(cm, a.chunks, mine);
            if ((int)threadIdx.x < a.chunks && rk == a.K - 1) atomicMax(&floor_key, (unsigned long long)mine);
        }
        __syncthreads();
    }
    stamp(21);
    const uint64_t fl = floor_key;
    for (int c0 = 0; c0 < n2; c0 += 8 * K6_THREADS) {
        uint64_t v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int i = c0 + q * K6_THREADS + threadIdx.x;
            v[q] = i < n2 ? __ldcg(cu + i) : 0ull;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const bool keep = v[q] != 0ull && v[q] >= fl;
            const unsigned bm = __ballot_sync(FULL, keep);
            if (bm) {
                int base = 0;
                if (lane == 0) base = atomicAdd(&count, __popc(bm));
                base = __shfl_sync(FULL, base, 0);
                PQ_DCHECK(base + __popc(bm) <= a.chunks * a.K);   // mk holds >= chunks * K keys (plan)
                if (keep) mk[base + __popc(bm & lanemask_lt())] = v[q];
            }
        }
    }
    __syncthreads();
    stamp(22);
    int n3 = count;
    if (n3 <= K6_THREADS) {
        uint64_t mine;
        const int rk = block_rank(mk, n3, mine);
        if ((int)threadIdx.x < n3 && rk < a.K) {
            a.ids[(int64_t)u * a.K + rk] = key_id(mine);
            a.scores[(int64_t)u * a.K + rk] = key_score(mine);
        }
        for (int j = n3 + (int)threadIdx.x; j < a.K; j += K6_THREADS) {
            a.ids[(int64_t)u * a.K + j] = -1;
            a.scores[(int64_t)u * a.K + j] = -INFINITY;
        }
    } else {
        if (n3 > 2048) {                               // rare: cut to the K best first
            const uint64_t kth = k6_block_kth(mk, n3, (uint32_t)a.K, hist, sc);
            __syncthreads();
            if (threadIdx.x == 0) count = 0;
            __syncthreads();
            for (int c0 = 0; c0 < n3; c0 += K6_THREADS) {
                const int i = c0 + threadIdx.x;
                const uint64_t v = i < n3 ? mk[i] : 0ull;
                const bool keep = i < n3 && v >= kth;
                const unsigned bm = __ballot_sync(FULL, keep);
                __syncthreads();                       // everyone read before anyone writes
                if (bm) {
                    int base = 0;
                    if (lane == 0) base = atomicAdd(&count, __popc(bm));
                    base = __shfl_sync(FULL, base, 0);
                    if (keep) mk[base + __popc(bm & lanemask_lt())] = v;
                }
                __syncthreads();
            }
            n3 = count;
        }
        const int np2 = pow2_ceil(max(n3, a.K));
        for (int j = n3 + threadIdx.x; j < np2; j += K6_THREADS) mk[j] = 0ull;
        __syncthreads();
        k6_block_sort(mk, np2);
        for (int j = threadIdx.x; j < a.K; j += K6_THREADS) {
            const uint64_t v = mk[j];
            a.ids[(int64_t)u * a.K + j] = v ? key_id(v) : -1;
            a.scores[(int64_t)u * a.K + j] = v ? key_score(v) : -INFINITY;
        }
    }
    stamp(23);
    if (threadIdx.x == 0 && a.trace) {
        a.trace[(int64_t)blockIdx.x * 32 + 31] = n3;
        a.trace[(int64_t)blockIdx.x * 32 + 30] = (long long)fl;
    }
    if (threadIdx.x == 0) a.done[u] = 0u;
    stamp(6);
}

// Zeroes the call's completion counters; lets the K6 launch that follows start
// at once (programmatic dependent launch) -- K6 waits (griddepcontrol.wait)
// only before its first counter access, after its prologue.
__global__ void k6_reset(unsigned int* c, int n) {
    asm volatile("griddepcontrol.launch_dependents;");
    for (int i = threadIdx.x; i < n; i += blockDim.x) c[i] = 0u;
}

// ---------------------------------------------------------------- host side
typedef void (*K6Fn)(const K6Args);

template <int M>
static K6Fn query_fn_g(int G, int b) {
    switch (G) {
        case 16: return b == 256 && M <= 8 ? k6_query<M, 16, 256> : k6_query<M, 16, 0>;
        case 8: return b == 256 && M == 16 ? k6_query<M, 8, 256> : k6_query<M, 8, 0>;
        case 4: return k6_query<M, 4, 0>;
        case 2: return k6_query<M, 2, 0>;
        default: return k6_query<M, 1, 0>;
    }
}
static K6Fn query_fn(int m, int G, int b) {
    switch (m) {
        case 4: return query_fn_g<4>(G, b);
        case 8: return query_fn_g<8>(G, b);
        case 16: return query_fn_g<16>(G, b);
        default: return nullptr;
    }
}
static int query_mp(int m) { return (m + 3) / 4 * 4; }
static int query_cap(int m) { return k6_cap(K6_STAGE / query_mp(m)); }
static size_t query_smem(int m, int b, int G, int nst, int d, int B) {
    return align_up((size_t)m * b * G * 4, 128) + (size_t)nst * K6_STAGE + k6_pro_bytes(query_cap(m), d, m * b, B) +
           256 * 4;
}
// keys the merge scratch (ring + prologue region) holds
static int64_t query_merge_keys(int m, int b, int nst, int d, int B) {
    return (int64_t)(((size_t)nst * K6_STAGE + k6_pro_bytes(query_cap(m), d, m * b, B)) / 8) - K6_THREADS;
}

// CL > 0: thread-block clusters of CL CTAs; CL == 0: cooperative grid (grid mode)
static void query_launch_cfg(cudaLaunchConfig_t& cfg, cudaLaunchAttribute* at, int grid, size_t smem,
                             int CL, cudaStream_t st, bool pdl = false) {
    cfg = cudaLaunchConfig_t{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(K6_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    if (CL > 0) {
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)CL;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
    } else {
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
    }
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (pdl) {
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.numAttrs = 2;
    }
}

static bool plan_uncached(const pq_index_s* idx, int B, int d, int K, K6Plan& p) {
    p = K6Plan{};
    const int m = idx->m;
    if (B < 1 || B > 4 || K < 1 || K > 512 || d % m) return false;
    if (!query_fn(m, 1, idx->b)) return false;
    const pq_tuning& t = idx->tuning;
    int G = 16, nst = 4;
    if (t.users_per_row > 0) G = std::min(16, pow2_ceil(t.users_per_row));   // tuning: table copies
    const size_t budget = idx->smem_optin;
    while (G > 1 && query_smem(m, idx->b, G, 2, d, B) > budget) G >>= 1;
    if (query_smem(m, idx->b, G, 2, d, B) > budget) return false;
    while (nst > 2 && query_smem(m, idx->b, G, nst, d, B) > budget) --nst;
    p.G = G; p.nst = nst;
    // colour-paired rows (one wavefront per lookup instead of two) for long
    // streams: c7 (10^9 items) 3.16 -> 2.64 ms; short ones (C1) lose more to the
    // row -> id loads of the seeding and the candidates than they gain
    static const bool no_pair = getenv("PQTOPK_NO_PAIRED") != nullptr;   // diagnostics (A/B)
    p.paired = idx->d_codes_p && G == 16 && !no_pair && idx->p_rows >= (int64_t)idx->num_sms * 65536 ? 1 : 0;
    p.smem = query_smem(m, idx->b, G, nst, d, B);
    K6Fn fn = query_fn(m, G, idx->b);
    ensure_max_smem(reinterpret_cast<const void*>(fn), (int)p.smem);
    // Cluster size CL: the CTAs of a cluster split one user's sub-id score work
    // (E * L fp64 fmas, E = m * b, L = d / m) -- a larger CL shortens that
    // prologue but packs fewer CTAs (clusters are placed within a GPC).  The
    // model picks the CL minimising prologue + rounds of the slowest CTA:
    //   t(CL) = E * L / CL / 8 clk + ceil(N / (chunks * items per round)) * 2400 clk
    // (about 8 fp64 fmas per clock per SM with the conversions; ~2400 clocks per
    // 16 KB round, measured); tuning.cluster forces one size.
    const int64_t N = p.paired ? idx->p_rows : idx->N;
    const int64_t ipr = K6_STAGE / query_mp(m);
    const int64_t merge_cap = query_merge_keys(m, idx->b, nst, d, B);
    if (merge_cap < 2048) return false;
    // Grid mode (default): one cooperative wave, S computed once per user by the
    // whole grid and shared through L2 behind a grid barrier -- no per-cluster
    // recomputation.  tuning.cluster > 0 selects the cluster mode instead.
    if (t.cluster == 0) {
        int per_sm = 0;
        PQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, K6_THREADS, p.smem));
        const int64_t cap_ctas = (int64_t)per_sm * idx->num_sms;
        if (cap_ctas >= B) {
            int64_t want = std::max<int64_t>(1, ceil_div(N, 512));   // >= 512 items per CTA
            if (t.chunks > 0) want = t.chunks;
            int64_t ch = std::max<int64_t>(1, std::min<int64_t>(want, cap_ctas / B));
            while (ch > 1 && ch * K > merge_cap) --ch;
            if (ch * K <= merge_cap) {
                p.gridsync = 1;
                p.CL = 0;
                p.chunks = (int)ch;
                p.chunk_items = (int64_t)align_up((size_t)ceil_div(N, ch), 16);
                p.grid = B * (int)ch;
                p.cand_bytes = (size_t)B * ch * K * 8;
                return true;
            }
        }
    }
    const int cands[4] = {8, 4, 2, 1};
    double best_t = 0.0;
    int CL = 0, chunks = 0;
    for (int ci = 0; ci < 4; ++ci) {
        const int cl = cands[ci];
        if (t.cluster > 0 && t.cluster != cl) continue;
        cudaLaunchConfig_t cfg;
        cudaLaunchAttribute at[1];
        query_launch_cfg(cfg, at, cl, p.smem, cl, nullptr);
        int max_cl = 0;
        PQ_CUDA(cudaOccupancyMaxActiveClusters(&max_cl, fn, &cfg));
        if (max_cl < B) continue;
        // chunks per user: >= one round each, a multiple of cl, one wave for the
        // batch, and a merge the last CTA can hold in shared memory
        int64_t want = std::max<int64_t>(1, ceil_div(N, ipr));
        if (t.chunks > 0) want = t.chunks;
        int64_t per_user_cl = std::max<int64_t>(1, std::min<int64_t>(ceil_div(want, cl), max_cl / B));
        while (per_user_cl > 1 && per_user_cl * cl * K > merge_cap) --per_user_cl;
        if (per_user_cl * cl * K > merge_cap) continue;
        const int64_t ch = per_user_cl * cl;
        const double tm = (double)m * idx->b * (d / m) / cl / 8.0 + (double)ceil_div(N, ch * ipr) * 2400.0;
        if (CL == 0 || tm < best_t) { best_t = tm; CL = cl; chunks = (int)ch; }
    }
    if (CL == 0) return false;
    const int64_t chunk_items = (int64_t)align_up((size_t)ceil_div(N, chunks), 16);
    p.CL = CL;
    p.chunks = chunks;
    p.chunk_items = chunk_items;
    p.grid = B * chunks;
    p.cand_bytes = (size_t)B * chunks * K * 8;
    return true;
}

// Plans are cached per index (the cluster-occupancy query costs host time on
// every call otherwise); the key includes the tuning fields the plan reads.
struct K6CacheEnt {
    int B, d, K;
    pq_tuning t;
    bool ok;
    K6Plan p;
};
static std::mutex g_k6_mu;

bool k6_query_plan(pq_index_s* idx, int B, int d, int K, K6Plan& p) {
    std::lock_guard<std::mutex> lk(g_k6_mu);
    auto* v = static_cast<std::vector<K6CacheEnt>*>(idx->k6_cache);
    if (!v) idx->k6_cache = v = new std::vector<K6CacheEnt>();
    for (const auto& e : *v)
        if (e.B == B && e.d == d && e.K == K && memcmp(&e.t, &idx->tuning, sizeof(pq_tuning)) == 0) {
            p = e.p;
            return e.ok;
        }
    // K7 (codes of each CTA's chunk resident in shared memory) whenever it
    // applies, unless the tuning forces K6 (variant 5); K6 otherwise
    bool ok = idx->tuning.variant != 5 && k7_resident_plan(idx, B, d, K, p);
    if (!ok && idx->tuning.variant != 7) ok = plan_uncached(idx, B, d, K, p);
    v->push_back(K6CacheEnt{B, d, K, idx->tuning, ok, p});
    return ok;
}

void k6_cache_free(pq_index_s* idx) {
    std::lock_guard<std::mutex> lk(g_k6_mu);
    delete static_cast<std::vector<K6CacheEnt>*>(idx->k6_cache);
    idx->k6_cache = nullptr;
}

size_t k6_query_ws_bytes(const K6Plan& p, int B, int E) {
    if (p.resident) return k7_resident_ws_bytes(p, B, E);
    return align_up(p.cand_bytes, 256) + 2 * align_up((size_t)B * p.chunks * 8, 256) +
           align_up((size_t)(B + 1) * 4, 256) + align_up((size_t)B * E * 4, 256);
}

void launch_k6_query(const pq_index_s* idx, const K6Plan& p, const float* phi, const float* psi, int B,
                     int d, int K, void* ws, float* S_out, int32_t* ids, float* scores, cudaStream_t st) {
    if (p.resident) {
        launch_k7_resident(idx, p, phi, psi, B, d, K, ws, S_out, ids, scores, st);
        return;
    }
    K6Args a{};
    a.codes = p.paired ? idx->d_codes_p : idx->d_codes;
    a.perm = p.paired ? idx->d_perm3 : (idx->lay.paired ? idx->d_perm : nullptr);
    a.cmap = p.paired ? idx->d_cmap3 : nullptr;
    a.phi = phi; a.psi = psi; a.S_out = S_out;
    a.N = p.paired ? idx->p_rows : idx->N;
    a.mp = idx->lay.mp; a.b = idx->b; a.B = B; a.K = K; a.d = d; a.L = d / idx->m;
    a.id_base = (uint32_t)idx->id_base;
    a.chunks = p.chunks; a.chunk_items = p.chunk_items;
    char* w = static_cast<char*>(ws);
    a.cand = reinterpret_cast<uint64_t*>(w);
    const size_t kb = align_up((size_t)B * p.chunks * 8, 256);
    a.kth = reinterpret_cast<uint64_t*>(w + align_up(p.cand_bytes, 256));
    a.kmax = reinterpret_cast<uint64_t*>(w + align_up(p.cand_bytes, 256) + kb);
    a.done = reinterpret_cast<unsigned int*>(w + align_up(p.cand_bytes, 256) + 2 * kb);
    a.Sg = S_out ? S_out
                 : reinterpret_cast<float*>(w + align_up(p.cand_bytes, 256) + 2 * kb + align_up((size_t)(B + 1) * 4, 256));
    a.gridsync = p.gridsync;
    if (p.gridsync) a.S_out = nullptr;              // written through Sg
    a.ids = ids; a.scores = scores;
    a.nst = p.nst;
    static const bool no_pdl = getenv("PQTOPK_K6_NO_PDL") != nullptr;   // diagnostics: plain memset + launch
    if (no_pdl) {
        PQ_CUDA(cudaMemsetAsync(a.done, 0, (size_t)(B + 1) * 4, st));
    } else {
        k6_reset<<<1, 32, 0, st>>>(a.done, B + 1);
        count_launch();
        check_launch("k6_reset");
    }
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute at[2];
    query_launch_cfg(cfg, at, p.grid, p.smem, p.CL, st, !no_pdl);
    const char* tf = getenv("PQTOPK_K6_TRACE");
    if (tf && *tf) {
        PQ_CUDA(cudaMalloc(&a.trace, (size_t)p.grid * 32 * 8));
        PQ_CUDA(cudaMemsetAsync(a.trace, 0, (size_t)p.grid * 32 * 8, st));
    }
    PQ_CUDA(cudaLaunchKernelEx(&cfg, query_fn(idx->m, p.G, idx->b), a));
    count_launch();
    check_launch("k6_query");
    if (a.trace) {                       // diagnostics only: per-CTA phase stamps
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
