// K2 — fused gather-sum-select (Eq. 5; Algorithm 1).
//
// For every (user u, item i) of a work unit:
//     r = ((+0.0f + S[u][0][g_i0]) + S[u][1][g_i1]) + ... + S[u][m-1][g_i,m-1]
// in fp32, k ascending (R1, R2), then keep r only if its ranking key beats the
// lane's running threshold.  No N-length score array is ever written (BJ).
//
// Layout ("row groups", variant 1).  A CTA owns Ug users (a user group) and a
// contiguous item chunk.  Shared memory holds the users' sub-id score tables
// interleaved by user: row (k, g) is G consecutive fp32 words, word w holding
// S[user(w % Ug)][k][g] (Ug < G: the G/Ug copies are replicas).  Lane l of a
// warp reads row word l % G and takes item slot l / Ug, so the P = 32/Ug slots
// of a warp look up P different items in the same split: one LDS per lane per
// split.  G = 32 makes every warp access
// bank-conflict free (32 distinct users, one row); smaller G trades conflicts
// for capacity (m*b*G*4 bytes must fit in shared memory; SURVEY §7 hard part 1).
//
// Selection.  Each lane keeps a private candidate buffer of `cap` 64-bit keys
// in global memory (L2-resident; appends are rare: ~K(1+ln(n/K)) per stream)
// and a threshold tau = the K-th best key it has proved.  When any lane's
// buffer could overflow on the next step, the warp cooperatively radix-selects
// that lane's K-th key, compacts the buffer to K keys and raises tau (and the
// CTA-shared per-user threshold, which other lanes of the same user adopt).
// Dropping a key below a proved threshold is safe: >= K larger keys exist.
// At the end of a unit every lane shrinks to <= K keys and the CTA merges the
// lanes of each user into one list of K keys (the unit's exact top-K) for K3.
#include "k2_common.cuh"

namespace pq {

template <int G, int M, int J>
__global__ void __launch_bounds__(512, 1) k2_score_select(const K2Args a) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    const int W = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int m = (M > 0) ? M : a.m;
    const int mp = (M > 0) ? M : a.mp;
    const int b = a.b;
    const size_t tbl_words = (size_t)m * b * G;
    float* T = reinterpret_cast<float*>(sm_raw);
    uint32_t* hist_all = reinterpret_cast<uint32_t*>(sm_raw + align_up(tbl_words * 4, 16));
    uint32_t* hist = hist_all + warp * 256;
    unsigned long long* tau_sh = reinterpret_cast<unsigned long long*>(hist_all + W * 256);
    int* ucnt = reinterpret_cast<int*>(tau_sh + 32);
    int* ucur = ucnt + 32;

    // Lane l reads row word l % G (user l % Ug, since Ug | G) and takes item
    // slot l / Ug: lanes of the same user (replicas when Ug < G) get distinct
    // items, lanes of distinct users share one item.
    const int Ug = a.Ug;
    const int P = 32 / Ug;
    const int slot = lane / Ug;
    const int lw = lane % G;
    const int my_u = lane & (Ug - 1);
    uint64_t* wbuf = a.lanebuf + ((int64_t)blockIdx.x * W + warp) * 32 * a.cap;
    uint64_t* mybuf = wbuf + (int64_t)lane * a.cap;
    const float* Tl = T + lw;
    const int64_t units = (int64_t)a.n_groups * a.chunks;

    for (int64_t unit = blockIdx.x; unit < units; unit += gridDim.x) {
        // chunk-major: concurrently running CTAs read the same code chunk (L2 reuse)
        const int chunk = (int)(unit / a.n_groups);
        const int grp = (int)(unit - (int64_t)chunk * a.n_groups);
        const int64_t i0 = (int64_t)chunk * a.chunk_items;
        const int64_t i1 = min(a.N, i0 + a.chunk_items);

        // ---- stage the group's S tables (interleaved by user) --------------
        __syncthreads();
        for (size_t x = threadIdx.x; x < tbl_words; x += blockDim.x) {
            const int row = (int)(x / G), w = (int)(x % G);
            const int user = grp * Ug + (w & (Ug - 1));
            T[x] = user < a.B ? a.S[(int64_t)user * m * b + row] : 0.0f;
        }
        if (threadIdx.x < 32) { tau_sh[threadIdx.x] = 0ull; ucnt[threadIdx.x] = 0; ucur[threadIdx.x] = 0; }
        __syncthreads();

        const int user = grp * Ug + my_u;
        const bool active = user < a.B;
        uint64_t tau = active ? 0ull : ~0ull;
        float tau_f = active ? -INFINITY : INFINITY;
        int cnt = 0;

        // ---- stream the chunk ---------------------------------------------
        const int64_t per_step = (int64_t)W * P * J;
        int64_t base = i0 + (int64_t)warp * P * J;
        constexpr int MW = (M > 0) ? (M + 3) / 4 : 1;
        uint32_t cw[J][MW];
        auto load = [&](int64_t bs, uint32_t (&dst)[J][MW]) {
#pragma unroll
            for (int j = 0; j < J; ++j) {
                int64_t row = bs + j * P + slot;
                row = row < i1 ? row : i1 - 1;
                const uint8_t* p = a.codes + row * mp;
                if constexpr (MW == 4) {
                    uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
                    dst[j][0] = v.x; dst[j][1] = v.y; dst[j][2] = v.z; dst[j][3] = v.w;
                } else if constexpr (MW == 2) {
                    uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
                    dst[j][0] = v.x; dst[j][1] = v.y;
                } else if constexpr (M > 0) {
#pragma unroll
                    for (int q = 0; q < MW; ++q) dst[j][q] = __ldg(reinterpret_cast<const uint32_t*>(p) + q);
                } else {
                    dst[j][0] = (uint32_t)(row);      // generic path: reload bytes below
                }
            }
        };
        if (base < i1) load(base, cw);
        int step = 0;
        for (; base < i1; base += per_step, ++step) {
            uint32_t nx[J][MW];
            const int64_t nb = base + per_step;
            if (nb < i1) load(nb, nx);
            float acc[J];
#pragma unroll
            for (int j = 0; j < J; ++j) acc[j] = 0.0f;            // +0.0f start (R2)
            if constexpr (M > 0) {
#pragma unroll
                for (int k = 0; k < M; ++k) {
#pragma unroll
                    for (int j = 0; j < J; ++j) {
                        const uint32_t g = (cw[j][k >> 2] >> (8 * (k & 3))) & 0xFFu;
                        acc[j] = acc[j] + Tl[((size_t)k * b + g) * G];   // k ascending (R1)
                    }
                }
            } else {
                for (int k = 0; k < m; ++k) {
#pragma unroll
                    for (int j = 0; j < J; ++j) {
                        int64_t row = base + j * P + slot;
                        row = row < i1 ? row : i1 - 1;
                        const uint32_t g = a.codes[row * mp + k];
                        acc[j] = acc[j] + Tl[((size_t)k * b + g) * G];
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const int64_t row = base + j * P + slot;
                if (row < i1 && acc[j] >= tau_f) {                  // rare slow path
                    const uint32_t lid = a.perm ? (uint32_t)a.perm[row] : (uint32_t)row;
                    const uint64_t key = make_key(acc[j], a.id_base + lid);
                    if (key > tau) mybuf[cnt++] = key;
                }
            }
            if (__any_sync(FULL, cnt > a.cap - J))
                warp_flush(wbuf, a.cap, cnt, tau, tau_f, a.K, a.cap - J, hist, &tau_sh[my_u]);
            if ((step & 7) == 7 && active) {
                const uint64_t t = *reinterpret_cast<volatile unsigned long long*>(&tau_sh[my_u]);
                if (t > tau) { tau = t; tau_f = key_score(t); }
            }
            if constexpr (M > 0) {
#pragma unroll
                for (int j = 0; j < J; ++j)
#pragma unroll
                    for (int q = 0; q < MW; ++q) cw[j][q] = nx[j][q];
            }
        }

        // ---- end of unit: every lane to <= K keys, then per-user CTA merge --
        if (__any_sync(FULL, cnt > a.K))
            warp_flush(wbuf, a.cap, cnt, tau, tau_f, a.K, a.K, hist, &tau_sh[my_u]);
        __syncthreads();
        cta_merge(a, mybuf, cnt, active, my_u, Ug, grp, chunk, tau_sh, ucnt, ucur,
                  a.mscr + (int64_t)blockIdx.x * 32 * W * a.K, (32 / Ug) * W * a.K, hist);
    }
}

// ---------------------------------------------------------------------------
// Host side: plan + dispatch
// ---------------------------------------------------------------------------
typedef void (*K2Fn)(const K2Args);

template <int G, int J>
static K2Fn pick_m(int m) {
    switch (m) {
        case 4: return k2_score_select<G, 4, J>;
        case 8: return k2_score_select<G, 8, J>;
        case 16: return k2_score_select<G, 16, J>;
        default: return k2_score_select<G, 0, J>;
    }
}
static K2Fn pick(int G, int m) {
    switch (G) {
        case 1: return pick_m<1, 4>(m);
        case 2: return pick_m<2, 4>(m);
        case 4: return pick_m<4, 4>(m);
        case 8: return pick_m<8, 4>(m);
        case 16: return pick_m<16, 4>(m);
        default: return pick_m<32, 4>(m);
    }
}

static size_t k2_smem(int m, int b, int G, int W) {
    return align_up((size_t)m * b * G * 4, 16) + (size_t)W * 256 * 4 + 32 * 8 + 64 * 4;
}

static int choose_chunks(int64_t n_items, int n_groups, int grid_full, int64_t min_items) {
    const int64_t max_c = std::max<int64_t>(1, std::min<int64_t>(4096, n_items / min_items));
    int best = 1;
    double best_eff = -1.0;
    for (int64_t c = 1; c <= max_c; ++c) {
        int64_t units = (int64_t)n_groups * c;
        int64_t waves = ceil_div(units, grid_full);
        double eff = (double)units / (double)(waves * grid_full);
        if (eff > best_eff + 1e-9) { best_eff = eff; best = (int)c; }
        if (eff >= 0.97) break;
    }
    return best;
}

K2Plan plan_k2(const pq_index_s* idx, int B, int K) {
    pq_tuning tt = idx->tuning;
    if (tt.variant == 5) tt.variant = 0;               // 5 selects K6 in pq_search only
    if (idx->v3_ok && (tt.variant == 3 || (tt.variant == 0 && tt.users_per_row == 0 && B >= 16))) {
        K2Plan p;
        plan_k2_tiled(idx, B, K, p);
        return p;
    }
    if ((tt.variant == 4 || (tt.variant == 0 && tt.users_per_row == 0)) && k2_latency_supported(idx, B, K)) {
        K2Plan p;
        plan_k2_latency(idx, B, K, p);
        return p;
    }
    K2Plan p;
    const int m = idx->m, b = idx->b;
    const pq_tuning& t = idx->tuning;
    p.W = t.warps > 0 ? std::min(t.warps, 16) : 8;
    p.J = 4;
    const size_t budget = idx->smem_optin;
    int G = 32;
    if (t.users_per_row > 0) G = std::min(32, pow2_ceil(t.users_per_row));
    while (G > 1 && k2_smem(m, b, G, p.W) > budget) G >>= 1;
    if (k2_smem(m, b, G, p.W) > budget) fail(PQ_ERR_UNSUPPORTED, "sub-id table does not fit in shared memory");
    p.G = G;
    p.Ug = std::min(G, pow2_ceil(std::max(B, 1)));
    p.n_groups = (int)ceil_div(B, p.Ug);
    p.cap = (int)align_up((size_t)std::max(2 * K, K + 4 * p.J), 32);
    p.smem = k2_smem(m, b, G, p.W);

    K2Fn fn = pick(G, m);
    ensure_max_smem(reinterpret_cast<const void*>(fn), (int)p.smem);
    int occ = 0;
    PQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, p.W * 32, p.smem));
    if (occ < 1) fail(PQ_ERR_UNSUPPORTED, "scoring kernel cannot be resident (occupancy 0)");
    // lane buffers: keep them under ~2 GiB
    const size_t per_cta = (size_t)p.W * 32 * p.cap * 8 + (size_t)32 * p.W * K * 8;
    const int occ_mem = (int)std::max<size_t>(1, ((size_t)2 << 30) / (per_cta * idx->num_sms));
    occ = std::min(occ, occ_mem);
    const int grid_full = idx->num_sms * occ;

    const int64_t N = idx->N;
    p.chunks = t.chunks > 0 ? t.chunks : choose_chunks(N, p.n_groups, grid_full, 1 << 15);
    p.chunk_items = ceil_div(N, p.chunks);
    p.chunks = (int)ceil_div(N, p.chunk_items);
    const int64_t units = (int64_t)p.n_groups * p.chunks;
    p.grid = (int)std::min<int64_t>(units, t.ctas > 0 ? t.ctas : grid_full);
    p.lanebuf_bytes = (size_t)p.grid * p.W * 32 * p.cap * 8;
    p.cand_bytes = (size_t)B * p.chunks * K * 8;
    p.mscr_bytes = (size_t)p.grid * 32 * p.W * K * 8;
    return p;
}

void launch_k2(const pq_index_s* idx, const K2Plan& p, const float* S, int B, int K,
               uint64_t* lanebuf, uint64_t* cand, cudaStream_t st) {
    K2Args a{};
    a.codes = idx->d_codes;
    a.perm = idx->lay.paired ? idx->d_perm : nullptr;
    a.S = S;
    a.N = idx->N;
    a.m = idx->m; a.b = idx->b; a.mp = idx->lay.mp;
    a.B = B; a.K = K;
    a.id_base = (uint32_t)idx->id_base;
    a.Ug = p.Ug; a.n_groups = p.n_groups; a.chunks = p.chunks; a.chunk_items = p.chunk_items;
    a.lanebuf = lanebuf; a.cap = p.cap; a.cand = cand;
    a.mscr = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(lanebuf) + align_up(p.lanebuf_bytes, 256));
    K2Fn fn = pick(p.G, idx->m);
    fn<<<p.grid, p.W * 32, p.smem, st>>>(a);
    count_launch();
    check_launch("k2_score_select");
}

}  // namespace pq
