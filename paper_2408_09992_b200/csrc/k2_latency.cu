// K2 v4 — small-batch (B <= 4) fused gather-sum-select: the paper's serving
// case is one user (mRT per user; elbow below 1e5 items, P:259;
// SURVEY §8(f) row f4).
//
// Lane = item (one user per work unit): every lane scores its own items, so a
// warp-wide table lookup touches up to 32 random rows.  The user's table is
// replicated G times in shared memory (row (k, g) = G copies; lane l reads
// copy l % G), which caps the bank conflict degree at ~32/G... (G = 16: two
// lanes per bank at most -> 2 wavefronts per lookup; measured simulation
// SURVEY App. A).  Staging the table costs m*b*G*4 bytes of shared-memory
// writes per work unit (C2a: 128 KB), negligible next to the items.
//
// Selection is CTA-wide and exact: items whose score reaches the CTA's
// threshold append their 64-bit key (R3) to a shared buffer with a
// warp-aggregated atomic; after every round (blockDim * J items) the CTA
// shrinks the buffer to its K best keys (radix select in shared memory) when
// the next round could overflow it, which raises the threshold.  A work unit
// (user, item chunk) ends with its exact top-K list for K3.  Sum order as
// everywhere: acc = S[0] + S[1] + ... + S[m-1] in fp32, +0.0f when keyed (R1/R2).
#include "k2_common.cuh"

namespace pq {

struct K2LArgs {
    const uint8_t* codes;      // [N][mp] item-order uint8 rows (K0 layout)
    const int32_t* perm;       // row -> local item id (subset scoring), or null (identity)
    const float* S;            // [B][m][b]
    int64_t N;
    int mp, b, B, K;
    uint32_t id_base;
    int chunks;
    int64_t chunk_items;
    uint64_t* cand;            // [B][chunks][K]
};

constexpr int K2L_THREADS = 256;
constexpr int K2L_J = 4;                              // items per thread per round
constexpr int K2L_CAP = 2 * K2L_THREADS * K2L_J;      // shared candidate buffer (keys)

template <int M, int G>
__global__ void __launch_bounds__(K2L_THREADS) k2_latency(const K2LArgs a) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    float* T = reinterpret_cast<float*>(sm_raw);                      // [M][b][G]
    uint64_t* cbuf = reinterpret_cast<uint64_t*>(sm_raw + align_up((size_t)M * a.b * G * 4, 16));
    uint32_t* hist = reinterpret_cast<uint32_t*>(cbuf + K2L_CAP);     // [256]
    __shared__ int count;
    __shared__ unsigned long long tau;
    __shared__ unsigned long long sc[4];
    __shared__ int wsum[K2L_THREADS / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int rep = lane % G;
    const int64_t units = (int64_t)a.B * a.chunks;

    for (int64_t unit = blockIdx.x; unit < units; unit += gridDim.x) {
        const int u = (int)(unit % a.B);
        const int chunk = (int)(unit / a.B);
        const int64_t i0 = (int64_t)chunk * a.chunk_items;
        const int64_t i1 = min(a.N, i0 + a.chunk_items);
        __syncthreads();
        {   // stage the user's table, G copies per row (rows loaded once, independent loads)
            const float* Su = a.S + (int64_t)u * M * a.b;
            const int rows = M * a.b;
            for (int r0 = 0; r0 < rows; r0 += 4 * K2L_THREADS) {
                float v[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int r = r0 + q * K2L_THREADS + threadIdx.x;
                    v[q] = r < rows ? __ldg(&Su[r]) : 0.0f;
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int r = r0 + q * K2L_THREADS + threadIdx.x;
                    if (r < rows) {
                        if constexpr (G >= 4) {
#pragma unroll
                            for (int c = 0; c < G; c += 4)
                                *reinterpret_cast<float4*>(&T[(size_t)r * G + c]) = make_float4(v[q], v[q], v[q], v[q]);
                        } else {
#pragma unroll
                            for (int c = 0; c < G; ++c) T[(size_t)r * G + c] = v[q];
                        }
                    }
                }
            }
        }
        if (threadIdx.x == 0) { count = 0; tau = 0ull; }
        __syncthreads();
        float tf = -INFINITY;
        const float* Tl = T + rep;
        constexpr int NW = (M + 3) / 4;                   // code words per item row
        auto load_codes = [&](int64_t r0, uint32_t (&cw)[K2L_J][NW]) {
#pragma unroll
            for (int j = 0; j < K2L_J; ++j) {
                const int64_t item = r0 + (int64_t)j * K2L_THREADS + threadIdx.x;
                const uint8_t* row = a.codes + (item < i1 ? item : i0) * a.mp;
#pragma unroll
                for (int q = 0; q < NW; ++q) cw[j][q] = __ldg(reinterpret_cast<const uint32_t*>(row) + q);
            }
        };
        uint32_t cw[K2L_J][NW];
        load_codes(i0, cw);
        int round = 0;
        for (int64_t r0 = i0; r0 < i1; r0 += (int64_t)K2L_THREADS * K2L_J, ++round) {
            uint32_t nx[K2L_J][NW];                        // next round's codes (prefetch)
            const int64_t r1 = r0 + (int64_t)K2L_THREADS * K2L_J;
            if (r1 < i1) load_codes(r1, nx);
            uint64_t keys[K2L_J];
#pragma unroll
            for (int j = 0; j < K2L_J; ++j) {
                const int64_t item = r0 + (int64_t)j * K2L_THREADS + threadIdx.x;
                float acc = Tl[(cw[j][0] & 0xFFu) * G];
#pragma unroll
                for (int k = 1; k < M; ++k) {
                    const uint32_t g = (cw[j][k >> 2] >> (8 * (k & 3))) & 0xFFu;
                    acc = acc + Tl[((size_t)k * a.b + g) * G];
                }
                const uint32_t lid = (item < i1 && a.perm) ? (uint32_t)a.perm[item] : (uint32_t)item;
                keys[j] = (item < i1 && acc >= tf) ? make_key(acc + 0.0f, a.id_base + lid) : 0ull;
            }
            // append this round's candidates (warp-aggregated slots)
#pragma unroll
            for (int j = 0; j < K2L_J; ++j) {
                const bool c = keys[j] != 0ull && keys[j] > tau;
                const unsigned bm = __ballot_sync(FULL, c);
                if (bm) {
                    int base = 0;
                    if (lane == 0) base = atomicAdd(&count, __popc(bm));
                    base = __shfl_sync(FULL, base, 0);
                    if (c) cbuf[base + __popc(bm & lanemask_lt())] = keys[j];
                }
            }
            __syncthreads();
            const int n_now = count;                       // same value in every thread
            // shrink after the first round (it ran without a threshold) and
            // whenever the next round could overflow the buffer
            if (((round == 0 && r1 < i1) || n_now > K2L_CAP - K2L_THREADS * K2L_J) && n_now > a.K) {
                const uint64_t kth = block_kth(cbuf, n_now, (uint32_t)a.K, hist, sc);
                // compact in place: block-wide ballot prefix over chunks of blockDim
                int base = 0;
                for (int i0c = 0; i0c < n_now; i0c += K2L_THREADS) {
                    const int i = i0c + threadIdx.x;
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
            __syncthreads();                               // nobody appends before all read count
            tf = tau ? key_score(tau) : -INFINITY;
            if (r1 < i1) {
#pragma unroll
                for (int j = 0; j < K2L_J; ++j)
#pragma unroll
                    for (int q = 0; q < NW; ++q) cw[j][q] = nx[j][q];
            }
        }

        // ---- end of unit: the unit's exact top-K list ---------------------
        __syncthreads();
        const int n = count;
        const uint64_t kth = n > a.K ? block_kth(cbuf, n, (uint32_t)a.K, hist, sc) : 1ull;
        if (warp == 0) {
            uint64_t* out = a.cand + ((int64_t)u * a.chunks + chunk) * a.K;
            int pos = 0;
            for (int b0 = 0; b0 < n; b0 += 32) {
                const int i = b0 + lane;
                const uint64_t v = i < n ? cbuf[i] : 0ull;
                const bool keep = i < n && v >= kth;
                const unsigned bm = __ballot_sync(FULL, keep);
                if (keep) out[pos + __popc(bm & lanemask_lt())] = v;
                pos += __popc(bm);
            }
            for (int j = pos + lane; j < a.K; j += 32) out[j] = 0ull;
        }
    }
}

// ---------------------------------------------------------------- host side
typedef void (*K2LFn)(const K2LArgs);

template <int M>
static K2LFn latency_fn_g(int G) {
    switch (G) {
        case 16: return k2_latency<M, 16>;
        case 8: return k2_latency<M, 8>;
        case 4: return k2_latency<M, 4>;
        case 2: return k2_latency<M, 2>;
        default: return k2_latency<M, 1>;
    }
}
static K2LFn latency_fn(int m, int G) {
    switch (m) {
        case 4: return latency_fn_g<4>(G);
        case 8: return latency_fn_g<8>(G);
        case 16: return latency_fn_g<16>(G);
        default: return nullptr;
    }
}
static size_t latency_smem(int m, int b, int G) {
    return align_up((size_t)m * b * G * 4, 16) + (size_t)K2L_CAP * 8 + 256 * 4;
}

bool k2_latency_supported(const pq_index_s* idx, int B, int K) {
    return B >= 1 && B <= 4 && K <= 512 && latency_fn(idx->m, 1) != nullptr &&
           latency_smem(idx->m, idx->b, 1) <= idx->smem_optin;
}

void plan_k2_latency(const pq_index_s* idx, int B, int K, K2Plan& p) {
    p.variant = 4;
    const pq_tuning& t = idx->tuning;
    int G = 16;
    while (G > 1 && latency_smem(idx->m, idx->b, G) > std::min<size_t>(idx->smem_optin, 200 * 1024)) G >>= 1;
    p.G = G; p.Ug = 1; p.W = K2L_THREADS / 32; p.J = K2L_J; p.tm = 0;
    p.n_groups = B;
    p.smem = latency_smem(idx->m, idx->b, G);
    K2LFn fn = latency_fn(idx->m, G);
    PQ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
    // chunks: about one wave of CTAs, >= one round (blockDim * J items) each
    const int64_t N = idx->N;
    const int64_t want = std::max<int64_t>(1, std::min<int64_t>(ceil_div(idx->num_sms, B),
                                                               ceil_div(N, (int64_t)K2L_THREADS * K2L_J)));
    p.chunks = t.chunks > 0 ? t.chunks : (int)want;
    p.chunk_items = ceil_div(N, p.chunks);
    p.chunks = (int)ceil_div(N, p.chunk_items);
    const int64_t units = (int64_t)B * p.chunks;
    p.grid = (int)std::min<int64_t>(units, t.ctas > 0 ? t.ctas : (int64_t)idx->num_sms);
    p.cap = K2L_CAP;
    p.lanebuf_bytes = 0; p.mscr_bytes = 0; p.ghist_bytes = 0; p.st_bytes = 0;
    p.cand_bytes = (size_t)B * p.chunks * K * 8;
}

void launch_k2_latency(const pq_index_s* idx, const K2Plan& p, const float* S, int B, int K,
                       uint64_t* cand, cudaStream_t st) {
    K2LArgs a{};
    a.codes = idx->d_codes;
    a.perm = idx->lay.paired ? idx->d_perm : nullptr;
    a.S = S;
    a.N = idx->N;
    a.mp = idx->lay.mp; a.b = idx->b; a.B = B; a.K = K;
    a.id_base = (uint32_t)idx->id_base;
    a.chunks = p.chunks; a.chunk_items = p.chunk_items;
    a.cand = cand;
    K2LFn fn = latency_fn(idx->m, p.G);
    fn<<<p.grid, K2L_THREADS, p.smem, st>>>(a);
    count_launch();
    check_launch("k2_latency");
}

}  // namespace pq
