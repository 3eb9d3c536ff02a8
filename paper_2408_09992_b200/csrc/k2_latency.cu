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
#include "ptx_dev.cuh"

namespace pq {

struct K2LArgs {
    const uint8_t* codes;      // [N][mp] item-order uint8 rows (K0 layout)
    const int32_t* perm;       // row -> local item id (subset scoring), or null (identity)
    const float* S;            // [B][m][b]
    int64_t N;
    int mp, b, B, K;
    uint32_t id_base;
    int chunks;
    int64_t chunk_items;       // multiple of 16 (16-byte aligned code stages)
    uint64_t* cand;            // [B][chunks][K]
    int nst;                   // code stages in flight (TMA ring)
};

constexpr int K2L_THREADS = 256;
constexpr int K2L_STAGE = 16384;                      // code bytes per round (one TMA stage)

// M splits (row = MP bytes), G table copies, NST code stages in flight.
template <int M, int G>
__global__ void __launch_bounds__(K2L_THREADS) k2_latency(const K2LArgs a) {
    constexpr int MP = (M + 3) / 4 * 4;               // bytes per item row
    constexpr int NW = MP / 4;                        // code words per row
    constexpr int IPR = K2L_STAGE / MP;               // items per round
    constexpr int J = IPR / K2L_THREADS;              // items per thread per round
    constexpr int CAP = 2 * IPR;                      // shared candidate buffer (keys)
    extern __shared__ __align__(128) unsigned char sm_raw[];
    float* T = reinterpret_cast<float*>(sm_raw);                      // [M][b][G]
    unsigned char* ring = sm_raw + align_up((size_t)M * a.b * G * 4, 128);       // [nst][K2L_STAGE]
    uint64_t* cbuf = reinterpret_cast<uint64_t*>(ring + (size_t)a.nst * K2L_STAGE);
    uint32_t* hist = reinterpret_cast<uint32_t*>(cbuf + CAP);         // [256]
    __shared__ int count;
    __shared__ unsigned long long tau;
    __shared__ unsigned long long sc[4];
    __shared__ int wsum[K2L_THREADS / 32];
    __shared__ __align__(8) unsigned long long mbar[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int rep = lane % G;
    const int64_t units = (int64_t)a.B * a.chunks;
    const uint32_t bar0 = smem_u32(mbar), ring0 = smem_u32(ring);
    if (threadIdx.x == 0) {
        for (int i = 0; i < a.nst; ++i) mbar_init(bar0 + 8u * i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    int64_t g = 0;                                    // rounds consumed by this CTA (ring position)

    for (int64_t unit = blockIdx.x; unit < units; unit += gridDim.x) {
        const int u = (int)(unit % a.B);
        const int chunk = (int)(unit / a.B);
        const int64_t i0 = (int64_t)chunk * a.chunk_items;
        const int64_t i1 = min(a.N, i0 + a.chunk_items);
        const int64_t rounds = (i1 - i0 + IPR - 1) / IPR;
        __syncthreads();
        // stream this unit's code rows through the ring: the unit's round r is ring
        // position g0 + r (slot (g0 + r) % nst), g0 = rounds consumed before the unit
        const int64_t g0 = g;
        auto issue = [&](int64_t r) {
            const int slot = (int)((uint32_t)(g0 + r) % (uint32_t)a.nst);   // rounds per CTA < 2^32
            const int64_t s0 = i0 + r * IPR;
            const uint32_t bytes = (uint32_t)align_up((size_t)(min((int64_t)IPR, i1 - s0) * MP), 16);
            const uint32_t bar = bar0 + 8u * slot;
            fence_proxy_async();
            mbar_expect_tx(bar, bytes);
            bulk_g2s(ring0 + (uint32_t)slot * K2L_STAGE, a.codes + s0 * MP, bytes, bar);
        };
        if (threadIdx.x == 0)
            for (int64_t r = 0; r < min((int64_t)a.nst, rounds); ++r) issue(r);
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

        for (int64_t r = 0; r < rounds; ++r, ++g) {
            const uint32_t gq = (uint32_t)g / (uint32_t)a.nst;     // 32-bit: no 64-bit division call
            const int slot = (int)((uint32_t)g - gq * (uint32_t)a.nst);
            mbar_wait(bar0 + 8u * slot, gq & 1u);
            const unsigned char* cs = ring + (size_t)slot * K2L_STAGE;
            const int64_t r0 = i0 + r * IPR;
            uint64_t keys[J];
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const int li = j * K2L_THREADS + threadIdx.x;            // item within the round
                const int64_t item = r0 + li;
                uint32_t cw[NW];
                if constexpr (NW == 1) {
                    cw[0] = *reinterpret_cast<const uint32_t*>(cs + (size_t)li * MP);
                } else if constexpr (NW == 2) {
                    const uint2 t = *reinterpret_cast<const uint2*>(cs + (size_t)li * MP);
                    cw[0] = t.x; cw[1] = t.y;
                } else {
                    const uint4 t = *reinterpret_cast<const uint4*>(cs + (size_t)li * MP);
                    cw[0] = t.x; cw[1] = t.y; cw[2] = t.z; cw[3] = t.w;
                }
                float acc = Tl[(cw[0] & 0xFFu) * G];
#pragma unroll
                for (int k = 1; k < M; ++k) {
                    const uint32_t gk = (cw[k >> 2] >> (8 * (k & 3))) & 0xFFu;
                    acc = acc + Tl[((size_t)k * a.b + gk) * G];
                }
                const bool in = item < i1;
                const uint32_t lid = (in && a.perm) ? (uint32_t)a.perm[item] : (uint32_t)item;
                keys[j] = (in && acc >= tf) ? make_key(acc + 0.0f, a.id_base + lid) : 0ull;
            }
            // append this round's candidates (warp-aggregated slots)
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const bool c = keys[j] != 0ull && keys[j] > tau;
                const unsigned bm = __ballot_sync(FULL, c);
                if (bm) {
                    int base = 0;
                    if (lane == 0) base = atomicAdd(&count, __popc(bm));
                    base = __shfl_sync(FULL, base, 0);
                    if (base + __popc(bm) > CAP) __trap();     // invariant: shrink before overflow
                    if (c) cbuf[base + __popc(bm & lanemask_lt())] = keys[j];
                }
            }
            __syncthreads();                               // every thread is done with this slot
            if (threadIdx.x == 0 && r + a.nst < rounds) issue(r + a.nst);
            const int n_now = count;                       // same value in every thread
            // shrink after the first round (it ran without a threshold) and
            // whenever the next round could overflow the buffer
            if (((r == 0 && rounds > 1) || n_now > CAP - IPR) && n_now > a.K) {
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
static int latency_mp(int m) { return (m + 3) / 4 * 4; }
static size_t latency_smem(int m, int b, int G, int nst) {
    const int ipr = K2L_STAGE / latency_mp(m);
    return align_up((size_t)m * b * G * 4, 128) + (size_t)nst * K2L_STAGE + (size_t)2 * ipr * 8 + 256 * 4;
}

bool k2_latency_supported(const pq_index_s* idx, int B, int K) {
    return B >= 1 && B <= 4 && K <= 512 && latency_fn(idx->m, 1) != nullptr &&
           latency_smem(idx->m, idx->b, 1, 2) <= idx->smem_optin;
}

void plan_k2_latency(const pq_index_s* idx, int B, int K, K2Plan& p) {
    p.variant = 4;
    const pq_tuning& t = idx->tuning;
    // table copies (bank-conflict relief) first, then code stages in flight
    int G = 16, nst = 4;
    const size_t budget = idx->smem_optin;
    while (G > 1 && latency_smem(idx->m, idx->b, G, 2) > budget) G >>= 1;
    while (nst > 2 && latency_smem(idx->m, idx->b, G, nst) > budget) --nst;
    p.G = G; p.Ug = 1; p.W = K2L_THREADS / 32; p.J = nst; p.tm = 0;
    p.n_groups = B;
    p.smem = latency_smem(idx->m, idx->b, G, nst);
    K2LFn fn = latency_fn(idx->m, G);
    ensure_max_smem(reinterpret_cast<const void*>(fn), (int)p.smem);
    // chunks: about one wave of CTAs, >= one round each, 16-item aligned
    const int64_t N = idx->N;
    const int64_t ipr = K2L_STAGE / latency_mp(idx->m);
    const int64_t want = std::max<int64_t>(1, std::min<int64_t>(ceil_div(idx->num_sms, B), ceil_div(N, ipr)));
    p.chunks = t.chunks > 0 ? t.chunks : (int)want;
    p.chunk_items = (int64_t)align_up((size_t)ceil_div(N, p.chunks), 16);
    p.chunks = (int)ceil_div(N, p.chunk_items);
    const int64_t units = (int64_t)B * p.chunks;
    p.grid = (int)std::min<int64_t>(units, t.ctas > 0 ? t.ctas : (int64_t)idx->num_sms);
    p.cap = 0;
    p.lanebuf_bytes = 0; p.mscr_bytes = 0; p.st_bytes = 0;
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
    a.nst = p.J;
    K2LFn fn = latency_fn(idx->m, p.G);
    fn<<<p.grid, K2L_THREADS, p.smem, st>>>(a);
    count_launch();
    check_launch("k2_latency");
}

}  // namespace pq
