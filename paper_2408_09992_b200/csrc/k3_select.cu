// K3 — exact segmented top-K on 64-bit ranking keys (TopK of Alg. 1).
//
// One block selects the K largest keys of one segment of <= K3_SEG entries
// that it stages in shared memory (8-bit MSD radix select: 8 histogram passes
// over shared memory, then a compaction of the keys above the K-th).  The
// survivors are either written as an unsorted key list (an intermediate
// level) or bitonic-sorted and decoded into ids/scores (the final level).
// Keys are unique (score bits + id), so the selected set — and hence the
// output — is unique: any segmentation / level structure gives the same bits.
#include "select_dev.cuh"
#include "ptx_dev.cuh"

namespace pq {

constexpr int K3_THREADS = 512;
static_assert(K3_SEG >= 2 * PQTOPK_MAX_K, "each merge level must at least halve the candidate list");

struct SrcKeys {        // keys[u][e], row length L
    const uint64_t* keys;
    int64_t L;
    __device__ __forceinline__ uint64_t get(int u, int64_t e) const { return keys[(int64_t)u * L + e]; }
};
struct SrcKeysCnt {     // keys[u][e], e = p*K + j: lists of K keys, lcnt[u][p] of them written
    const uint64_t* keys;
    int64_t L;
    const int32_t* lcnt;
    int K, P;
    __device__ __forceinline__ uint64_t get(int u, int64_t e) const {
        const int p = (int)((uint32_t)e / (uint32_t)K), j = (int)(e - (int64_t)p * K);   // e < P * K < 2^32
        return j < __ldg(&lcnt[(int64_t)u * P + p]) ? keys[(int64_t)u * L + e] : 0ull;
    }
};
struct SrcPairs {       // (ids, scores)[p][u][j] at p*pstride + u*K + j, e = p*K + j
    const int32_t* ids;
    const float* sc;
    int64_t pstride;    // elements between consecutive lists (B*K plain, 2*B*K packed)
    int K;
    __device__ __forceinline__ uint64_t get(int u, int64_t e) const {
        int p = (int)((uint32_t)e / (uint32_t)K), j = (int)(e - (int64_t)p * K);   // e < P * K < 2^32
        int64_t o = (int64_t)p * pstride + (int64_t)u * K + j;
        int32_t id = ids[o];
        if (id < 0) return 0ull;
        return make_key(sc[o] + 0.0f, (uint32_t)id);     // + 0.0f: -0 -> +0 (R2)
    }
};
struct SrcRows {        // score row R[u][e], global id = id0 + e
    const float* R;
    int64_t ld;
    uint32_t id0;
    __device__ __forceinline__ uint64_t get(int u, int64_t e) const {
        return make_key(R[(int64_t)u * ld + e] + 0.0f, id0 + (uint32_t)e);
    }
};

// grid (B, n_sub).  Segment s of user u = entries [s*SEG, min(L, (s+1)*SEG)).
// Final mode (out_ids != null, n_sub must be 1): sorted ids/scores [B][K].
// Level mode: unsorted keys at out_keys[(u*out_lists + list_off + s)*K + j].
template <class Src>
__global__ void __launch_bounds__(K3_THREADS)
k3_select(Src src, int64_t L, int K, int Kp, uint64_t* __restrict__ out_keys,
          int64_t out_lists, int64_t list_off, int32_t* __restrict__ out_ids,
          float* __restrict__ out_sc) {
    extern __shared__ uint64_t smk[];
    pdl_wait();                                   // the keys come from the predecessor (PDL launch)
    pdl_trigger();
    const int u = blockIdx.x;
    const int s = blockIdx.y;
    const int64_t e0 = (int64_t)s * K3_SEG;
    const int n = (int)(L - e0 < (int64_t)K3_SEG ? L - e0 : (int64_t)K3_SEG);
    uint64_t* keys = smk;                         // [n]
    uint64_t* sel = smk + K3_SEG;                 // [Kp]  (Kp = pow2ceil(min(K, SEG)))
    uint32_t* hist = reinterpret_cast<uint32_t*>(sel + Kp);   // [256]
    uint32_t* sh = hist + 256;                    // [4]
    const int tid = threadIdx.x;

    for (int i = tid; i < n; i += blockDim.x) keys[i] = src.get(u, e0 + i);
    if (n <= (int)blockDim.x) {
        // very short lists: thread i ranks key i against all (keys are unique; the
        // empty key 0 ranks last) and writes it straight to its sorted position
        __syncthreads();
        const uint64_t mine = tid < n ? keys[tid] : 0ull;
        // keys are unique for valid inputs; the index tie-break only keeps the
        // output slots distinct (memory-safe, every slot written) if a caller
        // passes a repeated (id, score) pair, which the contract forbids
        const int rk = tid < n ? rank_in_smem(keys, n, tid) : n;
        const int nz = __syncthreads_count(mine != 0ull);
        if (mine != 0ull && rk < K) {
            if (out_ids) {
                out_ids[(int64_t)u * K + rk] = key_id(mine);
                out_sc[(int64_t)u * K + rk] = key_score(mine);
            } else {
                out_keys[((int64_t)u * out_lists + list_off + s) * K + rk] = mine;
            }
        }
        for (int j = nz + tid; j < K; j += blockDim.x) {
            if (out_ids) {
                out_ids[(int64_t)u * K + j] = -1;
                out_sc[(int64_t)u * K + j] = -INFINITY;
            } else {
                out_keys[((int64_t)u * out_lists + list_off + s) * K + j] = 0ull;
            }
        }
        return;
    }
    if (n <= 1024) {
        // short lists (small batches, the B x P x K merges): sort them whole
        const int P = pow2_ceil(n > 0 ? n : 1);
        for (int i = n + tid; i < P; i += blockDim.x) keys[i] = 0ull;
        __syncthreads();
        block_bitonic_desc(keys, P);
        if (out_ids) {
            for (int j = tid; j < K; j += blockDim.x) {
                const uint64_t v = j < P ? keys[j] : 0ull;
                out_ids[(int64_t)u * K + j] = v ? key_id(v) : -1;
                out_sc[(int64_t)u * K + j] = v ? key_score(v) : -INFINITY;
            }
        } else {
            uint64_t* o = out_keys + ((int64_t)u * out_lists + list_off + s) * K;
            for (int j = tid; j < K; j += blockDim.x) o[j] = j < P ? keys[j] : 0ull;
        }
        return;
    }
    for (int i = tid; i < Kp; i += blockDim.x) sel[i] = 0ull;
    if (tid == 0) sh[2] = 0;
    __syncthreads();

    // the K-th largest key: MSD radix select with an early exit once the digit
    // bin holding it contains exactly the keys still to take (select_dev.cuh)
    __shared__ unsigned long long sc3[4];
    const uint64_t kth = n > K ? block_kth(keys, n, (uint32_t)K, hist, sc3) : 0ull;
    // keep keys > kth, plus kth itself when it is a real key (unique); the empty
    // key 0 is never collected (padding is 0 anyway)
    for (int i = tid; i < n; i += blockDim.x) {
        uint64_t v = keys[i];
        if (v != 0ull && v >= kth) {
            uint32_t pos = atomicAdd(&sh[2], 1u);
            if (pos < (uint32_t)Kp) sel[pos] = v;    // > K only with repeated input keys (caller error)
        }
    }
    __syncthreads();
    if (out_ids) {
        block_bitonic_desc(sel, Kp);
        for (int j = tid; j < K; j += blockDim.x) {
            uint64_t v = j < Kp ? sel[j] : 0ull;
            out_ids[(int64_t)u * K + j] = v ? key_id(v) : -1;
            out_sc[(int64_t)u * K + j] = v ? key_score(v) : -INFINITY;
        }
    } else {
        uint64_t* o = out_keys + ((int64_t)u * out_lists + list_off + s) * K;
        for (int j = tid; j < K; j += blockDim.x) o[j] = j < Kp ? sel[j] : 0ull;
    }
}

static size_t k3_smem(int K) {
    int Kp = pow2_ceil(std::min(K, K3_SEG));
    return (size_t)K3_SEG * 8 + (size_t)Kp * 8 + 256 * 4 + 16;
}

template <class Src>
static void launch_k3(Src src, int64_t L, int B, int K, uint64_t* out_keys, int64_t out_lists,
                      int64_t list_off, int32_t* ids, float* sc, cudaStream_t st) {
    size_t smem = k3_smem(K);
    ensure_max_smem(reinterpret_cast<const void*>(k3_select<Src>), (int)(K3_SEG * 8 + PQTOPK_MAX_K * 8 + 256 * 4 + 16));
    int n_sub = (int)ceil_div(L, K3_SEG);
    dim3 grid((unsigned)B, (unsigned)n_sub);
    int Kp = pow2_ceil(std::min(K, K3_SEG));
    launch_pdl(k3_select<Src>, grid, dim3(K3_THREADS), smem, st, src, L, K, Kp, out_keys, out_lists, list_off,
               ids, sc);
    count_launch();
    check_launch("k3_select");
}

size_t k3_reduce_scratch_bytes(int64_t L, int B, int K) {
    if (L <= K3_SEG) return 0;
    int64_t n_sub = ceil_div(L, K3_SEG);
    return 2 * align_up((size_t)B * n_sub * K * 8, 256);
}

void k3_keys_to_topk(const uint64_t* keys, int64_t L, int B, int K, void* scratch,
                     int32_t* ids, float* scores, cudaStream_t st, const int32_t* lcnt) {
    if (B <= 0 || K <= 0) return;
    const uint64_t* cur = keys;
    int64_t curL = L;
    size_t half = L > K3_SEG ? align_up((size_t)B * ceil_div(L, K3_SEG) * K * 8, 256) : 0;
    uint64_t* bufs[2] = {reinterpret_cast<uint64_t*>(scratch),
                         reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(scratch) + half)};
    int pp = 0;
    if (lcnt) {                                        // first level reads the counted lists
        const SrcKeysCnt src{keys, L, lcnt, K, (int)(L / K)};
        if (L <= K3_SEG) {
            launch_k3(src, L, B, K, nullptr, 0, 0, ids, scores, st);
            return;
        }
        const int64_t n_sub = ceil_div(L, K3_SEG);
        launch_k3(src, L, B, K, bufs[pp], n_sub, 0, nullptr, nullptr, st);
        cur = bufs[pp];
        curL = n_sub * K;
        pp ^= 1;
    }
    while (curL > K3_SEG) {
        int64_t n_sub = ceil_div(curL, K3_SEG);
        uint64_t* out = bufs[pp];
        launch_k3(SrcKeys{cur, curL}, curL, B, K, out, n_sub, 0, nullptr, nullptr, st);
        cur = out;
        curL = n_sub * K;
        pp ^= 1;
    }
    launch_k3(SrcKeys{cur, curL}, curL, B, K, nullptr, 0, 0, ids, scores, st);
}

size_t k3_pairs_scratch_bytes(int P, int B, int K) {
    int64_t L = (int64_t)P * K;
    if (L <= K3_SEG) return 0;
    int64_t n_sub = ceil_div(L, K3_SEG);
    size_t first = align_up((size_t)B * n_sub * K * 8, 256);
    return first + k3_reduce_scratch_bytes(n_sub * K, B, K);
}

void k3_pairs_to_topk(const int32_t* ids_in, const float* sc_in, int64_t pstride, int P, int B,
                      int K, void* scratch, int32_t* ids, float* scores, cudaStream_t st) {
    if (B <= 0 || K <= 0) return;
    int64_t L = (int64_t)P * K;
    SrcPairs src{ids_in, sc_in, pstride, K};
    if (L <= K3_SEG) {
        launch_k3(src, L, B, K, nullptr, 0, 0, ids, scores, st);
        return;
    }
    int64_t n_sub = ceil_div(L, K3_SEG);
    uint64_t* lvl = reinterpret_cast<uint64_t*>(scratch);
    size_t first = align_up((size_t)B * n_sub * K * 8, 256);
    launch_k3(src, L, B, K, lvl, n_sub, 0, nullptr, nullptr, st);
    k3_keys_to_topk(lvl, n_sub * K, B, K, reinterpret_cast<char*>(scratch) + first, ids, scores, st);
}

int k3_rows_lists(int64_t n) { return (int)ceil_div(n, K3_SEG); }

void k3_rows_to_keys(const float* R, int64_t ld, int64_t n, int B, int K, uint32_t id0,
                     uint64_t* out, int64_t out_lists_per_user, int64_t list_off,
                     cudaStream_t st) {
    if (B <= 0 || K <= 0 || n <= 0) return;
    launch_k3(SrcRows{R, ld, id0}, n, B, K, out, out_lists_per_user, list_off, nullptr, nullptr, st);
}

}  // namespace pq
