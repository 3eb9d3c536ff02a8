// K0b — the K2 v3 catalogue layout built on the GPU (pq_create; one-time,
// outside the timed region).  Input: the validated item-order code rows of K0
// (d_codes [N][mp]; Eq. 1).  Output: the phase-blocked stored codes
// d_codes3, the row -> item map d_perm3 and the stored -> original sub-id map
// d_cmap3 that k2_tiled.cu streams.
//
// R = 32 (item order): row r = item r, stored code = sub-id (or, for the exact
// first-pair tables of b = 16, g0 + 16 g1 then splits 2..).
// R = 16 (colour pairing, see k2_tiled.cu): every split's sub-ids are
// 2-coloured (balanced by item frequency; stored parity = colour); an item's
// signature is its colour bit at the first min(m, 20) splits; items of
// complementary signatures are paired (rows 2p, 2p+1), so the two 64-byte
// table rows a quarter-warp reads lie in opposite bank halves.
//   1. k0_hist      per-split sub-id histograms               (GPU)
//   2. colouring    greedy, b sub-ids per split              (host, m x 256)
//   3. k0_sig       signatures                                (GPU)
//   4. k0_classkey  key = 2 * class + side with class c = min(s, ~s), side = s > ~s;
//                   a stable radix sort of the item ids by key (CUB, one-time
//                   build step) puts each (class, side) group in id order (GPU)
//   5. pair offsets exclusive scans of the group sizes and of min(n0, n1) per
//                   class                                      (host, 2^19 classes)
//   6. k0_emit      the j-th items of a class's two sides -> rows 2p, 2p+1;
//                   the rest -> leftover list, in sorted order (GPU)
//   7. leftovers    sorted by (signature, id); pairs whose signatures differ
//                   from a complement in one split, then the rest in order
//                   (host; ~2% of the items at C4)
//   8. k0_v3_codes  stored codes -> [tile][phase][slot pair][row][2][pss] (GPU)
//   9. k0_check     every item on exactly one row              (GPU)
// The layout is deterministic (and equal to the round-1 host builder's for the
// exact pairs); the scores and the top-K never depend on it (R3/R4).
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstring>
#include <numeric>
#include <vector>

#include "pq_internal.cuh"

namespace pq {

__global__ void k0_hist(const uint8_t* __restrict__ codes, int64_t N, int mp, int m,
                        unsigned int* __restrict__ hist) {
    extern __shared__ unsigned int sh[];              // [m][256]
    for (int x = threadIdx.x; x < m * 256; x += blockDim.x) sh[x] = 0u;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t* row = reinterpret_cast<const uint32_t*>(codes + i * mp);
        for (int w = 0; w < mp / 4; ++w) {
            const uint32_t v = row[w];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int k = 4 * w + q;
                if (k < m) atomicAdd(&sh[k * 256 + ((v >> (8 * q)) & 0xFFu)], 1u);
            }
        }
    }
    __syncthreads();
    for (int x = threadIdx.x; x < m * 256; x += blockDim.x)
        if (sh[x]) atomicAdd(&hist[x], sh[x]);
}

__global__ void k0_sig(const uint8_t* __restrict__ codes, int64_t N, int mp, int sm,
                       const uint8_t* __restrict__ color, uint32_t* __restrict__ sig) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t* row = codes + i * mp;
        uint32_t s = 0;
        for (int k = 0; k < sm; ++k) s |= (uint32_t)color[k * 256 + row[k]] << k;
        sig[i] = s;
    }
}

// sort key 2 * class + side (and the item id as the value), group sizes
__global__ void k0_classkey(const uint32_t* __restrict__ sig, int64_t N, uint32_t mask,
                            uint32_t* __restrict__ key, int32_t* __restrict__ val, unsigned int* __restrict__ cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t s = sig[i], c = s ^ mask;
        const uint32_t k = 2u * (s < c ? s : c) + (s < c ? 0u : 1u);
        key[i] = k;
        val[i] = (int32_t)i;
        atomicAdd(&cnt[k], 1u);
    }
}

// sorted position p (item val[p] of group key[p], rank p - gstart[key]): the
// first min(n0, n1) items of each side of a class are paired in order
__global__ void k0_emit(const uint32_t* __restrict__ key, const int32_t* __restrict__ val, int64_t N,
                        const unsigned int* __restrict__ cnt, const int64_t* __restrict__ gstart,
                        const int64_t* __restrict__ poff, const int64_t* __restrict__ loff,
                        int32_t* __restrict__ rowitem, int32_t* __restrict__ left) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < N; p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = key[p], cls = k >> 1, side = k & 1u;
        const uint32_t npc = min(cnt[2 * cls], cnt[2 * cls + 1]);
        const int64_t r = p - gstart[k];
        if (r < (int64_t)npc) rowitem[2 * (poff[cls] + r) + side] = val[p];
        else left[loff[k] + (r - npc)] = val[p];      // leftovers in sorted (class, side, id) order
    }
}

// colour-paired row-order codes for K6 / K7: row r = item perm[r] in stored codes
__global__ void k0_pair_rows(const uint8_t* __restrict__ codes, int mp, int m, const int32_t* __restrict__ perm,
                             int64_t rows, const uint8_t* __restrict__ stored, uint8_t* __restrict__ out) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t it = perm[r];
        for (int k = 0; k < mp; ++k)
            out[r * mp + k] = (it >= 0 && k < m) ? stored[k * 256 + codes[(int64_t)it * mp + k]] : (uint8_t)0;
    }
}

__global__ void k0_iota(int32_t* __restrict__ perm, int64_t N) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        perm[i] = (int32_t)i;
}

__global__ void k0_gather_sig(const uint32_t* __restrict__ sig, const int32_t* __restrict__ ids, int64_t n,
                              uint32_t* __restrict__ out) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        out[j] = sig[ids[j]];
}

// One thread per layout row: the row's stored codes into the phase-blocked
// buffer.  Inside a phase block slot pairs are interleaved: logical row
// rr = slot * RPS + r is stored at ((slot / 2) * RPS + r) * 2 + slot % 2
// (k2_tiled.cu, CodePair).  Padding rows (perm -1) keep zero codes.
__global__ void k0_v3_codes(const uint8_t* __restrict__ codes, int mp, int m, const int32_t* __restrict__ perm,
                            int64_t rows, const uint8_t* __restrict__ stored, int pair, int ps, int pss, int np,
                            int RPS, int64_t TR, uint8_t* __restrict__ c3) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t it = perm[r];
        if (it < 0) continue;
        const int64_t t = r / TR, rr = r - t * TR;
        const int64_t gs = rr / RPS, ri = rr - gs * RPS;
        const int64_t sr = ((gs >> 1) * RPS + ri) * 2 + (gs & 1);
        const uint8_t* ci = codes + (int64_t)it * mp;
        const int mv = pair ? m - 1 : m;
        for (int v = 0; v < mv; ++v) {
            uint32_t c;
            if (pair) c = v == 0 ? (uint32_t)ci[0] + 16u * ci[1] : ci[v + 1];
            else c = stored ? stored[v * 256 + ci[v]] : ci[v];
            const int ph = v / ps, kk = v - ph * ps;
            c3[((t * np + ph) * TR + sr) * pss + kk] = (uint8_t)c;
        }
    }
}

__global__ void k0_check(const int32_t* __restrict__ perm, int64_t rows, int64_t N, unsigned int* __restrict__ bits,
                         unsigned long long* __restrict__ bad) {
    unsigned int nvalid = 0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t it = perm[r];
        if (it < 0) continue;
        if (it >= N) { atomicAdd(bad, 1ull); continue; }
        const unsigned old = atomicOr(&bits[it >> 5], 1u << (it & 31));
        if (old & (1u << (it & 31))) atomicAdd(bad, 1ull);           // item on two rows
        ++nvalid;                                                     // rows holding an item
    }
    nvalid = __reduce_add_sync(0xFFFFFFFFu, nvalid);
    if ((threadIdx.x & 31) == 0 && nvalid) atomicAdd(bad + 1, (unsigned long long)nvalid);
}

namespace {
// device buffers freed on every exit path
struct DevBufs {
    std::vector<void*> p;
    template <class T> T* alloc(size_t n) {
        void* q = nullptr;
        if (cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(T)) != cudaSuccess) {
            cudaGetLastError();
            fail(PQ_ERR_OUT_OF_MEMORY, "cudaMalloc failed while building the catalogue layout");
        }
        p.push_back(q);
        return static_cast<T*>(q);
    }
    ~DevBufs() { for (void* q : p) cudaFree(q); }
};
int grid_for(int64_t n, int num_sms) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), (int64_t)num_sms * 16));
}
}  // namespace

void build_v3_layout_gpu(pq_index_s* idx, cudaStream_t st) {
    const int m = idx->m, b = idx->b, mp = idx->lay.mp;
    const int64_t N = idx->N;
    const TiledShape sh = k2_tiled_shape(m, b);
    const int R = sh.R;
    if (!R || k2_tiled_smem(sh, 16) > idx->smem_optin) return;
    if (k2_tiled_code_bytes() != 1) fail(PQ_ERR_UNSUPPORTED, "GPU layout builder: 1-byte stored codes only");
    const int sms = idx->num_sms;
    DevBufs db;
    std::vector<uint8_t> cmap((size_t)m * b);
    int32_t* d_rowitem = nullptr;                      // layout rows -> item (-1 padding), tiles * TR
    int64_t rows = 0, matched = 0, leftover = 0;
    uint8_t* d_stored = nullptr;
    const int64_t TR = k2_tiled_rows_per_tile(R);

    if (R == 32) {                                     // item order
        for (int k = 0; k < m; ++k)
            for (int g = 0; g < b; ++g) cmap[(size_t)k * b + g] = (uint8_t)g;
        rows = N;
    } else {
        // 1-2. histograms -> colouring (greedy, largest first, b/2 sub-ids per colour)
        unsigned int* d_hist = db.alloc<unsigned int>((size_t)m * 256);
        PQ_CUDA(cudaMemsetAsync(d_hist, 0, (size_t)m * 256 * 4, st));
        const int hsm = m * 256 * 4;
        ensure_max_smem(reinterpret_cast<const void*>(k0_hist), hsm);
        k0_hist<<<grid_for(N, sms), 256, hsm, st>>>(idx->d_codes, N, mp, m, d_hist);
        count_launch();
        check_launch("k0_hist");
        std::vector<unsigned int> hist((size_t)m * 256);
        PQ_CUDA(cudaMemcpyAsync(hist.data(), d_hist, hist.size() * 4, cudaMemcpyDeviceToHost, st));
        PQ_CUDA(cudaStreamSynchronize(st));
        std::vector<uint8_t> color((size_t)m * 256, 0), stored((size_t)m * 256, 0);
        for (int k = 0; k < m; ++k) {
            std::vector<int> order(b);
            std::iota(order.begin(), order.end(), 0);
            std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
                return hist[(size_t)k * 256 + x] > hist[(size_t)k * 256 + y];
            });
            const int cap0 = (b + 1) / 2, cap1 = b / 2;
            int n0 = 0, n1 = 0;
            int64_t m0 = 0, m1 = 0;
            for (int g : order) {
                const int64_t w = hist[(size_t)k * 256 + g];
                const int c = (n1 >= cap1) ? 0 : (n0 >= cap0) ? 1 : (m0 <= m1 ? 0 : 1);
                color[(size_t)k * 256 + g] = (uint8_t)c;
                const int pos = c == 0 ? 2 * n0++ : 2 * n1++ + 1;
                stored[(size_t)k * 256 + g] = (uint8_t)pos;
                cmap[(size_t)k * b + pos] = (uint8_t)g;
                (c == 0 ? m0 : m1) += w;
            }
        }
        uint8_t* d_color = db.alloc<uint8_t>((size_t)m * 256);
        d_stored = db.alloc<uint8_t>((size_t)m * 256);
        PQ_CUDA(cudaMemcpyAsync(d_color, color.data(), color.size(), cudaMemcpyHostToDevice, st));
        PQ_CUDA(cudaMemcpyAsync(d_stored, stored.data(), stored.size(), cudaMemcpyHostToDevice, st));
        // 3-4. signatures over the first sm splits; items stably sorted by (class, side)
        const int sm = m < 20 ? m : 20;
        const uint32_t mask = (1u << sm) - 1u;
        const uint32_t ncls = 1u << (sm - 1);          // min(s, ~s) has its top bit clear
        const uint32_t nkey = 2 * ncls;
        uint32_t* d_sig = db.alloc<uint32_t>((size_t)N);
        uint32_t* d_key = db.alloc<uint32_t>((size_t)N);
        uint32_t* d_key2 = db.alloc<uint32_t>((size_t)N);
        int32_t* d_val = db.alloc<int32_t>((size_t)N);
        int32_t* d_val2 = db.alloc<int32_t>((size_t)N);
        unsigned int* d_cnt = db.alloc<unsigned int>(nkey);
        PQ_CUDA(cudaMemsetAsync(d_cnt, 0, (size_t)nkey * 4, st));
        k0_sig<<<grid_for(N, sms), 256, 0, st>>>(idx->d_codes, N, mp, sm, d_color, d_sig);
        k0_classkey<<<grid_for(N, sms), 256, 0, st>>>(d_sig, N, mask, d_key, d_val, d_cnt);
        count_launch(2);
        check_launch("k0_sig / k0_classkey");
        {
            size_t tmp_bytes = 0;
            PQ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, d_key, d_key2, d_val, d_val2, (int)N, 0, sm,
                                                    st));
            void* d_tmp = db.alloc<unsigned char>(tmp_bytes);
            PQ_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp, tmp_bytes, d_key, d_key2, d_val, d_val2, (int)N, 0, sm,
                                                    st));
            count_launch();
        }
        // 5. group starts, pair offsets per class, leftover offsets per group
        std::vector<unsigned int> cnt(nkey);
        PQ_CUDA(cudaMemcpyAsync(cnt.data(), d_cnt, cnt.size() * 4, cudaMemcpyDeviceToHost, st));
        PQ_CUDA(cudaStreamSynchronize(st));
        std::vector<int64_t> gstart(nkey), poff(ncls), loff(nkey);
        int64_t P = 0, G0 = 0, L0 = 0;
        for (uint32_t c = 0; c < ncls; ++c) {
            const int64_t n0 = cnt[2 * c], n1 = cnt[2 * c + 1], np = std::min(n0, n1);
            gstart[2 * c] = G0; gstart[2 * c + 1] = G0 + n0; G0 += n0 + n1;
            poff[c] = P; P += np;
            loff[2 * c] = L0; loff[2 * c + 1] = L0 + (n0 - np); L0 += (n0 - np) + (n1 - np);
        }
        matched = P;
        leftover = N - 2 * P;
        int64_t* d_gstart = db.alloc<int64_t>(nkey);
        int64_t* d_poff = db.alloc<int64_t>(ncls);
        int64_t* d_loff = db.alloc<int64_t>(nkey);
        PQ_CUDA(cudaMemcpyAsync(d_gstart, gstart.data(), gstart.size() * 8, cudaMemcpyHostToDevice, st));
        PQ_CUDA(cudaMemcpyAsync(d_poff, poff.data(), poff.size() * 8, cudaMemcpyHostToDevice, st));
        PQ_CUDA(cudaMemcpyAsync(d_loff, loff.data(), loff.size() * 8, cudaMemcpyHostToDevice, st));
        // 6. matched items -> rows 0 .. 2P-1, the rest -> leftover list
        const int64_t max_rows = align_up((size_t)(2 * P + leftover + 1), (size_t)TR);
        d_rowitem = db.alloc<int32_t>((size_t)max_rows);
        PQ_CUDA(cudaMemsetAsync(d_rowitem, 0xFF, (size_t)max_rows * 4, st));
        int32_t* d_left = db.alloc<int32_t>((size_t)std::max<int64_t>(leftover, 1));
        k0_emit<<<grid_for(N, sms), 256, 0, st>>>(d_key2, d_val2, N, d_cnt, d_gstart, d_poff, d_loff, d_rowitem,
                                                  d_left);
        count_launch();
        check_launch("k0_emit");
        // 7. leftovers on the host, in the round-1 builder's order (signature
        // classes ascending; a class with one side present at that side's
        // signature; inside a class the smaller signature's items first, ids
        // ascending): pairs whose signatures differ from a complement in one
        // split (conflict on that split only), then the rest pairwise
        std::vector<int32_t> left((size_t)leftover);
        std::vector<uint32_t> lsig((size_t)leftover);
        if (leftover > 0) {
            uint32_t* d_lsig = db.alloc<uint32_t>((size_t)leftover);
            k0_gather_sig<<<grid_for(leftover, sms), 256, 0, st>>>(d_sig, d_left, leftover, d_lsig);
            count_launch();
            check_launch("k0_gather_sig");
            PQ_CUDA(cudaMemcpyAsync(left.data(), d_left, (size_t)leftover * 4, cudaMemcpyDeviceToHost, st));
            PQ_CUDA(cudaMemcpyAsync(lsig.data(), d_lsig, (size_t)leftover * 4, cudaMemcpyDeviceToHost, st));
            PQ_CUDA(cudaStreamSynchronize(st));
        }
        std::vector<int64_t> ord((size_t)leftover);
        std::iota(ord.begin(), ord.end(), (int64_t)0);
        auto visit = [&](int64_t x) -> uint32_t {       // (the list arrives in (class, side, id) order)
            const uint32_t sg = lsig[x], cls = std::min(sg, sg ^ mask);
            return (cnt[2 * cls] > 0 && cnt[2 * cls + 1] > 0) ? cls : sg;
        };
        std::stable_sort(ord.begin(), ord.end(), [&](int64_t x, int64_t y) { return visit(x) < visit(y); });
        std::vector<int32_t> lrows;                   // rows 2P .. in pairs
        lrows.reserve((size_t)leftover + 1);
        {
            const size_t nb = (size_t)1 << sm;
            std::vector<int64_t> head(nb, -1), nxt((size_t)leftover, -1);
            for (size_t t = ord.size(); t-- > 0;) {
                const uint32_t sg = lsig[ord[t]];
                nxt[t] = head[sg];
                head[sg] = (int64_t)t;
            }
            std::vector<uint8_t> used((size_t)leftover, 0);
            std::vector<int32_t> rest;
            for (size_t t = 0; t < ord.size(); ++t) {
                if (used[t]) continue;
                const uint32_t sg = lsig[ord[t]];
                int64_t mate = -1;
                for (int j = 0; j < sm && mate < 0; ++j) {
                    const uint32_t c = (sg ^ mask) ^ (1u << j);
                    int64_t& h = head[c];
                    while (h >= 0 && used[h]) h = nxt[h];
                    if (h >= 0 && (size_t)h != t) mate = h;
                }
                used[t] = 1;
                if (mate >= 0) {
                    used[mate] = 1;
                    lrows.push_back(left[ord[t]]);
                    lrows.push_back(left[ord[mate]]);
                } else {
                    rest.push_back(left[ord[t]]);
                }
            }
            for (int32_t it : rest) lrows.push_back(it);
            if (lrows.size() % 2) lrows.push_back(-1);
        }
        if (!lrows.empty())
            PQ_CUDA(cudaMemcpyAsync(d_rowitem + 2 * P, lrows.data(), lrows.size() * 4, cudaMemcpyHostToDevice, st));
        rows = 2 * P + (int64_t)lrows.size();
        PQ_CUDA(cudaStreamSynchronize(st));            // lrows is a host temporary
    }
    // 8. phase-blocked stored codes + the row map
    const int64_t tiles = ceil_div(rows, TR);
    const int64_t rows_pad = tiles * TR;
    const int mv = sh.m_v, ps = sh.ps, pss = sh.pss, np = mv / ps;
    const size_t c3b = (size_t)rows_pad * np * pss;
    const size_t cbytes = c3b + V3_CODE_PAD;
    PQ_CUDA(cudaMalloc(&idx->d_codes3, cbytes));
    idx->v3_code_bytes = (int64_t)cbytes;
    PQ_CUDA(cudaMalloc(&idx->d_perm3, (size_t)rows_pad * 4));
    PQ_CUDA(cudaMalloc(&idx->d_cmap3, (size_t)m * b));
    PQ_CUDA(cudaMemsetAsync(idx->d_codes3, 0, cbytes, st));
    if (R == 32) {
        PQ_CUDA(cudaMemsetAsync(idx->d_perm3, 0xFF, (size_t)rows_pad * 4, st));
        k0_iota<<<grid_for(N, sms), 256, 0, st>>>(idx->d_perm3, N);
        count_launch();
        check_launch("k0_iota");
    } else {
        PQ_CUDA(cudaMemcpyAsync(idx->d_perm3, d_rowitem, (size_t)rows * 4, cudaMemcpyDeviceToDevice, st));
        if (rows_pad > rows)
            PQ_CUDA(cudaMemsetAsync(idx->d_perm3 + rows, 0xFF, (size_t)(rows_pad - rows) * 4, st));
    }
    PQ_CUDA(cudaMemcpyAsync(idx->d_cmap3, cmap.data(), cmap.size(), cudaMemcpyHostToDevice, st));
    const int RPS = 32 / (R / 4);
    k0_v3_codes<<<grid_for(rows_pad, sms), 256, 0, st>>>(idx->d_codes, mp, m, idx->d_perm3, rows_pad, d_stored,
                                                         sh.pair, ps, pss, np, RPS, TR, static_cast<uint8_t*>(idx->d_codes3));
    count_launch();
    check_launch("k0_v3_codes");
    // 8b. colour-paired row-order codes for the small-batch kernels (m they support)
    if (R == 16 && (m == 4 || m == 8 || m == 16) && d_stored) {
        int32_t last = 0;
        PQ_CUDA(cudaMemcpyAsync(&last, idx->d_perm3 + rows - 1, 4, cudaMemcpyDeviceToHost, st));
        PQ_CUDA(cudaStreamSynchronize(st));
        idx->p_rows = last < 0 ? rows - 1 : rows;     // only the last leftover slot can be empty
        PQ_CUDA(cudaMalloc(&idx->d_codes_p, (size_t)rows_pad * mp + 64));
        PQ_CUDA(cudaMemsetAsync(idx->d_codes_p, 0, (size_t)rows_pad * mp + 64, st));
        k0_pair_rows<<<grid_for(rows_pad, sms), 256, 0, st>>>(idx->d_codes, mp, m, idx->d_perm3, rows_pad, d_stored,
                                                              idx->d_codes_p);
        count_launch();
        check_launch("k0_pair_rows");
    }
    // 9. every item exactly once
    {
        unsigned int* d_bits = db.alloc<unsigned int>((size_t)ceil_div(N, 32));
        unsigned long long* d_bad = db.alloc<unsigned long long>(2);
        PQ_CUDA(cudaMemsetAsync(d_bits, 0, (size_t)ceil_div(N, 32) * 4, st));
        PQ_CUDA(cudaMemsetAsync(d_bad, 0, 16, st));
        k0_check<<<grid_for(rows_pad, sms), 256, 0, st>>>(idx->d_perm3, rows_pad, N, d_bits, d_bad);
        count_launch();
        check_launch("k0_check");
        unsigned long long h[2] = {0, 0};
        PQ_CUDA(cudaMemcpyAsync(h, d_bad, 16, cudaMemcpyDeviceToHost, st));
        PQ_CUDA(cudaStreamSynchronize(st));
        if (h[0] != 0 || (int64_t)h[1] != N) fail(PQ_ERR_CUDA, "internal error: catalogue layout is not a permutation");
    }
    idx->v3_ok = 1;
    idx->v3_R = R;
    idx->v3_tiles = tiles;
    idx->v3_matched = matched;
    idx->v3_leftover = leftover;
}

}  // namespace pq
