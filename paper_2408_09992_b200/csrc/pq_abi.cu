// pq_abi.cu — the extern "C" boundary of libpqtopk.so (include/pqtopk.h).
// Argument validation, index lifetime, workspace planning and dispatch to the
// kernels K0..K4.  No exception crosses the ABI.
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "pq_internal.cuh"
#include <mutex>

namespace pq {

static thread_local std::string t_err;
std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { t_err = msg; }
void clear_error() { t_err.clear(); }
[[noreturn]] void fail(pq_status st, const std::string& msg) { throw Error{st, msg}; }
void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(PQ_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
void check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(PQ_ERR_CUDA, std::string("launch ") + what + ": " + cudaGetErrorString(e));
}

void ensure_max_smem(const void* fn, int bytes) {
    struct Ent { int dev; const void* fn; int bytes; };
    static std::mutex mu;
    static std::vector<Ent> done;
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    {
        std::lock_guard<std::mutex> lk(mu);
        for (const Ent& e : done)
            if (e.dev == dev && e.fn == fn && e.bytes >= bytes) return;
    }
    check_cuda(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
               "cudaFuncSetAttribute(MaxDynamicSharedMemorySize)");
    std::lock_guard<std::mutex> lk(mu);
    for (Ent& e : done)
        if (e.dev == dev && e.fn == fn) { if (bytes > e.bytes) e.bytes = bytes; return; }
    done.push_back(Ent{dev, fn, bytes});
}

static bool is_device_ptr(const void* p) {
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) { cudaGetLastError(); return false; }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}


static void need(bool c, const char* msg) {
    if (!c) fail(PQ_ERR_INVALID_ARG, msg);
}

static int round_up4(int m) { return (m + 3) / 4 * 4; }

// Workspace carving helper.
struct Carve {
    char* base;
    size_t off = 0;
    explicit Carve(void* p) : base(static_cast<char*>(p)) {}
    template <class T> T* take(size_t bytes) {
        T* r = reinterpret_cast<T*>(base ? base + off : nullptr);
        off += align_up(bytes, 256);
        return r;
    }
};

struct TopkWs {
    K2Plan plan;
    size_t lanebuf, cand, k3, total;
};
static TopkWs topk_ws(const pq_index_s* idx, int B, int K) {
    TopkWs w{};
    w.plan = plan_k2(idx, B, K);
    w.lanebuf = align_up(w.plan.lanebuf_bytes, 256) +
                align_up(w.plan.mscr_bytes, 256) + align_up(w.plan.st_bytes, 256);
    w.cand = align_up(w.plan.cand_bytes, 256);
    w.k3 = align_up(k3_reduce_scratch_bytes((int64_t)w.plan.chunks * K, B, K), 256);
    w.total = w.lanebuf + w.cand + w.k3;
    return w;
}

static void run_score_topk(pq_index_s* idx, const float* S, int B, int K, void* ws, size_t ws_bytes,
                           int32_t* ids, float* scores, cudaStream_t st) {
    TopkWs w = topk_ws(idx, B, K);
    if (!ws || ws_bytes < w.total)
        fail(PQ_ERR_WORKSPACE, "workspace too small: need " + std::to_string(w.total) + " bytes");
    Carve c(ws);
    uint64_t* lanebuf = c.take<uint64_t>(w.lanebuf);     // lane buffers
    uint64_t* cand = c.take<uint64_t>(w.plan.cand_bytes);
    void* k3s = c.take<char>(k3_reduce_scratch_bytes((int64_t)w.plan.chunks * K, B, K));
    char* lb = reinterpret_cast<char*>(lanebuf);
    uint64_t* mscr = reinterpret_cast<uint64_t*>(lb + align_up(w.plan.lanebuf_bytes, 256));
    float* St = reinterpret_cast<float*>(lb + align_up(w.plan.lanebuf_bytes, 256) +
                                         align_up(w.plan.mscr_bytes, 256));
    if (w.plan.variant == 3) launch_k2_tiled_prep(idx, w.plan, S, B, St, st);   // S -> tiled tables
    pq_index_s::EvTriple ev{};
    if (idx->timing) {
        PQ_CUDA(cudaEventCreate(&ev.a)); PQ_CUDA(cudaEventCreate(&ev.b)); PQ_CUDA(cudaEventCreate(&ev.c));
        PQ_CUDA(cudaEventRecord(ev.a, st));
    }
    if (w.plan.variant == 3) launch_k2_tiled(idx, w.plan, B, K, lanebuf, mscr, St, cand, st);
    else if (w.plan.variant == 4) launch_k2_latency(idx, w.plan, S, B, K, cand, st);
    else launch_k2(idx, w.plan, S, B, K, lanebuf, cand, st);
    if (idx->timing) PQ_CUDA(cudaEventRecord(ev.b, st));
    k3_keys_to_topk(cand, (int64_t)w.plan.chunks * K, B, K, k3s, ids, scores, st,
                    w.plan.variant == 3 ? k2_tiled_list_counts(idx, w.plan, St) : nullptr);
    if (idx->timing) {
        PQ_CUDA(cudaEventRecord(ev.c, st));
        std::lock_guard<std::mutex> lk(*idx->ev_mu);
        idx->events->push_back(ev);
    }
}

// A temporary item-order catalogue over the subset V (k5_subset.cu): row r is
// item V[r]; only the generic (v1) and small-batch (v4) kernels read it.
static pq_index_s subset_index(const pq_index_s* idx, int64_t nV, uint8_t* codesV, const int32_t* V) {
    pq_index_s t{};
    t.N = nV; t.m = idx->m; t.b = idx->b; t.id_base = idx->id_base;
    t.device = idx->device; t.num_sms = idx->num_sms; t.smem_optin = idx->smem_optin;
    t.lay.mp = idx->lay.mp;
    t.lay.paired = 1;                                  // rows -> items through d_perm (= V)
    t.d_codes = codesV;
    t.d_perm = const_cast<int32_t*>(V);
    t.n_rows = nV;
    t.tuning = idx->tuning;
    if (t.tuning.variant == 3) t.tuning.variant = 0;
    return t;
}
static size_t subset_codes_bytes(const pq_index_s* idx, int64_t nV) {
    return align_up((size_t)nV * idx->lay.mp + 64, 256) + 256;
}

static void check_topk_args(int B, int K) {
    need(B >= 0, "B must be >= 0");
    need(K >= 0, "K must be >= 0");
    if (K > PQTOPK_MAX_K) fail(PQ_ERR_UNSUPPORTED, "K exceeds PQTOPK_MAX_K (4096)");
}

static int64_t dense_chunk(int64_t N, int B) {
    const int64_t budget = (int64_t)1 << 30;             // bytes of fp32 scores per chunk
    int64_t nc = budget / ((int64_t)std::max(B, 1) * 4);
    nc = std::max<int64_t>(nc / K3_SEG * K3_SEG, K3_SEG);
    return std::min(N, nc);
}
static int64_t dense_lists(int64_t N, int64_t nc) {
    int64_t lists = 0;
    for (int64_t c0 = 0; c0 < N; c0 += nc) lists += k3_rows_lists(std::min(nc, N - c0));
    return lists;
}

// Host-side state of one pq_create's layout builder: the codes on the host
// (copied once if the caller passed device memory) and the colour pairing.
struct CreateCtx {
    std::vector<uint8_t> hbuf;
    const uint8_t* hc = nullptr;
    bool have_pair = false;
    PairLayout pair0;                                  // pairing with every split in shared memory
};
static const uint8_t* host_codes(CreateCtx& cx, const pq_index_s* idx, const uint8_t* codes_in,
                                 const uint8_t* dev_src, cudaStream_t st) {
    if (!cx.hc) {
        if (is_device_ptr(codes_in)) {
            cx.hbuf.resize((size_t)idx->N * idx->m);
            PQ_CUDA(cudaMemcpyAsync(cx.hbuf.data(), dev_src, cx.hbuf.size(), cudaMemcpyDeviceToHost, st));
            PQ_CUDA(cudaStreamSynchronize(st));
            cx.hc = cx.hbuf.data();
        } else {
            cx.hc = codes_in;
        }
    }
    return cx.hc;
}
static const PairLayout& pairing0(CreateCtx& cx, const pq_index_s* idx, const uint8_t* codes_in,
                                  const uint8_t* dev_src, cudaStream_t st) {
    if (!cx.have_pair) {
        cx.pair0 = build_pairing(host_codes(cx, idx, codes_in, dev_src, st), idx->N, idx->m, idx->b, 0);
        cx.have_pair = true;
    }
    return cx.pair0;
}

// K2 v3 layout (k2_tiled.cu).  R = 16: the colour pairing (every split in
// shared memory); R = 32: item order; with an exact first-pair table (b = 16)
// split 0's stored code is g0 + 16 g1 and splits 2.. follow.  Rows are padded
// to whole tiles and the codes phase-blocked ([tile][phase][row][pss], pss >=
// ps stored bytes per row per phase).
static void free_index_buffers(pq_index_s* idx) {
    void* bufs[] = {idx->d_codes, idx->d_perm, idx->d_cmap, idx->d_codes3, idx->d_perm3, idx->d_cmap3,
                    idx->d_codes_p};
    for (void* p : bufs)
        if (p) cudaFree(p);
}

static void build_v3_layout(pq_index_s* idx, CreateCtx& cx, const uint8_t* codes_in, const uint8_t* dev_src,
                            cudaStream_t st) {
    const int m = idx->m, b = idx->b;
    const TiledShape sh = k2_tiled_shape(m, b);
    const int R = sh.R;
    if (!R || k2_tiled_smem(sh, 16) > idx->smem_optin) return;
    const int64_t N = idx->N;
    const uint8_t* hc = host_codes(cx, idx, codes_in, dev_src, st);
    const int mv = sh.m_v;                             // stored splits per row
    PairLayout Lio;
    const PairLayout* Lp = &Lio;
    if (R == 16) {                                     // colour pairing (m > 20: on 20 splits)
        Lp = &pairing0(cx, idx, codes_in, dev_src, st);
    } else {                                           // item order, codes * (R * 4)
        PairLayout& L = Lio;
        L.rows = N;
        L.perm.resize((size_t)N);
        L.codes16.resize((size_t)N * mv);
        L.cmap.resize((size_t)m * b);
        for (int k = 0; k < m; ++k)
            for (int g = 0; g < b; ++g) L.cmap[(size_t)k * b + g] = (uint8_t)g;
        for (int64_t i = 0; i < N; ++i) {
            L.perm[(size_t)i] = (int32_t)i;
            const uint8_t* ci = hc + i * m;
            for (int k = 0; k < mv; ++k) {
                const uint32_t c = sh.pair ? (k == 0 ? ci[0] + 16u * ci[1] : ci[k + 1]) : ci[k];
                L.codes16[(size_t)i * mv + k] = (uint16_t)(c * (uint32_t)(R * 4));
            }
        }
    }
    const PairLayout& L = *Lp;
    const int64_t TR = k2_tiled_rows_per_tile(R);
    const int64_t tiles = ceil_div(L.rows, TR);
    const int ps = sh.ps, pss = sh.pss, np = mv / ps;
    const int cb = k2_tiled_code_bytes();             // 1: sub-id byte, 2: pre-shifted row offset
    std::vector<uint8_t> c3((size_t)tiles * TR * np * pss * cb, 0);
    std::vector<int32_t> p3((size_t)tiles * TR, -1);
    // inside a phase block, slot pairs are interleaved: logical row rr = slot * RPS + r
    // is stored at ((slot / 2) * RPS + r) * 2 + slot % 2 (k2_tiled.cu, CodePair)
    const int64_t RPS = 32 / (R / 4);
    for (int64_t r = 0; r < L.rows; ++r) {
        const int64_t t = r / TR, rr = r % TR;
        const int64_t gs = rr / RPS, ri = rr % RPS;
        const int64_t sr = ((gs >> 1) * RPS + ri) * 2 + (gs & 1);
        p3[(size_t)r] = L.perm[(size_t)r];
        for (int ph = 0; ph < np; ++ph)
            for (int kk = 0; kk < ps; ++kk) {
                const uint16_t v = L.codes16[(size_t)r * mv + ph * ps + kk];    // stored code * R * 4
                const size_t at = (size_t)(((t * np + ph) * TR + sr) * pss + kk);
                if (cb == 1) c3[at] = (uint8_t)(v / (uint32_t)(R * 4));
                else reinterpret_cast<uint16_t*>(c3.data())[at] = v;
            }
    }
    const size_t cbytes = c3.size() + V3_CODE_PAD;
    PQ_CUDA(cudaMalloc(&idx->d_codes3, cbytes));
    idx->v3_code_bytes = (int64_t)cbytes;
    PQ_CUDA(cudaMalloc(&idx->d_perm3, p3.size() * 4));
    PQ_CUDA(cudaMalloc(&idx->d_cmap3, (size_t)m * b));
    PQ_CUDA(cudaMemsetAsync(idx->d_codes3, 0, cbytes, st));
    PQ_CUDA(cudaMemcpyAsync(idx->d_codes3, c3.data(), c3.size(), cudaMemcpyHostToDevice, st));
    PQ_CUDA(cudaMemcpyAsync(idx->d_perm3, p3.data(), p3.size() * 4, cudaMemcpyHostToDevice, st));
    PQ_CUDA(cudaMemcpyAsync(idx->d_cmap3, L.cmap.data(), (size_t)m * b, cudaMemcpyHostToDevice, st));
    PQ_CUDA(cudaStreamSynchronize(st));
    idx->v3_ok = 1;
    idx->v3_R = R;
    idx->v3_tiles = tiles;
    idx->v3_matched = L.matched_pairs;
    idx->v3_leftover = L.leftover;
}

static int recjpq_users(int64_t N, int B) {
    int64_t bc = ((int64_t)1 << 30) / (N * 4);
    return (int)std::max<int64_t>(1, std::min<int64_t>(B, bc));
}

}  // namespace pq

using namespace pq;

#define PQ_API_BEGIN try { clear_error();
#define PQ_API_END                                                         \
    }                                                                      \
    catch (const pq::Error& e) { set_error(e.msg); return e.st; }          \
    catch (const std::bad_alloc&) { set_error("host out of memory"); return PQ_ERR_OUT_OF_MEMORY; } \
    catch (const std::exception& e) { set_error(e.what()); return PQ_ERR_CUDA; } \
    catch (...) { set_error("unknown error"); return PQ_ERR_CUDA; }         \
    return PQ_OK;

extern "C" {

int32_t pq_abi_version(void) { return PQTOPK_ABI_VERSION; }
const char* pq_last_error(void) { return t_err.c_str(); }
int64_t pq_launch_count(void) { return g_launches.load(); }

pq_status pq_create(const uint8_t* codes, int64_t N, int32_t m, int32_t b, int64_t id_base,
                    void* stream, pq_index* out) {
    return pq_create_ex(codes, N, m, b, id_base, 0, stream, out);
}

pq_status pq_create_ex(const uint8_t* codes, int64_t N, int32_t m, int32_t b, int64_t id_base,
                       int32_t flags, void* stream, pq_index* out) {
    PQ_API_BEGIN
    need(out != nullptr, "out is NULL");
    *out = nullptr;
    need(codes != nullptr, "codes is NULL");
    need(N >= 1, "N must be >= 1");
    need(m >= 1 && m <= 64, "m must be in [1, 64]");
    need(b >= 1 && b <= 256, "b must be in [1, 256] (uint8 codes)");
    need(id_base >= 0 && id_base + N <= 2147483647LL, "id_base + N must be <= 2^31 - 1");
    cudaStream_t st = static_cast<cudaStream_t>(stream);

    pq_index_s* idx = new pq_index_s();
    uint8_t* tmp = nullptr;
    unsigned long long* d_bad = nullptr;
    try {
        idx->N = N; idx->m = m; idx->b = b; idx->id_base = id_base;
        PQ_CUDA(cudaGetDevice(&idx->device));
        PQ_CUDA(cudaDeviceGetAttribute(&idx->num_sms, cudaDevAttrMultiProcessorCount, idx->device));
        int optin = 0;
        PQ_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, idx->device));
        idx->smem_optin = (size_t)optin;
        idx->lay.mp = round_up4(m);
        idx->lay.paired = 0;
        idx->n_rows = N;
        const size_t bytes = (size_t)N * idx->lay.mp + 64;
        if (cudaMalloc(&idx->d_codes, bytes) != cudaSuccess) {
            cudaGetLastError();
            idx->d_codes = nullptr;
            fail(PQ_ERR_OUT_OF_MEMORY, "cudaMalloc of " + std::to_string(bytes) + " code bytes failed");
        }
        PQ_CUDA(cudaMemsetAsync(idx->d_codes, 0, bytes, st));
        const uint8_t* src = codes;
        if (!is_device_ptr(codes)) {
            if (cudaMalloc(&tmp, (size_t)N * m) != cudaSuccess) {
                cudaGetLastError();
                tmp = nullptr;
                fail(PQ_ERR_OUT_OF_MEMORY, "cudaMalloc of the code staging buffer failed");
            }
            PQ_CUDA(cudaMemcpyAsync(tmp, codes, (size_t)N * m, cudaMemcpyHostToDevice, st));
            src = tmp;
        }
        PQ_CUDA(cudaMalloc(&d_bad, sizeof(unsigned long long)));
        PQ_CUDA(cudaMemsetAsync(d_bad, 0xFF, sizeof(unsigned long long), st));
        launch_relayout(src, N, m, b, idx->d_codes, idx->lay.mp, d_bad, st);
        unsigned long long bad = 0;
        PQ_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, st));
        PQ_CUDA(cudaStreamSynchronize(st));
        if (bad != ~0ull) {
            uint8_t v = 0;
            PQ_CUDA(cudaMemcpy(&v, src + bad, 1, cudaMemcpyDeviceToHost));
            char msg[160];
            snprintf(msg, sizeof msg, "code out of range: item %lld split %lld has code %u >= b = %d",
                     (long long)(bad / m), (long long)(bad % m), (unsigned)v, b);
            fail(PQ_ERR_CODE_RANGE, msg);
        }
        need((flags & ~PQ_CREATE_SMALL_BATCH_ONLY) == 0, "unknown pq_create flags");
        if (!(flags & PQ_CREATE_SMALL_BATCH_ONLY)) {
            if (getenv("PQTOPK_HOST_LAYOUT")) {        // the host builder (A/B and cross-check only)
                CreateCtx cx;
                build_v3_layout(idx, cx, codes, src, st);
            } else {
                build_v3_layout_gpu(idx, st);          // k0_layout.cu
            }
        }
        if (tmp) { cudaFree(tmp); tmp = nullptr; }
        cudaFree(d_bad);
        d_bad = nullptr;
    } catch (...) {
        if (tmp) cudaFree(tmp);
        if (d_bad) cudaFree(d_bad);
        free_index_buffers(idx);
        delete idx;
        throw;
    }
    *out = idx;
    PQ_API_END
}

pq_status pq_destroy(pq_index idx) {
    PQ_API_BEGIN
    if (!idx) return PQ_OK;
    cudaDeviceSynchronize();
    free_index_buffers(idx);
    if (idx->events) {
        for (auto& e : *idx->events) { cudaEventDestroy(e.a); cudaEventDestroy(e.b); cudaEventDestroy(e.c); }
        delete idx->events;
        delete idx->ev_mu;
    }
    k6_cache_free(idx);
    delete idx;
    PQ_API_END
}

pq_status pq_index_info(pq_index idx, int64_t* N, int32_t* m, int32_t* b, int64_t* id_base) {
    PQ_API_BEGIN
    need(idx != nullptr, "index is NULL");
    if (N) *N = idx->N;
    if (m) *m = idx->m;
    if (b) *b = idx->b;
    if (id_base) *id_base = idx->id_base;
    PQ_API_END
}

pq_status pq_index_layout(pq_index idx, int32_t* paired, int32_t* tmem_splits,
                          int64_t* pairs_matched, int64_t* leftover_items) {
    PQ_API_BEGIN
    need(idx != nullptr, "index is NULL");
    // the colour pairing of the v3 layout (pq_create); for m > 20 it pairs
    // complementary colours on the first 20 splits
    const bool p3 = idx->v3_ok && idx->v3_R == 16;
    if (paired) *paired = p3 ? 1 : 0;
    if (tmem_splits) *tmem_splits = 0;
    if (pairs_matched) *pairs_matched = p3 ? idx->v3_matched : 0;
    if (leftover_items) *leftover_items = p3 ? idx->v3_leftover : 0;
    PQ_API_END
}

pq_status pq_index_variants(pq_index idx, int32_t* mask) {
    PQ_API_BEGIN
    need(idx != nullptr && mask != nullptr, "NULL argument");
    *mask = 2 | (idx->v3_ok ? 8 : 0) | (k2_latency_supported(idx, 1, 1) ? 16 : 0);
    PQ_API_END
}

pq_status pq_plan_info(pq_index idx, int32_t B, int32_t K, int64_t out[8]) {
    PQ_API_BEGIN
    need(idx != nullptr && out != nullptr, "NULL argument");
    check_topk_args(B, K);
    need(B > 0 && K > 0, "B and K must be > 0");
    K2Plan p = plan_k2(idx, B, K);
    out[0] = p.variant; out[1] = p.G; out[2] = p.Ug; out[3] = p.W;
    out[4] = p.grid; out[5] = p.chunks; out[6] = p.tm; out[7] = (int64_t)p.smem;
    PQ_API_END
}

pq_status pq_set_tuning(pq_index idx, const pq_tuning* t) {
    PQ_API_BEGIN
    need(idx != nullptr, "index is NULL");
    if (t) {
        need(t->warps >= 0 && t->warps <= 32, "tuning.warps must be in [0, 32]");
        need(t->ctas >= 0 && t->chunks >= 0 && t->variant >= 0, "tuning values must be >= 0");
        need(t->users_per_row >= 0 && t->users_per_row <= 32, "tuning.users_per_row must be in [0, 32]");
        need(t->shrink_watermark >= 0, "tuning.shrink_watermark must be >= 0");
        need(t->cluster == 0 || t->cluster == 1 || t->cluster == 2 || t->cluster == 4 || t->cluster == 8,
             "tuning.cluster must be 0, 1, 2, 4 or 8");
        idx->tuning = *t;
    } else {
        idx->tuning = pq_tuning{};
    }
    PQ_API_END
}

pq_status pq_subscores(const float* seq_emb, const float* subitem_emb, int32_t B, int32_t d,
                       int32_t m, int32_t b, float* S, void* stream) {
    PQ_API_BEGIN
    need(B >= 0, "B must be >= 0");
    need(m >= 1 && m <= 64, "m must be in [1, 64]");
    need(b >= 1 && b <= 256, "b must be in [1, 256]");
    need(d >= m && d % m == 0, "d must be a positive multiple of m");
    if (B == 0) return PQ_OK;
    need(seq_emb && subitem_emb && S, "NULL pointer");
    launch_subscores(seq_emb, subitem_emb, B, d, m, b, S, static_cast<cudaStream_t>(stream));
    PQ_API_END
}

size_t pq_topk_workspace_bytes(pq_index idx, int32_t B, int32_t K) {
    try {
        if (!idx || B <= 0 || K <= 0 || K > PQTOPK_MAX_K) return 0;
        return topk_ws(idx, B, K).total;
    } catch (const pq::Error& e) {
        set_error(e.msg);
        return 0;
    }
}

pq_status pq_score_topk(pq_index idx, const float* S, int32_t B, int32_t K, void* ws,
                        size_t ws_bytes, int32_t* ids, float* scores, void* stream) {
    PQ_API_BEGIN
    need(idx != nullptr, "index is NULL");
    check_topk_args(B, K);
    if (B == 0 || K == 0) return PQ_OK;
    need(S && ids && scores, "NULL pointer");
    run_score_topk(idx, S, B, K, ws, ws_bytes, ids, scores, static_cast<cudaStream_t>(stream));
    PQ_API_END
}

// pq_search runs the fused K6 kernel when it applies (B <= 4) unless the
// caller or the tuning asks for the multi-kernel path.
static bool use_k6(pq_index_s* idx, int B, int d, int K, int flags, K6Plan& p) {
    if (flags & PQ_SEARCH_NO_FUSED) return false;
    const int v = idx->tuning.variant;
    if (v != 0 && v != 5 && v != 7) return false;
    return k6_query_plan(idx, B, d, K, p);
}

size_t pq_search_workspace_bytes(pq_index idx, int32_t B, int32_t d, int32_t K) {
    try {
        if (!idx || B <= 0 || K <= 0 || K > PQTOPK_MAX_K || d < idx->m || d % idx->m) return 0;
        size_t s = 0;
        s += align_up((size_t)B * idx->m * idx->b * 4, 256);      // S
        s += align_up((size_t)B * d * 4, 256);                     // phi staging
        s += align_up((size_t)idx->b * d * 4, 256);                // psi staging
        s += 2 * align_up((size_t)B * K * 4, 256);                 // output staging
        size_t rest = topk_ws(idx, B, K).total;
        K6Plan kp;
        if (use_k6(idx, B, d, K, 0, kp)) rest = std::max(rest, k6_query_ws_bytes(kp, B, idx->m * idx->b));
        return s + rest;
    } catch (const pq::Error& e) {
        set_error(e.msg);
        return 0;
    }
}

pq_status pq_search(pq_index idx, const float* seq_emb, const float* subitem_emb, int32_t B,
                    int32_t d, int32_t K, void* ws, size_t ws_bytes, int32_t* ids, float* scores,
                    void* stream) {
    return pq_search_ex(idx, seq_emb, subitem_emb, B, d, K, 0, ws, ws_bytes, ids, scores, nullptr, stream);
}

pq_status pq_search_ex(pq_index idx, const float* seq_emb, const float* subitem_emb, int32_t B,
                       int32_t d, int32_t K, int32_t flags, void* ws, size_t ws_bytes, int32_t* ids,
                       float* scores, float* S_out, void* stream) {
    PQ_API_BEGIN
    need(idx != nullptr, "index is NULL");
    check_topk_args(B, K);
    need(d >= idx->m && d % idx->m == 0, "d must be a positive multiple of m");
    need((flags & ~PQ_SEARCH_NO_FUSED) == 0, "unknown pq_search_ex flags");
    if (B == 0 || K == 0) return PQ_OK;
    need(seq_emb && subitem_emb && ids && scores, "NULL pointer");
    need(!S_out || is_device_ptr(S_out), "S_out must be device memory");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t need_bytes = pq_search_workspace_bytes(idx, B, d, K);
    if (!ws || ws_bytes < need_bytes)
        fail(PQ_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need_bytes) + " bytes");
    const int m = idx->m, b = idx->b;
    Carve c(ws);
    float* S = c.take<float>((size_t)B * m * b * 4);
    float* phi_st = c.take<float>((size_t)B * d * 4);
    float* psi_st = c.take<float>((size_t)b * d * 4);
    int32_t* ids_st = c.take<int32_t>((size_t)B * K * 4);
    float* sc_st = c.take<float>((size_t)B * K * 4);
    char* rest = c.base + c.off;
    const float* phi = seq_emb;
    const float* psi = subitem_emb;
    K6Plan kp;
    const bool fused = use_k6(idx, B, d, K, flags, kp);
    // K7 writes pinned host ids / scores in place (zero copy: 8 B per result over
    // the host link instead of a DMA per buffer and its API call); pinned host
    // phi is read in place only when PQTOPK_ZC_PHI=1 (diagnostics: the kernel's
    // many small host reads measured slower than one DMA)
    static const bool zc_phi = [] { const char* e = getenv("PQTOPK_ZC_PHI"); return e && atoi(e) == 1; }();
    static const bool zc_off = getenv("PQTOPK_ZC_OFF") != nullptr;
    const bool zc = fused && kp.resident && !zc_off;
    cudaPointerAttributes pa;
    auto kind = [&](const void* p) -> int {            // 0 device, 1 pinned host (pa.devicePointer), 2 pageable
        if (cudaPointerGetAttributes(&pa, p) != cudaSuccess) { cudaGetLastError(); return 2; }
        if (pa.type == cudaMemoryTypeDevice || pa.type == cudaMemoryTypeManaged) return 0;
        return pa.type == cudaMemoryTypeHost && pa.devicePointer ? 1 : 2;
    };
    const int k_phi = kind(seq_emb);
    if (k_phi == 1 && zc && zc_phi) {
        phi = static_cast<const float*>(pa.devicePointer);
    } else if (k_phi != 0) {
        PQ_CUDA(cudaMemcpyAsync(phi_st, seq_emb, (size_t)B * d * 4, cudaMemcpyHostToDevice, st));
        phi = phi_st;
    }
    if (kind(subitem_emb) != 0) {
        PQ_CUDA(cudaMemcpyAsync(psi_st, subitem_emb, (size_t)b * d * 4, cudaMemcpyHostToDevice, st));
        psi = psi_st;
    }
    const int k_ids = kind(ids);
    void* m_ids = k_ids == 1 ? pa.devicePointer : nullptr;
    const int k_sc = kind(scores);
    void* m_sc = k_sc == 1 ? pa.devicePointer : nullptr;
    bool host_ids = k_ids != 0, host_sc = k_sc != 0;
    int32_t* ids_d = host_ids ? ids_st : ids;
    float* sc_d = host_sc ? sc_st : scores;
    bool sync_out = false;                             // host outputs written in place: sync only
    if (zc && m_ids && m_sc) {
        ids_d = static_cast<int32_t*>(m_ids);
        sc_d = static_cast<float*>(m_sc);
        host_ids = host_sc = false;
        sync_out = true;
    }
    if (fused) {
        pq_index_s::EvTriple ev{};
        if (idx->timing) {
            PQ_CUDA(cudaEventCreate(&ev.a)); PQ_CUDA(cudaEventCreate(&ev.b)); PQ_CUDA(cudaEventCreate(&ev.c));
            PQ_CUDA(cudaEventRecord(ev.a, st));
        }
        launch_k6_query(idx, kp, phi, psi, B, d, K, rest, S_out, ids_d, sc_d, st);
        if (idx->timing) {
            PQ_CUDA(cudaEventRecord(ev.b, st));
            PQ_CUDA(cudaEventRecord(ev.c, st));
            std::lock_guard<std::mutex> lk(*idx->ev_mu);
            idx->events->push_back(ev);
        }
    } else {
        launch_subscores(phi, psi, B, d, m, b, S, st);
        if (S_out) PQ_CUDA(cudaMemcpyAsync(S_out, S, (size_t)B * m * b * 4, cudaMemcpyDeviceToDevice, st));
        run_score_topk(idx, S, B, K, rest, ws_bytes - c.off, ids_d, sc_d, st);
    }
    if (host_ids) PQ_CUDA(cudaMemcpyAsync(ids, ids_st, (size_t)B * K * 4, cudaMemcpyDeviceToHost, st));
    if (host_sc) PQ_CUDA(cudaMemcpyAsync(scores, sc_st, (size_t)B * K * 4, cudaMemcpyDeviceToHost, st));
    if (host_ids || host_sc || sync_out) PQ_CUDA(cudaStreamSynchronize(st));
    PQ_API_END
}

pq_status pq_search_plan_info(pq_index idx, int32_t B, int32_t d, int32_t K, int64_t out[8]) {
    PQ_API_BEGIN
    need(idx != nullptr && out != nullptr, "NULL argument");
    check_topk_args(B, K);
    need(B > 0 && K > 0, "B and K must be > 0");
    need(d >= idx->m && d % idx->m == 0, "d must be a positive multiple of m");
    K6Plan kp;
    if (use_k6(idx, B, d, K, 0, kp)) {
        out[0] = kp.resident ? 7 : 5; out[1] = kp.G;
        out[2] = kp.resident ? kp.cl : (kp.gridsync ? 0 : kp.CL);
        out[3] = kp.resident ? 16 : 8;
        out[4] = kp.grid; out[5] = kp.chunks; out[6] = 0; out[7] = (int64_t)kp.smem;
    } else {
        K2Plan p = plan_k2(idx, B, K);
        out[0] = p.variant; out[1] = p.G; out[2] = p.Ug; out[3] = p.W;
        out[4] = p.grid; out[5] = p.chunks; out[6] = p.tm; out[7] = (int64_t)p.smem;
    }
    PQ_API_END
}

size_t pq_merge_workspace_bytes(int32_t P, int32_t B, int32_t K) {
    if (P <= 0 || B <= 0 || K <= 0 || K > PQTOPK_MAX_K) return 0;
    return k3_pairs_scratch_bytes(P, B, K);
}

pq_status pq_merge_topk(const int32_t* ids, const float* scores, int32_t P, int32_t B, int32_t K,
                        void* ws, size_t ws_bytes, int32_t* out_ids, float* out_scores,
                        void* stream) {
    PQ_API_BEGIN
    need(P >= 1, "P must be >= 1");
    check_topk_args(B, K);
    if (B == 0 || K == 0) return PQ_OK;
    need(ids && scores && out_ids && out_scores, "NULL pointer");
    const size_t nb = pq_merge_workspace_bytes(P, B, K);
    if (nb && (!ws || ws_bytes < nb))
        fail(PQ_ERR_WORKSPACE, "workspace too small: need " + std::to_string(nb) + " bytes");
    k3_pairs_to_topk(ids, scores, (int64_t)B * K, P, B, K, ws, out_ids, out_scores,
                     static_cast<cudaStream_t>(stream));
    PQ_API_END
}

pq_status pq_merge_topk_packed(const int32_t* lists, int32_t P, int32_t B, int32_t K, void* ws,
                               size_t ws_bytes, int32_t* out_ids, float* out_scores, void* stream) {
    PQ_API_BEGIN
    need(P >= 1, "P must be >= 1");
    check_topk_args(B, K);
    if (B == 0 || K == 0) return PQ_OK;
    need(lists && out_ids && out_scores, "NULL pointer");
    const size_t nb = pq_merge_workspace_bytes(P, B, K);
    if (nb && (!ws || ws_bytes < nb))
        fail(PQ_ERR_WORKSPACE, "workspace too small: need " + std::to_string(nb) + " bytes");
    const int64_t BK = (int64_t)B * K;
    k3_pairs_to_topk(lists, reinterpret_cast<const float*>(lists + BK), 2 * BK, P, B, K, ws, out_ids,
                     out_scores, static_cast<cudaStream_t>(stream));
    PQ_API_END
}

pq_status pq_reconstruct(pq_index idx, const float* subitem_emb, int32_t d, float* W, void* stream) {
    PQ_API_BEGIN
    need(idx != nullptr, "index is NULL");
    need(d >= idx->m && d % idx->m == 0, "d must be a positive multiple of m");
    need(subitem_emb && W, "NULL pointer");
    launch_reconstruct(idx, subitem_emb, d, W, static_cast<cudaStream_t>(stream));
    PQ_API_END
}

size_t pq_dense_workspace_bytes(int64_t N, int32_t B, int32_t K) {
    if (N <= 0 || B <= 0 || K <= 0 || K > PQTOPK_MAX_K) return 0;
    const int64_t nc = dense_chunk(N, B);
    const int64_t lists = dense_lists(N, nc);
    return align_up((size_t)B * nc * 4, 256) + align_up((size_t)B * lists * K * 8, 256) +
           k3_reduce_scratch_bytes(lists * K, B, K);
}

pq_status pq_dense_topk(const float* W, int64_t N, int32_t d, const float* seq_emb, int32_t B,
                        int32_t K, int64_t id_base, void* ws, size_t ws_bytes, int32_t* ids,
                        float* scores, void* stream) {
    PQ_API_BEGIN
    need(N >= 1 && d >= 1, "N and d must be >= 1");
    need(id_base >= 0 && id_base + N <= 2147483647LL, "id_base + N must be <= 2^31 - 1");
    check_topk_args(B, K);
    if (B == 0 || K == 0) return PQ_OK;
    need(W && seq_emb && ids && scores, "NULL pointer");
    const size_t nb = pq_dense_workspace_bytes(N, B, K);
    if (!ws || ws_bytes < nb) fail(PQ_ERR_WORKSPACE, "workspace too small: need " + std::to_string(nb) + " bytes");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t nc = dense_chunk(N, B);
    const int64_t lists = dense_lists(N, nc);
    Carve c(ws);
    float* R = c.take<float>((size_t)B * nc * 4);
    uint64_t* keys = c.take<uint64_t>((size_t)B * lists * K * 8);
    void* k3s = c.take<char>(k3_reduce_scratch_bytes(lists * K, B, K));
    int64_t off = 0;
    for (int64_t c0 = 0; c0 < N; c0 += nc) {
        const int64_t n = std::min(nc, N - c0);
        dense_sgemm(W + c0 * d, n, d, seq_emb, B, R, st);
        k3_rows_to_keys(R, n, n, B, K, (uint32_t)(id_base + c0), keys, lists, off, st);
        off += k3_rows_lists(n);
    }
    k3_keys_to_topk(keys, lists * K, B, K, k3s, ids, scores, st);
    PQ_API_END
}

size_t pq_recjpq_workspace_bytes(pq_index idx, int32_t B, int32_t K) {
    if (!idx || B <= 0 || K <= 0 || K > PQTOPK_MAX_K) return 0;
    const int bc = recjpq_users(idx->N, B);
    const int64_t lists = k3_rows_lists(idx->N);
    return align_up((size_t)bc * idx->N * 4, 256) + align_up((size_t)B * lists * K * 8, 256) +
           k3_reduce_scratch_bytes(lists * K, B, K);
}

pq_status pq_recjpq_topk(pq_index idx, const float* S, int32_t B, int32_t K, void* ws,
                         size_t ws_bytes, int32_t* ids, float* scores, void* stream) {
    PQ_API_BEGIN
    need(idx != nullptr, "index is NULL");
    check_topk_args(B, K);
    if (B == 0 || K == 0) return PQ_OK;
    need(S && ids && scores, "NULL pointer");
    const size_t nb = pq_recjpq_workspace_bytes(idx, B, K);
    if (!ws || ws_bytes < nb) fail(PQ_ERR_WORKSPACE, "workspace too small: need " + std::to_string(nb) + " bytes");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int bc = recjpq_users(idx->N, B);
    const int64_t lists = k3_rows_lists(idx->N);
    Carve c(ws);
    float* R = c.take<float>((size_t)bc * idx->N * 4);
    uint64_t* keys = c.take<uint64_t>((size_t)B * lists * K * 8);
    void* k3s = c.take<char>(k3_reduce_scratch_bytes(lists * K, B, K));
    for (int u0 = 0; u0 < B; u0 += bc) {
        const int n = std::min(bc, B - u0);
        PQ_CUDA(cudaMemsetAsync(R, 0, (size_t)n * idx->N * 4, st));    // "initialised to 0"
        for (int k = 0; k < idx->m; ++k)                                  // "Not parallelised"
            launch_recjpq_split(idx, S, B, u0, n, k, R, st);
        k3_rows_to_keys(R, idx->N, idx->N, n, K, (uint32_t)idx->id_base, keys + (size_t)u0 * lists * K,
                        lists, 0, st);
    }
    k3_keys_to_topk(keys, lists * K, B, K, k3s, ids, scores, st);
    PQ_API_END
}

size_t pq_subset_workspace_bytes(pq_index idx, int64_t nV, int32_t B, int32_t K) {
    try {
        if (!idx || nV <= 0 || B <= 0 || K <= 0 || K > PQTOPK_MAX_K) return 0;
        pq_index_s t = subset_index(idx, nV, nullptr, nullptr);
        return subset_codes_bytes(idx, nV) + topk_ws(&t, B, K).total;
    } catch (const pq::Error& e) {
        set_error(e.msg);
        return 0;
    }
}

pq_status pq_score_topk_subset(pq_index idx, const float* S, int32_t B, int32_t K, const int32_t* V,
                               int64_t nV, void* ws, size_t ws_bytes, int32_t* ids, float* scores,
                               void* stream) {
    return pq_score_topk_subset_ex(idx, S, B, K, V, nV, 0, ws, ws_bytes, ids, scores, stream);
}

pq_status pq_score_topk_subset_ex(pq_index idx, const float* S, int32_t B, int32_t K, const int32_t* V,
                                  int64_t nV, int32_t flags, void* ws, size_t ws_bytes, int32_t* ids,
                                  float* scores, void* stream) {
    PQ_API_BEGIN
    need(idx != nullptr, "index is NULL");
    check_topk_args(B, K);
    need(nV >= 0, "nV must be >= 0");
    need((flags & ~PQ_SUBSET_VALIDATE) == 0, "unknown pq_score_topk_subset_ex flags");
    if (B == 0 || K == 0) return PQ_OK;
    need(S && ids && scores, "NULL pointer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (nV == 0) {                                     // empty subset: all padding (R11), on the device
        launch_fill_padding(ids, scores, (int64_t)B * K, st);
        return PQ_OK;
    }
    need(V != nullptr, "V is NULL");
    const size_t nb = pq_subset_workspace_bytes(idx, nV, B, K);
    if (!ws || ws_bytes < nb) fail(PQ_ERR_WORKSPACE, "workspace too small: need " + std::to_string(nb) + " bytes");
    Carve c(ws);
    uint8_t* codesV = c.take<uint8_t>((size_t)nV * idx->lay.mp + 64);
    unsigned long long* bad = c.take<unsigned long long>(8);
    if (flags & PQ_SUBSET_VALIDATE) {                  // debug / untrusted V: synchronous check
        need(is_device_ptr(V), "V must be a device array of nV item ids");
        PQ_CUDA(cudaMemsetAsync(bad, 0xFF, 8, st));
        launch_check_subset(V, nV, idx->N, bad, st);
        unsigned long long hbad = 0;
        PQ_CUDA(cudaMemcpyAsync(&hbad, bad, 8, cudaMemcpyDeviceToHost, st));
        PQ_CUDA(cudaStreamSynchronize(st));
        if (hbad != ~0ull)
            fail(PQ_ERR_INVALID_ARG, "V must hold strictly increasing local item ids in [0, N): first bad "
                                     "position " + std::to_string(hbad));
    }
    launch_gather_codes(idx->d_codes, idx->lay.mp, idx->N, V, nV, codesV, st);
    pq_index_s t = subset_index(idx, nV, codesV, V);
    run_score_topk(&t, S, B, K, c.base + c.off, ws_bytes - c.off, ids, scores, st);
    PQ_API_END
}

size_t pq_exclude_workspace_bytes(pq_index idx, int32_t B, int32_t K, int32_t max_excl) {
    try {
        if (!idx || B <= 0 || K <= 0 || max_excl < 0 || K + max_excl > PQTOPK_MAX_K) return 0;
        const int K2 = K + max_excl;
        return 2 * align_up((size_t)B * K2 * 4, 256) + topk_ws(idx, B, K2).total;
    } catch (const pq::Error& e) {
        set_error(e.msg);
        return 0;
    }
}

pq_status pq_score_topk_exclude(pq_index idx, const float* S, int32_t B, int32_t K, const int32_t* excl,
                                const int64_t* excl_off, int32_t max_excl, void* ws, size_t ws_bytes,
                                int32_t* ids, float* scores, void* stream) {
    PQ_API_BEGIN
    need(idx != nullptr, "index is NULL");
    check_topk_args(B, K);
    need(max_excl >= 0, "max_excl must be >= 0");
    if (K + max_excl > PQTOPK_MAX_K) fail(PQ_ERR_UNSUPPORTED, "K + max_excl exceeds PQTOPK_MAX_K (4096)");
    if (B == 0 || K == 0) return PQ_OK;
    need(S && ids && scores && excl_off, "NULL pointer");
    need(max_excl == 0 || excl != nullptr, "excl is NULL");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t nb = pq_exclude_workspace_bytes(idx, B, K, max_excl);
    if (!ws || ws_bytes < nb) fail(PQ_ERR_WORKSPACE, "workspace too small: need " + std::to_string(nb) + " bytes");
    const int K2 = K + max_excl;
    Carve c(ws);
    int32_t* ids2 = c.take<int32_t>((size_t)B * K2 * 4);
    float* sc2 = c.take<float>((size_t)B * K2 * 4);
    run_score_topk(idx, S, B, K2, c.base + c.off, ws_bytes - c.off, ids2, sc2, st);
    launch_exclude(ids2, sc2, B, K2, excl, excl_off, K, ids, scores, st);
    PQ_API_END
}

pq_status pq_timing_enable(pq_index idx, int32_t on) {
    PQ_API_BEGIN
    need(idx != nullptr, "index is NULL");
    if (on && !idx->events) {
        idx->ev_mu = new std::mutex();
        idx->events = new std::vector<pq_index_s::EvTriple>();
    }
    idx->timing = on ? 1 : 0;
    PQ_API_END
}

pq_status pq_timing_read(pq_index idx, double* k2_ms, double* k3_ms, int64_t* launches) {
    PQ_API_BEGIN
    need(idx != nullptr, "index is NULL");
    double t2 = 0.0, t3 = 0.0;
    int64_t n = 0;
    if (idx->events) {
        std::lock_guard<std::mutex> lk(*idx->ev_mu);
        for (auto& e : *idx->events) {
            float a = 0.f, c = 0.f;
            PQ_CUDA(cudaEventSynchronize(e.c));
            PQ_CUDA(cudaEventElapsedTime(&a, e.a, e.b));
            PQ_CUDA(cudaEventElapsedTime(&c, e.b, e.c));
            t2 += a; t3 += c; ++n;
            cudaEventDestroy(e.a); cudaEventDestroy(e.b); cudaEventDestroy(e.c);
        }
        idx->events->clear();
    }
    if (k2_ms) *k2_ms = t2;
    if (k3_ms) *k3_ms = t3;
    if (launches) *launches = n;
    PQ_API_END
}

}  // extern "C"
