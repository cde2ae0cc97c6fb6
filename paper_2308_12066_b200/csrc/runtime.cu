// runtime.cu — the model object, the pre-gated decoder loop and the C ABI.
//
// Mirrors core.py:342-383 (decoder_iteration wiring) and the pre_gated
// branch of scheduler.py:287-373 on real hardware: block b's lookahead gate
// (K1) decides block b+L's experts; the host reads the active list as soon
// as K1 finishes and streams exactly those experts from pinned host memory
// into an (L+1)-slot HBM expert cache on a dedicated copy stream while
// block b's experts (K2) and dense layer (K3) run on the compute stream.
// CUDA events order slot reuse (a slot is refilled only after the block
// that consumed it finished, tiers.py "expert lifetime") and expert
// execution after arrival.  Block 0's fetch is exposed, as in the paper's
// footnote (scheduler.py:344-351).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cuda.h>

#include "common.cuh"
#include "decode.h"
#include "expert_cache.h"
#include "kernels.h"
#include "rng.h"
#include "route_common.cuh"

namespace pgmoe {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
// Debug probes: each launch of kind k takes the next `ctas` rows of the
// installed buffer (wrapping at its capacity), so one decoder iteration
// leaves every launch's stamps side by side.
static unsigned long long *g_probe[2] = {nullptr, nullptr};
static long long g_probe_rows[2] = {0, 0}, g_probe_next[2] = {0, 0};
unsigned long long *probe_buffer(int kind, int ctas) {
    if (kind < 0 || kind >= 2 || !g_probe[kind]) return nullptr;
    if (g_probe_next[kind] + ctas > g_probe_rows[kind]) g_probe_next[kind] = 0;
    unsigned long long *b = g_probe[kind] + (size_t)g_probe_next[kind] * kProbeSlots;
    g_probe_next[kind] += ctas;
    return b;
}

int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}

// SMs the CURRENT context may use: a green context (or any context carved
// out of the device's SMs) reports its own share through cuCtxGetDevResource;
// otherwise the device attribute.  Cached per context.  PGMOE_SM_LIMIT caps
// it (testing the persistent kernels on fewer co-resident CTAs).
int device_sm_count() {
    using GetCur = CUresult (*)(CUcontext *);
    using GetRes = CUresult (*)(CUcontext, CUdevResource *, CUdevResourceType);
    static std::mutex mu;
    static std::vector<std::pair<CUcontext, int>> cache;
    static GetCur get_cur = nullptr;
    static GetRes get_res = nullptr;
    static bool looked = false;
    std::lock_guard<std::mutex> lock(mu);
    if (!looked) {
        looked = true;
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuCtxGetCurrent", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            get_cur = reinterpret_cast<GetCur>(p);
        p = nullptr;
        if (cudaGetDriverEntryPoint("cuCtxGetDevResource", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            get_res = reinterpret_cast<GetRes>(p);
    }
    CUcontext ctx = nullptr;
    if (get_cur) get_cur(&ctx);
    if (!ctx && get_cur) {  // no context yet: create the primary one (never reached during stream capture)
        cudaFree(nullptr);
        get_cur(&ctx);
    }
    for (auto &e : cache)
        if (e.first == ctx) return e.second;
    int n = 0;
    CUdevResource res;
    memset(&res, 0, sizeof(res));
    if (ctx && get_res && get_res(ctx, &res, CU_DEV_RESOURCE_TYPE_SM) == CUDA_SUCCESS) n = (int)res.sm.smCount;
    if (n <= 0 && (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, current_device()) != cudaSuccess || n <= 0))
        n = kNumSMs;
    if (const char *e = getenv("PGMOE_SM_LIMIT")) {
        const int lim = atoi(e);
        if (lim > 0) n = std::min(n, lim);
    }
    cache.emplace_back(ctx, n);
    return n;
}

void set_error(const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
}

struct RoutingBuf {
    pgmoe_routing r{};
    void *mem = nullptr;
    int32_t *act_host = nullptr;  // pinned mirror of act[E] + n_act
};

struct BlockW {
    void *gate = nullptr, *pre_gate = nullptr, *dense = nullptr;
    unsigned char *experts = nullptr;  // device (resident) or pinned host (offloaded)
};

struct TimelineEv {
    const char *lane;
    std::string label;
    int block;
    cudaEvent_t a, b;
};

}  // namespace pgmoe

using namespace pgmoe;

struct pgmoe_model {
    pgmoe_config cfg{};
    int wdtype = PGMOE_BF16, placement = PGMOE_RESIDENT, max_tokens = 0, kernel = PGMOE_KERNEL_AUTO;
    int e_begin = 0, e_local = 0;  // expert range held by this model (expert parallelism)
    int strategy = PGMOE_PRE_GATED;  // offloaded migration policy (scheduler.py:36-49)
    // optional HBM expert cache (cache.py): entries live in `cache_region`; a
    // hit is a D2D copy into the block's working slot, an inserted miss is
    // copied on from the slot, all on the copy stream (FIFO: no slot hazards)
    ExpertCacheIndex *cache = nullptr;
    unsigned char *cache_region = nullptr;
    int64_t cache_seq = 0;
    size_t sw = 2, gate_bytes = 0, dense_bytes = 0, w1_bytes = 0, rec_bytes = 0;
    std::vector<BlockW> blocks;
    unsigned char *dev_pool = nullptr;   // gates + dense (+ experts when resident)
    unsigned char *host_pool = nullptr;  // pinned experts (offloaded)
    size_t dev_pool_bytes = 0, host_pool_bytes = 0;
    // work buffers
    float *act_buf[2] = {nullptr, nullptr};
    float *h = nullptr, *yw = nullptr;
    uint16_t *xb = nullptr, *hb = nullptr, *mixb = nullptr;  // bf16 tcgen05 operands
    std::vector<RoutingBuf> routing;  // ring of L+1 decisions
    void *route_ws = nullptr;
    void *tc_ws = nullptr;
    size_t tc_ws_bytes = 0;
    // offload
    unsigned char *slots = nullptr;
    size_t slot_capacity = 0;  // bytes per slot
    int slot_experts = 0;
    // expert slots: L+1 (one per routing decision in flight); prefetch_all
    // needs max(L+1, 2) because block b+1's set streams while b computes
    int nslots = 0;
    cudaStream_t copy = nullptr;
    std::vector<cudaEvent_t> ready, done, routed;
    cudaEvent_t gated = nullptr;  // on_demand: compute reached the block
    std::vector<bool> slot_used;
    // stats
    pgmoe_stats stats{};
    std::vector<int> nact_iter;  // per block, last iteration (offloaded)
    std::vector<cudaEvent_t> cp_a, cp_b, ffn_b;  // per block timing events
    bool timeline = false;
    std::vector<TimelineEv> tl;
    cudaEvent_t t0 = nullptr;
    bool t0_recorded = false;
    // resident decoder iterations are replayed from a CUDA graph per buffer set
    bool use_graph = true;
    cudaStream_t cap = nullptr;
    struct GraphEntry {
        cudaGraphExec_t exec = nullptr;
        const float *x = nullptr;
        float *y = nullptr;
        int T = -1;
        pgmoe_iteration_io io{};
        unsigned long long last_use = 0;
        long long launches = 0;  // kernels per replay (benchmark evidence)
    };
    GraphEntry graphs[8];  // small LRU: callers' output buffers rotate through the allocator
    unsigned long long graph_clock = 0;
    int64_t fused_blocks = 0;  // blocks whose dense layer ran inside the expert launch
    int64_t fused_routes = 0;  // pre-gates computed inside the block launch
    // small batches (T <= decode_max_t): one persistent launch per decoder
    // iteration (decode_tc.cu); per-block descriptors built at creation
    bool decode = true;          // pgmoe_model_set_decode / PGMOE_DECODE=0
    int decode_max_t = 1;        // PGMOE_DECODE_MAX_T (measured: the per-block launches win from T = 2)
    DecodeBlock *dec_blocks = nullptr;
    int *dec_sync = nullptr;
    int64_t decode_iters = 0;
    // low-latency decoder (decode_ll.cu) for T <= ll_max_t: LL-word phase exchanges
    bool ll_decode = true;       // pgmoe_model_set_ll_decode / PGMOE_LLDECODE=0
    int ll_max_t = kLLMaxT;      // PGMOE_LLDECODE_MAX_T
    void *ll_ws = nullptr;
    size_t ll_ws_bytes = 0;
    int64_t ll_iters = 0;
    bool fuse_route = true;    // resident: route inside the block launch (pgmoe_model_set_fused_route)
    long long fuse_max_t = 0;  // largest T routed inside the block launch (0: d_ff / 8; PGMOE_FUSE_MAX_T)
    // fused: launches chained on the previous dense phase instead of its
    // completion (PGMOE_CHAIN=1).  Measured: saves the ~4.5 us completion
    // latency but pays ~3-4 us of atomic + fence + poll, net -1 % at T=256
    // and +2 % at T=1 (tools/gpu_ab_chain.sh), so off by default.
    bool chain_launches = true;  // PGMOE_CHAIN=0: PDL completion only
    int *epoch = nullptr;        // device counter of chained launches
    // host-buffer entry point
    cudaStream_t io_stream = nullptr;
    float *io_x = nullptr, *io_y = nullptr, *io_w = nullptr;
    int32_t *io_ids = nullptr;
    int32_t *io_status = nullptr;  // pinned mirror of every routing buffer's status [R][4]
    int32_t *status_dev = nullptr; // the routing buffers' status words [R][4] (routing[i].r.status)
    std::mutex mu;
};

namespace pgmoe {

static bool has_conv_gate(const pgmoe_config &c, int b) {
    if (c.activation_level == 0) return true;
    return b < c.activation_level;
}
static bool has_pre_gate(const pgmoe_config &c, int b) {
    if (c.activation_level == 0) return false;
    return b < c.num_blocks - c.activation_level;
}

static int validate_config(const pgmoe_config *c) {
    PG_REQUIRE(c != nullptr, PGMOE_E_CONFIG, "null config");
    const int32_t v[5] = {c->d_model, c->d_ff, c->num_blocks, c->num_experts, c->top_k};
    const char *names[5] = {"d_model", "d_ff", "num_blocks", "num_experts", "top_k"};
    for (int i = 0; i < 5; ++i)
        PG_REQUIRE(v[i] >= 1, PGMOE_E_CONFIG, "%s must be a positive int, got %d", names[i], v[i]);
    PG_REQUIRE(c->top_k <= c->num_experts, PGMOE_E_CONFIG, "top_k=%d exceeds num_experts=%d",
               c->top_k, c->num_experts);
    PG_REQUIRE(c->activation_level >= 0 && c->activation_level < c->num_blocks, PGMOE_E_CONFIG,
               "activation_level=%d must be in [0, num_blocks=%d)", c->activation_level, c->num_blocks);
    PG_REQUIRE(c->top_k <= 8, PGMOE_E_CONFIG, "top_k=%d unsupported by the device path (<= 8)", c->top_k);
    PG_REQUIRE(c->num_experts <= 1024, PGMOE_E_CONFIG, "num_experts=%d unsupported (<= 1024)",
               c->num_experts);
    return PGMOE_OK;
}

static int alloc_routing(RoutingBuf &rb, int T, int E, int k) {
    const size_t n = (size_t)T * k;
    // layout: ids | w | perm | w_perm | inv | hist | off | act | n_act | status
    size_t bytes = n * 4 * 5 + (size_t)E * 4 + (size_t)(E + 1) * 4 + (size_t)(E + 1) * 4 + 16 + 256;
    PG_CUDA(cudaMalloc(&rb.mem, bytes));
    PG_CUDA(cudaMemset(rb.mem, 0, bytes));
    char *p = static_cast<char *>(rb.mem);
    rb.r.ids = reinterpret_cast<int32_t *>(p); p += n * 4;
    rb.r.w = reinterpret_cast<float *>(p); p += n * 4;
    rb.r.perm = reinterpret_cast<int32_t *>(p); p += n * 4;
    rb.r.w_perm = reinterpret_cast<float *>(p); p += n * 4;
    rb.r.inv = reinterpret_cast<int32_t *>(p); p += n * 4;
    rb.r.hist = reinterpret_cast<int32_t *>(p); p += (size_t)E * 4;
    rb.r.off = reinterpret_cast<int32_t *>(p); p += (size_t)(E + 1) * 4;
    rb.r.act = reinterpret_cast<int32_t *>(p);
    rb.r.n_act = rb.r.act + E;  // contiguous with act: one D2H copy
    p += (size_t)(E + 1) * 4;
    p = reinterpret_cast<char *>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
    rb.r.status = reinterpret_cast<int32_t *>(p);
    PG_CUDA(cudaHostAlloc(&rb.act_host, sizeof(int32_t) * (E + 1), cudaHostAllocDefault));
    return PGMOE_OK;
}

static void *mat_ptr(pgmoe_model *m, const std::string &name, int b, int e, size_t *bytes,
                     bool *on_host) {
    const auto &c = m->cfg;
    if (b < 0 || b >= c.num_blocks) return nullptr;
    BlockW &bw = m->blocks[b];
    *on_host = false;
    if (name == "gate") { *bytes = m->gate_bytes; return bw.gate; }
    if (name == "pre_gate") { *bytes = m->gate_bytes; return bw.pre_gate; }
    if (name == "non_moe") { *bytes = m->dense_bytes; return bw.dense; }
    if (name == "w1" || name == "w2") {
        const int le = e - m->e_begin;
        if (le < 0 || le >= m->e_local) return nullptr;
        *on_host = (m->placement == PGMOE_OFFLOADED);
        *bytes = m->w1_bytes;
        return bw.experts + (size_t)le * m->rec_bytes + (name == "w2" ? m->w1_bytes : 0);
    }
    return nullptr;
}

static bool use_tc(const pgmoe_model *m) {
    return m->wdtype == PGMOE_BF16 && m->kernel != PGMOE_KERNEL_SIMT && tc_supported(m->cfg.d_model, m->cfg.d_ff);
}

// xb_ready: the previous block's dense epilogue already wrote this block's
// packed bf16 operand (its routing was known before that dense ran).
int run_ffn(pgmoe_model *m, const float *x, int T, const void *experts, int indexed,
            const pgmoe_routing *r, cudaStream_t s, bool xb_ready = false) {
    const auto &c = m->cfg;
    const bool tc = use_tc(m);
    if (m->kernel == PGMOE_KERNEL_TCGEN05)
        PG_REQUIRE(tc, PGMOE_E_CONFIG, "tcgen05 kernels need bf16 weights and d, f multiples of 128");
    if (tc)
        return expert_ffn_tc2(x, T, c.d_model, c.d_ff, c.top_k, experts, m->rec_bytes, indexed, r, m->xb, m->hb,
                              m->yw, c.top_k == 1 ? m->mixb : nullptr, m->tc_ws, m->tc_ws_bytes, s, xb_ready);
    return expert_ffn_simt(x, T, c.d_model, c.d_ff, c.top_k, experts, m->rec_bytes, m->wdtype, indexed,
                           r, m->h, m->yw, s);
}

// next (optional): the following block's routing, for the fused operand pack.
int run_dense(pgmoe_model *m, int T, const void *dense, float *y, cudaStream_t s,
              const pgmoe_routing *next = nullptr) {
    const auto &c = m->cfg;
    if (use_tc(m))
        return dense_tc2(m->yw, c.top_k == 1 ? m->mixb : nullptr, T, c.d_model, c.top_k, dense, y, m->mixb,
                         m->tc_ws, m->tc_ws_bytes, s, next ? m->xb : nullptr, next ? next->inv : nullptr);
    return dense_simt(m->yw, T, c.d_model, c.top_k, dense, m->wdtype, y, s);
}

static void tl_begin(pgmoe_model *m, const char *lane, const std::string &label, int block,
                     cudaStream_t s) {
    if (!m->timeline) return;
    TimelineEv ev{lane, label, block, nullptr, nullptr};
    cudaEventCreate(&ev.a);
    cudaEventCreate(&ev.b);
    cudaEventRecord(ev.a, s);
    m->tl.push_back(ev);
}
static void tl_end(pgmoe_model *m, cudaStream_t s) {
    if (!m->timeline) return;
    cudaEventRecord(m->tl.back().b, s);
}

// Cached fetch of `n` experts (ids `ids`, in access order) of block `tb` into
// the working slot `dst`: the reference's cache.access per expert
// (scheduler.py:295-311), hits copied from the cache region (D2D), misses
// from pinned host memory, inserted misses copied on into the cache.
static int fetch_cached(pgmoe_model *m, int tb, const int32_t *ids, int n, unsigned char *dst, int *misses) {
    const unsigned char *src = m->blocks[tb].experts;
    const size_t rec = m->rec_bytes;
    int miss = 0;
    for (int i = 0; i < n; ++i) {
        const CacheOutcome o = m->cache->access(ExpertCacheIndex::key(tb, ids[i]), m->cache_seq++);
        unsigned char *w = dst + (size_t)i * rec;
        if (o.hit) {
            PG_CUDA(cudaMemcpyAsync(w, m->cache_region + (size_t)o.slot * rec, rec, cudaMemcpyDeviceToDevice, m->copy));
            m->stats.d2d_bytes += (int64_t)rec;
            continue;
        }
        ++miss;
        PG_CUDA(cudaMemcpyAsync(w, src + (size_t)ids[i] * rec, rec, cudaMemcpyHostToDevice, m->copy));
        m->stats.h2d_copies++;
        if (o.inserted) {
            PG_CUDA(cudaMemcpyAsync(m->cache_region + (size_t)o.slot * rec, w, rec, cudaMemcpyDeviceToDevice, m->copy));
            m->stats.d2d_bytes += (int64_t)rec;
        }
    }
    m->stats.cache_hits = m->cache->hits();
    m->stats.cache_misses = m->cache->misses();
    *misses = miss;
    return PGMOE_OK;
}

// Issue the H2D migration of block `tb`'s routed experts into slot `ri`
// (scheduler.py:287-330 `issue`, made real).  Waits on the host for K1's
// active list (pinned mirror), then enqueues one DMA per expert on the copy
// stream after the slot's previous consumer finished.
static int issue_fetch(pgmoe_model *m, int tb, int ri, int si) {
    const auto &c = m->cfg;
    RoutingBuf &rb = m->routing[ri];
    PG_CUDA(cudaEventSynchronize(m->routed[ri]));
    const int n = rb.act_host[c.num_experts];
    PG_REQUIRE(n >= 0 && n <= m->slot_experts, PGMOE_E_OOM,
               "block %d routes to %d experts but the HBM slot holds %d", tb, n, m->slot_experts);
    if (m->slot_used[si]) PG_CUDA(cudaStreamWaitEvent(m->copy, m->done[si], 0));
    if (!m->cp_a.empty()) PG_CUDA(cudaEventRecord(m->cp_a[tb], m->copy));
    tl_begin(m, "transfer", "fetch[" + std::to_string(n) + "]", tb, m->copy);
    unsigned char *dst = m->slots + (size_t)si * m->slot_capacity;
    const unsigned char *src = m->blocks[tb].experts;
    int misses = n;
    if (m->cache) {
        PG_TRY(fetch_cached(m, tb, rb.act_host, n, dst, &misses));
    } else {
        for (int i = 0; i < n;) {  // coalesce runs of consecutive experts into one DMA
            int j = i + 1;
            while (j < n && rb.act_host[j] == rb.act_host[j - 1] + 1) ++j;
            PG_CUDA(cudaMemcpyAsync(dst + (size_t)i * m->rec_bytes, src + (size_t)rb.act_host[i] * m->rec_bytes,
                                    (size_t)(j - i) * m->rec_bytes, cudaMemcpyHostToDevice, m->copy));
            m->stats.h2d_copies++;
            i = j;
        }
    }
    tl_end(m, m->copy);
    if (!m->cp_b.empty()) PG_CUDA(cudaEventRecord(m->cp_b[tb], m->copy));
    PG_CUDA(cudaEventRecord(m->ready[si], m->copy));
    m->stats.h2d_bytes += (int64_t)misses * (int64_t)m->rec_bytes;
    m->slot_used[si] = true;
    if ((int)m->nact_iter.size() == c.num_blocks) m->nact_iter[tb] = n;
    return PGMOE_OK;
}

// prefetch_all (scheduler.py:336-342): the whole expert set of block `tb`
// (one contiguous DMA of E records) into slot `ri`, indexed by expert id.
static int issue_fetch_all(pgmoe_model *m, int tb, int si) {
    const int E = m->e_local;
    if (m->slot_used[si]) PG_CUDA(cudaStreamWaitEvent(m->copy, m->done[si], 0));
    if (!m->cp_a.empty()) PG_CUDA(cudaEventRecord(m->cp_a[tb], m->copy));
    tl_begin(m, "transfer", "fetch[" + std::to_string(E) + "]", tb, m->copy);
    int misses = E;
    if (m->cache) {
        std::vector<int32_t> all(E);
        for (int e = 0; e < E; ++e) all[e] = e;
        PG_TRY(fetch_cached(m, tb, all.data(), E, m->slots + (size_t)si * m->slot_capacity, &misses));
    } else {
        PG_CUDA(cudaMemcpyAsync(m->slots + (size_t)si * m->slot_capacity, m->blocks[tb].experts,
                                (size_t)E * m->rec_bytes, cudaMemcpyHostToDevice, m->copy));
        m->stats.h2d_copies++;
    }
    tl_end(m, m->copy);
    if (!m->cp_b.empty()) PG_CUDA(cudaEventRecord(m->cp_b[tb], m->copy));
    PG_CUDA(cudaEventRecord(m->ready[si], m->copy));
    m->stats.h2d_bytes += (int64_t)misses * (int64_t)m->rec_bytes;
    m->slot_used[si] = true;
    if ((int)m->nact_iter.size() == m->cfg.num_blocks) m->nact_iter[tb] = E;
    return PGMOE_OK;
}

// Routing decision of block `target` into ring buffer `ri`: the gate (K1)
// on x, or — supplied decisions — the given ids/w of that block.
static int route_into(pgmoe_model *m, const float *x, int T, const void *G, int ri, bool mirror,
                      cudaStream_t s, const char *label, int block, const pgmoe_iteration_io &io, int target) {
    const auto &c = m->cfg;
    RoutingBuf &rb = m->routing[ri];
    tl_begin(m, "compute", label, block, s);
    if (io.ids_supplied) {
        const size_t o = (size_t)target * T * c.top_k;
        PG_TRY(pgmoe_route_from_decisions(io.ids_supplied + o, io.w_supplied + o, T, c.num_experts, c.top_k, &rb.r,
                                          reinterpret_cast<pgmoe_stream_t>(s)));
    } else {
        PG_TRY(pgmoe_gate_forward(x, T, c.d_model, G, m->wdtype, c.num_experts, c.top_k, &rb.r, m->route_ws,
                                  reinterpret_cast<pgmoe_stream_t>(s)));
    }
    tl_end(m, s);
    if (mirror) {
        PG_CUDA(cudaMemcpyAsync(rb.act_host, rb.r.act, sizeof(int32_t) * (c.num_experts + 1),
                                cudaMemcpyDeviceToHost, s));
        PG_CUDA(cudaEventRecord(m->routed[ri], s));
    }
    return PGMOE_OK;
}

// The pre-gate of block b, computed inside block b's tcgen05 launch (route
// workspace layout: counter @0, done flag @64, tile counters @256, partials
// after kFusedRouteHead).
static FusedRoute fused_route_args(pgmoe_model *m, const float *x, int T, const void *G, const pgmoe_routing &out,
                                   int parity) {
    const auto &c = m->cfg;
    FusedRoute r{};
    r.active = 1;
    r.gt_bf16 = m->wdtype == PGMOE_BF16;
    r.d = c.d_model;
    r.E = c.num_experts;
    r.T = T;
    r.k = c.top_k;
    route_bound_constants(r.d, &r.gam, &r.bscale);
    r.splits = fused_route_splits(T, c.d_model, device_sm_count());
    r.tiles = (T + kRouterTok - 1) / kRouterTok;
    r.x = x;
    r.G = G;
    r.out = out;
    char *ws = static_cast<char *>(m->route_ws);
    r.counter = reinterpret_cast<int *>(ws);
    r.done = reinterpret_cast<int *>(ws + 64 + 4 * (parity & 1));  // re-armed at its launch's exit
    r.tile_counter = reinterpret_cast<int *>(ws + 256);
    char *q = ws + kFusedRouteHead;
    r.plogit = reinterpret_cast<double *>(q);
    q += ((size_t)r.splits * T * c.num_experts * 8 + 255) & ~(size_t)255;
    r.pcmax = reinterpret_cast<float *>(q);
    q += ((size_t)r.tiles * r.splits * c.num_experts * 4 + 255) & ~(size_t)255;
    r.pxsum = reinterpret_cast<double *>(q);
    return r;
}

// Small batches: block 0's gate (K1) and operand pack, then ONE persistent
// launch runs every block (decode_tc.cu), the pre-gates included.
static int decode_iteration(pgmoe_model *m, const float *x_in, int T, float *y_out, const pgmoe_iteration_io &io,
                            cudaStream_t s) {
    const auto &c = m->cfg;
    const int nb = c.num_blocks;
    PG_CUDA(cudaMemsetAsync(m->dec_sync, 0, (size_t)nb * kDecodeSyncInts * 4, s));
    PG_TRY(route_into(m, x_in, T, m->blocks[0].gate, 0, false, s, "gate", 0, io, 0));
    PG_TRY(tc_pack_rows(x_in, m->routing[0].r.perm, T, c.d_model, 1, m->xb, s));
    DecodeArgs a{};
    a.T = T;
    a.d = c.d_model;
    a.f = c.d_ff;
    a.E = c.num_experts;
    a.nb = nb;
    a.blocks = m->dec_blocks;
    a.sync = m->dec_sync;
    a.x_in = x_in;
    a.y_out = y_out;
    a.xb = m->xb;
    a.hb = m->hb;
    a.mixb = m->mixb;
    a.route = fused_route_args(m, x_in, T, m->blocks[0].pre_gate, m->routing[1].r, 0);
    a.experts = m->blocks[0].experts;
    a.nrec = nb * c.num_experts;
    a.rec_bytes = m->rec_bytes;
    a.pool = m->dev_pool;
    a.pool_rows = (long long)(m->dev_pool_bytes / (2 * (size_t)c.d_model));
    a.x_trace = io.x_trace;
    a.ids_trace = io.ids_trace;
    a.w_trace = io.w_trace;
    tl_begin(m, "compute", "experts", 0, s);  // every block's experts, dense layers and pre-gates: one launch
    PG_TRY(decode_iteration_tc(a, s));
    tl_end(m, s);
    m->fused_blocks += nb;
    m->fused_routes += nb - 1;
    m->decode_iters++;
    return PGMOE_OK;
}

// Small batches, low-latency form: ONE persistent launch per decoder iteration
// (decode_ll.cu), block 0's gate included; its phases exchange LL words.
static int ll_decode_iteration(pgmoe_model *m, const float *x_in, int T, float *y_out, const pgmoe_iteration_io &io,
                               cudaStream_t s) {
    const auto &c = m->cfg;
    LLDecodeArgs a{};
    a.gate0 = m->blocks[0].gate;  // block 0's gate is routed inside the launch too: one launch per iteration
    a.gate0_out = m->routing[0].r;
    a.T = T;
    a.d = c.d_model;
    a.f = c.d_ff;
    a.E = c.num_experts;
    a.nb = c.num_blocks;
    a.blocks = m->dec_blocks;
    a.experts = m->blocks[0].experts;
    a.rec_bytes = m->rec_bytes;
    a.pool = reinterpret_cast<const uint16_t *>(m->dev_pool);
    a.x_in = x_in;
    a.y_out = y_out;
    a.ws = m->ll_ws;
    a.ws_bytes = m->ll_ws_bytes;
    a.x_trace = io.x_trace;
    a.ids_trace = io.ids_trace;
    a.w_trace = io.w_trace;
    tl_begin(m, "compute", "experts", 0, s);  // every block's experts, dense layers and pre-gates: one launch
    PG_TRY(ll_decode_iteration(a, s));
    tl_end(m, s);
    m->fused_blocks += c.num_blocks;
    m->fused_routes += c.num_blocks - 1;
    m->ll_iters++;
    return PGMOE_OK;
}

int decoder_iteration(pgmoe_model *m, const float *x_in, int T, float *y_out, const pgmoe_iteration_io &io,
                      cudaStream_t s) {
    const auto &c = m->cfg;
    int32_t *ids_trace = io.ids_trace;
    float *w_trace = io.w_trace;
    PG_REQUIRE((io.ids_supplied == nullptr) == (io.w_supplied == nullptr), PGMOE_E_ROUTING,
               "supplied decisions need both expert ids and combine weights");
    PG_REQUIRE(T >= 0 && T <= m->max_tokens, PGMOE_E_SHAPE, "T=%d exceeds max_tokens=%d", T,
               m->max_tokens);
    PG_REQUIRE(m->e_local == c.num_experts, PGMOE_E_CONFIG,
               "model holds experts [%d, %d) only: expert-parallel decoding runs through ep.py", m->e_begin,
               m->e_begin + m->e_local);
    if (T == 0) return PGMOE_OK;
    const int L = c.activation_level, R = L + 1, nb = c.num_blocks;
    const int NS = std::max(1, m->nslots);  // expert slots (offloaded)
    const bool off = m->placement == PGMOE_OFFLOADED;
    const size_t tk = (size_t)T * c.top_k;
    if (m->timeline && !m->t0_recorded) {  // events accumulate until set_timeline() resets them
        PG_CUDA(cudaEventRecord(m->t0, s));
        m->t0_recorded = true;
    }
    if (off) m->nact_iter.assign(nb, 0);
    // Migration policy (scheduler.py:287-373), offloaded placement only:
    //   pre_gated    : block b+L's routed experts leave as soon as K1 decides
    //                  them, overlapping block b; block 0's fetch is exposed
    //   on_demand    : block b's routed experts are fetched when block b
    //                  starts, serial with its compute
    //   prefetch_all : block b+1's whole expert set streams during block b;
    //                  block 0's set is an exposed head transfer
    const int strat = off ? m->strategy : PGMOE_PRE_GATED;
    const bool prefetch_all = off && strat == PGMOE_PREFETCH_ALL;
    bool xb_ready = false;
    // Resident top-1 blocks compute their pre-gate inside the block launch
    // (it depends only on the block input); offloaded blocks keep the
    // separate K1 launch because the host needs the active list at once.
    // The routing role (4 warps per CTA) keeps up with the expert GEMMs while
    // its work (~T·d·E fp64 FMAs + the permutation) is small next to theirs
    // (~E·d·f weight bytes): measured crossover T ≈ f/8 (Base-64 fused
    // better through T=384, separate at 512; Large-128 fused through 768,
    // even at 1024; tools/gpu_env_sweep.sh VAR=PGMOE_FUSE_MAX_T).
    // (any lookahead L >= 1: block b's launch routes block b+L into ring entry (b+L) % (L+1))
    const bool fuse_route = !off && !io.ids_supplied && use_tc(m) && c.top_k == 1 && L >= 1 && m->fuse_route &&
                            fused_route_supported(c.num_experts) &&
                            (long long)T <= (m->fuse_max_t > 0 ? m->fuse_max_t : c.d_ff / 8);
    if (m->ll_decode && m->ll_ws && !off && !io.ids_supplied && use_tc(m) && m->fuse_route && T <= m->ll_max_t &&
        ll_decode_supported(T, c.d_model, c.d_ff, c.num_experts, c.top_k, L, nb))
        return ll_decode_iteration(m, x_in, T, y_out, io, s);
    if (m->decode && m->dec_blocks && !off && !io.ids_supplied && use_tc(m) && m->fuse_route &&
        T <= m->decode_max_t && decode_supported(T, c.d_model, c.d_ff, c.num_experts, c.top_k, L, nb))
        return decode_iteration(m, x_in, T, y_out, io, s);
    const float *cur = x_in;
    // Chained block launches (fused routing): each launch waits for its
    // predecessor's dense phase through a device counter instead of for its
    // completion; the counter restarts every iteration.
    const bool chain = fuse_route && m->chain_launches;
    if (chain) PG_CUDA(cudaMemsetAsync(m->epoch, 0, sizeof(int), s));
    for (int b = 0; b < nb; ++b) {
        const BlockW &bw = m->blocks[b];
        const int ri = b % R;   // routing buffer of the decision block b consumes
        const int si = b % NS;  // expert slot of block b (offloaded)
        int pending_fetch = -1;
        if (prefetch_all) {  // NS >= 2: block b+1's set never lands in the slot block b reads
            if (b == 0) PG_TRY(issue_fetch_all(m, 0, 0));
            if (b + 1 < nb) PG_TRY(issue_fetch_all(m, b + 1, (b + 1) % NS));
        }
        if (io.x_trace)  // the block input, for teacher-forced parity at this exact launch sequence
            PG_CUDA(cudaMemcpyAsync(io.x_trace + (size_t)b * T * c.d_model, cur, (size_t)T * c.d_model * 4,
                                    cudaMemcpyDeviceToDevice, s));
        if (has_conv_gate(c, b)) {
            PG_TRY(route_into(m, cur, T, bw.gate, ri, off && !prefetch_all, s, "gate", b, io, b));
            if (off && strat == PGMOE_PRE_GATED) PG_TRY(issue_fetch(m, b, ri, si));  // exposed serial fetch
        }
        FusedRoute fr{};
        if (has_pre_gate(c, b)) {
            const int tr = (b + L) % R;
            if (fuse_route) {
                fr = fused_route_args(m, cur, T, bw.pre_gate, m->routing[tr].r, b & 1);
            } else {
                PG_TRY(route_into(m, cur, T, bw.pre_gate, tr, off && !prefetch_all, s, "pre_gate", b, io, b + L));
            }
            if (off && strat == PGMOE_PRE_GATED) pending_fetch = b + L;
        }
        if (off && strat == PGMOE_ON_DEMAND) {  // fetch starts once compute reaches block b
            PG_CUDA(cudaEventRecord(m->gated, s));
            PG_CUDA(cudaStreamWaitEvent(m->copy, m->gated, 0));
            PG_TRY(issue_fetch(m, b, ri, si));
        }
        const RoutingBuf &rb = m->routing[ri];
        const void *experts = off ? (const void *)(m->slots + (size_t)si * m->slot_capacity)
                                  : (const void *)bw.experts;
        if (off) PG_CUDA(cudaStreamWaitEvent(s, m->ready[si], 0));
        float *nxt = (b == nb - 1) ? y_out : m->act_buf[b & 1];
        // Pre-gating at work: block b+1's routing is already on the device
        // (unless b+1 carries a conventional gate), so this block's dense
        // epilogue also writes b+1's packed up-projection operand.
        const bool fuse_next = use_tc(m) && b + 1 < nb && !has_conv_gate(c, b + 1);
        const pgmoe_routing *next_r = fuse_next ? &m->routing[(b + 1) % R].r : nullptr;
        const int indexed = (off && !prefetch_all) ? 1 : 0;
        LaunchChain lc{m->epoch, b > 0 ? b : 0, b + 1, b & 1,
                       reinterpret_cast<unsigned long long *>(reinterpret_cast<char *>(m->epoch) + 256)};
        if (use_tc(m) && c.top_k == 1) {
            // one launch: up, down(+combine), dense — phases behind grid barriers
            tl_begin(m, "compute", "experts", b, s);
            PG_TRY(block_tc(cur, T, c.d_model, c.d_ff, 1, experts, m->rec_bytes, indexed, &rb.r, m->xb, m->hb, m->yw,
                            m->mixb, xb_ready, bw.dense, nxt, next_r ? m->xb : nullptr, next_r ? next_r->inv : nullptr,
                            m->tc_ws, m->tc_ws_bytes, s, fr.active ? &fr : nullptr,
                            chain ? &lc : nullptr, m->e_local));
            if (fr.active) m->fused_routes++;
            tl_end(m, s);
            if (off) {
                PG_CUDA(cudaEventRecord(m->done[si], s));
                if (!m->ffn_b.empty()) PG_CUDA(cudaEventRecord(m->ffn_b[b], s));
            }
            tl_begin(m, "compute", "non_moe", b, s);  // fused into the launch above
            tl_end(m, s);
            m->fused_blocks++;
        } else {
            tl_begin(m, "compute", "experts", b, s);
            PG_TRY(run_ffn(m, cur, T, experts, indexed, &rb.r, s, xb_ready));
            tl_end(m, s);
            if (off) {
                PG_CUDA(cudaEventRecord(m->done[si], s));
                if (!m->ffn_b.empty()) PG_CUDA(cudaEventRecord(m->ffn_b[b], s));
            }
            tl_begin(m, "compute", "non_moe", b, s);
            PG_TRY(run_dense(m, T, bw.dense, nxt, s, next_r));
            tl_end(m, s);
        }
        xb_ready = fuse_next;
        if (ids_trace) {
            PG_CUDA(cudaMemcpyAsync(ids_trace + (size_t)b * tk, rb.r.ids, tk * 4, cudaMemcpyDeviceToDevice, s));
            PG_CUDA(cudaMemcpyAsync(w_trace + (size_t)b * tk, rb.r.w, tk * 4, cudaMemcpyDeviceToDevice, s));
        }
        if (pending_fetch >= 0) PG_TRY(issue_fetch(m, pending_fetch, pending_fetch % R, pending_fetch % NS));
        cur = nxt;
    }
    return PGMOE_OK;
}

}  // namespace pgmoe

// =============================================================== C ABI ====

extern "C" const char *pgmoe_last_error(void) { return g_last_error.c_str(); }
extern "C" const char *pgmoe_version(void) { return "pgmoe-b200 0.1.0 (sm_100a)"; }
extern "C" int64_t pgmoe_launch_count(void) { return g_launches.load(); }
extern "C" int pgmoe_debug_set_probe(int32_t kind, void *device_buffer, int64_t rows) {
    PG_REQUIRE(kind >= 0 && kind < 2, PGMOE_E_CONFIG, "probe kind %d", kind);
    g_probe[kind] = static_cast<unsigned long long *>(device_buffer);
    g_probe_rows[kind] = device_buffer ? rows : 0;
    g_probe_next[kind] = 0;
    return PGMOE_OK;
}

// Debug: a green context of at least `min_sms` SMs (cuDevSmResourceSplitByCount)
// made current on the calling thread, so the persistent kernels can be run on
// a context with fewer co-resident CTAs than the device has SMs.
extern "C" int pgmoe_debug_green_context(int32_t min_sms, int32_t *sms_out) {
#define PG_DRV(name)                                                                                      \
    decltype(&name) p_##name = nullptr;                                                                   \
    {                                                                                                     \
        void *fp = nullptr;                                                                               \
        cudaDriverEntryPointQueryResult q;                                                                \
        if (cudaGetDriverEntryPoint(#name, &fp, cudaEnableDefault, &q) != cudaSuccess ||                  \
            q != cudaDriverEntryPointSuccess) {                                                           \
            set_error("driver entry point %s unavailable", #name);                                       \
            return PGMOE_E_CUDA;                                                                          \
        }                                                                                                 \
        p_##name = reinterpret_cast<decltype(&name)>(fp);                                                 \
    }
    PG_DRV(cuDeviceGetDevResource)
    PG_DRV(cuDevSmResourceSplitByCount)
    PG_DRV(cuDevResourceGenerateDesc)
    PG_DRV(cuGreenCtxCreate)
    PG_DRV(cuCtxFromGreenCtx)
    PG_DRV(cuCtxSetCurrent)
#undef PG_DRV
    const CUdevice dev = (CUdevice)current_device();
    CUdevResource input, result, remaining;
    memset(&input, 0, sizeof(input));
    memset(&result, 0, sizeof(result));
    memset(&remaining, 0, sizeof(remaining));
    unsigned int n = 1;
    CUdevResourceDesc desc = nullptr;
    CUgreenCtx g = nullptr;
    CUcontext ctx = nullptr;
    CUresult r = p_cuDeviceGetDevResource(dev, &input, CU_DEV_RESOURCE_TYPE_SM);
    if (r == CUDA_SUCCESS) r = p_cuDevSmResourceSplitByCount(&result, &n, &input, &remaining, 0, (unsigned)min_sms);
    if (r == CUDA_SUCCESS) r = p_cuDevResourceGenerateDesc(&desc, &result, 1);
    if (r == CUDA_SUCCESS) r = p_cuGreenCtxCreate(&g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM);
    if (r == CUDA_SUCCESS) r = p_cuCtxFromGreenCtx(&ctx, g);
    if (r == CUDA_SUCCESS) r = p_cuCtxSetCurrent(ctx);
    PG_REQUIRE(r == CUDA_SUCCESS, PGMOE_E_CUDA, "green context of %d SMs failed (CUresult %d)", min_sms, (int)r);
    if (sms_out) *sms_out = (int32_t)result.sm.smCount;
    return PGMOE_OK;
}

// Workspaces of the standalone (model-less) tcgen05 entry points: split-K
// tickets and partials, re-armed by each launch's last CTA, so calls that
// share one must be stream-ordered.  Allocated once per process, under a
// lock (EP ranks may be threads of one process).
// One set per device: models or EP ranks on other GPUs of the same process
// must not share device-0 memory.
constexpr size_t kSharedWsBytes = 64ull << 20;
static int shared_tc_ws(int slot, void **out) {
    static std::mutex mu;
    static void *ws[64][3] = {};
    const int dev = current_device();
    PG_REQUIRE(dev >= 0 && dev < 64, PGMOE_E_CONFIG, "device ordinal %d unsupported", dev);
    std::lock_guard<std::mutex> lock(mu);
    if (!ws[dev][slot]) {
        void *p = nullptr;
        PG_CUDA(cudaMalloc(&p, kSharedWsBytes));
        PG_CUDA(cudaMemset(p, 0, kSharedWsBytes));
        PG_CUDA(cudaDeviceSynchronize());
        ws[dev][slot] = p;
    }
    *out = ws[dev][slot];
    return PGMOE_OK;
}

extern "C" int pgmoe_expert_forward(const float *x, int32_t T, int32_t d, int32_t f, int32_t k,
                                    const void *experts, size_t expert_stride, int32_t wdtype,
                                    int32_t indexed_by_act, const pgmoe_routing *r, float *h, float *yw,
                                    int32_t kernel, pgmoe_stream_t stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (T == 0) return PGMOE_OK;
    const bool tc = wdtype == PGMOE_BF16 && kernel != PGMOE_KERNEL_SIMT && tc_supported(d, f);
    if (kernel == PGMOE_KERNEL_TCGEN05)
        PG_REQUIRE(tc, PGMOE_E_CONFIG, "tcgen05 kernels need bf16 weights and d, f multiples of 128");
    if (tc) {
        void *ws = nullptr;
        const size_t ws_bytes = kSharedWsBytes;
        PG_TRY(shared_tc_ws(0, &ws));
        return expert_ffn_tc(x, T, d, f, k, experts, expert_stride, indexed_by_act, r, h, yw, ws, ws_bytes, s);
    }
    return expert_ffn_simt(x, T, d, f, k, experts, expert_stride, wdtype, indexed_by_act, r, h, yw, s);
}

extern "C" int pgmoe_expert_forward_packed(const uint16_t *xb, int32_t n_max, int32_t d, int32_t f,
                                           const void *experts, size_t expert_stride, const pgmoe_routing *r,
                                           uint16_t *hb, float *y, pgmoe_stream_t stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (n_max == 0) return PGMOE_OK;
    PG_REQUIRE(tc_supported(d, f), PGMOE_E_CONFIG, "tcgen05 kernels need d, f multiples of 128");
    void *ws = nullptr;
    const size_t ws_bytes = kSharedWsBytes;
    PG_TRY(shared_tc_ws(1, &ws));
    return expert_ffn_tc2(nullptr, n_max, d, f, 1, experts, expert_stride, 0, r, const_cast<uint16_t *>(xb), hb, y,
                          nullptr, ws, ws_bytes, s, true);
}

extern "C" int pgmoe_dense_forward(const float *yw, int32_t T, int32_t d, int32_t k, const void *dense_w,
                                   int32_t wdtype, float *y, int32_t kernel, pgmoe_stream_t stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (T == 0) return PGMOE_OK;
    const bool tc = wdtype == PGMOE_BF16 && kernel != PGMOE_KERNEL_SIMT && d % 128 == 0;
    if (kernel == PGMOE_KERNEL_TCGEN05)
        PG_REQUIRE(tc, PGMOE_E_CONFIG, "tcgen05 dense needs bf16 weights and d multiple of 128");
    if (tc) {
        void *ws = nullptr;
        const size_t ws_bytes = kSharedWsBytes;
        PG_TRY(shared_tc_ws(2, &ws));
        return dense_tc(yw, T, d, k, dense_w, y, ws, ws_bytes, s);
    }
    return dense_simt(yw, T, d, k, dense_w, wdtype, y, s);
}

extern "C" int pgmoe_dense_forward_packed(const uint16_t *mixb, int32_t T, int32_t d, const void *dense_w,
                                          float *y, pgmoe_stream_t stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (T == 0) return PGMOE_OK;
    PG_REQUIRE(d % 128 == 0, PGMOE_E_CONFIG, "tcgen05 dense needs d multiple of 128");
    void *ws = nullptr;
    PG_TRY(shared_tc_ws(2, &ws));
    return dense_tc2(nullptr, mixb, T, d, 1, dense_w, y, nullptr, ws, kSharedWsBytes, s, nullptr, nullptr);
}

extern "C" int pgmoe_model_create(const pgmoe_config *cfg, int32_t wdtype, int32_t placement,
                                  int32_t max_tokens, pgmoe_model **out) {
    PG_TRY(validate_config(cfg));
    return pgmoe_model_create_ex(cfg, wdtype, placement, max_tokens, 0, cfg->num_experts, out);
}

extern "C" int pgmoe_model_create_ex(const pgmoe_config *cfg, int32_t wdtype, int32_t placement,
                                     int32_t max_tokens, int32_t expert_begin, int32_t expert_end,
                                     pgmoe_model **out) {
    PG_TRY(validate_config(cfg));
    PG_REQUIRE(0 <= expert_begin && expert_begin < expert_end && expert_end <= cfg->num_experts, PGMOE_E_CONFIG,
               "expert range [%d, %d) outside [0, %d)", expert_begin, expert_end, cfg->num_experts);
    PG_REQUIRE(out != nullptr, PGMOE_E_CONFIG, "null output handle");
    PG_REQUIRE(wdtype == PGMOE_F32 || wdtype == PGMOE_BF16, PGMOE_E_CONFIG, "unknown weight dtype %d", wdtype);
    PG_REQUIRE(placement == PGMOE_RESIDENT || placement == PGMOE_OFFLOADED, PGMOE_E_CONFIG,
               "unknown placement %d", placement);
    PG_REQUIRE(max_tokens >= 1, PGMOE_E_CONFIG, "max_tokens must be >= 1");
    auto *m = new pgmoe_model();
    m->cfg = *cfg;
    m->wdtype = wdtype;
    m->placement = placement;
    m->max_tokens = max_tokens;
    m->e_begin = expert_begin;
    m->e_local = expert_end - expert_begin;
    const auto &c = m->cfg;
    const size_t d = c.d_model, f = c.d_ff, E = m->e_local, nb = c.num_blocks, k = c.top_k;
    m->sw = dtype_bytes(wdtype);
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    m->gate_bytes = al(d * (size_t)c.num_experts * m->sw);  // gates span all experts, also on an EP shard
    m->dense_bytes = al(d * d * m->sw);
    m->w1_bytes = f * d * m->sw;
    m->rec_bytes = al(2 * f * d * m->sw);
    m->blocks.resize(nb);
    size_t pinned = 0;
    for (size_t b = 0; b < nb; ++b)
        pinned += (has_conv_gate(c, b) + has_pre_gate(c, b)) * m->gate_bytes + m->dense_bytes;
    const size_t experts_all = nb * E * m->rec_bytes;
    m->dev_pool_bytes = pinned + (placement == PGMOE_RESIDENT ? experts_all : 0);
    int st = PGMOE_OK;
    auto fail = [&](int code) {
        pgmoe_model_destroy(m);
        return code;
    };
    if (cudaMalloc(&m->dev_pool, m->dev_pool_bytes) != cudaSuccess) {
        set_error("OOM: %zu B of HBM for %s weights", m->dev_pool_bytes,
                  placement == PGMOE_RESIDENT ? "resident" : "pinned (gate/dense)");
        return fail(PGMOE_E_OOM);
    }
    unsigned char *p = m->dev_pool;
    for (size_t b = 0; b < nb; ++b) {
        BlockW &bw = m->blocks[b];
        if (has_conv_gate(c, b)) { bw.gate = p; p += m->gate_bytes; }
        if (has_pre_gate(c, b)) { bw.pre_gate = p; p += m->gate_bytes; }
        bw.dense = p;
        p += m->dense_bytes;
    }
    if (placement == PGMOE_RESIDENT) {
        for (size_t b = 0; b < nb; ++b) { m->blocks[b].experts = p; p += E * m->rec_bytes; }
    } else {
        m->host_pool_bytes = experts_all;
        if (cudaHostAlloc(&m->host_pool, experts_all, cudaHostAllocDefault) != cudaSuccess) {
            set_error("cannot pin %zu B of host memory for offloaded experts", experts_all);
            return fail(PGMOE_E_OOM);
        }
        for (size_t b = 0; b < nb; ++b) m->blocks[b].experts = m->host_pool + b * E * m->rec_bytes;
        const int R = c.activation_level + 1;
        m->nslots = R;
        m->slot_experts = (int)std::min<size_t>(E, (size_t)max_tokens * k);
        m->slot_capacity = (size_t)m->slot_experts * m->rec_bytes;
        if (cudaMalloc(&m->slots, m->slot_capacity * R) != cudaSuccess) {
            set_error("OOM: %zu B of HBM for %d expert slots", m->slot_capacity * R, R);
            return fail(PGMOE_E_OOM);
        }
        if (cudaStreamCreateWithFlags(&m->copy, cudaStreamNonBlocking) != cudaSuccess) return fail(PGMOE_E_CUDA);
        m->ready.resize(R); m->done.resize(R); m->slot_used.assign(R, false);
        cudaEventCreateWithFlags(&m->gated, cudaEventDisableTiming);
        for (int i = 0; i < R; ++i) {
            cudaEventCreateWithFlags(&m->ready[i], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&m->done[i], cudaEventDisableTiming);
        }
        m->cp_a.resize(nb); m->cp_b.resize(nb); m->ffn_b.resize(nb);
        for (size_t b = 0; b < nb; ++b) {
            cudaEventCreate(&m->cp_a[b]); cudaEventCreate(&m->cp_b[b]); cudaEventCreate(&m->ffn_b[b]);
        }
    }
    const int R = c.activation_level + 1;
    m->routing.resize(R);
    m->routed.resize(R);
    for (int i = 0; i < R; ++i) {
        if ((st = alloc_routing(m->routing[i], max_tokens, c.num_experts, (int)k)) != PGMOE_OK) return fail(st);
        cudaEventCreateWithFlags(&m->routed[i], cudaEventDisableTiming);
    }
    // every routing buffer's status words side by side: the host-buffer entry
    // point fetches them with one copy
    if (cudaMalloc(&m->status_dev, (size_t)R * 4 * sizeof(int32_t)) != cudaSuccess ||
        cudaMemset(m->status_dev, 0, (size_t)R * 4 * sizeof(int32_t)) != cudaSuccess)
        return fail(PGMOE_E_OOM);
    for (int i = 0; i < R; ++i) m->routing[i].r.status = m->status_dev + 4 * i;
    size_t rws = pgmoe_route_workspace_bytes(max_tokens, c.num_experts);
    for (int t = 1; t <= max_tokens; ++t)  // the routing role fused into the block kernel (resident)
        rws = std::max(rws, kFusedRouteHead + fused_route_ws_bytes(t, d, c.num_experts, device_sm_count()));
    if (cudaMalloc(&m->route_ws, rws) != cudaSuccess || cudaMemset(m->route_ws, 0, rws) != cudaSuccess)
        return fail(PGMOE_E_OOM);
    const size_t T = max_tokens;
    if (cudaMalloc(&m->act_buf[0], T * d * 4) != cudaSuccess ||
        cudaMalloc(&m->act_buf[1], T * d * 4) != cudaSuccess ||
        cudaMalloc(&m->h, T * k * f * 4) != cudaSuccess || cudaMalloc(&m->yw, T * k * d * 4) != cudaSuccess ||
        cudaMalloc(&m->xb, T * k * d * 2) != cudaSuccess || cudaMalloc(&m->hb, T * k * f * 2) != cudaSuccess ||
        cudaMalloc(&m->mixb, T * d * 2) != cudaSuccess) {
        set_error("OOM: activation buffers for max_tokens=%d", max_tokens);
        return fail(PGMOE_E_OOM);
    }
    m->tc_ws_bytes = 64ull << 20;
    if (cudaMalloc(&m->tc_ws, m->tc_ws_bytes) != cudaSuccess || cudaMemset(m->tc_ws, 0, m->tc_ws_bytes) != cudaSuccess)
        return fail(PGMOE_E_OOM);
    // [0] launch-chain epoch; bytes 256..: dense-end stamps per block (pgmoe_model_block_stamps)
    if (cudaMalloc(&m->epoch, 1024) != cudaSuccess || cudaMemset(m->epoch, 0, 1024) != cudaSuccess)
        return fail(PGMOE_E_OOM);
    if (const char *e = getenv("PGMOE_CHAIN")) m->chain_launches = (e[0] != '0');
    if (const char *e = getenv("PGMOE_FUSED_ROUTE")) m->fuse_route = (e[0] == '1');
    if (const char *e = getenv("PGMOE_FUSE_MAX_T")) m->fuse_max_t = atoll(e);
    if (const char *e = getenv("PGMOE_DECODE")) m->decode = (e[0] != '0');
    if (const char *e = getenv("PGMOE_DECODE_MAX_T")) m->decode_max_t = std::max(0, std::min(kDecodeMaxT, atoi(e)));
    if (placement == PGMOE_RESIDENT && wdtype == PGMOE_BF16 && m->e_local == c.num_experts &&
        decode_supported(1, (int)d, (int)f, c.num_experts, (int)k, c.activation_level, (int)nb) &&
        m->dev_pool_bytes % (2 * d) == 0) {
        std::vector<DecodeBlock> db(nb);
        for (size_t b = 0; b < nb; ++b) {
            const pgmoe_routing &r = m->routing[b % 2].r;
            DecodeBlock &x = db[b];
            x.act = r.act; x.n_act = r.n_act; x.hist = r.hist; x.off = r.off; x.perm = r.perm; x.inv = r.inv;
            x.w_perm = r.w_perm; x.ids = r.ids; x.w = r.w;
            x.next_inv = b + 1 < nb ? m->routing[(b + 1) % 2].r.inv : nullptr;
            x.wrec0 = (int)(b * E);
            x.dense_row0 = (int)((static_cast<unsigned char *>(m->blocks[b].dense) - m->dev_pool) / (2 * d));
            x.has_pre_gate = has_pre_gate(c, (int)b) ? 1 : 0;
            x.x = b >= 1 ? m->act_buf[(b - 1) & 1] : nullptr;
            x.y = b + 1 < nb ? m->act_buf[b & 1] : nullptr;
            x.pre_gate = m->blocks[b].pre_gate;
            x.out = m->routing[(b + 1) % 2].r;
        }
        if (cudaMalloc(&m->dec_blocks, nb * sizeof(DecodeBlock)) != cudaSuccess ||
            cudaMemcpy(m->dec_blocks, db.data(), nb * sizeof(DecodeBlock), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMalloc(&m->dec_sync, nb * kDecodeSyncInts * 4) != cudaSuccess ||
            cudaMemset(m->dec_sync, 0, nb * kDecodeSyncInts * 4) != cudaSuccess)
            return fail(PGMOE_E_OOM);
        if (ll_decode_supported(1, (int)d, (int)f, c.num_experts, (int)k, c.activation_level, (int)nb)) {
            const int tmax = std::min(max_tokens, kLLMaxT);
            m->ll_ws_bytes = ll_decode_ws_bytes(tmax, (int)d, (int)f, c.num_experts, (int)nb);
            if (cudaMalloc(&m->ll_ws, m->ll_ws_bytes) != cudaSuccess ||
                cudaMemset(m->ll_ws, 0, m->ll_ws_bytes) != cudaSuccess)
                return fail(PGMOE_E_OOM);
            m->ll_max_t = tmax;
            if ((st = ll_decode_prepare(m->ll_ws, nullptr)) != PGMOE_OK)
                return fail(st);
        }
    }
    if (const char *e = getenv("PGMOE_LLDECODE")) m->ll_decode = (e[0] != '0');
    if (const char *e = getenv("PGMOE_LLDECODE_MAX_T")) m->ll_max_t = std::max(0, std::min(m->ll_max_t, atoi(e)));
    cudaEventCreate(&m->t0);
    m->stats.pinned_hbm_bytes = (int64_t)pinned;
    m->stats.slot_capacity_bytes = (int64_t)m->slot_capacity;
    if (const char *e = getenv("PGMOE_NO_GRAPH")) m->use_graph = (e[0] == '0');
    *out = m;
    return PGMOE_OK;
}

extern "C" int pgmoe_model_destroy(pgmoe_model *m) {
    if (!m) return PGMOE_OK;
    cudaDeviceSynchronize();
    for (auto &rb : m->routing) {
        if (rb.mem) cudaFree(rb.mem);
        if (rb.act_host) cudaFreeHost(rb.act_host);
    }
    for (auto e : m->ready) cudaEventDestroy(e);
    for (auto e : m->done) cudaEventDestroy(e);
    for (auto e : m->routed) cudaEventDestroy(e);
    if (m->gated) cudaEventDestroy(m->gated);
    for (auto e : m->cp_a) cudaEventDestroy(e);
    for (auto e : m->cp_b) cudaEventDestroy(e);
    for (auto e : m->ffn_b) cudaEventDestroy(e);
    for (auto &e : m->tl) { cudaEventDestroy(e.a); cudaEventDestroy(e.b); }
    if (m->t0) cudaEventDestroy(m->t0);
    delete m->cache;
    cudaFree(m->cache_region);
    for (auto &g : m->graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    if (m->io_stream) cudaStreamDestroy(m->io_stream);
    cudaFree(m->io_x);
    cudaFree(m->io_y);
    cudaFree(m->io_ids);
    cudaFree(m->io_w);
    if (m->io_status) cudaFreeHost(m->io_status);
    if (m->status_dev) cudaFree(m->status_dev);
    if (m->cap) cudaStreamDestroy(m->cap);
    if (m->copy) cudaStreamDestroy(m->copy);
    cudaFree(m->dev_pool);
    if (m->host_pool) cudaFreeHost(m->host_pool);
    cudaFree(m->slots);
    cudaFree(m->route_ws);
    cudaFree(m->dec_blocks);
    cudaFree(m->dec_sync);
    cudaFree(m->ll_ws);
    cudaFree(m->tc_ws);
    cudaFree(m->epoch);
    cudaFree(m->act_buf[0]);
    cudaFree(m->act_buf[1]);
    cudaFree(m->h);
    cudaFree(m->yw);
    cudaFree(m->xb);
    cudaFree(m->hb);
    cudaFree(m->mixb);
    delete m;
    return PGMOE_OK;
}

extern "C" int pgmoe_model_config(pgmoe_model *m, pgmoe_config *cfg, int32_t *wdtype) {
    PG_REQUIRE(m != nullptr, PGMOE_E_CONFIG, "null model");
    if (cfg) *cfg = m->cfg;
    if (wdtype) *wdtype = m->wdtype;
    return PGMOE_OK;
}

extern "C" int pgmoe_model_set_strategy(pgmoe_model *m, int32_t strategy) {
    PG_REQUIRE(m != nullptr, PGMOE_E_CONFIG, "null model");
    PG_REQUIRE(strategy >= PGMOE_PRE_GATED && strategy <= PGMOE_PREFETCH_ALL, PGMOE_E_CONFIG,
               "unknown strategy %d", strategy);
    PG_REQUIRE(m->placement == PGMOE_OFFLOADED, PGMOE_E_CONFIG, "migration strategies need an offloaded model");
    PG_REQUIRE(strategy != PGMOE_PRE_GATED || m->cfg.activation_level >= 1, PGMOE_E_CONFIG,
               "pre_gated strategy requires a model with activation_level >= 1");
    std::lock_guard<std::mutex> g(m->mu);
    // prefetch_all: slots hold a whole block, and there are at least two of
    // them (block b+1's set streams in while block b reads its own)
    const int ns_need = std::max(m->cfg.activation_level + 1, 2);
    if (strategy == PGMOE_PREFETCH_ALL && (m->slot_experts < m->e_local || m->nslots < ns_need)) {
        PG_CUDA(cudaDeviceSynchronize());
        const size_t cap = (size_t)m->e_local * m->rec_bytes;
        unsigned char *ns = nullptr;
        if (cudaMalloc(&ns, cap * ns_need) != cudaSuccess) {
            set_error("OOM: %zu B of HBM for %d whole-block expert slots", cap * ns_need, ns_need);
            return PGMOE_E_OOM;
        }
        cudaFree(m->slots);
        m->slots = ns;
        m->slot_capacity = cap;
        m->slot_experts = m->e_local;
        m->stats.slot_capacity_bytes = (int64_t)cap;
        for (int i = m->nslots; i < ns_need; ++i) {
            m->ready.push_back(nullptr);
            m->done.push_back(nullptr);
            cudaEventCreateWithFlags(&m->ready.back(), cudaEventDisableTiming);
            cudaEventCreateWithFlags(&m->done.back(), cudaEventDisableTiming);
        }
        m->nslots = ns_need;
        m->slot_used.assign(ns_need, false);
    }
    m->strategy = strategy;
    return PGMOE_OK;
}

extern "C" int pgmoe_model_set_cache(pgmoe_model *m, int32_t policy, double capacity_fraction) {
    PG_REQUIRE(m != nullptr, PGMOE_E_CONFIG, "null model");
    PG_REQUIRE(policy >= kCacheNone && policy <= kCacheLru, PGMOE_E_CONFIG, "unknown cache policy %d", policy);
    PG_REQUIRE(capacity_fraction >= 0.0 && capacity_fraction <= 1.0, PGMOE_E_CONFIG,
               "capacity_fraction must be in [0, 1]");
    PG_REQUIRE(m->placement == PGMOE_OFFLOADED, PGMOE_E_CONFIG, "the expert cache serves offloaded models");
    std::lock_guard<std::mutex> g(m->mu);
    PG_CUDA(cudaDeviceSynchronize());
    delete m->cache;
    m->cache = nullptr;
    cudaFree(m->cache_region);
    m->cache_region = nullptr;
    m->stats.cache_bytes = 0;
    if (policy == kCacheNone) return PGMOE_OK;
    // cache.py: capacity = fraction of all expert bytes (scheduler.py:269-271)
    const double total = (double)m->cfg.num_blocks * m->e_local * (double)(2.0 * m->cfg.d_model * m->cfg.d_ff *
                                                                          (double)m->sw);
    const int records = (int)((capacity_fraction * total) / (double)(2.0 * m->cfg.d_model * m->cfg.d_ff * m->sw));
    if (records > 0 && cudaMalloc(&m->cache_region, (size_t)records * m->rec_bytes) != cudaSuccess) {
        set_error("OOM: %d expert records of HBM cache", records);
        return PGMOE_E_OOM;
    }
    m->cache = new ExpertCacheIndex(records, policy);
    m->cache_seq = 0;
    m->stats.cache_bytes = (int64_t)records * (int64_t)m->rec_bytes;
    return PGMOE_OK;
}

extern "C" int pgmoe_cache_replay(int32_t policy, int32_t capacity_records, const int32_t *blocks,
                                  const int32_t *experts, int32_t n, int32_t *hit, int32_t *n_evicted) {
    PG_REQUIRE(policy >= kCacheLifo && policy <= kCacheLru, PGMOE_E_CONFIG, "unknown cache policy %d", policy);
    ExpertCacheIndex c(capacity_records, policy);
    for (int i = 0; i < n; ++i) {
        const CacheOutcome o = c.access(ExpertCacheIndex::key(blocks[i], experts[i]), i);
        hit[i] = o.hit ? 1 : 0;
        n_evicted[i] = (int32_t)o.evicted.size();
    }
    return PGMOE_OK;
}

// Captured decoder graphs bake the launch sequence: drop them when it changes.
static void drop_graphs(pgmoe_model *m) {
    cudaDeviceSynchronize();
    for (auto &g : m->graphs) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        g = pgmoe_model::GraphEntry{};
    }
}

extern "C" int pgmoe_model_set_kernel(pgmoe_model *m, int32_t kernel) {
    PG_REQUIRE(kernel >= PGMOE_KERNEL_AUTO && kernel <= PGMOE_KERNEL_TCGEN05, PGMOE_E_CONFIG, "bad kernel %d", kernel);
    if (m->kernel != kernel) drop_graphs(m);
    m->kernel = kernel;
    return PGMOE_OK;
}

extern "C" int pgmoe_model_set_fused_route(pgmoe_model *m, int32_t enabled) {
    PG_REQUIRE(m != nullptr, PGMOE_E_CONFIG, "null model");
    if (m->fuse_route != (enabled != 0)) drop_graphs(m);
    m->fuse_route = enabled != 0;
    return PGMOE_OK;
}

extern "C" int pgmoe_model_set_decode(pgmoe_model *m, int32_t enabled, int32_t max_tokens) {
    PG_REQUIRE(m != nullptr, PGMOE_E_CONFIG, "null model");
    PG_REQUIRE(max_tokens >= 0 && max_tokens <= kDecodeMaxT, PGMOE_E_CONFIG,
               "decode kernel serves 1..%d tokens per iteration", kDecodeMaxT);
    drop_graphs(m);
    m->decode = enabled != 0;
    if (max_tokens > 0) m->decode_max_t = max_tokens;
    return PGMOE_OK;
}

extern "C" int64_t pgmoe_model_decode_iterations(pgmoe_model *m) { return m ? m->decode_iters : 0; }

extern "C" int pgmoe_model_set_ll_decode(pgmoe_model *m, int32_t enabled, int32_t max_tokens) {
    PG_REQUIRE(m != nullptr, PGMOE_E_CONFIG, "null model");
    PG_REQUIRE(max_tokens >= 0 && max_tokens <= kLLMaxT, PGMOE_E_CONFIG,
               "low-latency decoder serves 1..%d tokens per iteration", kLLMaxT);
    drop_graphs(m);
    m->ll_decode = enabled != 0;
    if (max_tokens > 0) m->ll_max_t = max_tokens;
    return PGMOE_OK;
}

extern "C" int64_t pgmoe_model_ll_decode_iterations(pgmoe_model *m) { return m ? m->ll_iters : 0; }

extern "C" int pgmoe_model_block_stamps(pgmoe_model *m, int64_t *out, int32_t n) {
    PG_REQUIRE(m != nullptr && out != nullptr, PGMOE_E_CONFIG, "null argument");
    PG_REQUIRE(n >= 0 && n <= 96, PGMOE_E_CONFIG, "at most 96 stamps");
    PG_CUDA(cudaDeviceSynchronize());
    PG_CUDA(cudaMemcpy(out, reinterpret_cast<char *>(m->epoch) + 256, (size_t)n * 8, cudaMemcpyDeviceToHost));
    return PGMOE_OK;
}

extern "C" int pgmoe_model_init_weights(pgmoe_model *m) {
    const auto &c = m->cfg;
    const int nb = c.num_blocks, E = m->e_local, e0 = m->e_begin;
    const int64_t d = c.d_model, f = c.d_ff;
    cudaStream_t s = nullptr;
    PG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    std::vector<GenJob> jobs;
    for (int b = 0; b < nb; ++b) {
        BlockW &bw = m->blocks[b];
        if (bw.gate) jobs.push_back({bw.gate, matrix_seed(c.seed, kTagGate, b, -1), d * c.num_experts});
        if (bw.pre_gate) jobs.push_back({bw.pre_gate, matrix_seed(c.seed, kTagPreGate, b, -1), d * c.num_experts});
        jobs.push_back({bw.dense, matrix_seed(c.seed, kTagDense, b, -1), d * d});
    }
    const bool off = m->placement == PGMOE_OFFLOADED;
    unsigned char *stage = nullptr;
    int chunk = 1;
    if (off) {  // stage as many blocks as comfortably fit in HBM, then D2H
        size_t free_b = 0, total_b = 0;
        PG_CUDA(cudaMemGetInfo(&free_b, &total_b));
        const size_t blk = (size_t)E * m->rec_bytes;
        chunk = (int)std::max<size_t>(1, std::min<size_t>(nb, (free_b / 2) / blk));
        PG_CUDA(cudaMalloc(&stage, (size_t)chunk * blk));
    }
    GenJob *dj = nullptr;
    const size_t max_jobs = std::max<size_t>(jobs.size(), (size_t)2 * E * (off ? chunk : nb));
    PG_CUDA(cudaMalloc(&dj, sizeof(GenJob) * max_jobs));
    auto run = [&](std::vector<GenJob> &js) -> int {
        PG_CUDA(cudaMemcpyAsync(dj, js.data(), sizeof(GenJob) * js.size(), cudaMemcpyHostToDevice, s));
        PG_TRY(gen_matrices(dj, (int)js.size(), m->wdtype, s));
        PG_CUDA(cudaStreamSynchronize(s));
        return PGMOE_OK;
    };
    int st = run(jobs);
    if (st == PGMOE_OK && !off) {
        std::vector<GenJob> ej;
        for (int b = 0; b < nb; ++b)
            for (int e = 0; e < E; ++e) {
                unsigned char *rec = m->blocks[b].experts + (size_t)e * m->rec_bytes;
                ej.push_back({rec, matrix_seed(c.seed, kTagW1, b, e0 + e), f * d});
                ej.push_back({rec + m->w1_bytes, matrix_seed(c.seed, kTagW2, b, e0 + e), d * f});
            }
        st = run(ej);
    } else if (st == PGMOE_OK) {
        for (int b0 = 0; b0 < nb && st == PGMOE_OK; b0 += chunk) {
            const int b1 = std::min(nb, b0 + chunk);
            std::vector<GenJob> ej;
            for (int b = b0; b < b1; ++b)
                for (int e = 0; e < E; ++e) {
                    unsigned char *rec = stage + ((size_t)(b - b0) * E + e) * m->rec_bytes;
                    ej.push_back({rec, matrix_seed(c.seed, kTagW1, b, e0 + e), f * d});
                    ej.push_back({rec + m->w1_bytes, matrix_seed(c.seed, kTagW2, b, e0 + e), d * f});
                }
            st = run(ej);
            if (st == PGMOE_OK && cudaMemcpy(m->blocks[b0].experts, stage, (size_t)(b1 - b0) * E * m->rec_bytes,
                                             cudaMemcpyDeviceToHost) != cudaSuccess) {
                set_error("D2H of generated experts failed");
                st = PGMOE_E_CUDA;
            }
        }
    }
    cudaFree(dj);
    if (stage) cudaFree(stage);
    cudaStreamDestroy(s);
    return st;
}

extern "C" int pgmoe_model_set_matrix(pgmoe_model *m, const char *name, int32_t block, int32_t expert,
                                      const void *host_data, size_t nbytes) {
    size_t bytes = 0;
    bool on_host = false;
    void *dst = mat_ptr(m, name ? name : "", block, expert, &bytes, &on_host);
    PG_REQUIRE(dst != nullptr, PGMOE_E_CONFIG, "no matrix %s block %d expert %d", name, block, expert);
    const size_t want = (std::string(name) == "w1" || std::string(name) == "w2")
                            ? m->w1_bytes
                            : (std::string(name) == "non_moe" ? (size_t)m->cfg.d_model * m->cfg.d_model * m->sw
                                                              : (size_t)m->cfg.d_model * m->cfg.num_experts * m->sw);
    PG_REQUIRE(nbytes == want, PGMOE_E_SHAPE, "matrix %s expects %zu bytes, got %zu", name, want, nbytes);
    if (on_host) memcpy(dst, host_data, nbytes);
    else PG_CUDA(cudaMemcpy(dst, host_data, nbytes, cudaMemcpyHostToDevice));
    return PGMOE_OK;
}

extern "C" int pgmoe_model_get_matrix(pgmoe_model *m, const char *name, int32_t block, int32_t expert,
                                      void *host_data, size_t nbytes) {
    size_t bytes = 0;
    bool on_host = false;
    void *src = mat_ptr(m, name ? name : "", block, expert, &bytes, &on_host);
    PG_REQUIRE(src != nullptr, PGMOE_E_CONFIG, "no matrix %s block %d expert %d", name, block, expert);
    PG_REQUIRE(nbytes <= bytes, PGMOE_E_SHAPE, "matrix %s holds %zu bytes, asked %zu", name, bytes, nbytes);
    if (on_host) memcpy(host_data, src, nbytes);
    else PG_CUDA(cudaMemcpy(host_data, src, nbytes, cudaMemcpyDeviceToHost));
    return PGMOE_OK;
}

extern "C" const void *pgmoe_model_matrix_ptr(pgmoe_model *m, const char *name, int32_t block, int32_t expert) {
    size_t bytes = 0;
    bool on_host = false;
    return mat_ptr(m, name ? name : "", block, expert, &bytes, &on_host);
}

// Resident iterations have no host round trip, so the whole block loop
// (route, pack, up, down, dense per block; PDL edges between them) is
// captured once per buffer set and replayed as one graph launch.
static bool same_io(const pgmoe_iteration_io &a, const pgmoe_iteration_io &b) {
    return a.ids_trace == b.ids_trace && a.w_trace == b.w_trace && a.x_trace == b.x_trace &&
           a.ids_supplied == b.ids_supplied && a.w_supplied == b.w_supplied;
}

static int decoder_iteration_graph(pgmoe_model *m, const float *x_in, int T, float *y_out,
                                   const pgmoe_iteration_io &io, cudaStream_t s) {
    ++m->graph_clock;
    pgmoe_model::GraphEntry *victim = &m->graphs[0];
    for (auto &g : m->graphs) {
        if (g.exec && g.x == x_in && g.y == y_out && g.T == T && same_io(g.io, io)) {
            g.last_use = m->graph_clock;
            PG_CUDA(cudaGraphLaunch(g.exec, s));
            count_launch((int)g.launches);
            return PGMOE_OK;
        }
        if (!g.exec || g.last_use < victim->last_use) victim = &g;
    }
    if (victim->exec) {
        cudaGraphExecDestroy(victim->exec);
        victim->exec = nullptr;
    }
    if (!m->cap) PG_CUDA(cudaStreamCreateWithFlags(&m->cap, cudaStreamNonBlocking));
    const long long l0 = g_launches.load();
    PG_CUDA(cudaStreamBeginCapture(m->cap, cudaStreamCaptureModeThreadLocal));
    const int st = decoder_iteration(m, x_in, T, y_out, io, m->cap);
    victim->launches = g_launches.load() - l0;
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(m->cap, &graph);
    if (st != PGMOE_OK) {
        if (graph) cudaGraphDestroy(graph);
        return st;
    }
    PG_CUDA(ce);
    const cudaError_t ie = cudaGraphInstantiate(&victim->exec, graph, 0);
    cudaGraphDestroy(graph);
    PG_CUDA(ie);
    victim->x = x_in;
    victim->y = y_out;
    victim->T = T;
    victim->io = io;
    victim->last_use = m->graph_clock;
    PG_CUDA(cudaGraphLaunch(victim->exec, s));
    return PGMOE_OK;
}

extern "C" int pgmoe_decoder_iteration_ex(pgmoe_model *m, const float *x_in, int32_t T, float *y_out,
                                          const pgmoe_iteration_io *io_in, pgmoe_stream_t stream) {
    PG_REQUIRE(m != nullptr, PGMOE_E_CONFIG, "null model");
    std::lock_guard<std::mutex> g(m->mu);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const pgmoe_iteration_io io = io_in ? *io_in : pgmoe_iteration_io{};
    if (m->placement == PGMOE_RESIDENT && m->use_graph && !m->timeline && T > 0 && T <= m->max_tokens &&
        m->e_local == m->cfg.num_experts)
        return decoder_iteration_graph(m, x_in, T, y_out, io, s);
    return decoder_iteration(m, x_in, T, y_out, io, s);
}

extern "C" int pgmoe_decoder_iteration(pgmoe_model *m, const float *x_in, int32_t T, float *y_out,
                                       int32_t *ids_trace, float *w_trace, pgmoe_stream_t stream) {
    pgmoe_iteration_io io{};
    io.ids_trace = ids_trace;
    io.w_trace = w_trace;
    return pgmoe_decoder_iteration_ex(m, x_in, T, y_out, &io, stream);
}

// Surfaces (and clears) a device-detected routing error of any ring buffer:
// the error belongs to the iteration that raised it, not to later ones.
static int check_all_routing(pgmoe_model *m) {
    int first = PGMOE_OK;
    std::string msg;
    for (auto &rb : m->routing) {
        int32_t fb = 0;
        int st = pgmoe_check_routing(&rb.r, &fb);
        m->stats.route_fallbacks = std::max<int64_t>(m->stats.route_fallbacks, fb);
        if (st != PGMOE_OK) {
            if (first == PGMOE_OK) {
                first = st;
                msg = g_last_error;
            }
            PG_CUDA(cudaMemset(rb.r.status, 0, sizeof(int32_t)));
        }
    }
    if (first != PGMOE_OK) g_last_error = msg;
    return first;
}

extern "C" int pgmoe_model_check_routing(pgmoe_model *m) {
    PG_REQUIRE(m != nullptr, PGMOE_E_CONFIG, "null model");
    std::lock_guard<std::mutex> g(m->mu);
    PG_CUDA(cudaDeviceSynchronize());
    return check_all_routing(m);
}

extern "C" int pgmoe_decoder_iteration_host(pgmoe_model *m, const float *x_in, int32_t T, float *y_out,
                                            int32_t *ids_trace, float *w_trace) {
    PG_REQUIRE(m != nullptr, PGMOE_E_CONFIG, "null model");
    const auto &c = m->cfg;
    PG_REQUIRE(T >= 0 && T <= m->max_tokens, PGMOE_E_SHAPE, "T=%d exceeds max_tokens=%d", T, m->max_tokens);
    if (T == 0) return PGMOE_OK;
    const size_t xb = (size_t)T * c.d_model * 4, tb = (size_t)c.num_blocks * T * c.top_k * 4;
    {
        std::lock_guard<std::mutex> g(m->mu);
        if (!m->io_stream) {  // persistent I/O buffers: the graph path keys on their addresses
            const size_t cap_x = (size_t)m->max_tokens * c.d_model * 4;
            const size_t cap_t = (size_t)c.num_blocks * m->max_tokens * c.top_k * 4;
            PG_CUDA(cudaStreamCreateWithFlags(&m->io_stream, cudaStreamNonBlocking));
            PG_CUDA(cudaMalloc(&m->io_x, cap_x));
            PG_CUDA(cudaMalloc(&m->io_y, cap_x));
            PG_CUDA(cudaMalloc(&m->io_ids, cap_t));
            PG_CUDA(cudaMalloc(&m->io_w, cap_t));
            PG_CUDA(cudaHostAlloc(&m->io_status, m->routing.size() * 4 * sizeof(int32_t), cudaHostAllocDefault));
        }
    }
    cudaStream_t s = m->io_stream;
    PG_CUDA(cudaMemcpyAsync(m->io_x, x_in, xb, cudaMemcpyHostToDevice, s));
    int st = pgmoe_decoder_iteration(m, m->io_x, T, m->io_y, ids_trace ? m->io_ids : nullptr,
                                     ids_trace ? m->io_w : nullptr, reinterpret_cast<pgmoe_stream_t>(s));
    if (st == PGMOE_OK) {
        PG_CUDA(cudaMemcpyAsync(y_out, m->io_y, xb, cudaMemcpyDeviceToHost, s));
        if (ids_trace) {
            PG_CUDA(cudaMemcpyAsync(ids_trace, m->io_ids, tb, cudaMemcpyDeviceToHost, s));
            PG_CUDA(cudaMemcpyAsync(w_trace, m->io_w, tb, cudaMemcpyDeviceToHost, s));
        }
        // routing statuses ride along (one synchronisation per call instead
        // of a blocking copy per routing buffer afterwards)
        PG_CUDA(cudaMemcpyAsync(m->io_status, m->status_dev, m->routing.size() * 4 * sizeof(int32_t),
                                cudaMemcpyDeviceToHost, s));
    }
    if (cudaStreamSynchronize(s) != cudaSuccess && st == PGMOE_OK) {
        set_error("decoder iteration failed: %s", cudaGetErrorString(cudaGetLastError()));
        st = PGMOE_E_CUDA;
    }
    if (st == PGMOE_OK) {
        std::lock_guard<std::mutex> g(m->mu);
        bool clean = true;
        for (size_t i = 0; i < m->routing.size(); ++i) {
            clean &= m->io_status[4 * i] == 0;
            m->stats.route_fallbacks = std::max<int64_t>(m->stats.route_fallbacks, m->io_status[4 * i + 1]);
        }
        if (!clean) st = check_all_routing(m);  // error path: message, reset
    }
    return st;
}

extern "C" int pgmoe_moe_block_forward(pgmoe_model *m, int32_t block, const float *x, int32_t T,
                                       const pgmoe_routing *r_in, float *y, const pgmoe_routing *r_out,
                                       pgmoe_stream_t stream) {
    PG_REQUIRE(m != nullptr, PGMOE_E_CONFIG, "null model");
    std::lock_guard<std::mutex> g(m->mu);
    const auto &c = m->cfg;
    PG_REQUIRE(block >= 0 && block < c.num_blocks, PGMOE_E_CONFIG, "block %d out of range", block);
    PG_REQUIRE(T >= 0 && T <= m->max_tokens, PGMOE_E_SHAPE, "T=%d exceeds max_tokens=%d", T, m->max_tokens);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const BlockW &bw = m->blocks[block];
    if (r_out && has_pre_gate(c, block))
        PG_TRY(pgmoe_gate_forward(x, T, c.d_model, bw.pre_gate, m->wdtype, c.num_experts, c.top_k, r_out,
                                  m->route_ws, stream));
    PG_REQUIRE(r_in != nullptr, PGMOE_E_ROUTING, "no routing decision available");
    if (T == 0) return PGMOE_OK;
    const void *experts = bw.experts;
    int indexed = 0;
    if (m->placement == PGMOE_OFFLOADED) {  // on-demand fetch into slot 0
        PG_CUDA(cudaStreamSynchronize(m->copy));  // no decoder migration still writing the slot
        int32_t nact = 0;
        PG_CUDA(cudaMemcpyAsync(m->routing[0].act_host, r_in->act, sizeof(int32_t) * (c.num_experts + 1),
                                cudaMemcpyDeviceToHost, s));
        PG_CUDA(cudaStreamSynchronize(s));
        nact = m->routing[0].act_host[c.num_experts];
        PG_REQUIRE(nact <= m->slot_experts, PGMOE_E_OOM, "slot overflow");
        for (int i = 0; i < nact; ++i)
            PG_CUDA(cudaMemcpyAsync(m->slots + (size_t)i * m->rec_bytes,
                                    bw.experts + (size_t)m->routing[0].act_host[i] * m->rec_bytes, m->rec_bytes,
                                    cudaMemcpyHostToDevice, s));
        experts = m->slots;
        indexed = 1;
        m->slot_used[0] = false;
    }
    PG_TRY(run_ffn(m, x, T, experts, indexed, r_in, s));
    return run_dense(m, T, bw.dense, y, s);
}

extern "C" int pgmoe_model_expert_records(pgmoe_model *m, int32_t block, const void **base, size_t *stride,
                                          int32_t *expert_begin, int32_t *n_local) {
    PG_REQUIRE(m && block >= 0 && block < m->cfg.num_blocks, PGMOE_E_CONFIG, "bad block %d", block);
    *base = m->blocks[block].experts;
    *stride = m->rec_bytes;
    *expert_begin = m->e_begin;
    *n_local = m->e_local;
    return PGMOE_OK;
}

extern "C" int pgmoe_model_stats(pgmoe_model *m, pgmoe_stats *out) {
    PG_REQUIRE(m && out, PGMOE_E_CONFIG, "null argument");
    std::lock_guard<std::mutex> g(m->mu);
    PG_CUDA(cudaDeviceSynchronize());
    const auto &c = m->cfg;
    if (m->placement == PGMOE_OFFLOADED && (int)m->nact_iter.size() == c.num_blocks) {
        // Eq.1 (tiers.py:68-86) over the last iteration's measured active sets
        int64_t best = 0;
        const int L = c.activation_level;
        for (int n = 0; n < c.num_blocks; ++n) {
            int64_t win = 0;
            for (int q = n; q <= n + L && q < c.num_blocks; ++q) win += (int64_t)m->nact_iter[q] * m->rec_bytes;
            best = std::max(best, win);
        }
        m->stats.eq1_peak_bytes = m->stats.pinned_hbm_bytes + best;
        // Ledger from real event times: expert bytes of block b live over
        // [copy start, experts done] (half-open; releases first at ties).
        struct Ev { float t; int kind; int64_t bytes; };
        std::vector<Ev> evs;
        double busy = 0;
        for (int b = 0; b < c.num_blocks; ++b) {
            float ta = 0, tb = 0, te = 0;
            if (cudaEventElapsedTime(&ta, m->cp_a[0], m->cp_a[b]) != cudaSuccess) continue;
            cudaEventElapsedTime(&tb, m->cp_a[0], m->cp_b[b]);
            cudaEventElapsedTime(&te, m->cp_a[0], m->ffn_b[b]);
            busy += (tb - ta) * 1e-3;
            const int64_t by = (int64_t)m->nact_iter[b] * m->rec_bytes;
            evs.push_back({ta, 1, by});
            evs.push_back({std::max(te, ta), 0, -by});
        }
        cudaGetLastError();
        std::sort(evs.begin(), evs.end(), [](const Ev &a, const Ev &b) {
            return a.t < b.t || (a.t == b.t && a.kind < b.kind);
        });
        int64_t cur = 0, peak = 0;
        for (auto &e : evs) { cur += e.bytes; peak = std::max(peak, cur); }
        m->stats.ledger_peak_bytes = m->stats.pinned_hbm_bytes + peak;
        m->stats.h2d_seconds = busy;
    }
    int32_t fb = 0;
    for (auto &rb : m->routing) {
        int32_t st[4];
        if (cudaMemcpy(st, rb.r.status, sizeof(st), cudaMemcpyDeviceToHost) == cudaSuccess) fb += st[1];
    }
    m->stats.route_fallbacks = fb;
    m->stats.fused_blocks = m->fused_blocks;
    m->stats.fused_routes = m->fused_routes;
    *out = m->stats;
    return PGMOE_OK;
}

extern "C" int pgmoe_model_reset_stats(pgmoe_model *m) {
    std::lock_guard<std::mutex> g(m->mu);
    const int64_t pinned = m->stats.pinned_hbm_bytes, slot = m->stats.slot_capacity_bytes;
    const int64_t cb = m->stats.cache_bytes;
    m->stats = pgmoe_stats{};
    m->stats.pinned_hbm_bytes = pinned;
    m->stats.slot_capacity_bytes = slot;
    m->stats.cache_bytes = cb;
    m->fused_blocks = 0;
    m->fused_routes = 0;
    return PGMOE_OK;
}

extern "C" int pgmoe_model_set_timeline(pgmoe_model *m, int32_t enabled) {
    std::lock_guard<std::mutex> g(m->mu);
    cudaDeviceSynchronize();
    for (auto &e : m->tl) { cudaEventDestroy(e.a); cudaEventDestroy(e.b); }
    m->tl.clear();
    m->t0_recorded = false;
    m->timeline = enabled != 0;
    return PGMOE_OK;
}

extern "C" int64_t pgmoe_model_timeline_jsonl(pgmoe_model *m, char *buf, int64_t cap) {
    std::lock_guard<std::mutex> g(m->mu);
    cudaDeviceSynchronize();
    std::string outs;
    for (auto &e : m->tl) {
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, m->t0, e.a);
        cudaEventElapsedTime(&b, m->t0, e.b);
        char line[256];
        snprintf(line, sizeof(line), "{\"lane\": \"%s\", \"label\": \"%s\", \"block\": %d, \"start_s\": %.9g, \"end_s\": %.9g}\n",
                 e.lane, e.label.c_str(), e.block, std::max(0.f, a) * 1e-3, std::max(0.f, b) * 1e-3);
        outs += line;
    }
    cudaGetLastError();
    if (buf && cap > 0) {
        const int64_t n = std::min<int64_t>(cap - 1, (int64_t)outs.size());
        memcpy(buf, outs.data(), n);
        buf[n] = 0;
    }
    return (int64_t)outs.size();
}
