// decode_ll.cu — low-latency small-batch decoder (T <= 8 tokens, top-1,
// lookahead 1, bf16 weights, resident experts): ONE persistent launch runs
// the block loop of decoder_iteration (core.py:342-383), one CTA per SM.
//
// At decode batch sizes a block is three dependent GEMV-shaped contractions
// (up, down + combine, dense) plus the next pre-gate; its weights (Base-64
// T=1: 10.6 MB) are tiny next to the time a global round trip costs, so the
// block latency is the number of serial round trips, not the weight stream.
// This kernel spends one round trip per phase:
//   * rows, not K, are split over the CTAs: every CTA finishes whole output
//     values (no partial sums between CTAs, no split-K tickets);
//   * phase outputs travel as LL words — {fp32 payload, 32-bit flag} in one
//     8-byte store — so a consumer polls the data itself: no fence, no
//     counter, no second round trip (flag = launch epoch x 64 + block);
//   * a CTA's weight slice of a phase is bulk-copied (cp.async.bulk) into a
//     3-slot shared-memory ring as soon as the block's routing is known, so
//     it is on chip before the phase input arrives; the dense slices and
//     pre-gate rows (static) have their own buffer;
//   * the dense CTAs also compute the next pre-gate's partial fp64 logits of
//     their rows from the y values in registers (exact products), so routing
//     costs one more LL hop: T reducer CTAs sum the partials in producer
//     order, certify and select (route_common.cuh, the K1 arithmetic
//     contract: certified ranking, serial reference-order recompute), and
//     publish the decision as LL words the weight producers poll.
// Per CTA: warp 0 expert-slice producer (decisions -> schedule -> copies),
// warp 1 dense-slice producer, warps 2-9 compute (mma.sync m16n8k16 bf16 ->
// fp32, K split over the warps and summed in a fixed order), warps 10-11
// reducer (the last T CTAs only).  Deterministic.
#include <cstdlib>

#include "common.cuh"
#include "decode.h"
#include "kernels.h"
#include "route_common.cuh"
#include "tc_common.cuh"

namespace pgmoe {
namespace ll {
using tc::bf16_bits;
using tc::mbar_arrive;
using tc::mbar_expect_tx;
using tc::mbar_init;
using tc::mbar_wait;
using tc::named_sync;
using tc::smem_u32;

constexpr int kThreads = 384;
constexpr int kCW0 = 2, kCWarps = 8, kCThreads = kCWarps * 32;  // compute warps
constexpr int kRW0 = 10, kRThreads = 64;                        // reducer warps
constexpr int kMaxSlots = 6;  // weight-slice ring: as many slots as shared memory allows (>= 3)
constexpr int kSlotBytes = 33792;  // the smallest ring slot (one row of K = 4096 needs 8208 B)
constexpr int kDRows = 16;  // dense rows per dense CTA
constexpr int kMaxE = 128;

struct Piece {
    int b, phase, e, row0, nrows, ng, end;
    int tok[kLLMaxT];
    float w[kLLMaxT];
};

struct Params {
    int T, d, f, E, nb, nd;           // nd: dense CTAs (d / kDRows)
    int nslots, slot_bytes;           // weight-slice ring: slots x bytes (pick_ring)
    const DecodeBlock *blocks;
    const unsigned char *experts;     // records [nb][E]: W1 [f][d] then W2 [d][f]
    size_t rec_bytes;
    const uint16_t *pool;             // weight pool: dense(b) = pool + blocks[b].dense_row0 * d
    const float *x_in;
    float *y_out;
    const uint16_t *gate0;            // block 0's conventional gate [d][E] (core.py:362-366)
    pgmoe_routing gate0_out;          // the decision it writes (block 0 consumes it)
    unsigned long long *llx;          // [2][T][d]
    unsigned long long *llh;          // [T][f]
    unsigned long long *llmix;        // [T][d]
    unsigned long long *llpart;       // [2][nd][T][E + 2] x 2 words (fp64 halves): logits, sum|x|, max|G|;
                                      // gate g (0: block 0's gate, b + 1: block b's pre-gate) uses [g & 1]
    unsigned long long *lllog;        // [2][T][E] x 2 words: the reducers' logits
    unsigned long long *lldec;        // [nb][kLLMaxT] x 2 words (id, weight)
    unsigned *ctr;                    // [0] epoch (>= 1), [1] CTAs finished
    double gam, bscale;
    float *x_trace;                   // optional [nb][T][d]
    int32_t *ids_trace;               // optional [nb][T]
    float *w_trace;
    unsigned long long *probe;
};

// flag of the words produced during block b (b = -1: the launch prologue; -2:
// block 0's conventional gate): never 0, the value of fresh memory
__device__ __forceinline__ uint32_t flag_of(uint32_t epoch, int b) { return (epoch << 7) + (uint32_t)(b + 2); }
__device__ __forceinline__ unsigned long long ll_word(uint32_t payload, uint32_t flag) {
    return ((unsigned long long)flag << 32) | payload;
}
__device__ __forceinline__ void st_ll(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_ll2(unsigned long long *p, unsigned long long a, unsigned long long b) {
    asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ unsigned long long ld_ll(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void ld_ll2(const unsigned long long *p, unsigned long long &a, unsigned long long &b) {
    asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
// poll one LL word until its flag matches; returns the payload
__device__ __forceinline__ uint32_t poll_ll(const unsigned long long *p, uint32_t flag) {
    unsigned long long v = ld_ll(p);
    while ((uint32_t)(v >> 32) != flag) v = ld_ll(p);
    return (uint32_t)v;
}
__device__ __forceinline__ double poll_ll_f64(const unsigned long long *p, uint32_t flag) {
    unsigned long long a, b;
    ld_ll2(p, a, b);
    while ((uint32_t)(a >> 32) != flag || (uint32_t)(b >> 32) != flag) ld_ll2(p, a, b);
    return __hiloint2double((int)(uint32_t)b, (int)(uint32_t)a);
}
// Poll U word pairs (one 16-byte load each) until every flag matches.  All
// pending loads are re-issued together, so a batch waits about one round
// trip after its data lands instead of one per word.
template <int U, typename Addr>
__device__ __forceinline__ void poll2(Addr addr, uint32_t valid, uint32_t flag, unsigned long long (&a)[U],
                                      unsigned long long (&b)[U]) {
    uint32_t pend = valid;
    while (pend) {
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (pend >> u & 1u) ld_ll2(addr(u), a[u], b[u]);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if ((pend >> u & 1u) && (uint32_t)(a[u] >> 32) == flag && (uint32_t)(b[u] >> 32) == flag)
                pend &= ~(1u << u);
    }
}
template <int U, typename Addr>
__device__ __forceinline__ void poll1(Addr addr, uint32_t valid, uint32_t flag, unsigned long long (&a)[U]) {
    uint32_t pend = valid;
    while (pend) {
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (pend >> u & 1u) a[u] = ld_ll(addr(u));
#pragma unroll
        for (int u = 0; u < U; ++u)
            if ((pend >> u & 1u) && (uint32_t)(a[u] >> 32) == flag) pend &= ~(1u << u);
    }
}

__device__ __forceinline__ void st_ll_f64(unsigned long long *p, double v, uint32_t flag) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    st_ll2(p, ll_word((uint32_t)bits, flag), ll_word((uint32_t)(bits >> 32), flag));
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

__device__ __forceinline__ void mma_bf16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Device-side stamps (tools/probe_ll.py) exist only in a -DPGMOE_LL_PROBE
// build: at T = 1 the launch is sensitive to every extra instruction on its
// serial path (a handful of disabled stamps measured +4 us per block).
#ifdef PGMOE_LL_PROBE
__device__ __forceinline__ void dprobe(const Params &p, int b, int k) {
    if (p.probe && b < 4) p.probe[(size_t)blockIdx.x * kProbeSlots + 1 + 8 * b + k] = gtimer();
}
// block 2's cycle accumulators (thread ct 0 of the compute group): slot 33 + 4 * phase + {wait for
// the slice, stage, gemv, epilogue}; 45 + phase: pieces
#define PCLK(v) long long v = clock64()
#define PACC(b, ph, k, t0)                                                                               \
    do {                                                                                                 \
        if (p.probe && (b) == 2 && ct == 0) p.probe[(size_t)blockIdx.x * kProbeSlots + 33 + 4 * (ph) + (k)] += \
            (unsigned long long)(clock64() - (t0));                                                      \
    } while (0)
#else
__device__ __forceinline__ void dprobe(const Params &, int, int) {}
#define PCLK(v)
#define PACC(b, ph, k, t0)
#endif
__device__ __forceinline__ void csync() { named_sync(1, kCThreads); }
__device__ __forceinline__ void rsync() { named_sync(2, kRThreads); }

// rows of a [rows][K] piece x the staged activations [8][K] -> fp32
// outputs in `red` (K split over the compute warps, summed in warp order).
// Returns through `out` (thread ct < mt*128 owns output (ct / 8, ct % 8) of
// its m-tile); rows past nrows repeat the last row (results discarded).
__device__ __forceinline__ void piece_gemv(const unsigned char *A, int apitch, int nrows, const unsigned char *B,
                                           int bpitch, int brows, int K, float *red, int ct, float &out, int &orow, int &otok,
                                           uint64_t *release = nullptr) {
    const int w = ct >> 5, lane = ct & 31, g = lane >> 2, t4 = lane & 3;
    const int mt = nrows > 16 ? 2 : 1, S = kCWarps / mt;
    const int m = w / S, s = w - m * S;
    const int KS = K / 16, k0 = KS * s / S, k1 = KS * (s + 1) / S;
    // A fragments with one ldmatrix.x4 per k-step: lanes 0-15 address rows
    // 0-15 of the m-tile at k, lanes 16-31 the same rows at k + 8
    const int lr = min(m * 16 + (lane & 15), nrows - 1);
    const uint32_t abase = (uint32_t)__cvta_generic_to_shared(A + (size_t)lr * apitch + (lane >> 4) * 16);
    const unsigned char *bp = B + (size_t)min(g, brows - 1) * bpitch + t4 * 4;  // staged rows only
    float c[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
    for (int ks = k0; ks < k1; ++ks) {
        const int o = ks * 32;
        uint32_t a0, a1, a2, a3;
        // not volatile (the k-steps' loads may be issued ahead of the mmas); the
        // memory clobber keeps it behind the slot's barrier wait
        asm("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
            : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
            : "r"(abase + o)
            : "memory");
        const uint32_t b0 = *reinterpret_cast<const uint32_t *>(bp + o);
        const uint32_t b1 = *reinterpret_cast<const uint32_t *>(bp + o + 16);
        mma_bf16(c, a0, a1, a2, a3, b0, b1);
    }
    if (release) {  // this warp is done reading the slot: the producer may refill it now
        __syncwarp();
        if (lane == 0) mbar_arrive(release);
    }
    // red[w][row 0..15][tok 0..7]
    float *rw = red + w * 128;
    rw[g * 8 + 2 * t4] = c[0];
    rw[g * 8 + 2 * t4 + 1] = c[1];
    rw[(g + 8) * 8 + 2 * t4] = c[2];
    rw[(g + 8) * 8 + 2 * t4 + 1] = c[3];
    csync();
    out = 0.f;
    orow = -1;
    otok = 0;
    if (ct < mt * 128) {
        const int mm = ct >> 7, q = ct & 127;
        float v = 0.f;
        for (int z = 0; z < S; ++z) v += red[(mm * S + z) * 128 + q];
        out = v;
        orow = mm * 16 + (q >> 3);
        otok = q & 7;
    }
    csync();  // red reusable
}

// Stage ng token vectors of K values as bf16 rows [8][K + 8] (tokens tok[n],
// or n itself when tok is null).  LL source (every word polled for `flag`)
// or plain fp32.  Loads are issued U at a time before any flag is checked,
// so a thread waits about one round trip, not one per word.  Rows >= ng are
// left as they are: a B column only feeds its own output column.
__device__ __forceinline__ void stage(unsigned char *act, int K, int ng, const int *tok,
                                      const unsigned long long *ll, size_t ll_stride, const float *plain,
                                      size_t plain_stride, uint32_t flag, int ct) {
    constexpr int U = 4;
    const int apitch = K * 2 + 16;
    const int npair = K / 2, n_all = ng * npair;
    for (int i0 = ct; i0 < n_all; i0 += U * kCThreads) {
        unsigned long long a[U], b[U];
        int n[U], k[U];
        uint32_t valid = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * kCThreads;
            n[u] = min(i, n_all - 1) / npair;
            k[u] = 2 * (min(i, n_all - 1) - n[u] * npair);
            if (i < n_all) valid |= 1u << u;
        }
        if (plain) {
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (valid >> u & 1u) {
                    const int t = tok ? tok[n[u]] : n[u];
                    const float2 v = __ldcg(reinterpret_cast<const float2 *>(plain + (size_t)t * plain_stride + k[u]));
                    a[u] = __float_as_uint(v.x);
                    b[u] = __float_as_uint(v.y);
                }
        } else {
            poll2<U>([&](int u) { return ll + (size_t)(tok ? tok[n[u]] : n[u]) * ll_stride + k[u]; }, valid, flag, a, b);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (valid >> u & 1u)
                *reinterpret_cast<uint32_t *>(act + (size_t)n[u] * apitch + k[u] * 2) =
                    (uint32_t)bf16_bits(__uint_as_float((uint32_t)a[u])) |
                    ((uint32_t)bf16_bits(__uint_as_float((uint32_t)b[u])) << 16);
    }
    csync();
}

// dense rows [r0, r0 + kDRows) of block b: pre-gate partials of the next
// block's pre-gate over those rows, from y [kDRows][8] in shared memory.
__device__ void pregate_partials(const Params &p, const float *ytile, const uint16_t *gsl, float *red, int c,
                                 int par, uint32_t flag, int ct) {
    const int E = p.E, T = p.T, W = E + 2;
    // max |G| over this slice (all experts): a valid column bound for every
    // expert (>= its column maximum), so no per-column maxima travel
    float gm = 0.f;
    for (int i = ct; i < kDRows * E; i += kCThreads) gm = fmaxf(gm, fabsf(bf16_to_f32(gsl[i])));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) gm = fmaxf(gm, __shfl_xor_sync(0xffffffffu, gm, o));
    if ((ct & 31) == 0) red[ct >> 5] = gm;
    csync();
    gm = red[0];
    for (int w = 1; w < kCWarps; ++w) gm = fmaxf(gm, red[w]);
    const int TPE = kCThreads / E;  // threads per expert (2 or 4)
    const int j = ct % E, tq = ct / E;
    unsigned long long *base = p.llpart + (size_t)par * p.nd * T * W * 2;
    for (int t = tq; t < T; t += TPE) {
        double acc = 0.0;
#pragma unroll
        for (int r = 0; r < kDRows; ++r)
            acc = fma((double)ytile[r * 8 + t], (double)bf16_to_f32(gsl[r * E + j]), acc);  // exact product
        st_ll_f64(base + (((size_t)c * T + t) * W + j) * 2, acc, flag);
    }
    if (ct < T) {  // sum |x_i| over the rows (bounds the logit error)
        double s = 0.0;
        for (int r = 0; r < kDRows; ++r) s += fabs((double)ytile[r * 8 + ct]);
        st_ll_f64(base + (((size_t)c * T + ct) * W + E) * 2, s, flag);
        st_ll_f64(base + (((size_t)c * T + ct) * W + E + 1) * 2, (double)gm, flag);
    }
}

__global__ void __launch_bounds__(kThreads, 1) ll_decode_kernel(const __grid_constant__ Params p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const int T = p.T, d = p.d, f = p.f, E = p.E, nb = p.nb;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int c = blockIdx.x, G = gridDim.x;
    const int dpitch = d * 2 + 16;
    // ---- shared memory layout ------------------------------------------
    const int kSlots = p.nslots;
    const int kSlotB = p.slot_bytes;
    unsigned char *slots = smem_raw;                                    // kSlots x kSlotB
    unsigned char *dbuf = slots + (size_t)kSlots * kSlotB;              // kDRows x dpitch
    uint16_t *gsl = reinterpret_cast<uint16_t *>(dbuf + kDRows * dpitch);  // kDRows x E pre-gate rows
    uint16_t *gsl0 = gsl + kDRows * E;                                     // block 0's gate rows (fill 0)
    unsigned char *act = reinterpret_cast<unsigned char *>(gsl0 + kDRows * E);  // T x (max(d,f) * 2 + 16)
    float *red = reinterpret_cast<float *>(act + (size_t)((T + 1) & ~1) * (f * 2 + 16));  // kCWarps x 128
    float *ytile = red + kCWarps * 128;                                         // kDRows x 8
    float *rx = ytile + kDRows * 8;                                             // reducer: x [d]
    double *rlg = reinterpret_cast<double *>(rx + d);                           // [kRThreads] chunk sums
    double *rsel = rlg + kRThreads;                                             // [kMaxE] logits
    float *rcm = reinterpret_cast<float *>(rsel + kMaxE);                       // [kMaxE]
    double *rsx = reinterpret_cast<double *>(rcm + kMaxE);                      // [kRThreads + 1]
    double *rgx = rsx + kRThreads + 1;                                          // [kRThreads]
    Piece *desc = reinterpret_cast<Piece *>(rgx + kRThreads);                   // [kSlots]
    uint64_t *bars = reinterpret_cast<uint64_t *>(
        (reinterpret_cast<uintptr_t>(desc + kSlots) + 15) & ~(uintptr_t)15);
    uint64_t *full = bars, *empty = full + kSlots, *dfull = empty + kSlots, *dempty = dfull + 1;
    int *sched = reinterpret_cast<int *>(dempty + 1);  // [2 * kLLMaxT] ids, weights (producer warp)
    __shared__ int s_ids[kRouterTok * 8];
    __shared__ float s_w[kRouterTok * 8];

    if (tid == 0) {
        for (int i = 0; i < kSlots; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kCWarps);  // each compute warp releases a slot after its last read
        }
        mbar_init(dfull, 1);
        mbar_init(dempty, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#ifdef PGMOE_LL_PROBE
        if (p.probe) p.probe[(size_t)c * kProbeSlots] = gtimer();
#endif
    }
    __syncthreads();
    const bool dense_cta = c < p.nd;
    const int dr0 = c * kDRows;

    if (warp == 1) {
        // ============ dense-slice producer (static weights) ================
        if (lane == 0 && dense_cta) {
            uint64_t pol;
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
            // fill 0: block 0's gate and pre-gate rows (both on x_in); fill
            // b+1: dense(b) rows + pre-gate(b+1) rows
            for (int fl = 0; fl <= nb; ++fl) {
                const int b = fl - 1;
                const bool has_d = b >= 0;
                const bool has_g = fl < nb && p.blocks[fl].has_pre_gate;
                if (fl > 0) mbar_wait(dempty, (fl - 1) & 1);
                const bool has_g0 = fl == 0;
                const uint32_t bytes = (has_d ? kDRows * d * 2 : 0) + (has_g ? kDRows * E * 2 : 0) +
                                       (has_g0 ? kDRows * E * 2 : 0);
                if (bytes == 0) {
                    mbar_arrive(dfull);
                    continue;
                }
                mbar_expect_tx(dfull, bytes);
                if (has_d)
                    for (int r = 0; r < kDRows; ++r)
                        bulk_g2s(dbuf + r * dpitch, p.pool + ((size_t)p.blocks[b].dense_row0 + dr0 + r) * d, d * 2,
                                 dfull, pol);
                if (has_g)
                    bulk_g2s(gsl, static_cast<const uint16_t *>(p.blocks[fl].pre_gate) + (size_t)dr0 * E,
                             kDRows * E * 2, dfull, pol);
                if (has_g0) bulk_g2s(gsl0, p.gate0 + (size_t)dr0 * E, kDRows * E * 2, dfull, pol);
            }
        }
        return;
    }
    pdl_wait();  // block 0's decision (K1) and x_in
    const uint32_t epoch = *reinterpret_cast<volatile unsigned *>(p.ctr);

    if (warp == 0) {
        // ============ expert-slice producer ================================
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        int pc = 0;  // pieces issued
        for (int b = 0; b < nb; ++b) {
            // the decision block b consumes, from the reducers (LL words): block 0's
            // gate (b = 0) or block b-1's pre-gate
            if (lane < T) {
                int id;
                float w;
                {
                    const unsigned long long *q = p.lldec + ((size_t)b * kLLMaxT + lane) * 2;
                    const uint32_t fl = flag_of(epoch, b == 0 ? -2 : b - 1);
                    id = (int)poll_ll(q, fl);
                    w = __uint_as_float(poll_ll(q + 1, fl));
                }
                sched[lane] = id;
                reinterpret_cast<float *>(sched)[kLLMaxT + lane] = w;
            }
            __syncwarp();
            // every lane walks the same schedule; lane 0 publishes the piece
            // descriptors and arms the barriers, the lanes issue one row copy each
            if (lane == 0) dprobe(p, b, 0);
            // active experts ascending; tokens of each in ascending order (stable)
            int ex[kLLMaxT], na = 0;
            for (int t = 0; t < T; ++t) {
                const int e = sched[t];
                int pos = 0;
                bool seen = false;
                for (int a = 0; a < na; ++a) {
                    seen |= ex[a] == e;
                    pos += ex[a] < e;
                }
                if (!seen) {
                    for (int a = na; a > pos; --a) ex[a] = ex[a - 1];
                    ex[pos] = e;
                    ++na;
                }
            }
            const unsigned char *recs = p.experts + (size_t)b * E * p.rec_bytes;
            for (int ph = 0; ph < 2; ++ph) {
                const int R = ph == 0 ? f : d, K = ph == 0 ? d : f;
                const int pitch = K * 2 + 16, prow = min(kSlotB / pitch, 32);
                const long long N = (long long)na * R;
                const long long lo = N * c / G, hi = N * (c + 1) / G;
                long long r = lo;
                do {
                    const int slot = pc % kSlots;
                    if (pc >= kSlots) mbar_wait(&empty[slot], ((pc / kSlots) - 1) & 1);
                    Piece &pd = desc[slot];
                    if (r < hi) {
                        const int a = (int)(r / R), rr = (int)(r - (long long)a * R);
                        const int n = (int)min((long long)min(R - rr, prow), hi - r);
                        const int e = ex[a];
                        r += n;
                        if (lane == 0) {
                            pd.b = b;
                            pd.phase = ph;
                            pd.e = e;
                            pd.row0 = rr;
                            pd.nrows = n;
                            int ng = 0;
                            for (int t = 0; t < T; ++t)
                                if (sched[t] == e) {
                                    pd.tok[ng] = t;
                                    pd.w[ng] = reinterpret_cast<const float *>(sched)[kLLMaxT + t];
                                    ++ng;
                                }
                            pd.ng = ng;
                            pd.end = r >= hi;
                            mbar_expect_tx(&full[slot], (uint32_t)(n * K * 2));
                        }
                        __syncwarp();
                        const unsigned char *src = recs + (size_t)e * p.rec_bytes +
                                                   (ph == 0 ? (size_t)rr * d * 2 : (size_t)f * d * 2 + (size_t)rr * f * 2);
                        for (int i = lane; i < n; i += 32)
                            bulk_g2s(slots + (size_t)slot * kSlotB + i * pitch, src + (size_t)i * K * 2, K * 2,
                                     &full[slot], pol);
                    } else if (lane == 0) {  // no rows of this phase here: an empty marker piece
                        pd.b = b;
                        pd.phase = ph;
                        pd.nrows = 0;
                        pd.ng = 0;
                        pd.end = 1;
                        mbar_arrive(&full[slot]);
                    }
                    __syncwarp();
                    ++pc;
                } while (r < hi);
            }
            __syncwarp();
        }
        return;
    }

    if (warp >= kRW0) {
        // ============ reducers (the last T x Q CTAs) ========================
        // CTA (t, q) sums, in producer order, the nd dense CTAs' partial
        // logits of experts [16q, 16q + 16) for token t and publishes them
        // (LL); CTA (t, 0) then reads the E logits, certifies and selects.
        const int Q = E / 16, r0c = G - T * Q;
        if (c < r0c) return;
        const int t = (c - r0c) / Q, q = (c - r0c) - t * Q;
        const int rt = tid - kRW0 * 32;
        const bool selector = q == 0;
        FusedRoute r{};
        r.active = 1;
        r.gt_bf16 = 1;
        r.d = d;
        r.E = E;
        r.T = T;
        r.k = 1;
        r.gam = p.gam;
        r.bscale = p.bscale;
        r.x = rx - (size_t)t * d;  // serial fallback reads x[tok * d + i]: this token's copy in shared memory
        if (selector && p.x_trace)
            for (int i = rt; i < d; i += kRThreads) p.x_trace[(size_t)t * d + i] = __ldcg(p.x_in + (size_t)t * d + i);
        const int W = E + 2, nd = p.nd;
        // thread (expert jj of 16, producer chunk k of 4)
        const int jj = rt % 16, kc = rt / 16, NK = kRThreads / 16;
        const int qp0 = nd * kc / NK, qp1 = nd * (kc + 1) / NK;
        // gate g: 0 = block 0's conventional gate on x_in (core.py:362-366), g = b + 1 =
        // block b's pre-gate on block b's input (core.py:327-329); decision for block g
        for (int g = 0; g < nb; ++g) {
            const int b = g - 1;  // the block whose pre-gate this is (-1: block 0's gate)
            if (g > 0 && !p.blocks[b].has_pre_gate) continue;
            // partials: written in the prologue (g <= 1) or by dense(g - 2); decision: flag of block b
            const uint32_t fin = flag_of(epoch, g <= 1 ? -1 : g - 2), fout = flag_of(epoch, g == 0 ? -2 : b);
            const int par = g & 1;
            const void *Gm = g == 0 ? static_cast<const void *>(p.gate0) : p.blocks[b].pre_gate;
            const pgmoe_routing rout = g == 0 ? p.gate0_out : p.blocks[b].out;
            const unsigned long long *base = p.llpart + (size_t)par * nd * T * W * 2;
            // 1. this CTA's 16 experts: partials of its producer chunk, in order
            {
                const int j = 16 * q + jj;
                double s = 0.0;
                for (int q0 = qp0; q0 < qp1; q0 += 16) {
                    unsigned long long lo[16], hi[16];
                    uint32_t valid = 0;
#pragma unroll
                    for (int u = 0; u < 16; ++u)
                        if (q0 + u < qp1) valid |= 1u << u;
                    poll2<16>([&](int u) { return base + (((size_t)(q0 + u) * T + t) * W + j) * 2; }, valid, fin, lo,
                              hi);
#pragma unroll
                    for (int u = 0; u < 16; ++u)
                        if (valid >> u & 1u) s += __hiloint2double((int)(uint32_t)hi[u], (int)(uint32_t)lo[u]);
                }
                rlg[kc * 16 + jj] = s;
            }
            rsync();
            if (rt < 16) {  // chunk order: deterministic
                double s = 0.0;
                for (int k = 0; k < NK; ++k) s += rlg[k * 16 + rt];
                st_ll_f64(p.lllog + (((size_t)par * T + t) * E + 16 * q + rt) * 2, s, fout);
            }
            if (!selector) {
                rsync();
                continue;
            }
            // 2. selector: this token's block input (the serial fallback's
            //    operand), the producers' sum|x| / max|G|, the E logits
            if (g <= 1) {
                for (int i = rt; i < d; i += kRThreads) rx[i] = __ldcg(p.x_in + (size_t)t * d + i);
            } else {
                const unsigned long long *xq = p.llx + ((size_t)(b & 1) * T + t) * d;
                for (int i0 = rt; i0 < d; i0 += 16 * kRThreads) {
                    unsigned long long v[16];
                    uint32_t valid = 0;
#pragma unroll
                    for (int u = 0; u < 16; ++u)
                        if (i0 + u * kRThreads < d) valid |= 1u << u;
                    poll1<16>([&](int u) { return xq + i0 + u * kRThreads; }, valid, fin, v);
#pragma unroll
                    for (int u = 0; u < 16; ++u)
                        if (valid >> u & 1u) rx[i0 + u * kRThreads] = __uint_as_float((uint32_t)v[u]);
                }
            }
            {   // the producers' sum|x| / max|G| words and the E logits: one batch
                unsigned long long lo[4], hi[4];
                const unsigned long long *pq = base + (((size_t)rt * T + t) * W + E) * 2;
                const unsigned long long *lq = p.lllog + ((size_t)par * T + t) * E * 2;
                auto addr = [&](int u) { return u < 2 ? pq + 2 * u : lq + (rt + (u - 2) * kRThreads) * 2; };
                uint32_t pend = (rt < nd ? 3u : 0u) | (rt < E ? 4u : 0u) | (rt + kRThreads < E ? 8u : 0u);
                const uint32_t valid = pend;
                while (pend) {
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (pend >> u & 1u) ld_ll2(addr(u), lo[u], hi[u]);
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint32_t fl = u < 2 ? fin : fout;
                        if ((pend >> u & 1u) && (uint32_t)(lo[u] >> 32) == fl && (uint32_t)(hi[u] >> 32) == fl)
                            pend &= ~(1u << u);
                    }
                }
                rsx[rt] = (valid & 1u) ? __hiloint2double((int)(uint32_t)hi[0], (int)(uint32_t)lo[0]) : 0.0;
                rgx[rt] = (valid & 2u) ? __hiloint2double((int)(uint32_t)hi[1], (int)(uint32_t)lo[1]) : 0.0;
                if (valid & 4u) rsel[rt] = __hiloint2double((int)(uint32_t)hi[2], (int)(uint32_t)lo[2]);
                if (valid & 8u) rsel[rt + kRThreads] = __hiloint2double((int)(uint32_t)hi[3], (int)(uint32_t)lo[3]);
            }
            rsync();
            if (rt < 32) {
                const double sxt = warp_sumd(rsx[rt] + rsx[rt + 32]);
                const double gxt = warp_max(fmax(rgx[rt], rgx[rt + 32]));
                for (int j = rt; j < E; j += 32) rcm[j] = (float)gxt;  // exact: a bf16 magnitude
                if (rt == 0) rsx[kRThreads] = sxt;
                __syncwarp();
                TileSums ts;
                ts.lgs = rsel;
                ts.cms = rcm;
                ts.sxs = rsx + kRThreads;
                r.G = Gm;
                r.out = rout;
                if (E == 64) router_select_token<uint16_t, 2>(r, ts, 0, t, lane, s_ids, s_w);
                else router_select_token<uint16_t, 4>(r, ts, 0, t, lane, s_ids, s_w);
                __syncwarp();
                if (lane == 0) {
                    unsigned long long *qd = p.lldec + ((size_t)g * kLLMaxT + t) * 2;
                    st_ll2(qd, ll_word((uint32_t)s_ids[0], fout), ll_word(__float_as_uint(s_w[0]), fout));
                    if (p.ids_trace) {
                        p.ids_trace[(size_t)g * T + t] = s_ids[0];
                        p.w_trace[(size_t)g * T + t] = s_w[0];
                    }
                    dprobe(p, b, 5);
                }
            }
            rsync();
        }
        return;
    }

    // ============ compute warps (2..9) ======================================
    const int ct = tid - kCW0 * 32;
    int pc = 0, dfill = 0;
    float out;
    int orow, otok;
    if (dense_cta) {  // prologue (fill 0): block 0's gate and block 0's pre-gate, both on x_in
        mbar_wait(dfull, 0);
        for (int i = ct; i < kDRows * 8; i += kCThreads) {
            const int rr = i >> 3, t = i & 7;
            ytile[i] = t < T ? __ldcg(p.x_in + (size_t)t * d + dr0 + rr) : 0.f;
        }
        csync();
        pregate_partials(p, ytile, gsl0, red, c, 0, flag_of(epoch, -1), ct);
        if (p.blocks[0].has_pre_gate) {
            csync();  // red is reused
            pregate_partials(p, ytile, gsl, red, c, 1, flag_of(epoch, -1), ct);
        }
        csync();
        if (ct == 0) mbar_arrive(dempty);
        dfill = 1;
    }
    for (int b = 0; b < nb; ++b) {
        const uint32_t fl = flag_of(epoch, b), fprev = flag_of(epoch, b - 1);
        // ---- expert phases: up (h = relu(W1 x)), down (mix = w * W2 h) ----
        for (int ph = 0; ph < 2; ++ph) {
            int staged = -1;
            bool first = true;
            for (;;) {
                const int slot = pc % kSlots;
                PCLK(tw);
                mbar_wait(&full[slot], (pc / kSlots) & 1);
                PACC(b, ph, 0, tw);
                const Piece &pd = desc[slot];
                const int nrows = pd.nrows, ng = pd.ng, e = pd.e, row0 = pd.row0, end = pd.end;
                if (nrows > 0) {
                    const int K = ph == 0 ? d : f;
                    // this thread's output column (piece_gemv: token ct & 7), read before the
                    // slot is released
                    const int my_t = (ct & 7) < ng ? pd.tok[ct & 7] : 0;
                    const float my_w = pd.w[ct & 7];
                    PCLK(ts);
                    if (e != staged) {
                        if (ph == 0)
                            stage(act, d, ng, pd.tok, p.llx + (size_t)(b & 1) * T * d, d,
                                  b == 0 ? p.x_in : nullptr, d, fprev, ct);
                        else
                            stage(act, f, ng, pd.tok, p.llh, f, nullptr, 0, fl, ct);
                        staged = e;
                        if (first && ct == 0) dprobe(p, b, ph == 0 ? 1 : 3);
                        first = false;
                    }
                    PACC(b, ph, 1, ts);
                    PCLK(tg);
                    piece_gemv(slots + (size_t)slot * kSlotB, K * 2 + 16, nrows, act, K * 2 + 16, ng, K, red, ct,
                               out, orow, otok, &empty[slot]);
                    PACC(b, ph, 2, tg);
                    PCLK(te);
                    if (orow >= 0 && orow < nrows && otok < ng) {
                        const int t = my_t;
                        if (ph == 0)
                            st_ll(p.llh + (size_t)t * f + row0 + orow,
                                  ll_word(__float_as_uint(fmaxf(out, 0.f)), fl));  // relu, linalg.py:41-42
                        else  // top-1 combine: mix = w * y (linalg.py:45-51)
                            st_ll(p.llmix + (size_t)t * d + row0 + orow, ll_word(__float_as_uint(my_w * out), fl));
                    }
                    PACC(b, ph, 3, te);
#ifdef PGMOE_LL_PROBE
                    if (p.probe && b == 2 && ct == 0) p.probe[(size_t)blockIdx.x * kProbeSlots + 45 + ph] += 1;
#endif
                } else {
                    __syncwarp();
                    if ((ct & 31) == 0) mbar_arrive(&empty[slot]);  // one arrival per compute warp
                }
                ++pc;
                if (end) break;
            }
            if (ct == 0) dprobe(p, b, ph == 0 ? 2 : 4);
        }
        // ---- dense layer (core.py:338) + the next pre-gate's partials ----
        if (dense_cta) {
            mbar_wait(dfull, dfill & 1);
            stage(act, d, T, nullptr, p.llmix, d, nullptr, 0, fl, ct);
            if (ct == 0) dprobe(p, b, 6);
            piece_gemv(dbuf, dpitch, kDRows, act, d * 2 + 16, T, d, red, ct, out, orow, otok);
            if (orow >= 0 && otok < T) {
                const int row = dr0 + orow;
                ytile[orow * 8 + otok] = out;
                if (b + 1 < nb) {
                    st_ll(p.llx + ((size_t)((b + 1) & 1) * T + otok) * d + row, ll_word(__float_as_uint(out), fl));
                    if (p.x_trace) p.x_trace[((size_t)(b + 1) * T + otok) * d + row] = out;
                } else {
                    p.y_out[(size_t)otok * d + row] = out;
                }
            }
            csync();
            if (b + 1 < nb && p.blocks[b + 1].has_pre_gate)  // gate g = b + 2
                pregate_partials(p, ytile, gsl, red, c, b & 1, fl, ct);
            csync();
            if (ct == 0) {
                mbar_arrive(dempty);
                dprobe(p, b, 7);
            }
            ++dfill;
        }
    }
    // ---- epoch: the last CTA to finish advances it for the next launch ----
    csync();
    if (ct == 0) {
        __threadfence();
        if (atomicAdd(p.ctr + 1, 1u) == (unsigned)G - 1) {
            p.ctr[1] = 0;
            p.ctr[0] = epoch + 1 > 0x1FFFFFFu ? 1u : epoch + 1;
            __threadfence();
        }
#ifdef PGMOE_LL_PROBE
        if (p.probe) p.probe[(size_t)c * kProbeSlots + 41] = gtimer();
#endif
    }
}

// Shared memory of a launch: the weight ring (nslots), the dense slice, the
// staged activations of T tokens (mma B rows past T are never read: columns
// repeat the last staged token) and small per-role buffers.
size_t smem_bytes(int T, int d, int f, int E, int nslots, int slot_bytes = kSlotBytes) {
    return (size_t)nslots * slot_bytes + (size_t)kDRows * (d * 2 + 16) + (size_t)2 * kDRows * E * 2 +
           (size_t)((T + 1) & ~1) * (f * 2 + 16) + (size_t)kCWarps * 128 * 4 + kDRows * 8 * 4 + (size_t)d * 4 +
           (kRThreads + kMaxE) * 8 + kMaxE * 4 + (2 * kRThreads + 1) * 8 + nslots * sizeof(Piece) + 16 +
           (2 * nslots + 2) * 8 + 2 * kLLMaxT * 4 + 64;
}
constexpr size_t kSmemCap = 226 * 1024;
// The ring: bigger slots mean fewer, larger pieces (each piece pays a fixed
// K-split reduction, two barriers and an epilogue).  Rule: the largest slot
// (65, 48, 33 KB) that still leaves at least 2 slots.  Measured (A/B of
// PGMOE_LL_SLOT_KB on one box, us per block, 33 KB -> chosen): Base-64
// T=1 10.6 -> 9.4, T=2 13.3 -> 11.8, T=4 18.6 -> 15.7, T=8 32.5 -> 28.3;
// Large-128 T=1 11.8 -> 10.1, T=2 16.9 -> 13.2, T=4 25.4 -> 20.6, T=8
// 51.9 -> 47.6 (48 KB: 64 KB slots do not fit twice there).
void pick_ring(int T, int d, int f, int E, int *nslots, int *slot_bytes) {
    static const int sizes[3] = {65536 + 1024, 49152, kSlotBytes};
    int force = 0;
    if (const char *e = getenv("PGMOE_LL_SLOT_KB")) force = atoi(e) * 1024;
    for (int i = 0; i < 3; ++i) {
        int sb = sizes[i];
        if (force && sb != (force >= 60 * 1024 ? sizes[0] : force >= 40 * 1024 ? sizes[1] : sizes[2])) continue;
        int n = kMaxSlots;
        while (n > 2 && smem_bytes(T, d, f, E, n, sb) > kSmemCap) --n;
        if (smem_bytes(T, d, f, E, n, sb) <= kSmemCap) {
            *nslots = n;
            *slot_bytes = sb;
            return;
        }
    }
    *nslots = 3;
    *slot_bytes = kSlotBytes;
}

}  // namespace ll

bool ll_decode_supported(int T, int d, int f, int E, int k, int L, int nb) {
    return T >= 1 && T <= kLLMaxT && k == 1 && L == 1 && d % ll::kDRows == 0 && d % 16 == 0 && f % 16 == 0 &&
           (E == 64 || E == 128) && nb >= 2 && nb <= kDecodeMaxBlocks && d * 2 + 16 <= ll::kSlotBytes &&
           f * 2 + 16 <= ll::kSlotBytes && ll::smem_bytes(kLLMaxT, d, f, E, 3) <= ll::kSmemCap &&
           d / ll::kDRows <= ll::kRThreads &&
           d / ll::kDRows + kLLMaxT * (E / 16) <= device_sm_count();
}

// Workspace: [epoch counter | llx | llh | llmix | llpart | lldec | lllog], 256-byte aligned parts.
static size_t ll_ws_layout(int T, int d, int f, int E, int nb, size_t *off) {
    const int nd = d / ll::kDRows;
    const size_t words[6] = {(size_t)2 * T * d, (size_t)T * f, (size_t)T * d, (size_t)2 * nd * T * (E + 2) * 2,
                             (size_t)nb * kLLMaxT * 2, (size_t)2 * T * E * 2};
    size_t o = 256;
    for (int i = 0; i < 6; ++i) {
        if (off) off[i] = o;
        o += (words[i] * 8 + 255) & ~(size_t)255;
    }
    return o;
}

size_t ll_decode_ws_bytes(int T, int d, int f, int E, int nb) { return ll_ws_layout(T, d, f, E, nb, nullptr); }

int ll_decode_prepare(void *ws, cudaStream_t s) {
    // the epoch counter starts at 1: flags are never 0, the value of fresh memory
    const unsigned init[2] = {1u, 0u};
    PG_CUDA(cudaMemcpyAsync(ws, init, sizeof(init), cudaMemcpyHostToDevice, s));
    PG_CUDA(cudaStreamSynchronize(s));
    return PGMOE_OK;
}

int ll_decode_iteration(const LLDecodeArgs &a, cudaStream_t s) {
    using namespace ll;
    int nslots = 3, slot_bytes = kSlotBytes;
    pick_ring(a.T, a.d, a.f, a.E, &nslots, &slot_bytes);
    const size_t smem = smem_bytes(a.T, a.d, a.f, a.E, nslots, slot_bytes);
    static size_t attr_smem[64] = {0};  // per device: dynamic shared memory the attribute allows
    static int grid_dev[64] = {0};
    const int dev = current_device();
    PG_REQUIRE(dev >= 0 && dev < 64, PGMOE_E_CONFIG, "device ordinal %d unsupported", dev);
    if (smem > attr_smem[dev]) {
        PG_CUDA(cudaFuncSetAttribute(ll_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        PG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ll_decode_kernel, kThreads, smem));
        // every CTA polls words other CTAs write: all must be co-resident
        PG_REQUIRE(per_sm >= 1, PGMOE_E_CUDA, "ll decode kernel: no CTA fits on an SM");
        grid_dev[dev] = device_sm_count();
        attr_smem[dev] = smem;
    }
    const int G = grid_dev[dev];
    const int nd = a.d / kDRows;
    PG_REQUIRE(nd + a.T * (a.E / 16) <= G, PGMOE_E_CONFIG, "ll decode: %d dense + %d reducer CTAs exceed the grid (%d)",
               nd, a.T * (a.E / 16), G);
    Params p{};
    p.T = a.T;
    p.d = a.d;
    p.f = a.f;
    p.E = a.E;
    p.nb = a.nb;
    p.nd = nd;
    p.nslots = nslots;
    p.slot_bytes = slot_bytes;
    p.blocks = a.blocks;
    p.experts = static_cast<const unsigned char *>(a.experts);
    p.rec_bytes = a.rec_bytes;
    p.pool = a.pool;
    p.x_in = a.x_in;
    p.y_out = a.y_out;
    p.gate0 = static_cast<const uint16_t *>(a.gate0);
    p.gate0_out = a.gate0_out;
    char *w = static_cast<char *>(a.ws);
    size_t off[6];
    const size_t need = ll_ws_layout(a.T, a.d, a.f, a.E, a.nb, off);
    PG_REQUIRE(need <= a.ws_bytes, PGMOE_E_CONFIG, "ll decode workspace too small (%zu > %zu)", need, a.ws_bytes);
    p.ctr = reinterpret_cast<unsigned *>(w);
    p.llx = reinterpret_cast<unsigned long long *>(w + off[0]);
    p.llh = reinterpret_cast<unsigned long long *>(w + off[1]);
    p.llmix = reinterpret_cast<unsigned long long *>(w + off[2]);
    p.llpart = reinterpret_cast<unsigned long long *>(w + off[3]);
    p.lldec = reinterpret_cast<unsigned long long *>(w + off[4]);
    p.lllog = reinterpret_cast<unsigned long long *>(w + off[5]);
    route_bound_constants(a.d, &p.gam, &p.bscale);
    p.x_trace = a.x_trace;
    p.ids_trace = a.ids_trace;
    p.w_trace = a.w_trace;
    p.probe = probe_buffer(1, G);
    // Cooperative: every CTA polls words other CTAs write, so the launch must
    // be all-or-nothing co-resident (another persistent kernel on a second
    // stream must not hold part of the SMs while this one spins on the rest).
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    PG_CUDA(cudaLaunchKernelEx(&cfg, ll_decode_kernel, p));
    count_launch();
    return PGMOE_OK;
}

}  // namespace pgmoe
