// ffn_tc.cu — K2/K3 on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// One persistent, warp-specialised kernel runs the dense contractions of a
// block as consecutive PHASES of a single launch (core.py:308-316, :338):
//   up   : hb[r][m]  = bf16(relu(W1_e[m] . xb[r]))              (M = f, K = d)
//   down : yw[perm[r]][m] = w_perm[r] * (W2_e[m] . hb[r])       (M = d, K = f)
//          (+ mixb[perm[r]][m] = bf16(that) when top_k == 1)
//   dense: y[t][m]  = D[m] . mixb[t]                            (M = d, K = d)
//          (+ the next block's packed operand, see next_xb)
// "Swap-AB": weight rows fill the 128-row UMMA M dimension and the few
// routed tokens of an expert are the N dimension (padded to 16), so every
// weight tile is streamed from HBM exactly once; the kernel is bound by
// weight bytes, which is the roofline at these shapes.
//
// Both operands arrive by TMA into 128-byte-swizzled K-major tiles: the
// weights through a 3-D map over the expert records (K, rows, record) and
// the activations (bf16 rows in routing order, so an expert's tokens are
// contiguous) through a 2-D map in 16-row boxes.  A phase's activations are
// the previous phase's output, so a grid-wide barrier separates phases; its
// latency is hidden because the producer keeps streaming the next phase's
// WEIGHT tiles into free pipeline stages and only defers their activation
// boxes until the barrier opens (the same trick hides the programmatic-
// dependent-launch wait of phase 0).
//
// Warp roles (224 threads, one CTA per SM, grid = #SMs so all CTAs are
// co-resident for the barrier):
//   warp 0      : weight TMA producer + unit scheduler (one lane)
//   warp 6      : gated activation TMA producer (one lane)
//   warp 1      : TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-5   : epilogue — tcgen05.ld the fp32 accumulator, ReLU / combine
//                 weight / scatter, or the split-K fix-up; signals phases
// Phases with few tiles split K across CTAs; the last CTA to finish a tile
// (atomic ticket) sums the partials in split order — deterministic — and
// runs the epilogue.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "route_common.cuh"
#include "tc_common.cuh"

namespace pgmoe {

namespace tc {

constexpr int kThreads = 352;  // 11 warps (3 per scheduler at most: 168 registers either way)
constexpr int kMaxGroups = 512;        // active experts per launch (smem schedule arrays)
constexpr int kMaxPhases = 3;
constexpr int kCounterInts = 8192;    // split-K tile tickets at the head of the workspace
constexpr int kSyncInts = 16 + kMaxGroups;  // phase barriers, exit ticket, unit counter; per-group up tiles done
constexpr int kUnitQ = 16;            // producer -> MMA / epilogue unit queue (shared memory ring)
constexpr int kMetaInts = 512;        // per-column epilogue metadata staged in shared memory
// split-K cost model (bytes per microsecond; microseconds)
constexpr float kSmBytesPerUs = 150e3f;   // one SM's TMA stream when few CTAs load
constexpr float kHbmBytesPerUs = 6.5e6f;  // whole-chip HBM stream
constexpr float kFixUs = 3.0f;            // split-K fix-up chain (stores, fence, ticket)
constexpr float kFixRoundUs = 1.0f;       // + one dependent partial-load round per kFixSplits splits
constexpr int kFixSplits = 4;

enum Mode { kUp = 0, kDown = 1, kDense = 2 };

struct PhaseDesc {
    int mode, M, K;
    float *out_f32;      // kDown: yw [T*k][M] ; kDense: y [T][M]
    uint16_t *out_bf16;  // kUp: hb [T*k][M] ; kDown (k == 1): mixb [T][M]
};

struct Params {
    int nphase, T, k;
    PhaseDesc ph[kMaxPhases];
    const int *act, *n_act, *off, *hist, *perm;
    const float *w_perm;
    int indexed_by_act;
    // dense epilogue: the next block's routing is already known (pre-gate),
    // so it also writes the next up-projection's packed bf16 operand:
    // next_xb[next_inv[t*k+s]][m] = bf16(y[t][m])
    uint16_t *next_xb;
    const int *next_inv;
    int *counters;   // [kCounterInts] split-K tickets
    int *sync;       // [kSyncInts] phase_done[kMaxPhases], exit ticket, unit counter, grp_done[kMaxGroups]
    float *partial;
    long long partial_cap;  // floats
    unsigned long long *probe;  // debug stamps [grid][kProbeSlots] or null
    FusedRoute route;           // the next block's routing, computed by warps 7-10 (resident)
    int max_inflight;           // weight stages the producer keeps in flight (<= STAGES)
    int max_split;              // cap on the split-K factor (0: cost model only)
    // Chained launches (resident decoder): instead of waiting for the previous
    // launch to COMPLETE (griddepcontrol.wait, ~4-6 us after its last CTA),
    // phase 0 and the routing role wait for its dense phase to be written:
    // *epoch >= epoch_wait.  This launch sets *epoch = epoch_set once its own
    // dense phase is complete.  Counters / partials alternate between two
    // parity buffers, so a launch never touches what its predecessor re-arms.
    int *epoch;                 // null: not chained
    int epoch_wait, epoch_set;
    unsigned long long *stamps;  // chained: stamps[epoch_set] = %globaltimer at dense-phase completion
};

struct PhaseSched {
    int mode, M, K, m_tiles, kb_total, kbs, S;
    int nw;               // token columns per tile (BN; narrower for the dense phase)
    int ctr0;             // first split-K ticket of this phase (phases may overlap)
    long long part0;      // first partial-tile float of this phase
    long long tiles, units, unit0;
};

struct Unit {
    int ph, g, m_tile, n0, n_valid, n_pad, kb0, kb1, tile, s, row0, rec;
};

struct Groups {
    int n;              // expert groups (routing)
    int T;              // tokens (dense)
    const int *ntp;     // [n + 1] prefix of N tiles per group (smem)
    const int *rec, *row0, *ng;  // per group (smem)
};

template <int BN>
__device__ __forceinline__ Unit decode_unit(const PhaseSched *ps, int nphase, const Groups &gr, long long u) {
    Unit x;
    int ph = 0;
    while (ph + 1 < nphase && u >= ps[ph + 1].unit0) ++ph;
    const PhaseSched &sc = ps[ph];
    const int lu = (int)(u - sc.unit0);  // 32-bit: a 64-bit divide is ~100 instructions per unit
    x.ph = ph;
    x.tile = lu / sc.S;
    x.s = lu - x.tile * sc.S;
    int ng;
    if (sc.mode == kDense) {
        x.g = 0;
        const int n_tile = x.tile / sc.m_tiles;
        x.m_tile = x.tile - n_tile * sc.m_tiles;
        x.n0 = n_tile * sc.nw;
        ng = gr.T;
        x.row0 = 0;
        x.rec = 0;
    } else {
        int lo = 0, hi = gr.n - 1;  // last g with ntp[g] * m_tiles <= tile
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (gr.ntp[mid] * sc.m_tiles <= x.tile) lo = mid;
            else hi = mid - 1;
        }
        x.g = lo;
        const int local = x.tile - gr.ntp[lo] * sc.m_tiles;
        const int n_tile = local / sc.m_tiles;
        x.m_tile = local - n_tile * sc.m_tiles;
        x.n0 = n_tile * BN;
        ng = gr.ng[lo];
        x.row0 = gr.row0[lo];
        x.rec = gr.rec[lo];
    }
    x.n_valid = min(sc.nw, ng - x.n0);
    x.n_pad = max(16, (x.n_valid + 15) & ~15);
    x.kb0 = x.s * sc.kbs;
    x.kb1 = min(sc.kb_total, x.kb0 + sc.kbs);
    return x;
}

// Epilogue stores.  Everything a stored column needs is in registers before
// the first store of a 16-column chunk: the per-unit constants (EpiRegs,
// loaded once per unit) and the per-column metadata (down: destination token
// and combine weight; dense: the next block's packed rows), which the
// epilogue threads stage in shared memory together while the MMA runs and
// each thread then reads for its chunk in one batch.  (Reading them between
// stores would serialise: every st.global is a compiler memory barrier, so
// shared-memory values would be re-read, one dependent LDS chain per
// column — measured at ~0.2 us per column.)
struct EpiRegs {
    int mode, M, k;
    bool staged;
    float *out_f32;
    uint16_t *out_bf16;
    uint16_t *next_xb;
    const int *perm, *next_inv;
    const float *w_perm;
};

__device__ __forceinline__ EpiRegs epi_regs(const Params &p, const PhaseDesc &pd, const Unit &x) {
    EpiRegs e;
    e.mode = pd.mode;
    e.M = pd.M;
    e.k = p.k;
    e.out_f32 = pd.out_f32;
    e.out_bf16 = pd.out_bf16;
    e.next_xb = pd.mode == kDense ? p.next_xb : nullptr;
    e.perm = p.perm;
    e.w_perm = p.w_perm;
    e.next_inv = p.next_inv;
    e.staged = (e.mode == kDown && x.n_valid <= kMetaInts / 2) ||
               (e.mode == kDense && e.next_xb != nullptr && x.n_valid * e.k <= kMetaInts);
    return e;
}

__device__ __forceinline__ void stage_meta(const EpiRegs &e, const Unit &x, int et, int *mi, float *mf) {
    if (!e.staged) return;
    if (e.mode == kDown) {
        for (int c = et; c < x.n_valid; c += 128) {
            const int r = x.row0 + x.n0 + c;
            mi[c] = __ldg(e.perm + r);
            mf[c] = __ldg(e.w_perm + r);
        }
    } else {
        for (int c = et; c < x.n_valid * e.k; c += 128) mi[c] = __ldg(e.next_inv + (size_t)x.n0 * e.k + c);
    }
}

// Columns [c0, c0 + 16) of the accumulator rows this warp owns (m0w + lane),
// only those < x.n_valid.  The warp transposes its 32 x 16 slice through a
// 2 KB shared staging tile so that every global store is a 16-byte vector of
// consecutive output rows (one thread per (column, row group)): a scalar
// st.global per column per thread costs ~40 cycles of LSU issue per warp.
__device__ __forceinline__ void store_chunk(const EpiRegs &e, const Unit &x, int c0, int m0w, int lane,
                                            const float (&v)[16], const int *mi, const float *mf, float *stg) {
    const int nv = min(16, x.n_valid - c0);
    if (e.mode == kDown) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {  // combine weight (linalg.py:45-51), one per column
            const float w = j < nv ? (e.staged ? mf[c0 + j] : __ldg(e.w_perm + x.row0 + x.n0 + c0 + j)) : 0.f;
            stg[j * 32 + lane] = w * v[j];
        }
    } else if (e.mode == kUp) {
#pragma unroll
        for (int j = 0; j < 16; ++j) stg[j * 32 + lane] = fmaxf(v[j], 0.f);  // relu, linalg.py:41-42
    } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) stg[j * 32 + lane] = v[j];
    }
    __syncwarp();
    // fp32 rows: down -> yw[perm[r]], dense -> y[token]; 8 float4 per column
    if (e.mode != kUp) {
        for (int i = lane; i < nv * 8; i += 32) {
            const int col = i >> 3, g = i & 7;
            const int row = e.mode == kDown
                                ? (e.staged ? mi[c0 + col] : __ldg(e.perm + x.row0 + x.n0 + c0 + col))
                                : x.n0 + c0 + col;
            const float4 val = *reinterpret_cast<const float4 *>(stg + col * 32 + g * 4);
            __stcg(reinterpret_cast<float4 *>(e.out_f32 + (size_t)row * e.M + m0w + g * 4), val);
        }
    }
    // bf16 rows: up -> hb[r], down (top-1) -> mixb[perm[r]], dense -> the next
    // block's packed rows next_xb[next_inv[t*k+s]]; 4 x 16 bytes per column
    uint16_t *ob = e.mode == kDense ? e.next_xb : e.out_bf16;
    if (ob != nullptr) {
        const int slots = e.mode == kDense ? e.k : 1;
        for (int i = lane; i < nv * 4 * slots; i += 32) {
            const int s = i / (nv * 4), rem = i - s * (nv * 4);
            const int col = rem >> 2, g = rem & 3;
            int row;
            if (e.mode == kUp) {
                row = x.row0 + x.n0 + c0 + col;
            } else if (e.mode == kDown) {
                row = e.staged ? mi[c0 + col] : __ldg(e.perm + x.row0 + x.n0 + c0 + col);
            } else {
                const int idx = (c0 + col) * e.k + s;
                row = e.staged ? mi[idx] : __ldg(e.next_inv + (size_t)x.n0 * e.k + idx);
            }
            const float4 a = *reinterpret_cast<const float4 *>(stg + col * 32 + g * 8);
            const float4 b = *reinterpret_cast<const float4 *>(stg + col * 32 + g * 8 + 4);
            uint4 o;
            o.x = bf16_bits(a.x) | ((uint32_t)bf16_bits(a.y) << 16);
            o.y = bf16_bits(a.z) | ((uint32_t)bf16_bits(a.w) << 16);
            o.z = bf16_bits(b.x) | ((uint32_t)bf16_bits(b.y) << 16);
            o.w = bf16_bits(b.z) | ((uint32_t)bf16_bits(b.w) << 16);
            __stcg(reinterpret_cast<uint4 *>(ob + (size_t)row * e.M + m0w + g * 8), o);
        }
    }
    __syncwarp();  // the staging tile is rewritten by the next chunk
}


template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
block_gemm_kernel(const __grid_constant__ CUtensorMap a0, const __grid_constant__ CUtensorMap b0,
                  const __grid_constant__ CUtensorMap a1, const __grid_constant__ CUtensorMap b1,
                  const __grid_constant__ CUtensorMap a2, const __grid_constant__ CUtensorMap b2,
                  const Params p_in) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // Kernel parameters live in the constant bank; the epilogue indexes the
    // phase descriptors dynamically and, under register pressure, the
    // compiler re-reads them per stored column (indexed LDC, slow on a miss).
    // One copy in shared memory makes every such read an LDS.
    __shared__ Params p_sh;
    __shared__ PhaseSched ps[kMaxPhases];
    __shared__ __align__(16) float r_xs[kRouterSmemFloats];  // routing role: x slice, reduction, permutation
    static_assert(kRouterSmemFloats >= kRouterTok * kRouterMaxKn, "routing x slice");
    __shared__ int r_flag;
    __shared__ long long s_total_units;
    static_assert(sizeof(Params) % 4 == 0 && sizeof(Params) / 4 <= kThreads, "Params copy");
    if (threadIdx.x < sizeof(Params) / 4)
        reinterpret_cast<int *>(&p_sh)[threadIdx.x] = reinterpret_cast<const int *>(&p_in)[threadIdx.x];
    __syncthreads();
    const Params &p = p_sh;
    // 1024-byte alignment by pointer arithmetic on the shared array (an
    // integer round trip would lose the state space and turn every shared
    // access below into a generic one that must order against global stores)
    unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    constexpr int kBBytes = BN * 128;
    unsigned char *sA = smem;
    unsigned char *sB = smem + STAGES * kABytes;
    uint64_t *full = reinterpret_cast<uint64_t *>(sB + STAGES * kBBytes);
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;
    uint64_t *tempty = tfull + 2;
    uint64_t *uq_full = tempty + 2;       // [kUnitQ]
    uint64_t *uq_empty = uq_full + kUnitQ;  // [kUnitQ]
    long long *unit_q = reinterpret_cast<long long *>(uq_empty + kUnitQ);  // [kUnitQ]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(unit_q + kUnitQ);
    int *s_flag = reinterpret_cast<int *>(tmem_slot + 1);
    int *ntp = s_flag + 4;
    int *g_rec = ntp + kMaxGroups + 1;
    int *g_row0 = g_rec + kMaxGroups;
    int *g_ng = g_row0 + kMaxGroups;
    int *meta_i = g_ng + kMaxGroups;                            // [kMetaInts]
    float *meta_f = reinterpret_cast<float *>(meta_i + kMetaInts);  // [kMetaInts / 2]
    unsigned char *stage_raw = reinterpret_cast<unsigned char *>(meta_f + kMetaInts / 2);
    float *stage_out = reinterpret_cast<float *>(stage_raw + ((16u - (smem_u32(stage_raw) & 15u)) & 15u));
    // ^ [4 warps][16 cols][32 rows], 16-byte aligned for the vector reads
    const CUtensorMap *amaps[3] = {&a0, &a1, &a2};
    const CUtensorMap *bmaps[3] = {&b0, &b1, &b2};

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        probe(p.probe, blockIdx.x, 0);  // entry
        if (p.probe) p.probe[(size_t)blockIdx.x * kProbeSlots + 21] = clock64();
    }
    bool has_expert_phase = false, has_dense = false;
    for (int i = 0; i < p.nphase; ++i) {
        has_expert_phase |= p.ph[i].mode != kDense;
        has_dense |= p.ph[i].mode == kDense;
    }

    // ---- schedule (identical in every CTA) --------------------------------
    Groups gr;
    gr.n = has_expert_phase ? __ldg(p.n_act) : 0;
    gr.T = p.T;
    gr.ntp = ntp;
    gr.rec = g_rec;
    gr.row0 = g_row0;
    gr.ng = g_ng;
    if (warp == 0) {
        int run = 0, mx = 16;
        for (int g0 = 0; g0 < gr.n; g0 += 32) {
            const int g = g0 + lane;
            int nt = 0;
            if (g < gr.n) {
                const int e = __ldg(p.act + g);
                const int ng = __ldg(p.hist + e);
                g_rec[g] = p.indexed_by_act ? g : e;
                g_row0[g] = __ldg(p.off + e);
                g_ng[g] = ng;
                nt = (ng + BN - 1) / BN;
                mx = max(mx, (min(ng, BN) + 15) & ~15);
            }
            int incl = nt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            if (g < gr.n) ntp[g] = run + incl - nt;
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0) {
            ntp[gr.n] = run;
            s_flag[1] = mx;
            s_flag[2] = run;
        }
    }
    if (warp == 1) {  // TMEM: two accumulator stages of BN fp32 columns
        constexpr uint32_t cols = (2 * BN < 32) ? 32 : 2 * BN;
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 64) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&full[i], 1);   // producer arrive.expect_tx (A + B bytes)
            mbar_init(&empty[i], 1);  // tcgen05.commit
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 128);
        }
        for (int i = 0; i < kUnitQ; ++i) {
            mbar_init(&uq_full[i], 1);   // producer
            mbar_init(&uq_empty[i], 3);  // MMA lane 0, activation producer, one epilogue thread
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid == 96) {
        for (int i = 0; i < p.nphase; ++i) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(amaps[i]) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(bmaps[i]) : "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (tid == 0) probe(p.probe, blockIdx.x, 1);  // prologue done
    const int max_npad_expert = s_flag[1], ntiles_expert = s_flag[2];

    // One warp: every lane prices one split factor (the cost model is on the
    // critical path of every CTA that enters after its dependency resolved)
    if (warp == 0) {
    long long total_units = 0, part_used = 0;
    int ctr_used = 0;
    const int grid = (int)gridDim.x;
    for (int i = 0; i < p.nphase; ++i) {
        PhaseSched sc;
        sc.mode = p.ph[i].mode;
        sc.M = p.ph[i].M;
        sc.K = p.ph[i].K;
        sc.m_tiles = sc.M / BM;
        sc.kb_total = sc.K / BK;
        int max_npad;
        if (sc.mode == kDense) {
            // The dense phase has few tiles (T / BN x d / 128) and a serial
            // epilogue per tile: 32-token tiles double the CTAs sharing it
            // (the 1-2 MB weight tile is re-read from L2, not HBM)
            sc.nw = (BN >= 64 && p.T > 32) ? 32 : BN;
            sc.tiles = (long long)((p.T + sc.nw - 1) / sc.nw) * sc.m_tiles;
            max_npad = max(16, (min(p.T, sc.nw) + 15) & ~15);
        } else {
            sc.tiles = (long long)ntiles_expert * sc.m_tiles;
            sc.nw = BN;
            max_npad = max_npad_expert;
        }
        // Split K only when it pays for its fix-up.  A split-K tile costs one
        // extra dependent chain (partials out, fence + ticket, partials in:
        // ~kFixUs) but spreads the tile's K stream over S CTAs.  Streaming
        // time of a unit = its bytes / per-CTA bandwidth, where the per-CTA
        // bandwidth is the single-SM TMA limit when few CTAs stream and the
        // HBM share when all do (measured on B200 with tools/probe.py).
        int s_cap = max(1, min(sc.kb_total, 8 * 16 / min(BN, max_npad)));
        if (p.max_split > 0) s_cap = min(s_cap, p.max_split);
        const float kb_bytes = (float)(kABytes + max_npad * 128);
        const int tiles = (int)sc.tiles;
        const int cand = lane + 1;
        float t = 3.4e38f;
        // Beyond 2, a split only pays as coverage (at most one unit per
        // CTA): the epilogue runs one split tile at a time, each paying the
        // fix-up chain, so more units per CTA serialise on it
        // (tools/gpu_split_sweep2.sh: Base-64 T=4..128 -3..10 % capped at 2)
        if (cand <= s_cap && tiles > 0 && !(cand > 2 && tiles * cand > grid)) {
            const int units = tiles * cand;
            const int kbs = (sc.kb_total + cand - 1) / cand;
            const int waves = (units + grid - 1) / grid;
            const float bw = fminf(kSmBytesPerUs, kHbmBytesPerUs / (float)min(units, grid));
            const float fix = cand > 1 ? kFixUs + kFixRoundUs * ((cand + kFixSplits - 1) / kFixSplits) : 0.f;
            t = (float)waves * kbs * kb_bytes / bw + fix;
        }
        int S = 1;
        float best = 3.4e38f;
        for (int c = 0; c < 32; ++c) {  // ascending: a larger split must win by 2 %
            const float tc = __shfl_sync(0xffffffffu, t, c);
            if (tc < best * 0.98f) { best = tc; S = c + 1; }
        }
        // phases can run concurrently (per-expert gating), so each phase's
        // tickets and partial tiles live in their own ranges
        while (S > 1 && (part_used + (long long)sc.tiles * S * BN * BM > p.partial_cap ||
                         ctr_used + sc.tiles > kCounterInts)) --S;
        sc.kbs = (sc.kb_total + S - 1) / S;
        sc.S = (sc.kb_total + sc.kbs - 1) / sc.kbs;
        sc.ctr0 = ctr_used;
        sc.part0 = part_used;
        if (sc.S > 1) {
            ctr_used += (int)sc.tiles;
            part_used += sc.tiles * sc.S * BN * BM;
        }
        sc.units = sc.tiles * sc.S;
        sc.unit0 = total_units;
        total_units += sc.units;
        if (lane == 0) ps[i] = sc;
    }
    if (lane == 0) {
        s_total_units = total_units;
        if (p.probe && blockIdx.x == 0)  // chosen split per phase (slots 23, 24, 31: values, not times)
            for (int i = 0; i < p.nphase; ++i) p.probe[(i == 2) ? 31 : 23 + i] = (unsigned long long)ps[i].S;
    }
    }
    __syncthreads();
    const long long total_units = s_total_units;
    int *phase_done = p.sync;                    // [kMaxPhases]
    int *unit_ctr = p.sync + kMaxPhases + 1;     // dynamic unit counter
    int *grp_done = p.sync + 16;                 // [kMaxGroups] up tiles finished per expert group
    // Down-projection units of group g wait only for g's own up tiles (not for
    // the whole up phase), so the two expert phases overlap at their boundary.
    const bool group_gated = p.nphase >= 2 && ps[0].mode == kUp && ps[1].mode == kDown;

    if (warp == 0) {
        // ================= weight producer (one thread) ====================
        // Units are handed out dynamically (the first one static, then an
        // atomic counter once the previous launch is complete) and published
        // to the other roles through a shared ring.  This thread streams the
        // weight tiles: they never depend on earlier work, so it runs up to
        // STAGES ahead of the MMA and arms each stage for the weight AND the
        // activation bytes.  The activation boxes come from the gated
        // producer (warp 6), so a gate wait never stalls the weight stream.
        if (lane == 0) {
            uint64_t policy, policy_keep;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
            // the dense weight tiles are re-read by every token tile: keep them
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(policy_keep));
            int stage = 0, qi = 0;
            uint32_t phase = 0, qphase = 0;
            bool pdl_done = false;
            long long cyc_empty = 0, cyc_atom = 0, n_units = 0;
            // Bytes in flight set the memory system's queueing delay for every
            // other access of the kernel (latency = in-flight / bandwidth once
            // HBM saturates), so streaming phases keep only as many stages
            // in flight as the bandwidth needs.
            const int lim = max(1, min(p.max_inflight, STAGES));
            long long kbi = 0;  // weight k-blocks issued by this CTA
            // chained: the unit counter lives in this launch's parity buffer,
            // re-armed two launches ago, so units are fetched without waiting
            const bool chained = p.epoch != nullptr;
            if (chained) pdl_done = true;
            long long u = blockIdx.x;
            while (u < total_units) {
                const Unit x = decode_unit<BN>(ps, p.nphase, gr, u);
                mbar_wait(&uq_empty[qi], qphase ^ 1);
                unit_q[qi] = u;
                mbar_arrive(&uq_full[qi]);
                if (++qi == kUnitQ) { qi = 0; qphase ^= 1; }
                // fetch the next unit early: the atomic's latency overlaps this unit
                int nxt = -1;
                if (pdl_done) nxt = atomicAdd(unit_ctr, 1);
                for (int kb = x.kb0; kb < x.kb1; ++kb, ++kbi) {
                    const long long c1 = clock64();
                    if (lim < STAGES && kbi >= lim) {  // k-block kbi - lim consumed
                        const long long o = kbi - lim;
                        mbar_wait(&empty[o % STAGES], (uint32_t)((o / STAGES) & 1));
                    }
                    mbar_wait(&empty[stage], phase ^ 1);
                    cyc_empty += clock64() - c1;
                    mbar_expect_tx(&full[stage], kABytes + x.n_pad * 128);
                    tma_load_3d(sA + stage * kABytes, amaps[x.ph], &full[stage], kb * BK, x.m_tile * BM, x.rec,
                                (ps[x.ph].mode == kDense && ps[x.ph].tiles > ps[x.ph].m_tiles) ? policy_keep : policy);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                if (!pdl_done) {  // the unit counter is re-armed by the previous launch
                    pdl_wait();
                    // with fused routing the next launch reads this launch's
                    // routing output: the routing role triggers it instead
                    if (!p.route.active) pdl_trigger();
                    pdl_done = true;
                    probe(p.probe, blockIdx.x, 2);  // PDL gate open
                    const long long c3 = clock64();
                    nxt = atomicAdd(unit_ctr, 1);
                    cyc_atom += clock64() - c3;
                }
                u = (long long)gridDim.x + nxt;
                ++n_units;
            }
            if (!pdl_done || (chained && !p.route.active)) {  // still honour PDL before exiting
                pdl_wait();
                if (!p.route.active) pdl_trigger();
            }
            mbar_wait(&uq_empty[qi], qphase ^ 1);
            unit_q[qi] = -1;
            mbar_arrive(&uq_full[qi]);
            probe(p.probe, blockIdx.x, 11);  // last weight load issued
            if (p.probe) {
                unsigned long long *pr = p.probe + (size_t)blockIdx.x * kProbeSlots;
                pr[17] = cyc_empty; pr[18] = cyc_atom; pr[19] = n_units;
            }
        }
    } else if (warp == 6) {
        // ================= activation producer (one thread) ================
        // Follows the unit ring; before a unit's activation boxes it waits for
        // the unit's gate: griddepcontrol.wait (PDL) for phase 0, the unit's
        // expert's up tiles for a down unit (so the expert phases overlap),
        // the whole previous phase for the dense phase.  Its boxes complete
        // the stage the weight producer armed for both (the transaction count
        // may briefly run ahead of the arming).
        if (lane == 0) {
            int stage = 0, qi = 0;
            uint32_t phase = 0, qphase = 0;
            long long cyc_gate = 0;
            // the activations of phase 0 come from the previous launch: its
            // dense phase (chained, epoch_wait > 0) or its completion (PDL) —
            // the first launch of a chain follows a non-chained producer (the
            // operand pack), whose writes only griddepcontrol.wait orders
            if (p.epoch && p.epoch_wait > 0) {
                while (ld_acquire(p.epoch) < p.epoch_wait) __nanosleep(32);
                asm volatile("fence.proxy.async.global;" ::: "memory");
            } else {
                pdl_wait();
            }
            int open_group = -1, open_phase = 0;
            for (;;) {
                mbar_wait(&uq_full[qi], qphase);
                const long long u = unit_q[qi];
                mbar_arrive(&uq_empty[qi]);
                if (++qi == kUnitQ) { qi = 0; qphase ^= 1; }
                if (u < 0) break;
                const Unit x = decode_unit<BN>(ps, p.nphase, gr, u);
                const long long c0 = clock64();
                if (x.ph > 0) {
                    if (group_gated && x.ph == 1) {
                        if (x.g != open_group) {
                            const int need = (gr.ntp[x.g + 1] - gr.ntp[x.g]) * ps[0].m_tiles;
                            while (ld_acquire(grp_done + x.g) < need) __nanosleep(32);
                            open_group = x.g;
                            asm volatile("fence.proxy.async.global;" ::: "memory");
                        }
                    } else if (x.ph > open_phase) {
                        while (ld_acquire(phase_done + x.ph - 1) < (int)gridDim.x) __nanosleep(32);
                        // the dense epilogue packs the next block's operand in
                        // its routing order: that routing must be complete
                        if (p.route.active && ps[x.ph].mode == kDense)
                            while (ld_acquire(p.route.done) == 0) __nanosleep(32);
                        open_phase = x.ph;
                        probe(p.probe, blockIdx.x, 2 + x.ph);  // phase gate open
                        // the previous phase's rows were written through the generic proxy
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                    }
                }
                cyc_gate += clock64() - c0;
                const int brow = x.row0 + x.n0;
                for (int kb = x.kb0; kb < x.kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    for (int j = 0; j < x.n_pad; j += kBRowsPerBox)
                        tma_load_2d(sB + stage * kBBytes + j * 128, bmaps[x.ph], &full[stage], kb * BK, brow + j);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
            if (p.probe) p.probe[(size_t)blockIdx.x * kProbeSlots + 16] = cyc_gate;
        }
    } else if (warp >= 7) {
        // ================= routing role (warps 7-10) =======================
        // The next block's pre-gated routing (route_common.cuh), overlapped
        // with this block's expert GEMMs; once it is complete the next launch
        // (which schedules from it) may start.
        if (p.route.active) {
            if (p.epoch && p.epoch_wait > 0) {  // the block input is the previous launch's dense output
                if (tid == 7 * 32)
                    while (ld_acquire(p.epoch) < p.epoch_wait) __nanosleep(32);
                router_sync();
            } else {
                pdl_wait();
            }
            if (tid == 7 * 32) probe(p.probe, blockIdx.x, 25);  // routing role past its gate
            router_run(p.route, tid - 7 * 32, r_xs, &r_flag, p.probe);
            if (tid == 7 * 32) {
                while (ld_acquire(p.route.done) == 0) __nanosleep(64);
                // the next launch may start once it can schedule from this
                // routing — and (chained: parity buffers) once the previous
                // launch has completed, so that launch k+2 never meets launch
                // k's re-arm
                pdl_wait();
                pdl_trigger();
                probe(p.probe, blockIdx.x, 30);  // dependents triggered
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer (single thread) ======================
        int stage = 0, cnt = 0, qi = 0;
        uint32_t phase = 0, qphase = 0;
        for (;; ++cnt) {
            mbar_wait(&uq_full[qi], qphase);
            const long long u = unit_q[qi];
            __syncwarp();
            if (lane == 0) mbar_arrive(&uq_empty[qi]);
            if (++qi == kUnitQ) { qi = 0; qphase ^= 1; }
            if (u < 0) break;
            const Unit x = decode_unit<BN>(ps, p.nphase, gr, u);
            const int acc = cnt & 1;
            mbar_wait(&tempty[acc], ((cnt >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t tmem_d = tmem_base + acc * BN;
            const uint32_t idesc = idesc_bf16(x.n_pad);
            for (int kb = x.kb0; kb < x.kb1; ++kb) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t a_s = smem_u32(sA + stage * kABytes);
                    const uint32_t b_s = smem_u32(sB + stage * kBBytes);
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk)
                        umma_bf16(tmem_d, sw128_desc(a_s + kk * 32), sw128_desc(b_s + kk * 32), idesc,
                                  (kb > x.kb0 || kk > 0) ? 1u : 0u);
                    umma_commit(&empty[stage]);
                }
                __syncwarp();
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
            if (lane == 0) umma_commit(&tfull[acc]);
            __syncwarp();
        }
    } else {
        // ================= epilogue: TMEM -> registers -> global ===========
        const int q = warp & 3;        // TMEM lane quarter this warp may access
        const int et = q * 32 + lane;  // accumulator row 0..127
        int cnt = 0, signalled = 0, qi = 0;  // phases [0, signalled) reported done
        bool route_seen = false;
        uint32_t qphase = 0;
        // The previous launch's last CTA re-arms the counters on its way out;
        // with programmatic dependent launch this grid may already be running,
        // so no signal may precede griddepcontrol.wait (chained launches use
        // the other parity's counters instead).
        if (!p.epoch) pdl_wait();
        auto signal_upto = [&](int ph_end) {
            for (; signalled < ph_end; ++signalled) {
                __threadfence();
                named_sync(1, 128);
                if (et == 0) {
                    probe(p.probe, blockIdx.x, 6 + signalled);  // this CTA's phase done
                    const int old = atomicAdd(phase_done + signalled, 1);
                    if (p.epoch && signalled == p.nphase - 1 && old == (int)gridDim.x - 1) {
                        // every CTA's last-phase rows are written: release the next launch
                        __threadfence();
                        asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p.epoch), "r"(p.epoch_set)
                                     : "memory");
                        // the reference's block latency is the time between consecutive
                        // blocks' dense-layer ends (scheduler.py:374-397): stamp it on the
                        // device, so graph-replayed timed iterations report it unperturbed
                        if (p.stamps) p.stamps[p.epoch_set] = gtimer();
                    }
                }
            }
        };
        // an up tile's hidden rows are complete: release its expert's down units
        auto tile_done = [&](const Unit &x) {
            if (!group_gated || x.ph != 0) return;
            __threadfence();
            named_sync(1, 128);
            if (et == 0) atomicAdd(grp_done + x.g, 1);
        };
        for (;; ++cnt) {
            mbar_wait(&uq_full[qi], qphase);
            const long long u = unit_q[qi];
            named_sync(1, 128);  // every epilogue thread has read the slot
            if (et == 0) mbar_arrive(&uq_empty[qi]);
            if (++qi == kUnitQ) { qi = 0; qphase ^= 1; }
            if (u < 0) break;
            const Unit x = decode_unit<BN>(ps, p.nphase, gr, u);
            signal_upto(x.ph);
            const EpiRegs e = epi_regs(p, p.ph[x.ph], x);
            const int S = ps[x.ph].S;
            const int acc = cnt & 1;
            if (e.mode == kDense && p.route.active && !route_seen) {  // next_inv comes from the routing role
                if (et == 0)
                    while (ld_acquire(p.route.done) == 0) __nanosleep(32);
                named_sync(1, 128);
                route_seen = true;
            }
            if (e.staged) {
                named_sync(1, 128);  // the previous unit's readers are done
                stage_meta(e, x, et, meta_i, meta_f);
                named_sync(1, 128);
            }
            mbar_wait(&tfull[acc], (cnt >> 1) & 1);
            tc_fence_after();
            if (et == 0) probe(p.probe, blockIdx.x, cnt == 0 ? 5 : 12);  // first / last accumulator ready
            const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
            if (S == 1) {
                for (int c0 = 0; c0 < x.n_valid; c0 += 16) {
                    float v[16];
                    tmem_ld16(taddr + c0, v);
                    store_chunk(e, x, c0, x.m_tile * BM + q * 32, lane, v, meta_i, meta_f, stage_out + q * 512);
                }
                tc_fence_before();
                mbar_arrive(&tempty[acc]);
                tile_done(x);
            } else {
                const PhaseSched &sc = ps[x.ph];
                float *part = p.partial + sc.part0 + ((size_t)x.tile * S + x.s) * (BN * BM);
                for (int c0 = 0; c0 < x.n_valid; c0 += 16) {
                    float v[16];
                    tmem_ld16(taddr + c0, v);
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (c0 + j < x.n_valid) __stcg(part + (size_t)(c0 + j) * BM + et, v[j]);
                }
                tc_fence_before();
                mbar_arrive(&tempty[acc]);  // accumulator free: the rest works from global
                if (et == 0) probe(p.probe, blockIdx.x, 13);  // partials stored (last unit)
                __threadfence();
                named_sync(1, 128);
                int *ticket = p.counters + sc.ctr0 + x.tile;
                if (et == 0) s_flag[0] = (atomicAdd(ticket, 1) == S - 1);
                named_sync(1, 128);
                if (s_flag[0]) {
                    __threadfence();
                    if (et == 0) probe(p.probe, blockIdx.x, 14);  // fix-up start (last unit)
                    const float *base = p.partial + sc.part0 + (size_t)x.tile * S * (BN * BM) + et;
                    // 64 partial loads in flight per thread: 16 columns x 4
                    // splits at a time (one dependent round for S <= 4),
                    // summed in split order (deterministic)
                    for (int n0 = 0; n0 < x.n_valid; n0 += 16) {
                        float a[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) a[j] = 0.f;
                        for (int s0 = 0; s0 < S; s0 += kFixSplits) {
                            float v[kFixSplits][16];
#pragma unroll
                            for (int h = 0; h < kFixSplits; ++h)
#pragma unroll
                                for (int j = 0; j < 16; ++j)
                                    v[h][j] = (s0 + h < S && n0 + j < x.n_valid)
                                                  ? __ldcg(base + ((size_t)(s0 + h) * BN + n0 + j) * BM)
                                                  : 0.f;
#pragma unroll
                            for (int h = 0; h < kFixSplits; ++h)
#pragma unroll
                                for (int j = 0; j < 16; ++j)
                                    if (s0 + h < S) a[j] += v[h][j];
                        }
                        store_chunk(e, x, n0, x.m_tile * BM + q * 32, lane, a, meta_i, meta_f, stage_out + q * 512);
                    }
                    if (et == 0) *ticket = 0;
                    tile_done(x);
                }
                named_sync(1, 128);
            }
            if (et == 0) probe(p.probe, blockIdx.x, 15);  // last unit finished
        }
        signal_upto(p.nphase);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        constexpr uint32_t cols = (2 * BN < 32) ? 32 : 2 * BN;
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(cols));
    }
    // the last CTA out re-arms the counters for the next launch
    if (tid == 0) {
        probe(p.probe, blockIdx.x, 9);  // exit
        if (p.probe) p.probe[(size_t)blockIdx.x * kProbeSlots + 22] = clock64();
        __threadfence();
        s_flag[3] = (atomicAdd(p.sync + kMaxPhases, 1) == (int)gridDim.x - 1);
    }
    __syncthreads();
    if (s_flag[3]) {
        for (int i = tid; i < gr.n; i += kThreads) grp_done[i] = 0;
        if (tid == 0) {
            for (int i = 0; i < kMaxPhases; ++i) phase_done[i] = 0;
            if (p.route.active) *p.route.done = 0;
            p.sync[kMaxPhases] = 0;
            *unit_ctr = 0;
        }
        __threadfence();
    }
}

// xb[r] = bf16(x[perm[r] / k])  (activation rows in routing order)
__global__ void pack_rows_bf16_kernel(const float *__restrict__ x, const int *__restrict__ perm, int n, int d, int k,
                                      uint16_t *__restrict__ xb) {
    pdl_wait();
    pdl_trigger();
    const int vec = d / 8;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)n * vec;
         i += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(i / vec), c = (int)(i - (long long)r * vec);
        const int row = perm ? __ldg(perm + r) / k : r;
        const float4 *s = reinterpret_cast<const float4 *>(x + (size_t)row * d) + 2 * c;
        const float4 a = __ldg(s), b = __ldg(s + 1);
        uint4 o;
        o.x = bf16_bits(a.x) | ((uint32_t)bf16_bits(a.y) << 16);
        o.y = bf16_bits(a.z) | ((uint32_t)bf16_bits(a.w) << 16);
        o.z = bf16_bits(b.x) | ((uint32_t)bf16_bits(b.y) << 16);
        o.w = bf16_bits(b.z) | ((uint32_t)bf16_bits(b.w) << 16);
        reinterpret_cast<uint4 *>(xb)[(size_t)r * vec + c] = o;
    }
}

// mixb[t] = bf16(sum_s yw[t*k+s]) in slot (routing) order, linalg.py:45-51
__global__ void sum_slots_bf16_kernel(const float *__restrict__ yw, int T, int d, int k, uint16_t *__restrict__ mixb) {
    pdl_wait();
    pdl_trigger();
    const int vec = d / 4;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)T * vec;
         i += (long long)gridDim.x * blockDim.x) {
        const int t = (int)(i / vec), c = (int)(i - (long long)t * vec);
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int s = 0; s < k; ++s) {
            const float4 v = __ldg(reinterpret_cast<const float4 *>(yw + ((size_t)t * k + s) * d) + c);
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        uint2 o;
        o.x = bf16_bits(acc.x) | ((uint32_t)bf16_bits(acc.y) << 16);
        o.y = bf16_bits(acc.z) | ((uint32_t)bf16_bits(acc.w) << 16);
        reinterpret_cast<uint2 *>(mixb)[(size_t)t * vec + c] = o;
    }
}

template <int BN, int STAGES>
constexpr size_t smem_bytes() {
    return 1024 + (size_t)STAGES * (kABytes + BN * 128) + (2 * STAGES + 4 + 3 * kUnitQ) * 8 + 32 +
           (4 * kMaxGroups + 1) * 4 +
           (kMetaInts + kMetaInts / 2) * 4 + 16 + 4 * 512 * 4;
}

struct PhaseMaps {
    CUtensorMap a, b;
};

template <int BN, int STAGES>
static int launch(const PhaseMaps *mp, const Params &p, cudaStream_t s) {
    constexpr size_t smem = smem_bytes<BN, STAGES>();
    static_assert(smem <= 227 * 1024, "shared memory budget");
    // Per device: the attribute and the co-residency check belong to the
    // device the launch goes to.  The kernel spins on grid-wide counters
    // (phase gates, split-K tickets), so every CTA must be resident at once:
    // one per SM of THIS device (cudaDevAttrMultiProcessorCount), and the
    // launch is refused — not hung — if even that does not fit (a reduced-SM
    // context, another kernel's shared-memory carve-out).
    static std::atomic<unsigned long long> attr_set{0};
    const int dev = current_device();
    PG_REQUIRE(dev >= 0 && dev < 64, PGMOE_E_CONFIG, "device ordinal %d unsupported", dev);
    if (!(attr_set.load() & (1ull << dev))) {
        PG_CUDA(cudaFuncSetAttribute(block_gemm_kernel<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
        int per_sm = 0;
        PG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, block_gemm_kernel<BN, STAGES>, kThreads, smem));
        PG_REQUIRE(per_sm >= 1, PGMOE_E_CUDA,
                   "the persistent tcgen05 block kernel does not fit on an SM (%zu B shared memory)", smem);
        attr_set.fetch_or(1ull << dev);
    }
    const int grid = device_sm_count();  // of the current context (green contexts: its own SMs)
    // unused phase slots repeat phase 0's maps (never dereferenced)
    const PhaseMaps &m0 = mp[0], &m1 = p.nphase > 1 ? mp[1] : mp[0], &m2 = p.nphase > 2 ? mp[2] : mp[0];
    PG_CUDA(launch_pdl(block_gemm_kernel<BN, STAGES>, dim3(grid), dim3(kThreads), smem, s, m0.a, m0.b, m1.a, m1.b,
                       m2.a, m2.b, p));
    count_launch();
    return PGMOE_OK;
}

// BN: widest N tile.  Token groups wider than BN are split into N tiles
// (each re-reads its weight tile), so BN follows the expected tokens per
// group: 64 covers decode batches, 256 the compute-bound stress shapes.
// Workspace: [parity 0: tickets | sync][parity 1: tickets | sync][partials 0][partials 1]
static int run(const PhaseMaps *mp, Params p, int bn, void *ws, size_t ws_bytes, cudaStream_t s, int parity = 0) {
    const size_t head = (size_t)(kCounterInts + kSyncInts) * 4;
    PG_REQUIRE(ws_bytes > 2 * head + 8192, PGMOE_E_CONFIG, "tcgen05 workspace too small");
    const size_t half = ((ws_bytes - 2 * head) / 2) & ~(size_t)255;
    p.counters = reinterpret_cast<int *>(static_cast<char *>(ws) + (size_t)parity * head);
    p.sync = p.counters + kCounterInts;
    p.partial = reinterpret_cast<float *>(static_cast<char *>(ws) + 2 * head + (size_t)parity * half);
    p.partial_cap = (long long)(half / 4);
    p.probe = probe_buffer(1, device_sm_count());
    if (p.max_inflight <= 0) p.max_inflight = 8;
    { const char *e = getenv("PGMOE_INFLIGHT"); if (e) p.max_inflight = atoi(e); }
    { const char *e = getenv("PGMOE_MAX_SPLIT"); if (e) p.max_split = atoi(e); }
    if (bn <= 64) return launch<64, 8>(mp, p, s);
    return launch<256, 4>(mp, p, s);
}

static int launch_grid(long long work) {
    return (int)std::min<long long>(kNumSMs * 8, std::max(1LL, (work + 255) / 256));
}

}  // namespace tc

bool tc_supported(int d, int f) { return d % 128 == 0 && f % 128 == 0 && d >= 128 && f >= d; }

int tc_pack_rows(const float *x, const int *perm, int n, int d, int k, uint16_t *xb, cudaStream_t s) {
    if (n == 0) return PGMOE_OK;
    PG_CUDA(launch_pdl(tc::pack_rows_bf16_kernel, dim3(tc::launch_grid((long long)n * d / 8)), dim3(256), 0, s, x,
                       perm, n, d, k, xb));
    count_launch();
    return PGMOE_OK;
}

// One launch for a block's expert FFN (up, down) and — when `dense_w` is
// given and top_k == 1 — its dense layer: phases separated by in-kernel grid
// barriers.  `xb_ready`: the packed bf16 operand was already written (by the
// previous block's dense epilogue).  next_xb/next_inv: see Params.
int block_tc(const float *x, int T, int d, int f, int k, const void *experts, size_t stride, int indexed_by_act,
             const pgmoe_routing *r, uint16_t *xb, uint16_t *hb, float *yw, uint16_t *mixb, bool xb_ready,
             const void *dense_w, float *y, uint16_t *next_xb, const int *next_inv, void *ws, size_t ws_bytes,
             cudaStream_t s, const FusedRoute *route, const LaunchChain *chain, int n_experts) {
    PG_REQUIRE(tc_supported(d, f), PGMOE_E_CONFIG, "tcgen05 path needs d, f multiples of 128 and f >= d");
    PG_REQUIRE((reinterpret_cast<uintptr_t>(experts) & 15) == 0 && stride % 16 == 0, PGMOE_E_CONFIG,
               "expert records must be 16-byte aligned");
    PG_REQUIRE(dense_w == nullptr || (k == 1 && mixb != nullptr), PGMOE_E_CONFIG,
               "the fused dense phase needs top_k == 1 (mix written by the down projection)");
    const int n = T * k;
    // Records addressed through the map are < E (resident) or < n_act (slot
    // cache), both <= 1024; the extent only bounds TMA address generation.
    const int rec_extent = 1024;
    if (!xb_ready) PG_TRY(tc_pack_rows(x, r->perm, n, d, k, xb, s));
    tc::Params p{};
    p.T = T;
    p.k = k;
    p.act = r->act; p.n_act = r->n_act; p.off = r->off; p.hist = r->hist; p.perm = r->perm; p.w_perm = r->w_perm;
    p.indexed_by_act = indexed_by_act;
    tc::PhaseMaps mp[3];
    PG_TRY(tc::make_wmap(&mp[0].a, experts, d, f, rec_extent, stride));
    PG_TRY(tc::make_bmap(&mp[0].b, xb, d, n));
    p.ph[0] = {tc::kUp, f, d, nullptr, hb};
    PG_TRY(tc::make_wmap(&mp[1].a, static_cast<const char *>(experts) + (size_t)f * d * 2, f, d, rec_extent, stride));
    PG_TRY(tc::make_bmap(&mp[1].b, hb, f, n));
    p.ph[1] = {tc::kDown, d, f, yw, (k == 1) ? mixb : nullptr};
    p.nphase = 2;
    if (dense_w) {
        PG_TRY(tc::make_wmap(&mp[2].a, dense_w, d, d, 1, (size_t)d * d * 2));
        PG_TRY(tc::make_bmap(&mp[2].b, mixb, d, T));
        p.ph[2] = {tc::kDense, d, d, y, nullptr};
        p.nphase = 3;
        p.next_xb = next_xb;
        p.next_inv = next_inv;
    }
    if (route && route->active) {
        PG_REQUIRE(dense_w != nullptr && fused_route_supported(route->E), PGMOE_E_CONFIG,
                   "fused routing needs the dense phase and E in {64, 128, 256}");
        p.route = *route;
        // (In-flight stage limits for the routing role's sake were measured
        // and dropped once the role ran on 4 warps: within 1 % at every T,
        // tools/gpu_env_sweep.sh VAR=PGMOE_INFLIGHT.)
    }
    int parity = 0;
    if (chain && chain->epoch) {
        PG_REQUIRE(dense_w != nullptr, PGMOE_E_CONFIG, "chained launches end with the dense phase");
        p.epoch = chain->epoch;
        p.epoch_wait = chain->epoch_wait;
        p.epoch_set = chain->epoch_set;
        p.stamps = chain->stamps;
        parity = chain->parity & 1;
    }
    // N tile: 64 tokens (8 weight stages) while the average expert holds at
    // most 64 routed tokens; 256 (4 stages) only for compute-heavy groups —
    // a group wider than the N tile re-reads its weight tile per N tile
    const bool wide = n_experts > 0 ? (long long)n > 64LL * n_experts : n >= 2048;
    return tc::run(mp, p, wide ? 256 : 64, ws, ws_bytes, s, parity);
}

int expert_ffn_tc2(const float *x, int T, int d, int f, int k, const void *experts, size_t stride, int indexed_by_act,
                   const pgmoe_routing *r, uint16_t *xb, uint16_t *hb, float *yw, uint16_t *mixb, void *ws,
                   size_t ws_bytes, cudaStream_t s, bool xb_ready) {
    return block_tc(x, T, d, f, k, experts, stride, indexed_by_act, r, xb, hb, yw, mixb, xb_ready, nullptr, nullptr,
                    nullptr, nullptr, ws, ws_bytes, s);
}

int dense_tc2(const float *yw, const uint16_t *mixb_ready, int T, int d, int k, const void *dense_w, float *y,
              uint16_t *mixb_scratch, void *ws, size_t ws_bytes, cudaStream_t s, uint16_t *next_xb,
              const int *next_inv) {
    PG_REQUIRE(d % 128 == 0, PGMOE_E_CONFIG, "tcgen05 dense needs d multiple of 128");
    const uint16_t *mixb = mixb_ready;
    if (!mixb) {
        if (T > 0) {
            PG_CUDA(launch_pdl(tc::sum_slots_bf16_kernel, dim3(tc::launch_grid((long long)T * d / 4)), dim3(256), 0, s,
                               yw, T, d, k, mixb_scratch));
            count_launch();
        }
        mixb = mixb_scratch;
    }
    tc::Params p{};
    p.T = T;
    p.k = k;
    p.nphase = 1;
    p.ph[0] = {tc::kDense, d, d, y, nullptr};
    p.next_xb = next_xb;
    p.next_inv = next_inv;
    tc::PhaseMaps mp[1];
    PG_TRY(tc::make_wmap(&mp[0].a, dense_w, d, d, 1, (size_t)d * d * 2));
    PG_TRY(tc::make_bmap(&mp[0].b, mixb, d, T));
    return tc::run(mp, p, T >= 2048 ? 256 : 64, ws, ws_bytes, s);
}

// Entry points with the fp32-scratch signatures: the bf16 operands live in
// the caller's fp32 h scratch ([T*k][f] floats hold hb [T*k][f] plus
// xb [T*k][d] bf16 since f >= d) and the mix in a temporary.
int expert_ffn_tc(const float *x, int T, int d, int f, int k, const void *experts, size_t stride,
                  int indexed_by_act, const pgmoe_routing *r, float *h, float *yw, void *ws, size_t ws_bytes,
                  cudaStream_t s) {
    uint16_t *hb = reinterpret_cast<uint16_t *>(h);
    uint16_t *xb = hb + (size_t)T * k * f;
    return expert_ffn_tc2(x, T, d, f, k, experts, stride, indexed_by_act, r, xb, hb, yw, nullptr, ws, ws_bytes, s,
                          false);
}

int dense_tc(const float *yw, int T, int d, int k, const void *dense_w, float *y, void *ws, size_t ws_bytes,
             cudaStream_t s) {
    uint16_t *mixb = nullptr;
    PG_CUDA(cudaMallocAsync(&mixb, (size_t)std::max(T, 1) * d * 2, s));
    int st = dense_tc2(yw, nullptr, T, d, k, dense_w, y, mixb, ws, ws_bytes, s, nullptr, nullptr);
    cudaFreeAsync(mixb, s);
    return st;
}

}  // namespace pgmoe
