// decode_tc.cu — small-batch resident decoder: ONE persistent launch per
// decoder iteration (the block loop of decoder_iteration, core.py:342-383,
// runs inside the kernel), for T <= 64 tokens, top-1, lookahead 1, bf16.
//
// At decode batch sizes a block is a chain of three dependent GEMV-shaped
// contractions (up, down + combine, dense) whose weights are small next to
// the 148 SMs' shared memory (Base-64 T=1: 10.6 MB vs ~26 MB), so the block
// latency is the dependency chain, not the weight stream.  This kernel
// shortens the chain:
//   * clusters of C = 8 CTAs; every weight tile (128 output rows x the full
//     K of one phase) is split K-wise over the C CTAs of one cluster, and
//     the C fp32 partial accumulators are summed through distributed shared
//     memory (mbarrier handshakes between the CTAs, no global partials, no
//     atomic tickets), each CTA finishing 128 / C rows of the tile;
//   * the schedule is static (tile i of a block -> cluster i mod #clusters),
//     so every CTA knows its weight tiles as soon as the block's routing is
//     known and streams them into its pipeline stages ahead of the data
//     dependency — including the NEXT block's tiles while this block still
//     runs (its routing is computed early by the pre-gate);
//   * no launch boundary between blocks: gates are per-block device
//     counters (expert group up tiles done -> its down tiles; all down tiles
//     -> dense; dense -> next block), the routing role of every CTA computes
//     the next block's pre-gate (route_common.cuh, certified fp64 logits)
//     while the expert phases run.
// Per CTA: warp 0 weight producer + schedule builder, warp 6 activation
// producer, warp 1 TMEM owner + MMA issuer, warps 2-5 epilogue (partial ->
// DSMEM reduction -> ReLU / combine weight / un-permute / dense stores),
// warps 7-10 routing role.
// Deterministic: the C partials of a tile are summed in rank order.
#include <cooperative_groups.h>
#include <cstdlib>

#include "common.cuh"
#include "decode.h"
#include "kernels.h"
#include "route_common.cuh"
#include "tc_common.cuh"

namespace pgmoe {
namespace dec {
using namespace tc;

constexpr int C = 8;                 // CTAs per cluster = K splits per tile
constexpr int BN = 16;               // token columns per tile (UMMA N)
constexpr int STAGES = 8;            // (16 KB weight + 2 KB activation) per stage
constexpr int kRouteGBytes = 32 * 1024;  // cluster routing: this CTA's rows of the pre-gate (bf16)
constexpr int kRouteMaxT = 8, kRouteMaxE = 128;
constexpr int kBBytes = BN * 128;    // one 16-row activation box per k-block
constexpr int kThreads = 352;
constexpr int kRows = BM / C;        // output rows each CTA finishes per tile
static_assert(BM % C == 0 && (kRows * BN) % 128 == 0, "epilogue slice");

struct Sched {          // one block's schedule (identical in every CTA)
    int n, mt_up, mt_dn, mt_ds, up_tiles, dn_tiles, ds_tiles, total, nt_ds;
    int ntp[kDecodeMaxAct + 1];   // prefix of 16-token tiles per expert group
    int rec[kDecodeMaxAct], row0[kDecodeMaxAct], ng[kDecodeMaxAct];
};

struct Tile {
    int ph, g, m, n0, n_valid, kb0, kb1, rec, row0;
};

__device__ __forceinline__ Tile decode_tile(const Sched &s, int i, int rank, int d, int f) {
    Tile t;
    int local, mt, kbt;
    if (i < s.up_tiles) {
        t.ph = 0; local = i; mt = s.mt_up; kbt = d / BK;
    } else if (i < s.up_tiles + s.dn_tiles) {
        t.ph = 1; local = i - s.up_tiles; mt = s.mt_dn; kbt = f / BK;
    } else {
        t.ph = 2; local = i - s.up_tiles - s.dn_tiles; mt = s.mt_ds; kbt = d / BK;
    }
    if (t.ph < 2) {
        int lo = 0, hi = s.n - 1;  // last group g with ntp[g] * mt <= local
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s.ntp[mid] * mt <= local) lo = mid;
            else hi = mid - 1;
        }
        t.g = lo;
        const int l2 = local - s.ntp[lo] * mt;
        const int nt = l2 / mt;
        t.m = l2 - nt * mt;
        t.n0 = nt * BN;
        t.n_valid = min(BN, s.ng[lo] - t.n0);
        t.rec = s.rec[lo];
        t.row0 = s.row0[lo];
    } else {
        t.g = 0;
        const int nt = local / mt;
        t.m = local - nt * mt;
        t.n0 = nt * BN;
        t.n_valid = -1;  // filled by the caller (T)
        t.rec = 0;
        t.row0 = 0;
    }
    t.kb0 = kbt * rank / C;
    t.kb1 = kbt * (rank + 1) / C;
    return t;
}

struct Params {
    int T, d, f, E, nb;
    const DecodeBlock *blocks;  // [nb]
    int *sync;                  // [nb][kDecodeSyncInts] zeroed before the launch
    const float *x_in;          // block 0 input (routing role of block 0)
    float *y_out;               // last block's output
    uint16_t *xb, *hb, *mixb;   // bf16 operands: packed up input, hidden, mix
    FusedRoute route;           // T-dependent routing-role fields (x, G, out, done per block below)
    float *x_trace;             // optional [nb][T][d] block inputs
    int32_t *ids_trace;         // optional [nb][T] consumed decisions
    float *w_trace;
    int cluster_route;          // 1: cluster 0 routes from shared-memory gate slices (T <= 8, E <= 128)
    unsigned long long *probe;
};

// sync layout per block
__device__ __forceinline__ int *s_down(int *s) { return s; }
__device__ __forceinline__ int *s_dense(int *s) { return s + 1; }
__device__ __forceinline__ int *s_route(int *s) { return s + 2; }
__device__ __forceinline__ int *s_up(int *s, int g) { return s + 4 + g; }

__device__ __forceinline__ void spin_ge(const int *p, int v) {
    while (ld_acquire(p) < v) __nanosleep(20);
}

__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
// arrive on the mbarrier at the same offset in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_remote(uint64_t *bar, uint32_t rank) {
    const uint32_t ra = mapa(smem_u32(bar), rank);
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAITC_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAITC_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ float ld_dsmem(uint32_t saddr_remote) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(saddr_remote) : "memory");
    return v;
}
__device__ __forceinline__ float2 ld_dsmem2(uint32_t saddr_remote) {
    float2 v;
    asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(saddr_remote) : "memory");
    return v;
}

// probe slots: 1 + 8*b + k for b < 5 (k: 0 schedule built, 1 first gate open,
// 2 first accumulator, 3 first partials summed, 4 last tile signalled,
// 5 routing done (role), 6 dense gate open, 7 first weight load issued); 41 exit
__device__ __forceinline__ void dprobe(const Params &p, int b, int k) {
    if (p.probe && b < 5) p.probe[(size_t)blockIdx.x * kProbeSlots + 1 + 8 * b + k] = gtimer();
}

__device__ __forceinline__ int dense_need(const Params &p) {
    return ((p.T + BN - 1) / BN) * (p.d / BM) * C;
}

// Schedule of block b from its routing (act / hist / off), built by one warp.
__device__ void build_sched(const Params &p, int b, Sched &s, int lane) {
    const DecodeBlock &bd = p.blocks[b];
    const int n = __ldcg(bd.n_act);
    int run = 0;
    for (int g0 = 0; g0 < n; g0 += 32) {
        const int g = g0 + lane;
        int nt = 0;
        if (g < n) {
            const int e = __ldcg(bd.act + g);
            const int ng = __ldcg(bd.hist + e);
            s.rec[g] = bd.wrec0 + e;
            s.row0[g] = __ldcg(bd.off + e);
            s.ng[g] = ng;
            nt = (ng + BN - 1) / BN;
        }
        int incl = nt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (g < n) s.ntp[g] = run + incl - nt;
        run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) {
        s.n = n;
        s.ntp[n] = run;
        s.mt_up = p.f / BM;
        s.mt_dn = p.d / BM;
        s.mt_ds = p.d / BM;
        s.nt_ds = (p.T + BN - 1) / BN;
        s.up_tiles = run * s.mt_up;
        s.dn_tiles = run * s.mt_dn;
        s.ds_tiles = s.nt_ds * s.mt_ds;
        s.total = s.up_tiles + s.dn_tiles + s.ds_tiles;
    }
    __syncwarp();
}

// ---------------------------------------------------------------------------
// Cluster routing (T <= 8, E <= 128): the pre-gate of the next block by the
// 8 CTAs of cluster 0.  CTA `rank` keeps rows [rank*d/8, (rank+1)*d/8) of
// the block's pre-gate in shared memory, loaded while the block input is
// still being produced (static weights), so the routing's critical path is:
// x slice -> partial fp64 logits (exact products, one rounding per FMA) ->
// handshake -> rank 0 sums the 8 partials over DSMEM in rank order ->
// certified selection + softmax (router_select_token) -> stable
// permutation (router_permute).  Same arithmetic contract as K1.
struct RouteSmem {
    uint32_t *gsl;   // [kn][E/2] bf16 pairs
    double *part;    // [kRouteMaxT][E] partial logits
    float *gcm;      // [E] column max |G| of the slice
    double *xs;      // [kRouteMaxT] sum |x| over the slice
    uint64_t *rfull, *rempty;
};

__device__ void route_prefetch(const Params &p, const DecodeBlock &bd, int rank, int rt, const RouteSmem &rs) {
    const int d = p.d, E = p.E, kn = d / C;
    const uint4 *src = reinterpret_cast<const uint4 *>(static_cast<const uint16_t *>(bd.pre_gate) + (size_t)rank * kn * E);
    uint4 *dst = reinterpret_cast<uint4 *>(rs.gsl);
    const int nv = kn * E * 2 / 16;
    for (int i0 = rt; i0 < nv; i0 += 8 * kRouterThreads) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (i0 + u * kRouterThreads < nv) v[u] = __ldg(src + i0 + u * kRouterThreads);
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (i0 + u * kRouterThreads < nv) dst[i0 + u * kRouterThreads] = v[u];
    }
}

template <int NJ>
__device__ void cluster_route(const Params &p, const FusedRoute &r, int rank, int rt, const RouteSmem &rs,
                              float *scratch, int use) {
    // fine stamps of the second routing round (slots 42..47)
    auto st = [&](int k) {
        if (p.probe && use == 1 && rt == 0) p.probe[(size_t)blockIdx.x * kProbeSlots + 42 + k] = gtimer();
    };
    namespace cg = cooperative_groups;
    const int d = p.d, E = p.E, T = p.T, kn = d / C, k0 = rank * kn;
    const int lane = rt & 31, w = rt >> 5;
    float *xsl = scratch;  // [T][kn] (the scratch holds the tile sums later, rank 0 only)
    for (int i = rt; i < T * kn; i += kRouterThreads) {
        const int t = i / kn;
        xsl[i] = __ldcg(r.x + (size_t)t * d + k0 + (i - t * kn));
    }
    st(0);
    if (use > 0) mbar_wait_cluster(rs.rempty, (use - 1) & 1);  // rank 0 done reading our last partials
    router_sync();
    for (int t = w; t < T; t += kRouterWarps) {  // sum |x_i| over the slice (bounds the logit error)
        double v = 0.0;
        for (int i = lane; i < kn; i += 32) v += fabs((double)xsl[t * kn + i]);
        v = warp_sumd(v);
        if (lane == 0) rs.xs[t] = v;
    }
    {   // partial logits: thread (g, pair) owns experts 2*pair, 2*pair+1; the TG thread groups
        // split the tokens, and groups left over (T < TG) split the rows, so every
        // dependent FP64 chain is as short as the batch allows (two accumulators
        // per expert, even / odd rows); partials are combined in a fixed order
        const int P = E / 2, TG = kRouterThreads / P;
        const int pr = rt % P, tg = rt / P;
        const int tgrp = min(T, TG);            // token groups in use
        const int RS = TG / tgrp;               // row slices per token group
        const int t0 = tg % tgrp, rsl = tg / tgrp;
        const int NT = (T + tgrp - 1) / tgrp;   // tokens per thread (<= 4)
        double acc[4][2][2];
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u][0][0] = acc[u][0][1] = acc[u][1][0] = acc[u][1][1] = 0.0;
        float cm0 = 0.f, cm1 = 0.f;
        const bool active = tg < tgrp * RS;
        const int i0 = active ? kn * rsl / RS : 0, i1 = active ? kn * (rsl + 1) / RS : 0;
        auto rows = [&](auto nb, int i) {
            constexpr int NB = decltype(nb)::value;
            uint32_t g[NB];
#pragma unroll
            for (int u = 0; u < NB; ++u) g[u] = rs.gsl[(size_t)(i + u) * P + pr];
#pragma unroll
            for (int u = 0; u < NB; ++u) {
                const float f0 = __uint_as_float(g[u] << 16), f1 = __uint_as_float(g[u] & 0xffff0000u);
                cm0 = fmaxf(cm0, fabsf(f0));
                cm1 = fmaxf(cm1, fabsf(f1));
                const double g0 = f0, g1 = f1;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int t = t0 + q * tgrp;
                    if (q < NT && t < T) {
                        const double xv = xsl[t * kn + i + u];
                        acc[q][u & 1][0] = fma(xv, g0, acc[q][u & 1][0]);  // exact product, one rounding
                        acc[q][u & 1][1] = fma(xv, g1, acc[q][u & 1][1]);
                    }
                }
            }
        };
        int i = i0;
        for (; i + 8 <= i1; i += 8) rows(std::integral_constant<int, 8>{}, i);
        for (; i + 2 <= i1; i += 2) rows(std::integral_constant<int, 2>{}, i);
        for (; i < i1; ++i) rows(std::integral_constant<int, 1>{}, i);
        // [row slice][t][E] partials; slice 0 goes straight to part, the others through
        // the scratch after the x slice, then added in slice order
        double *extra = reinterpret_cast<double *>(xsl + ((T * kn + 1) & ~1));
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int t = t0 + q * tgrp;
            if (active && q < NT && t < T) {
                double *dst = rsl == 0 ? rs.part : extra + (size_t)(rsl - 1) * T * E;
                dst[t * E + 2 * pr] = acc[q][0][0] + acc[q][1][0];
                dst[t * E + 2 * pr + 1] = acc[q][0][1] + acc[q][1][1];
            }
        }
        // column maxima: combine the row slices' maxima (max is order-free)
        float *cmx = reinterpret_cast<float *>(extra + (size_t)(RS - 1) * T * E);
        if (active && t0 == 0) {
            cmx[rsl * E + 2 * pr] = cm0;
            cmx[rsl * E + 2 * pr + 1] = cm1;
        }
        router_sync();
        if (RS > 1)
            for (int q = rt; q < T * E; q += kRouterThreads) {
                double v = rs.part[q];
                for (int z = 1; z < RS; ++z) v += extra[(size_t)(z - 1) * T * E + q];
                rs.part[q] = v;
            }
        for (int j = rt; j < E; j += kRouterThreads) {
            float m = cmx[j];
            for (int z = 1; z < RS; ++z) m = fmaxf(m, cmx[z * E + j]);
            rs.gcm[j] = m;
        }
    }
    st(1);
    router_sync();
    if (rt == 0) mbar_arrive_remote(rs.rfull, 0);  // our partials -> rank 0
    if (rank != 0) return;
    // ---- rank 0: cluster sums in rank order, selection, permutation -------
    mbar_wait_cluster(rs.rfull, use & 1);
    st(2);
    const TileSums ts = tile_sums_layout(scratch, E, kRouteMaxT);
    const uint32_t part_s = smem_u32(rs.part), gcm_s = smem_u32(rs.gcm), xs_s = smem_u32(rs.xs);
    for (int q = rt; q < T * E; q += kRouterThreads) {
        const int t = q / E, j = q - t * E;
        double pv[C];
        float cv[C];
#pragma unroll
        for (int z = 0; z < C; ++z) {
            double v;
            asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(mapa(part_s + q * 8, z)) : "memory");
            pv[z] = v;
            cv[z] = ld_dsmem(mapa(gcm_s + j * 4, z));
        }
        double sum = 0.0;
        float cm = 0.f;
#pragma unroll
        for (int z = 0; z < C; ++z) {
            sum += pv[z];
            cm = fmaxf(cm, cv[z]);
        }
        ts.lgs[q] = sum;
        ts.cms[q] = cm;
        (void)t;
    }
    if (rt < T) {
        double v = 0.0;
        for (int z = 0; z < C; ++z) {
            double x;
            asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(x) : "r"(mapa(xs_s + rt * 8, z)) : "memory");
            v += x;
        }
        ts.sxs[rt] = v;
    }
    router_sync();
    st(3);
    if (rt < C) mbar_arrive_remote(rs.rempty, (uint32_t)rt);  // every CTA may reuse its partials
    int *s_ids = reinterpret_cast<int *>(scratch + kRouterSmemFloats - 2 * kRouterTok * 8);
    float *s_w = scratch + kRouterSmemFloats - kRouterTok * 8;
    for (int t = w; t < T; t += kRouterWarps) router_select_token<uint16_t, NJ>(r, ts, t, t, lane, s_ids, s_w);
    router_sync();
    st(4);
    if (T * r.k <= 32) {
        if (w == 0) router_permute_small(r, lane, s_ids, s_w);
    } else {
        router_permute(r, rt, reinterpret_cast<int *>(scratch), s_ids, s_w);
    }
    router_sync();
    st(5);
    __threadfence();
    router_sync();
    if (rt == 0) asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(r.done), "r"(1) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1) decode_kernel(const __grid_constant__ CUtensorMap w1map,
                                                             const __grid_constant__ CUtensorMap w2map,
                                                             const __grid_constant__ CUtensorMap dmap,
                                                             const __grid_constant__ CUtensorMap xmap,
                                                             const __grid_constant__ CUtensorMap hmap,
                                                             const __grid_constant__ CUtensorMap mmap,
                                                             const Params p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    __shared__ __align__(16) float r_xs[kRouterSmemFloats];  // routing role scratch
    __shared__ int r_flag;
    unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char *sA = smem;
    unsigned char *sB = sA + STAGES * kABytes;
    float *part = reinterpret_cast<float *>(sB + STAGES * kBBytes);  // [2][BM][BN] fp32 partials
    Sched *sched = reinterpret_cast<Sched *>(part + 2 * BM * BN);     // [2]
    RouteSmem rs;
    rs.gsl = reinterpret_cast<uint32_t *>(sched + 2);
    rs.part = reinterpret_cast<double *>(reinterpret_cast<unsigned char *>(rs.gsl) + kRouteGBytes);
    rs.gcm = reinterpret_cast<float *>(rs.part + kRouteMaxT * kRouteMaxE);
    rs.xs = reinterpret_cast<double *>(rs.gcm + kRouteMaxE);
    uint64_t *bars = reinterpret_cast<uint64_t *>(rs.xs + kRouteMaxT);
    uint64_t *full = bars, *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES, *tempty = tfull + 2;
    uint64_t *pfull = tempty + 2, *pempty = pfull + 2;     // partial buffers: all C partials in / all C readers done
    uint64_t *sfull = pempty + 2, *sempty = sfull + 2;     // schedule buffers
    rs.rfull = sempty + 2;                                 // cluster routing: partials in (rank 0) / read (all)
    rs.rempty = rs.rfull + 1;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(rs.rempty + 1);

    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank();
    const int cluster = blockIdx.x / C, nclusters = gridDim.x / C;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int T = p.T, d = p.d, f = p.f, nb = p.nb;
    if (tid == 0) probe(p.probe, blockIdx.x, 0);
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(32));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 64) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 128);
            mbar_init(&pfull[i], C);
            mbar_init(&pempty[i], C);
            mbar_init(&sfull[i], 1);
            mbar_init(&sempty[i], 3);  // MMA, activation producer, epilogue
        }
        mbar_init(rs.rfull, C);
        mbar_init(rs.rempty, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid == 96) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&w1map) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&w2map) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&dmap) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&xmap) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&hmap) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mmap) : "memory");
    }
    tc_fence_before();
    cl.sync();  // barriers initialised cluster-wide before any remote arrive
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const CUtensorMap *amaps[3] = {&w1map, &w2map, &dmap};
    const CUtensorMap *bmaps[3] = {&xmap, &hmap, &mmap};

    if (warp == 0) {
        // ============ schedule builder + weight producer ===================
        uint64_t pol_first, pol_last;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
        int stage = 0;
        uint32_t phase = 0;
        for (int b = 0; b < nb; ++b) {
            const int sb = b & 1;
            // the block's routing: K1 before the launch (b = 0), else the
            // previous block's routing role
            if (b == 0) {
                pdl_wait();
            } else if (lane == 0) {
                spin_ge(s_route(p.sync + (size_t)(b - 1) * kDecodeSyncInts), 1);
            }
            __syncwarp();
            if (b >= 2) mbar_wait(&sempty[sb], ((b >> 1) - 1) & 1);
            build_sched(p, b, sched[sb], lane);
            if (lane == 0) {
                mbar_arrive(&sfull[sb]);
                dprobe(p, b, 0);
                const Sched &s = sched[sb];
                const DecodeBlock &bd = p.blocks[b];
                bool first = true;
                for (int i = cluster; i < s.total; i += nclusters) {
                    const Tile t = decode_tile(s, i, rank, d, f);
                    for (int kb = t.kb0; kb < t.kb1; ++kb) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        if (first) { dprobe(p, b, 7); first = false; }
                        mbar_expect_tx(&full[stage], kABytes + kBBytes);
                        if (t.ph == 2)  // dense rows of the weight pool, re-read by every token tile: keep in L2
                            tma_load_3d(sA + stage * kABytes, &dmap, &full[stage], kb * BK, bd.dense_row0 + t.m * BM,
                                        0, pol_last);
                        else
                            tma_load_3d(sA + stage * kABytes, amaps[t.ph], &full[stage], kb * BK, t.m * BM, t.rec,
                                        pol_first);
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                }
            }
            __syncwarp();
        }
    } else if (warp == 6) {
        // ============ activation producer: per tile gate, then its boxes ==
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            pdl_wait();  // xb of block 0 (operand pack before the launch)
            for (int b = 0; b < nb; ++b) {
                const int sb = b & 1;
                mbar_wait(&sfull[sb], (b >> 1) & 1);
                const Sched &s = sched[sb];
                int *sy = p.sync + (size_t)b * kDecodeSyncInts;
                int open_g = -1;
                bool up_open = (b == 0), ds_open = false, first = true;
                for (int i = cluster; i < s.total; i += nclusters) {
                    const Tile t = decode_tile(s, i, rank, d, f);
                    if (t.ph == 0 && !up_open) {  // the block input: the previous block's dense layer
                        spin_ge(s_dense(p.sync + (size_t)(b - 1) * kDecodeSyncInts), dense_need(p));
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                        up_open = true;
                    } else if (t.ph == 1 && t.g != open_g) {  // this expert's hidden rows
                        spin_ge(s_up(sy, t.g), (s.ntp[t.g + 1] - s.ntp[t.g]) * s.mt_up * C);
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                        open_g = t.g;
                    } else if (t.ph == 2 && !ds_open) {  // every expert's mix + the next block's routing
                        spin_ge(s_down(sy), s.dn_tiles * C);
                        if (b + 1 < nb) spin_ge(s_route(sy), 1);
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                        ds_open = true;
                    }
                    if (first) { dprobe(p, b, 1); first = false; }
                    if (t.ph == 2 && ds_open) dprobe(p, b, 6);
                    const int brow = t.ph == 2 ? t.n0 : t.row0 + t.n0;
                    for (int kb = t.kb0; kb < t.kb1; ++kb) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        tma_load_2d(sB + stage * kBBytes, bmaps[t.ph], &full[stage], kb * BK, brow);
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                }
                mbar_arrive(&sempty[sb]);
            }
        }
    } else if (warp >= 7) {
        // ============ routing role: the next block's pre-gate ==============
        const int rt = tid - 7 * 32;
        const bool tracing = p.x_trace != nullptr || p.ids_trace != nullptr;
        const bool croute = p.cluster_route && cluster == 0;
        int use = 0;
        for (int b = 0; b < nb; ++b) {
            const DecodeBlock &bd = p.blocks[b];
            if (!bd.has_pre_gate && !tracing) continue;
            if (p.cluster_route && !croute && !(tracing && blockIdx.x == 0)) continue;  // cluster 0 routes
            if (croute && bd.has_pre_gate) route_prefetch(p, bd, rank, rt, rs);  // static: before the input
            if (b == 0) {
                pdl_wait();
            } else {
                if (rt == 0) spin_ge(s_dense(p.sync + (size_t)(b - 1) * kDecodeSyncInts), dense_need(p));
                router_sync();
            }
            const float *xin = b == 0 ? p.x_in : bd.x;
            if (tracing && blockIdx.x == 0) {
                // block input and consumed decision, for teacher-forced parity
                // (this decision buffer is rewritten only once block b's dense
                // layer is done, after this CTA's routing work for block b)
                if (b > 0 && rt == 0) spin_ge(s_route(p.sync + (size_t)(b - 1) * kDecodeSyncInts), 1);
                router_sync();
                if (p.x_trace)
                    for (int i = rt; i < T * d / 4; i += kRouterThreads)
                        reinterpret_cast<float4 *>(p.x_trace + (size_t)b * T * d)[i] =
                            __ldcg(reinterpret_cast<const float4 *>(xin) + i);
                if (p.ids_trace)
                    for (int i = rt; i < T; i += kRouterThreads) {
                        p.ids_trace[(size_t)b * T + i] = __ldcg(bd.ids + i);
                        p.w_trace[(size_t)b * T + i] = __ldcg(bd.w + i);
                    }
            }
            if (!bd.has_pre_gate) continue;
            FusedRoute r = p.route;
            r.x = xin;
            r.G = bd.pre_gate;
            r.out = bd.out;
            r.done = s_route(p.sync + (size_t)b * kDecodeSyncInts);
            if (p.cluster_route) {
                if (croute) {
                    if (p.E == 64) cluster_route<2>(p, r, rank, rt, rs, r_xs, use);
                    else cluster_route<4>(p, r, rank, rt, rs, r_xs, use);
                    ++use;
                }
            } else {
                router_run(r, rt, r_xs, &r_flag, nullptr);
            }
            router_sync();
            if (rt == 0) dprobe(p, b, 5);
        }
    } else if (warp == 1) {
        // ============ MMA issuer ===========================================
        int stage = 0, cnt = 0;
        uint32_t phase = 0;
        for (int b = 0; b < nb; ++b) {
            const int sb = b & 1;
            mbar_wait(&sfull[sb], (b >> 1) & 1);
            const Sched &s = sched[sb];
            for (int i = cluster; i < s.total; i += nclusters, ++cnt) {
                const Tile t = decode_tile(s, i, rank, d, f);
                const int acc = cnt & 1;
                mbar_wait(&tempty[acc], ((cnt >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t tmem_d = tmem_base + acc * BN;
                const uint32_t idesc = idesc_bf16(BN);
                for (int kb = t.kb0; kb < t.kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    if (lane == 0) {
                        const uint32_t a_s = smem_u32(sA + stage * kABytes);
                        const uint32_t b_s = smem_u32(sB + stage * kBBytes);
#pragma unroll
                        for (int kk = 0; kk < BK / 16; ++kk)
                            umma_bf16(tmem_d, sw128_desc(a_s + kk * 32), sw128_desc(b_s + kk * 32), idesc,
                                      (kb > t.kb0 || kk > 0) ? 1u : 0u);
                        umma_commit(&empty[stage]);
                    }
                    __syncwarp();
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                if (lane == 0) {
                    if (t.kb1 > t.kb0) umma_commit(&tfull[acc]);
                    else mbar_arrive(&tfull[acc]);  // empty K slice: a zero partial
                }
                __syncwarp();
            }
            if (lane == 0) mbar_arrive(&sempty[sb]);
            __syncwarp();
        }
    } else {
        // ============ epilogue (warps 2-5): partial -> DSMEM sum -> stores =
        const int q = warp & 3;
        const int et = q * 32 + lane;  // accumulator row (TMEM lane)
        int cnt = 0;
        // this CTA's slice of every tile: rows [rank*kRows, +kRows); thread
        // et owns token column c = et / (kRows/2) and rows r0, r0+1
        constexpr int kPairs = kRows / 2;
        const int c = et / kPairs, rr = rank * kRows + 2 * (et % kPairs);
        for (int b = 0; b < nb; ++b) {
            const int sb = b & 1;
            mbar_wait(&sfull[sb], (b >> 1) & 1);
            const Sched &s = sched[sb];
            const DecodeBlock &bd = p.blocks[b];
            int *sy = p.sync + (size_t)b * kDecodeSyncInts;
            float *yb = b == nb - 1 ? p.y_out : bd.y;
            bool route_seen = false;
            for (int i = cluster; i < s.total; i += nclusters, ++cnt) {
                const Tile t = decode_tile(s, i, rank, d, f);
                const int acc = cnt & 1, pb = cnt & 1;
                float *pp = part + pb * (BM * BN);
                // 1. our partial -> shared memory (once every reader of the
                //    buffer's previous use is done)
                if (cnt >= 2) mbar_wait_cluster(&pempty[pb], ((cnt >> 1) - 1) & 1);
                mbar_wait(&tfull[acc], (cnt >> 1) & 1);
                tc_fence_after();
                if (et == 0 && i == cluster) dprobe(p, b, 2);
                float v[16];
                if (t.kb1 > t.kb0) {
                    tmem_ld16(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN, v);
                } else {
#pragma unroll
                    for (int j = 0; j < 16; ++j) v[j] = 0.f;
                }
                tc_fence_before();
                mbar_arrive(&tempty[acc]);
#pragma unroll
                for (int j = 0; j < 16; ++j) pp[j * BM + et] = v[j];  // [column][row]
                named_sync(1, 128);
                if (et < C) mbar_arrive_remote(&pfull[pb], (uint32_t)et);  // our partial -> every CTA
                // 2. the C partials of our rows, summed in rank order
                mbar_wait_cluster(&pfull[pb], (cnt >> 1) & 1);
                const uint32_t off = smem_u32(pp + c * BM + rr);
                float2 sum = make_float2(0.f, 0.f);
#pragma unroll
                for (int z = 0; z < C; ++z) {
                    const float2 a = ld_dsmem2(mapa(off, (uint32_t)z));
                    sum.x += a.x;
                    sum.y += a.y;
                }
                named_sync(1, 128);
                if (et == 0 && i == cluster) dprobe(p, b, 3);
                if (et < C) mbar_arrive_remote(&pempty[pb], (uint32_t)et);  // done reading every CTA's buffer
                // 3. epilogue of our slice
                const int nv = t.ph == 2 ? min(BN, T - t.n0) : t.n_valid;
                int *signal;
                if (t.ph == 0) {
                    if (c < nv) {
                        const size_t r = (size_t)(t.row0 + t.n0 + c);
                        const uint32_t o = bf16_bits(fmaxf(sum.x, 0.f)) | ((uint32_t)bf16_bits(fmaxf(sum.y, 0.f)) << 16);
                        *reinterpret_cast<uint32_t *>(p.hb + r * f + t.m * BM + rr) = o;  // relu, linalg.py:41-42
                    }
                    signal = s_up(sy, t.g);
                } else if (t.ph == 1) {
                    if (c < nv) {
                        const int r = t.row0 + t.n0 + c;
                        const float w = __ldcg(bd.w_perm + r);  // combine weight, linalg.py:45-51 (top-1)
                        const int tok = __ldcg(bd.perm + r);
                        const uint32_t o = bf16_bits(w * sum.x) | ((uint32_t)bf16_bits(w * sum.y) << 16);
                        *reinterpret_cast<uint32_t *>(p.mixb + (size_t)tok * d + t.m * BM + rr) = o;
                    }
                    signal = s_down(sy);
                } else {
                    if (bd.next_inv && !route_seen) {  // the next block's routing (operand order)
                        if (et == 0) spin_ge(s_route(sy), 1);
                        named_sync(1, 128);
                        route_seen = true;
                    }
                    if (c < nv) {
                        const int tok = t.n0 + c;
                        *reinterpret_cast<float2 *>(yb + (size_t)tok * d + t.m * BM + rr) = sum;
                        if (bd.next_inv) {
                            const int r = __ldcg(bd.next_inv + tok);
                            const uint32_t o = bf16_bits(sum.x) | ((uint32_t)bf16_bits(sum.y) << 16);
                            *reinterpret_cast<uint32_t *>(p.xb + (size_t)r * d + t.m * BM + rr) = o;
                        }
                    }
                    signal = s_dense(sy);
                }
                __threadfence();
                named_sync(1, 128);
                if (et == 0) {
                    atomicAdd(signal, 1);
                    dprobe(p, b, 4);
                }
            }
            if (et == 0) mbar_arrive(&sempty[sb]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(32));
    }
    if (tid == 0) probe(p.probe, blockIdx.x, 41);
    cl.sync();  // no CTA leaves while a peer may still read its shared memory
}

constexpr size_t smem_bytes() {
    return 1024 + (size_t)STAGES * (kABytes + kBBytes) + 2 * BM * BN * 4 + 2 * sizeof(Sched) + kRouteGBytes +
           (size_t)kRouteMaxT * kRouteMaxE * 8 + kRouteMaxE * 4 + kRouteMaxT * 8 + (2 * STAGES + 14) * 8 + 16;
}

}  // namespace dec

bool decode_supported(int T, int d, int f, int E, int k, int L, int nb) {
    return T >= 1 && T <= kDecodeMaxT && k == 1 && L == 1 && d % 128 == 0 && f % 128 == 0 && f >= d &&
           fused_route_supported(E) && nb <= kDecodeMaxBlocks;
}

int decode_iteration_tc(const DecodeArgs &a, cudaStream_t s) {
    using namespace dec;
    constexpr size_t smem = smem_bytes();
    static_assert(smem <= 227 * 1024, "decode kernel shared memory");
    static unsigned long long attr_set = 0;
    static int nclusters_dev[64] = {0};
    const int dev = current_device();
    PG_REQUIRE(dev >= 0 && dev < 64, PGMOE_E_CONFIG, "device ordinal %d unsupported", dev);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = C;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    if (!(attr_set & (1ull << dev))) {
        PG_CUDA(cudaFuncSetAttribute(decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        // every CTA spins on device counters: all clusters must be co-resident
        cfg.gridDim = dim3(C);
        int n = 0;
        PG_CUDA(cudaOccupancyMaxActiveClusters(&n, decode_kernel, &cfg));
        n = std::min(n, device_sm_count() / C);
        PG_REQUIRE(n >= 1, PGMOE_E_CUDA, "decode kernel: no co-resident %d-CTA cluster fits", C);
        nclusters_dev[dev] = n;
        attr_set |= 1ull << dev;
    }
    const int ncl = nclusters_dev[dev];
    cfg.gridDim = dim3(ncl * C);
    Params p{};
    p.T = a.T;
    p.d = a.d;
    p.f = a.f;
    p.E = a.E;
    p.nb = a.nb;
    p.blocks = a.blocks;
    p.sync = a.sync;
    p.x_in = a.x_in;
    p.y_out = a.y_out;
    p.xb = a.xb;
    p.hb = a.hb;
    p.mixb = a.mixb;
    p.route = a.route;
    p.x_trace = a.x_trace;
    p.ids_trace = a.ids_trace;
    p.w_trace = a.w_trace;
    p.cluster_route = (a.T <= kRouteMaxT && (a.E == 64 || a.E == 128) && a.d % (C * 8) == 0 &&
                       (size_t)(a.d / C) * a.E * 2 <= (size_t)kRouteGBytes && a.route.gt_bf16) ? 1 : 0;
    if (const char *e = getenv("PGMOE_DECODE_CROUTE")) p.cluster_route &= (e[0] != '0');
    p.probe = probe_buffer(1, ncl * C);
    CUtensorMap mw1, mw2, md, mx, mh, mm;
    PG_TRY(make_wmap(&mw1, a.experts, a.d, a.f, a.nrec, a.rec_bytes));
    PG_TRY(make_wmap(&mw2, static_cast<const char *>(a.experts) + (size_t)a.f * a.d * 2, a.f, a.d, a.nrec,
                     a.rec_bytes));
    PG_TRY(make_wmap(&md, a.pool, a.d, (int)a.pool_rows, 1, (size_t)a.pool_rows * a.d * 2));
    PG_TRY(make_bmap(&mx, a.xb, a.d, a.T));
    PG_TRY(make_bmap(&mh, a.hb, a.f, a.T));
    PG_TRY(make_bmap(&mm, a.mixb, a.d, a.T));
    PG_CUDA(cudaLaunchKernelEx(&cfg, decode_kernel, mw1, mw2, md, mx, mh, mm, p));
    count_launch();
    return PGMOE_OK;
}

}  // namespace pgmoe
