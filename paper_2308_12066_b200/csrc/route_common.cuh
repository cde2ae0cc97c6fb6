// route_common.cuh — certified-routing helpers shared by K1 (route.cu) and
// the routing role fused into the tcgen05 block kernel (ffn_tc.cu).
// Reference: gate_forward, core.py:284-305; matvec_columns, linalg.py:25-38.
#pragma once
#include <type_traits>
#include <algorithm>

#include "common.cuh"

namespace pgmoe {

__device__ __forceinline__ bool better(double fa, int ia, double fb, int ib) {
    // reference sort key (-logit, id): larger logit first, ties -> lower id
    return fa > fb || (fa == fb && ia < ib);
}

__device__ __forceinline__ void warp_argmax(double &f, int &id) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double of = __shfl_xor_sync(0xffffffffu, f, o);
        int oi = __shfl_xor_sync(0xffffffffu, id, o);
        if (oi >= 0 && (id < 0 || better(of, oi, f, id))) {
            f = of;
            id = oi;
        }
    }
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ double warp_sumd(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}


// Gate row loads of V adjacent experts as exact doubles (+ |g| for the
// column max that bounds the logit error).
template <typename GT> struct Vec;
template <> struct Vec<uint16_t> {
    static constexpr int N = 4;
    using Raw = uint2;
    __device__ __forceinline__ static Raw ld(const uint16_t *p) { return __ldg(reinterpret_cast<const uint2 *>(p)); }
    __device__ __forceinline__ static void cvt(Raw v, double (&d)[4], float (&a)[4]) {
        const float f[4] = {__uint_as_float(v.x << 16), __uint_as_float(v.x & 0xffff0000u),
                            __uint_as_float(v.y << 16), __uint_as_float(v.y & 0xffff0000u)};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            d[i] = f[i];
            a[i] = fabsf(f[i]);
        }
    }
    __device__ __forceinline__ static void load(const uint16_t *p, double (&d)[4], float (&a)[4]) {
        const uint2 v = __ldg(reinterpret_cast<const uint2 *>(p));
        const float f[4] = {__uint_as_float(v.x << 16), __uint_as_float(v.x & 0xffff0000u),
                            __uint_as_float(v.y << 16), __uint_as_float(v.y & 0xffff0000u)};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            d[i] = f[i];
            a[i] = fabsf(f[i]);
        }
    }
    __device__ __forceinline__ static double one(const uint16_t *p) { return bf16_to_f32(__ldg(p)); }
};
template <> struct Vec<float> {
    static constexpr int N = 4;
    using Raw = float4;
    __device__ __forceinline__ static Raw ld(const float *p) { return __ldg(reinterpret_cast<const float4 *>(p)); }
    __device__ __forceinline__ static void cvt(Raw v, double (&d)[4], float (&a)[4]) {
        d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
        a[0] = fabsf(v.x); a[1] = fabsf(v.y); a[2] = fabsf(v.z); a[3] = fabsf(v.w);
    }
    __device__ __forceinline__ static void load(const float *p, double (&d)[4], float (&a)[4]) {
        const float4 v = __ldg(reinterpret_cast<const float4 *>(p));
        d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
        a[0] = fabsf(v.x); a[1] = fabsf(v.y); a[2] = fabsf(v.z); a[3] = fabsf(v.w);
    }
    __device__ __forceinline__ static double one(const float *p) { return __ldg(p); }
};
// fp64 gate weights (the reference's own init_model matrices, unrounded):
// products are no longer exact, so the bound takes one more rounding
// (gamma_{d+1}); |g| is rounded UP to fp32 for the column max.
template <> struct Vec<double> {
    static constexpr int N = 2;
    __device__ __forceinline__ static void load(const double *p, double (&d)[2], float (&a)[2]) {
        const double2 v = __ldg(reinterpret_cast<const double2 *>(p));
        d[0] = v.x; d[1] = v.y;
        a[0] = __double2float_ru(fabs(v.x)); a[1] = __double2float_ru(fabs(v.y));
    }
    __device__ __forceinline__ static double one(const double *p) { return __ldg(p); }
};
template <typename GT> __device__ __forceinline__ double gval(const GT *G, size_t i) { return Vec<GT>::one(G + i); }
template <typename GT> __device__ __forceinline__ float gabs_up(const GT *G, size_t i) {
    return std::is_same<GT, double>::value ? __double2float_ru(fabs(gval(G, i))) : fabsf((float)gval(G, i));
}
// Two adjacent experts per load (the routing role's partial logits: 128
// threads x 2 experts cover a token group, so each warp's dependent FP64
// chain per gate row is half as long as with 4 experts per thread).
template <typename GT> struct Vec2;
template <> struct Vec2<uint16_t> {
    using Raw = uint32_t;
    __device__ __forceinline__ static Raw ld(const uint16_t *p) { return __ldg(reinterpret_cast<const uint32_t *>(p)); }
    __device__ __forceinline__ static void cvt(Raw v, double (&d)[2], float (&a)[2]) {
        const float f[2] = {__uint_as_float(v << 16), __uint_as_float(v & 0xffff0000u)};
        d[0] = f[0]; d[1] = f[1];
        a[0] = fabsf(f[0]); a[1] = fabsf(f[1]);
    }
};
template <> struct Vec2<float> {
    using Raw = float2;
    __device__ __forceinline__ static Raw ld(const float *p) { return __ldg(reinterpret_cast<const float2 *>(p)); }
    __device__ __forceinline__ static void cvt(Raw v, double (&d)[2], float (&a)[2]) {
        d[0] = v.x; d[1] = v.y;
        a[0] = fabsf(v.x); a[1] = fabsf(v.y);
    }
};


// Serial fp64 logit in the reference order (linalg.py:35-37): out += x_i*G_ij.
// Not inlined: the rare uncertified path would otherwise put NJ unrolled
// copies of this loop into the routing role's instruction stream.
template <typename GT, typename XT>
__device__ __noinline__ double serial_logit(const XT *x, const GT *G, int d, int E, int j) {
    double acc = 0.0;
    for (int i = 0; i < d; ++i) acc = __dadd_rn(acc, __dmul_rn((double)x[i], gval(G, (size_t)i * E + j)));
    return acc;
}

// ---------------------------------------------------------------------------
// Routing role fused into the tcgen05 block kernel (resident placement).
// The pre-gate of block b depends only on block b's INPUT, so the routing of
// block b+1 is computed by two extra warps per CTA while the expert GEMMs of
// block b stream their weights; only the dense epilogue (which packs block
// b+1's operand in b+1's routing order) and the next launch wait for it.
// Same arithmetic contract as route.cu: exact fp64 products, certified
// ranking with serial reference-order recompute, reference softmax.
// Work: units (token tile of kRouterTok tokens) x (K split) spread over the
// grid; the last split of a tile selects (one warp per token); the last
// tile builds histogram, scan, stable permutation and active list.
constexpr int kRouterThreads = 128;
constexpr int kRouterWarps = 4;
constexpr int kRouterTok = 8;
constexpr int kRouterMaxKn = 256;  // gate rows per split (x slice in shared memory)
// route workspace: [counter @0 | done @64 | tile counters @256 (8192 ints) | partials]
constexpr size_t kFusedRouteHead = 256 + 8192 * 4;

struct FusedRoute {
    int active;          // 0: this launch routes nothing
    int gt_bf16;         // gate dtype: 1 bf16, 0 fp32
    int d, E, T, k, splits, tiles;
    const float *x;      // block input [T][d]
    const void *G;       // pre-gate [d][E]
    pgmoe_routing out;
    int *counter;        // token tiles finished (reset by the last)
    int *tile_counter;   // [tiles] splits finished (reset by each tile's last)
    int *done;           // 1 once the permutation is written (re-armed at kernel exit)
    double *plogit;      // [splits][T][E]
    float *pcmax;        // [tiles][splits][E]
    double *pxsum;       // [splits][T]
    double gam, bscale;  // error-bound constants of d (route_bound_constants)
};

// gamma_d = d u / (1 - d u) and the certified-ranking bound scale, computed
// once on the host (IEEE double, the same values route.cu derives on device)
inline void route_bound_constants(int d, double *gam, double *bscale) {
    const double u = 1.1102230246251565e-16;  // 2^-53
    *gam = (double)d * u / (1.0 - (double)d * u);
    *bscale = 2.0 * *gam / (1.0 - *gam) * 1.001;
}

// Splits for a fused routing of T tokens: one unit per SM where possible,
// at most kRouterMaxKn gate rows per split.
inline int fused_route_splits(int T, int d, int grid) {
    const int tiles = (T + kRouterTok - 1) / kRouterTok;
    int s = std::max(1, grid / std::max(1, tiles));
    s = std::min(s, std::max(1, d / 64));
    s = std::min(s, 16);
    s = std::max(s, (d + kRouterMaxKn - 1) / kRouterMaxKn);
    return s;
}
inline size_t fused_route_ws_bytes(int T, int d, int E, int grid) {
    const int s = fused_route_splits(T, d, grid);
    const size_t tiles = (T + kRouterTok - 1) / kRouterTok;
    return (size_t)s * T * E * 8 + 256 + tiles * s * E * 4 + 256 + (size_t)s * T * 8 + 256;
}

__device__ __forceinline__ void router_sync() { asm volatile("bar.sync 2, %0;" ::"n"(kRouterThreads)); }

// Partial fp64 logits of one (tile, split) unit.  NJ = E / 32: each thread
// owns 2 adjacent experts x NJ tokens (128 threads cover 8 tokens x E; the
// loop is latency-bound per warp, so more, shorter chains finish sooner).  When
// the tile holds <= NJ tokens (small batches) the token groups take row
// slices instead and are summed in shared memory in a fixed order, so each
// thread has a quarter (E=64) or half (E=128) of the rows to load: at small T
// every gate load waits behind the block's weight prefetch, and the number
// of dependent load rounds is the routing role's critical path.
constexpr int kRouterSmemFloats = 3328;  // x slice + row-split reduction (13 KB)

template <typename GT, int NJ>
__device__ void router_logits(const FusedRoute &r, int unit, int rt, float *xs, unsigned long long *pr) {
    const int E = r.E, T = r.T, d = r.d;
    const int tile = unit / r.splits, split = unit - tile * r.splits;
    const int t0 = tile * kRouterTok, ntok = min(kRouterTok, T - t0);
    const int k0 = (int)((long)d * split / r.splits), k1 = (int)((long)d * (split + 1) / r.splits);
    const int kn = k1 - k0;
    constexpr int CG = 16 * NJ;                // E / 2 column groups (2 experts per thread)
    constexpr int TG = kRouterThreads / CG;    // token (or row) groups: TG x NJ = 8 tokens
    static_assert(TG * NJ == kRouterTok, "the role's threads cover a token tile");
    const bool rowsplit = TG > 1 && ntok <= NJ;
    const int tslots = rowsplit ? NJ : kRouterTok;
    for (int i0 = rt; i0 < tslots * kn; i0 += 8 * kRouterThreads) {  // 8 loads in flight
        float v[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const int i = i0 + b * kRouterThreads, t = i / kn;
            v[b] = (i < tslots * kn && t < ntok) ? __ldg(r.x + (size_t)(t0 + t) * d + k0 + (i - t * kn)) : 0.f;
        }
#pragma unroll
        for (int b = 0; b < 8; ++b)
            if (i0 + b * kRouterThreads < tslots * kn) xs[i0 + b * kRouterThreads] = v[b];
    }
    router_sync();
    const int lane = rt & 31, w = rt >> 5;
    for (int t = w; t < ntok; t += kRouterWarps) {  // sum |x_i| over the slice (bounds the error)
        double sx = 0.0;
        for (int i = lane; i < kn; i += 32) sx += fabs((double)xs[t * kn + i]);
        sx = warp_sumd(sx);
        if (lane == 0) r.pxsum[(size_t)split * T + t0 + t] = sx;
    }
    if (rt == 0) probe(pr, blockIdx.x, 40);  // x slice in shared memory
    const int cg = rt % CG, tg = rt / CG;
    const int tbase = rowsplit ? 0 : tg * NJ;
    const int rstart = rowsplit ? tg : 0, rstep = rowsplit ? TG : 1;
    const int nrows = rowsplit ? (kn - tg + TG - 1) / TG : kn;
    double acc[NJ][2];
    float cm[2] = {0.f, 0.f};
#pragma unroll
    for (int tt = 0; tt < NJ; ++tt)
#pragma unroll
        for (int v = 0; v < 2; ++v) acc[tt][v] = 0.0;
    const GT *G = static_cast<const GT *>(r.G) + (size_t)k0 * E + cg * 2;
    // 32 gate rows in flight per thread (raw, converted on use): this role
    // runs next to the expert GEMMs' weight stream, so every load sees the
    // loaded memory latency (in-flight bytes / bandwidth)
    using Raw = typename Vec2<GT>::Raw;
    // Batches of NB rows without a per-row guard: a guard per row made every
    // row its own basic block, so the scheduler could not overlap one row's
    // shared-memory load and conversions with the previous row's FMAs
    // (~160 cycles per row instead of a few).
    auto rows = [&](auto nb, int n0) {
        constexpr int NB = decltype(nb)::value;
        Raw raw[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) raw[b] = Vec2<GT>::ld(G + (size_t)(rstart + (n0 + b) * rstep) * E);
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const int i = rstart + (n0 + b) * rstep;
            double g[2];
            float a[2];
            Vec2<GT>::cvt(raw[b], g, a);
#pragma unroll
            for (int v = 0; v < 2; ++v) cm[v] = fmaxf(cm[v], a[v]);
#pragma unroll
            for (int tt = 0; tt < NJ; ++tt) {
                const double xv = xs[(tbase + tt) * kn + i];
#pragma unroll
                for (int v = 0; v < 2; ++v) acc[tt][v] = fma(xv, g[v], acc[tt][v]);  // exact product, one rounding
            }
        }
    };
    int n0 = 0;
    for (; n0 + 32 <= nrows; n0 += 32) rows(std::integral_constant<int, 32>{}, n0);  // rows in order: same sums
    for (; n0 + 8 <= nrows; n0 += 8) rows(std::integral_constant<int, 8>{}, n0);
    for (; n0 < nrows; ++n0) rows(std::integral_constant<int, 1>{}, n0);
    if (rt == 0) probe(pr, blockIdx.x, 41);  // gate rows consumed
    if (!rowsplit) {
#pragma unroll
        for (int tt = 0; tt < NJ; ++tt) {
            const int t = tbase + tt;
            if (t < ntok)
#pragma unroll
                for (int v = 0; v < 2; ++v) r.plogit[((size_t)split * T + t0 + t) * E + cg * 2 + v] = acc[tt][v];
        }
        if (tg == 0)
#pragma unroll
            for (int v = 0; v < 2; ++v) r.pcmax[((size_t)tile * r.splits + split) * E + cg * 2 + v] = cm[v];
    } else {
        // [TG][NJ][E] partial sums and [TG][E] column maxima after the x slice
        double *red = reinterpret_cast<double *>(xs + ((tslots * kn + 1) & ~1));
        float *cmr = reinterpret_cast<float *>(red + TG * NJ * E);
#pragma unroll
        for (int tt = 0; tt < NJ; ++tt)
#pragma unroll
            for (int v = 0; v < 2; ++v) red[(tg * NJ + tt) * E + cg * 2 + v] = acc[tt][v];
#pragma unroll
        for (int v = 0; v < 2; ++v) cmr[tg * E + cg * 2 + v] = cm[v];
        router_sync();
        for (int q = rt; q < ntok * E; q += kRouterThreads) {
            const int tt = q / E, j = q - tt * E;
            double sum = 0.0;
#pragma unroll
            for (int g = 0; g < TG; ++g) sum += red[(g * NJ + tt) * E + j];  // fixed order: deterministic
            r.plogit[((size_t)split * T + t0 + tt) * E + j] = sum;
        }
        for (int j = rt; j < E; j += kRouterThreads) {
            float m = 0.f;
#pragma unroll
            for (int g = 0; g < TG; ++g) m = fmaxf(m, cmr[g * E + j]);
            r.pcmax[((size_t)tile * r.splits + split) * E + j] = m;
        }
    }
    router_sync();  // the x slice is rewritten by the next unit
}

// Sum the K-split partials of a tile's tokens (all 128 role threads, loads
// of two (token, expert) entries = up to 64 partials in flight per thread,
// summed in split order) into shared memory: lgs[t][j] (fp64 logit),
// cms[t][j] (column max |G|), sxs[t] (sum |x|).  The per-token selection
// then works from shared memory, so the tile costs one or two dependent
// load rounds rather than one per 32 experts per token.
struct TileSums {
    double *lgs;  // [ntok][E]
    float *cms;   // [ntok][E]
    double *sxs;  // [kRouterTok]
};
// ch: tokens per chunk (the scratch holds ch rows of sums, see router_role)
__device__ __forceinline__ TileSums tile_sums_layout(float *xs, int E, int ch) {
    TileSums ts;
    ts.sxs = reinterpret_cast<double *>(xs);
    ts.lgs = ts.sxs + kRouterTok;
    ts.cms = reinterpret_cast<float *>(ts.lgs + ch * E);
    return ts;
}
static __device__ __noinline__ void router_reduce_tile(const FusedRoute &r, int tile, int t0, int ntok, int rt, const TileSums &ts,
                                                       unsigned long long *pr) {
    const int E = r.E, T = r.T, S = r.splits;
    // sum |x| per token: one (token, split) per lane, 16 lanes per token
    // (4 warps x 2 tokens = the tile), summed by a fixed butterfly; issued
    // before the first batch of partials so both share one load round
    static_assert(kRouterThreads >= 16 * kRouterTok, "16 lanes per token");
    const int st = rt >> 4, sz = rt & 15;
    double sxv = 0.0;
    if (st < ntok)
        for (int z = sz; z < S; z += 16) sxv += __ldcg(r.pxsum + (size_t)z * T + t0 + st);
    const int n = ntok * E;
    for (int q0 = rt; q0 < n; q0 += 2 * kRouterThreads) {
        double pl[2][16];
        float pc[2][16];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int q = q0 + h * kRouterThreads;
            const int t = q / E, j = q - t * E;
#pragma unroll
            for (int z = 0; z < 16; ++z) {
                const bool ok = q < n && z < S;
                pl[h][z] = ok ? __ldcg(r.plogit + ((size_t)z * T + t0 + t) * E + j) : 0.0;
                pc[h][z] = ok ? __ldcg(r.pcmax + ((size_t)tile * S + z) * E + j) : 0.f;
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int q = q0 + h * kRouterThreads;
            if (q >= n) continue;
            double sum = 0.0;
            float cm = 0.f;
#pragma unroll
            for (int z = 0; z < 16; ++z)  // split order: deterministic
                if (z < S) {
                    sum += pl[h][z];
                    cm = fmaxf(cm, pc[h][z]);
                }
            for (int z = 16; z < S; ++z) {  // S > 16 (not produced by fused_route_splits)
                sum += __ldcg(r.plogit + ((size_t)z * T + t0 + q / E) * E + (q % E));
                cm = fmaxf(cm, __ldcg(r.pcmax + ((size_t)tile * S + z) * E + (q % E)));
            }
            ts.lgs[q] = sum;
            ts.cms[q] = cm;
        }
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) sxv += __shfl_xor_sync(0xffffffffu, sxv, o);
    if (sz == 0 && st < ntok) ts.sxs[st] = sxv;
    if (rt == 0 && t0 == tile * kRouterTok) probe(pr, blockIdx.x, 35);  // sums in shared memory
    router_sync();
}

// One token's certified selection + softmax, by one warp (select_tile's
// per-token logic with the E logits in registers, NJ per lane).  `t`: the
// token's index in the tile (shared sums), `tok`: its global index.
template <typename GT, int NJ>
__device__ void router_select_token(const FusedRoute &r, const TileSums &ts, int t, int tok, int lane,
                                    int *s_ids, float *s_w, unsigned long long *pr = nullptr) {
    if (t != 0 || lane != 0) pr = nullptr;
    const int E = r.E, k = r.k, d = r.d;
    const double gam = r.gam, bscale = r.bscale;
    const double bpad = 1e-300;
    const double sx = ts.sxs[t] * (1.0 + 2.0 * gam);
    double lg[NJ], bd[NJ];
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj) {
        const int j = lane + 32 * jj;
        lg[jj] = ts.lgs[t * E + j];
        bd[jj] = bscale * sx * (double)ts.cms[t * E + j] + bpad;
    }
    auto pick = [&](const double (&a)[NJ], int bi) -> double {  // a[bi >> 5] of lane bi & 31
        double mine = 0.0;
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj)
            if (jj == (bi >> 5)) mine = a[jj];
        return __shfl_sync(0xffffffffu, mine, bi & 31);
    };
    probe(pr, blockIdx.x, 37);
    bool finite = true;
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj) finite &= (bool)isfinite(lg[jj]);
    finite = __all_sync(0xffffffffu, finite);
    if (!finite) {  // core.py:297
        if (lane == 0) atomicCAS(r.out.status, 0, (int)PGMOE_E_GATE_OVERFLOW);
        for (int s = lane; s < k; s += 32) {
            r.out.ids[(size_t)tok * k + s] = 0;
            r.out.w[(size_t)tok * k + s] = 0.f;
            s_ids[t * k + s] = 0;
            s_w[t * k + s] = 0.f;
        }
        return;
    }
    int sel[8];
    uint32_t taken = 0;
    bool certified = true;
    double minlow = INFINITY;
    double top = 0.0;  // the largest logit: the first selected one (the softmax shift)
    for (int s = 0; s < k; ++s) {
        double bf = -INFINITY;
        int bi = -1;
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj)
            if (!(taken >> jj & 1u) && (bi < 0 || better(lg[jj], lane + 32 * jj, bf, bi))) {
                bf = lg[jj];
                bi = lane + 32 * jj;
            }
        warp_argmax(bf, bi);
        if (s == 0) top = bf;
        sel[s] = bi;
        if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
        const double low = bf - pick(bd, bi);
        minlow = fmin(minlow, low);
        double up = -INFINITY;
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj)
            if (!(taken >> jj & 1u)) up = fmax(up, lg[jj] + bd[jj]);
        up = warp_max(up);
        certified &= (low > up);
    }
    if (!certified) {  // recompute the candidates in the reference's serial order
        uint32_t cand = 0;
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj)
            if (lg[jj] + bd[jj] >= minlow) cand |= 1u << jj;
        const GT *G = static_cast<const GT *>(r.G);
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj)
            if (cand >> jj & 1u) lg[jj] = serial_logit<GT, float>(r.x + (size_t)tok * d, G, d, E, lane + 32 * jj);
        for (int s = 0; s < k; ++s) {
            double bf = -INFINITY;
            int bi = -1;
#pragma unroll
            for (int jj = 0; jj < NJ; ++jj)
                if ((cand >> jj & 1u) && (bi < 0 || better(lg[jj], lane + 32 * jj, bf, bi))) {
                    bf = lg[jj];
                    bi = lane + 32 * jj;
                }
            warp_argmax(bf, bi);
            // the recomputed candidates bound every other logit from above
            // (those stay below minlow), so the maximum is still the first pick
            if (s == 0) top = bf;
            sel[s] = bi;
            if ((bi & 31) == lane) cand &= ~(1u << (bi >> 5));
        }
        if (lane == 0) atomicAdd(r.out.status + 1, 1);
    }
    probe(pr, blockIdx.x, 38);
    // softmax over all E (linalg.py:54-59), max-subtracted; same order as route.cu
    const double m = top;  // == max over all E logits (no extra warp reduction)
    double z = 0.0;
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj) z += exp(lg[jj] - m);
    z = warp_sumd(z);
    probe(pr, blockIdx.x, 39);
    for (int s = 0; s < k; ++s) {
        const double pr = exp(pick(lg, sel[s]) - m) / z;
        if (lane == 0) {
            if (!(pr > 0.0)) atomicCAS(r.out.status, 0, (int)PGMOE_E_GATE_UNDERFLOW);
            r.out.ids[(size_t)tok * k + s] = sel[s];
            r.out.w[(size_t)tok * k + s] = __double2float_rn(pr);
            s_ids[t * k + s] = sel[s];
            s_w[t * k + s] = __double2float_rn(pr);
        }
    }
}

// Histogram, exclusive scan, stable permutation, active list (permute_all
// of route.cu with the router's warps).  sm: >= (kRouterWarps + 1) * E ints.
static __device__ __noinline__ void router_permute(const FusedRoute &r, int rt, int *sm, const int *ids_src,
                                                   const float *w_src) {
    const int E = r.E, k = r.k, lane = rt & 31, w = rt >> 5;
    const int N = r.T * k;
    int *whist = sm;                        // [kRouterWarps][E] -> cursors
    int *tot = whist + kRouterWarps * E;    // [E]
    for (int i = rt; i < kRouterWarps * E; i += kRouterThreads) whist[i] = 0;
    router_sync();
    const int seg = (N + kRouterWarps - 1) / kRouterWarps;
    const int r0 = w * seg, r1 = min(N, r0 + seg);
    for (int i = r0 + lane; i < r1; i += 32) atomicAdd(&whist[w * E + ids_src[i]], 1);
    router_sync();
    for (int e = rt; e < E; e += kRouterThreads) {
        int s = 0;
        for (int ww = 0; ww < kRouterWarps; ++ww) s += whist[ww * E + e];
        tot[e] = s;
    }
    router_sync();
    if (w == 0) {
        int run = 0, nact = 0;
        for (int e0 = 0; e0 < E; e0 += 32) {
            const int e = e0 + lane;
            const int h = e < E ? tot[e] : 0;
            int incl = h;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            const unsigned am = __ballot_sync(0xffffffffu, h > 0);
            if (e < E) {
                const int ex = run + incl - h;
                r.out.hist[e] = h;
                r.out.off[e] = ex;
                tot[e] = ex;
                if (h > 0) r.out.act[nact + __popc(am & ((1u << lane) - 1u))] = e;
            }
            run += __shfl_sync(0xffffffffu, incl, 31);
            nact += __popc(am);
        }
        if (lane == 0) {
            r.out.off[E] = run;
            *r.out.n_act = nact;
        }
    }
    router_sync();
    for (int e = rt; e < E; e += kRouterThreads) {
        int base = tot[e];
        for (int ww = 0; ww < kRouterWarps; ++ww) {
            const int c = whist[ww * E + e];
            whist[ww * E + e] = base;
            base += c;
        }
    }
    router_sync();
    const unsigned ltmask = (1u << lane) - 1u;
    for (int c0 = r0; c0 < r1; c0 += 32) {
        const int i = c0 + lane;
        const bool valid = i < r1;
        const unsigned vm = __ballot_sync(0xffffffffu, valid);
        if (valid) {
            const int e = ids_src[i];
            const unsigned grp = __match_any_sync(vm, e);
            const int rank = __popc(grp & ltmask);
            const int pos = whist[w * E + e] + rank;
            r.out.perm[pos] = i;
            if (r.out.inv) r.out.inv[i] = pos;
            r.out.w_perm[pos] = w_src[i];
            __syncwarp(vm);
            if (rank == __popc(grp) - 1) whist[w * E + e] += __popc(grp);
        }
        __syncwarp();
    }
}

// The same permutation for N = T*k <= 32 rows by ONE warp (lane = row), with
// no shared-memory histogram and no barriers: row r goes to #{rows of a
// smaller expert} + #{earlier rows of its expert} — the stable order
// router_permute builds.
static __device__ __noinline__ void router_permute_small(const FusedRoute &r, int lane, const int *ids_src,
                                                         const float *w_src) {
    const int E = r.E, N = r.T * r.k;
    const bool v = lane < N;
    const int e = v ? ids_src[lane] : 0x7fffffff;
    const float wv = v ? w_src[lane] : 0.f;
    int less = 0, before = 0;
    for (int l = 0; l < N; ++l) {
        const int el = __shfl_sync(0xffffffffu, e, l);
        less += el < e;
        before += (el == e) & (l < lane);
    }
    if (v) {
        const int pos = less + before;
        r.out.perm[pos] = lane;
        if (r.out.inv) r.out.inv[lane] = pos;
        r.out.w_perm[pos] = wv;
    }
    int nact = 0;
    for (int e0 = 0; e0 < E; e0 += 32) {
        const int ex = e0 + lane;
        int h = 0, lt = 0;
        for (int l = 0; l < N; ++l) {
            const int el = __shfl_sync(0xffffffffu, e, l);
            h += el == ex;
            lt += el < ex;
        }
        const unsigned am = __ballot_sync(0xffffffffu, ex < E && h > 0);
        if (ex < E) {
            r.out.hist[ex] = h;
            r.out.off[ex] = lt;
            if (h > 0) r.out.act[nact + __popc(am & ((1u << lane) - 1u))] = ex;
        }
        nact += __popc(am);
    }
    if (lane == 0) {
        r.out.off[E] = N;
        *r.out.n_act = nact;
    }
}

// The whole routing role (64 threads, rt = 0..63) for one CTA.
template <typename GT, int NJ>
__device__ void router_role(const FusedRoute &r, int rt, float *xs, int *s_flag, unsigned long long *pr) {
    const int lane = rt & 31, w = rt >> 5;
    const int units = r.tiles * r.splits;
    for (int unit = blockIdx.x; unit < units; unit += gridDim.x) {
        router_logits<GT, NJ>(r, unit, rt, xs, unit == (int)blockIdx.x ? pr : nullptr);
        if (rt == 0) probe(pr, blockIdx.x, 26);  // partial logits written
        const int tile = unit / r.splits;
        __threadfence();
        router_sync();
        if (rt == 0) *s_flag = (atomicAdd(r.tile_counter + tile, 1) == r.splits - 1);
        router_sync();
        if (!*s_flag) continue;
        __threadfence();
        const int t0 = tile * kRouterTok, ntok = min(kRouterTok, r.T - t0);
        if (rt == 0) probe(pr, blockIdx.x, 27);  // tile select start

        // the tile's ids / weights also stay in shared memory (the end of the
        // scratch, clear of the sums and of the permutation's histograms)
        int *s_ids = reinterpret_cast<int *>(xs + kRouterSmemFloats - 2 * kRouterTok * 8);
        float *s_w = xs + kRouterSmemFloats - kRouterTok * 8;
        // token chunks whose sums fit the scratch (E=256: 4 tokens at a time)
        constexpr int kChunk = (kRouterSmemFloats - 2 * kRouterTok * 8 - 2 * kRouterTok) / (NJ * 32 * 3);
        constexpr int CH = kChunk < kRouterTok ? kChunk : kRouterTok;
        static_assert(CH >= 1, "routing scratch too small");
        static_assert(2 * kRouterTok + CH * NJ * 32 * 3 + 2 * kRouterTok * 8 <= kRouterSmemFloats,
                      "tile sums + ids / weights exceed the routing scratch");
        const TileSums ts = tile_sums_layout(xs, r.E, CH);
        for (int c0 = 0; c0 < ntok; c0 += CH) {
            const int nc = min(CH, ntok - c0);
            router_reduce_tile(r, tile, t0 + c0, nc, rt, ts, pr);
            if (rt == 0 && c0 == 0) probe(pr, blockIdx.x, 32);  // partials reduced
            for (int t = w; t < nc; t += kRouterWarps)
                router_select_token<GT, NJ>(r, ts, t, t0 + c0 + t, lane, s_ids + c0 * r.k, s_w + c0 * r.k,
                                            c0 == 0 ? pr : nullptr);
            if (rt == 0 && c0 == 0) probe(pr, blockIdx.x, 33);  // warp 0 selected
            router_sync();  // the sums are rewritten by the next chunk
        }
        __threadfence();
        router_sync();
        if (rt == 0) probe(pr, blockIdx.x, 28);  // tile selected
        const bool single = r.tiles == 1;  // this CTA holds every token's decision: no global ticket
        if (rt == 0) {
            r.tile_counter[tile] = 0;
            *s_flag = single ? 1 : (atomicAdd(r.counter, 1) == r.tiles - 1);
        }
        router_sync();
        if (!*s_flag) continue;
        if (!single) __threadfence();
        if (r.T * r.k <= 32) {
            if (w == 0) router_permute_small(r, lane, single ? s_ids : r.out.ids, single ? s_w : r.out.w);
        } else {
            router_permute(r, rt, reinterpret_cast<int *>(xs), single ? s_ids : r.out.ids, single ? s_w : r.out.w);
        }
        __threadfence();
        router_sync();
        if (rt == 0) probe(pr, blockIdx.x, 29);  // permutation written
        if (rt == 0) {
            if (!single) *r.counter = 0;
            asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(r.done), "r"(1) : "memory");
        }
    }
}

template <int NJ>
__device__ __forceinline__ void router_dispatch_gt(const FusedRoute &r, int rt, float *xs, int *s_flag,
                                                   unsigned long long *pr) {
    if (r.gt_bf16) router_role<uint16_t, NJ>(r, rt, xs, s_flag, pr);
    else router_role<float, NJ>(r, rt, xs, s_flag, pr);
}
__device__ __forceinline__ void router_run(const FusedRoute &r, int rt, float *xs, int *s_flag,
                                           unsigned long long *pr) {
    switch (r.E) {
        case 64: router_dispatch_gt<2>(r, rt, xs, s_flag, pr); break;
        case 128: router_dispatch_gt<4>(r, rt, xs, s_flag, pr); break;
        case 256: router_dispatch_gt<8>(r, rt, xs, s_flag, pr); break;
        default: break;  // the host only fuses E in {64, 128, 256}
    }
}
inline bool fused_route_supported(int E) { return E == 64 || E == 128 || E == 256; }

}  // namespace pgmoe
