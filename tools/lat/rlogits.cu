// Standalone timing of the routing role's partial-logit loop (route_common.cuh
// router_logits) without the GEMM roles: is it issue/compute-bound or does it
// wait on the co-resident warps?  One CTA per SM, 128 routing threads.
#include <cstdio>
#include <cstdint>
#include "../../paper_2308_12066_b200/csrc/common.cuh"
#include "../../paper_2308_12066_b200/csrc/route_common.cuh"
using namespace pgmoe;
__global__ void __launch_bounds__(kRouterThreads, 1) k(FusedRoute r, long long *cyc, unsigned long long *pr) {
    __shared__ __align__(16) float xs[kRouterSmemFloats];
    const int rt = threadIdx.x;
    long long t0 = clock64();
    if (rt == 0) probe(pr, blockIdx.x, 0);
    router_logits<uint16_t, 2>(r, blockIdx.x, rt, xs, pr);
    if (rt == 0) probe(pr, blockIdx.x, 1);
    long long t1 = clock64();
    if (rt == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    const int d = 768, E = 64, T = 8, S = 12;
    FusedRoute r{};
    r.active = 1; r.gt_bf16 = 1; r.d = d; r.E = E; r.T = T; r.k = 1; r.splits = S; r.tiles = 1;
    route_bound_constants(d, &r.gam, &r.bscale);
    float *x; uint16_t *G; double *pl, *px; float *pc; long long *cyc; unsigned long long *pr;
    cudaMalloc(&pr, 64 * 48 * 8);
    cudaMalloc(&x, T * d * 4); cudaMalloc(&G, d * E * 2); cudaMalloc(&pl, S * T * E * 8); cudaMalloc(&px, S * T * 8);
    cudaMalloc(&pc, S * E * 4); cudaMalloc(&cyc, 8 * S);
    cudaMemset(x, 0, T * d * 4); cudaMemset(G, 0x3f, d * E * 2);
    r.x = x; r.G = G; r.plogit = pl; r.pcmax = pc; r.pxsum = px;
    for (int it = 0; it < 3; ++it) {
        k<<<S, kRouterThreads>>>(r, cyc, pr);
        long long h[S]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        unsigned long long q[48]; cudaMemcpy(q, pr, sizeof(q), cudaMemcpyDeviceToHost);
        printf("  x+sx %.2f us, rows %.2f us, writes %.2f us\n", (q[40] - q[0]) / 1e3, (q[41] - q[40]) / 1e3, (q[1] - q[41]) / 1e3);
        printf("T=%d: %lld cycles (%.2f us at 1.965 GHz) for %d rows per split\n", T, h[0], h[0] / 1965.0, d / S);
    }
    r.T = 1;
    for (int it = 0; it < 2; ++it) {
        k<<<S, kRouterThreads>>>(r, cyc, pr);
        long long h[S]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        unsigned long long q[48]; cudaMemcpy(q, pr, sizeof(q), cudaMemcpyDeviceToHost);
        printf("  x+sx %.2f us, rows %.2f us, writes %.2f us\n", (q[40] - q[0]) / 1e3, (q[41] - q[40]) / 1e3, (q[1] - q[41]) / 1e3);
        printf("T=1: %lld cycles (%.2f us)\n", h[0], h[0] / 1965.0);
    }
    return 0;
}
