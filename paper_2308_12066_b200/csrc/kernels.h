// kernels.h — internal launch entry points shared by the runtime.
#pragma once
#include <cuda_runtime.h>

#include "../../include/pgmoe.h"

namespace pgmoe {

int expert_ffn_simt(const float *x, int T, int d, int f, int k, const void *experts, size_t stride,
                    int wdtype, int indexed_by_act, const pgmoe_routing *r, float *h, float *yw,
                    cudaStream_t s);
int dense_simt(const float *yw, int T, int d, int k, const void *dense_w, int wdtype, float *y,
               cudaStream_t s);

// tcgen05/TMA path (bf16 weights).  Returns PGMOE_E_CONFIG when the shape
// is outside what the kernel supports so callers can report it loudly.
int expert_ffn_tc(const float *x, int T, int d, int f, int k, const void *experts, size_t stride,
                  int indexed_by_act, const pgmoe_routing *r, float *h, float *yw, void *workspace,
                  size_t ws_bytes, cudaStream_t s);
int dense_tc(const float *yw, int T, int d, int k, const void *dense_w, float *y, void *workspace,
             size_t ws_bytes, cudaStream_t s);
bool tc_supported(int d, int f);
// xb[r] = bf16(x[perm[r] / k]): the up-projection operand in routing order
int tc_pack_rows(const float *x, const int *perm, int n, int d, int k, uint16_t *xb, cudaStream_t s);
// Fused-operand variants used by the runtime: bf16 activations packed once
// (xb), bf16 hidden (hb), and for top-1 the bf16 mix written by the down
// projection's epilogue so the dense layer reads it directly.
int expert_ffn_tc2(const float *x, int T, int d, int f, int k, const void *experts, size_t stride, int indexed_by_act,
                   const pgmoe_routing *r, uint16_t *xb, uint16_t *hb, float *yw, uint16_t *mixb, void *ws,
                   size_t ws_bytes, cudaStream_t s, bool xb_ready);
// One launch for up + down (+ the dense layer when dense_w != nullptr and
// top_k == 1), phases separated by in-kernel grid barriers.
struct FusedRoute;
// Chained resident launches (see tc::Params::epoch).
struct LaunchChain {
    int *epoch;       // device counter, zeroed at the start of each decoder iteration
    int epoch_wait;   // > 0: wait for *epoch >= epoch_wait; 0: for the previous launch to complete (PDL)
    int epoch_set;
    int parity;       // alternates between consecutive block launches
    unsigned long long *stamps;  // [epoch_set] %globaltimer when the launch's dense phase completes (or null)
};
int block_tc(const float *x, int T, int d, int f, int k, const void *experts, size_t stride, int indexed_by_act,
             const pgmoe_routing *r, uint16_t *xb, uint16_t *hb, float *yw, uint16_t *mixb, bool xb_ready,
             const void *dense_w, float *y, uint16_t *next_xb, const int *next_inv, void *ws, size_t ws_bytes,
             cudaStream_t s, const FusedRoute *route = nullptr, const LaunchChain *chain = nullptr,
             int n_experts = 0);
// next_xb / next_inv (optional): scatter y as the next block's packed bf16
// up-projection operand (the next block's routing is already known).
int dense_tc2(const float *yw, const uint16_t *mixb_ready, int T, int d, int k, const void *dense_w, float *y,
              uint16_t *mixb_scratch, void *ws, size_t ws_bytes, cudaStream_t s, uint16_t *next_xb,
              const int *next_inv);

}  // namespace pgmoe
