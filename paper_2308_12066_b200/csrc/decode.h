// decode.h — the small-batch persistent decoder (decode_tc.cu): per-block
// descriptors built once per resident model, and the launch arguments.
#pragma once
#include <cuda_runtime.h>

#include "route_common.cuh"

namespace pgmoe {

constexpr int kDecodeMaxT = 64;        // tokens per iteration (top-1: active experts <= T)
constexpr int kDecodeMaxAct = 64;
constexpr int kDecodeMaxBlocks = 64;
constexpr int kDecodeSyncInts = 4 + kDecodeMaxAct;  // per block: down, dense, route done, -, up per group

struct DecodeBlock {  // one decoder block, device memory (static per model)
    // the routing decision this block consumes
    const int *act, *n_act, *hist, *off, *perm, *inv;
    const float *w_perm;
    const int *ids;   // ids [T] and weights [T] of the decision (traces)
    const float *w;
    const int *next_inv;  // the next block's operand order (null: last block)
    int wrec0;            // first expert record of the block in the W1 / W2 maps
    int dense_row0;       // first row of the dense matrix in the weight-pool map
    int has_pre_gate;
    const float *x;       // block input (b >= 1)
    float *y;             // block output (b < nb - 1)
    const void *pre_gate;
    pgmoe_routing out;    // the decision this block's pre-gate writes
};

struct DecodeArgs {
    int T, d, f, E, nb;
    const DecodeBlock *blocks;
    int *sync;
    const float *x_in;
    float *y_out;
    uint16_t *xb, *hb, *mixb;
    FusedRoute route;               // T-dependent routing-role fields
    const void *experts;            // resident expert records [nb][E]
    int nrec;
    size_t rec_bytes;
    const void *pool;               // weight pool holding every dense matrix
    long long pool_rows;            // pool bytes / (2 d)
    // optional traces (null: off): block inputs [nb][T][d], decisions [nb][T]
    float *x_trace;
    int32_t *ids_trace;
    float *w_trace;
};

bool decode_supported(int T, int d, int f, int E, int k, int L, int nb);

// Low-latency small-batch decoder (decode_ll.cu): LL-word exchanges between
// row-split phases, T <= kLLMaxT tokens.
constexpr int kLLMaxT = 8;
struct LLDecodeArgs {
    int T, d, f, E, nb;
    const DecodeBlock *blocks;
    const void *experts;  // resident expert records [nb][E]
    size_t rec_bytes;
    const uint16_t *pool; // weight pool holding every dense matrix (DecodeBlock::dense_row0)
    const float *x_in;
    float *y_out;
    const void *gate0;        // block 0's conventional gate (bf16 [d][E]): routed inside the launch
    pgmoe_routing gate0_out;  // where its decision goes (the routing block 0 consumes)
    void *ws;             // ll_decode_ws_bytes(max T), prepared once by ll_decode_prepare
    size_t ws_bytes;
    float *x_trace;       // optional traces (as DecodeArgs)
    int32_t *ids_trace;
    float *w_trace;
};
bool ll_decode_supported(int T, int d, int f, int E, int k, int L, int nb);
size_t ll_decode_ws_bytes(int T, int d, int f, int E, int nb);
int ll_decode_prepare(void *ws, cudaStream_t s);
int ll_decode_iteration(const LLDecodeArgs &a, cudaStream_t s);
int decode_iteration_tc(const DecodeArgs &a, cudaStream_t s);

}  // namespace pgmoe
