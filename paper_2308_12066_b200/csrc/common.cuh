// common.cuh — shared helpers for the sm_100a pre-gated MoE library.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/pgmoe.h"

namespace pgmoe {

void set_error(const char *fmt, ...);
void count_launch(int n = 1);  // kernels launched by this library (bench evidence)

#define PG_CUDA(call)                                                                 \
    do {                                                                              \
        cudaError_t _e = (call);                                                      \
        if (_e != cudaSuccess) {                                                      \
            ::pgmoe::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,             \
                               cudaGetErrorString(_e));                               \
            return (_e == cudaErrorMemoryAllocation) ? PGMOE_E_OOM : PGMOE_E_CUDA;    \
        }                                                                             \
    } while (0)

#define PG_TRY(call)                  \
    do {                              \
        int _s = (call);              \
        if (_s != PGMOE_OK) return _s; \
    } while (0)

#define PG_REQUIRE(cond, code, ...)           \
    do {                                      \
        if (!(cond)) {                        \
            ::pgmoe::set_error(__VA_ARGS__);  \
            return (code);                    \
        }                                     \
    } while (0)

constexpr int kNumSMs = 148;  // B200; grid sizing heuristics only — persistent launches use device_sm_count()

// SMs of the current device (cudaDevAttrMultiProcessorCount, cached per
// device): the persistent kernels put one CTA on each and spin on grid-wide
// counters, so their grid must never exceed what is co-resident.
int device_sm_count();
int current_device();

__device__ __forceinline__ float bf16_to_f32(uint16_t h) {
    return __uint_as_float(static_cast<uint32_t>(h) << 16);
}

// Weight element -> fp32 / fp64 (exact for both storage types).
template <typename WT> struct WTraits;
template <> struct WTraits<float> {
    static constexpr int id = PGMOE_F32;
    __device__ __forceinline__ static float f32(float v) { return v; }
};
template <> struct WTraits<uint16_t> {
    static constexpr int id = PGMOE_BF16;
    __device__ __forceinline__ static float f32(uint16_t v) { return bf16_to_f32(v); }
};

inline size_t dtype_bytes(int dt) { return dt == PGMOE_BF16 ? 2 : 4; }

// Programmatic dependent launch: wait for the preceding kernel's memory /
// let the next kernel start its prologue.  No-ops without the launch attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Debug probes (tools/probe.py): per-CTA %globaltimer stamps written when a
// probe buffer is installed with pgmoe_debug_set_probe(); null otherwise.
constexpr int kProbeSlots = 48;
unsigned long long *probe_buffer(int kind, int ctas);  // 0: route, 1: tcgen05 block kernel
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void probe(unsigned long long *buf, int cta, int slot) {
    if (buf) buf[(size_t)cta * kProbeSlots + slot] = gtimer();
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace pgmoe
