// internal.h -- shared host/device helpers of libmcapq (NOT part of the ABI).
// Nothing here is shared with oracle/: the CUDA path has its own conversions
// (hardware intrinsics) and its own launch plumbing.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>

#include "../../include/mcapq.h"

namespace mcapq {

// ---------------------------------------------------------------- host side
void set_error(const char *fmt, ...);
void clear_error();

#define MCAPQ_REQUIRE(cond, code, ...)                                                                       \
    do {                                                                                                     \
        if (!(cond)) {                                                                                       \
            ::mcapq::set_error(__VA_ARGS__);                                                                 \
            return (code);                                                                                   \
        }                                                                                                    \
    } while (0)

#define MCAPQ_CUDA_TRY(expr)                                                                                 \
    do {                                                                                                     \
        cudaError_t e_ = (expr);                                                                             \
        if (e_ != cudaSuccess) {                                                                             \
            ::mcapq::set_error("%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__);         \
            return MCAPQ_ECUDA;                                                                              \
        }                                                                                                    \
    } while (0)

inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
// thread-local: API linears launch with programmatic dependent launch (mcapq_set_pdl)
bool api_pdl();
void set_api_pdl(bool on);
inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Launch a kernel with the programmatic-stream-serialization attribute (PDL):
// it may start before the previous kernel on the stream finishes; the kernel
// itself calls griddep_wait() before touching data the predecessor wrote.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       bool pdl, Args &&...args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Per-process device facts (cached per device ordinal).
int device_sms();
// cudaFuncSetAttribute(kernel, MaxDynamicSharedMemorySize = smem_bytes [, preferred
// carveout]) once per (kernel, current device): host-side, thread-safe, no stream work.
cudaError_t kernel_smem_attr(const void *kernel, int smem_bytes, int carveout = -1);

// Kernel launchers (kernels_*.cu).  All return cudaError_t of the launch.
cudaError_t launch_pack_w4(const void *w, int wdt, int64_t n, int64_t k, int64_t ldw, uint8_t *nib,
                           uint16_t *scale, uint32_t *dev_err, cudaStream_t s);
cudaError_t launch_quant_a8(const uint16_t *x, int64_t m, int64_t k, int64_t ldx, int8_t *q, float *sx,
                            int32_t *sq, cudaStream_t s, bool pdl);
cudaError_t launch_w4a8(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k, const int8_t *q,
                        const float *sx, const int32_t *sq, int64_t m, void *y, int ydt, int64_t ldy,
                        cudaStream_t s, bool pdl);
cudaError_t launch_w4a16(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k, const uint16_t *x,
                         int64_t m, int64_t ldx, void *y, int ydt, int64_t ldy, cudaStream_t s, bool pdl);
cudaError_t launch_w4a8_group_dots(const uint8_t *nib, int64_t n, int64_t k, const int8_t *q,
                                   const int32_t *sq, int64_t m, int32_t *D, int mode, cudaStream_t s);
int kernels_per_linear(int route, int64_t m);

// Workspace carve-up of a fused W4A8 call.
struct A8Workspace {
    int8_t *q;
    float *sx;
    int32_t *sq;
};
size_t a8_workspace_bytes(int64_t m, int64_t k);
A8Workspace a8_workspace(void *ws, int64_t m, int64_t k);

}  // namespace mcapq

// ---------------------------------------------------------------- device side
#ifdef __CUDACC__
namespace mcapq {
namespace dev {

// PDL controls (sm_90+): wait for the predecessor grid's memory, and allow the
// successor grid to launch early.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Streaming 128-bit read-only load that does not allocate in L1.
__device__ __forceinline__ uint4 ld_stream_128(const void *p)
{
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
// 32-bit read-only load through L1 (the quad-split fragment loads re-hit the line).
__device__ __forceinline__ uint32_t ld_nc_32(const void *p)
{
    uint32_t r;
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ uint16_t ld_nc_16(const void *p)
{
    uint16_t r;
    asm volatile("ld.global.nc.u16 %0, [%1];" : "=h"(r) : "l"(p));
    return r;
}

__device__ __forceinline__ float half_bits_to_float(uint16_t h)
{
    float f;
    asm("cvt.f32.f16 %0, %1;" : "=f"(f) : "h"(h));
    return f;
}
__device__ __forceinline__ float bf16_bits_to_float(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }
__device__ __forceinline__ uint16_t float_to_bf16_bits(float f)
{
    uint16_t r;
    asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(r) : "f"(f));
    return r;
}

__device__ __forceinline__ void store_out(void *y, int ydt, int64_t idx, float v)
{
    if (ydt == MCAPQ_F32)
        reinterpret_cast<float *>(y)[idx] = v;
    else
        reinterpret_cast<uint16_t *>(y)[idx] = float_to_bf16_bits(v);
}

}  // namespace dev
}  // namespace mcapq
#endif
