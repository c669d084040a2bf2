// diag.cu -- measurement probe (not on the hot path): the pure-read ceiling of HBM
// (SURVEY 8(d) D.2 denominator (iii)): a streaming LDG.128 read of a large buffer with
// L1 no-allocate and L2 evict-first, one CTA of 512 threads per SM x 4, each thread
// XOR-folding what it reads so the loads cannot be elided.
#include "internal.h"

namespace mcapq {
namespace {

__global__ void __launch_bounds__(512) read_bw_kernel(const uint4 *__restrict__ p, size_t n16, unsigned long long *sink)
{
    uint32_t acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    // four independent loads in flight per thread per iteration
    for (; i + 3 * stride < n16; i += 4 * stride) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                         : "l"(p + i + u * stride));
#pragma unroll
        for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    for (; i < n16; i += stride) {
        uint4 v;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(p + i));
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x9e3779b9u) *sink = acc;   // practically never: keeps the loads live
}

}  // namespace
}  // namespace mcapq

extern "C" mcapq_status mcapq_debug_read_bw(const void *buf, size_t bytes, unsigned long long *sink, void *stream)
{
    using namespace mcapq;
    clear_error();
    MCAPQ_REQUIRE(buf && sink && aligned16(buf) && bytes >= 16, MCAPQ_EINVAL, "bad read_bw arguments");
    read_bw_kernel<<<4 * device_sms(), 512, 0, as_stream(stream)>>>(reinterpret_cast<const uint4 *>(buf), bytes / 16, sink);
    MCAPQ_CUDA_TRY(cudaGetLastError());
    return MCAPQ_OK;
}
