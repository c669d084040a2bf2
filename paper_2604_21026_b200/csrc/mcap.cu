// mcap.cu -- the MCAP activation profiler on the GPU (Alg. 1,
// sec:mcap P:533-559): the per-layer importance score that the routing table (row a7)
// consumes, computed from the outputs the layer's linears already produce.
//
//   a_t^attn = || [Q x_t, V x_t] ||_2         (Alg. 1 line 5, the attention proxy)
//   a_t^ffn  = || FFN(x_t) ||_2               (line 6, the FFN magnitude)
//   s_i     += weight * sum_t (a_t^attn + a_t^ffn)     (line 10, weight = 1 / (k |p_j|))
//
// Two launches per call: one CTA per token computes a_t in fp64 (bf16 inputs are exact in
// fp32; squares summed per thread in fp64, a fixed tree over the CTA), then one CTA adds the
// weighted token sum in a fixed order -- the score is deterministic for a given M and
// shape (no atomics).  Normalisation, the degenerate branch and tau stay on the host
// (profile.cpp, Alg. 1 lines 11-17), fed by the profile JSON mcapq_profile_write_json emits.
#include <cuda_bf16.h>

#include <cmath>

#include "internal.h"

namespace mcapq {
namespace {

constexpr int kMcapThreads = 256;

__device__ __forceinline__ double sumsq_row(const uint16_t *y, int64_t n)
{
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += kMcapThreads) {
        const double v = (double)__uint_as_float((uint32_t)y[i] << 16);
        acc = fma(v, v, acc);
    }
    return acc;
}

// fixed-order CTA sum (warp butterfly, then warp 0 over the 8 warp totals)
__device__ __forceinline__ double cta_sum(double v, double *red)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double t = 0.0;
    if (warp == 0) {
        t = lane < kMcapThreads / 32 ? red[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    return t;   // valid in thread 0
}

__global__ void __launch_bounds__(kMcapThreads) mcap_token_kernel(const uint16_t *yq, int64_t ldq, int64_t nq,
                                                                const uint16_t *yv, int64_t ldv, int64_t nv,
                                                                const uint16_t *yf, int64_t ldf, int64_t nf,
                                                                double *tok)
{
    __shared__ double red[kMcapThreads / 32];
    const int64_t t = blockIdx.x;
    // || [Q x_t, V x_t] ||^2 = ||Q x_t||^2 + ||V x_t||^2
    const double attn = cta_sum(sumsq_row(yq + t * ldq, nq) + sumsq_row(yv + t * ldv, nv), red);
    const double ffn = cta_sum(sumsq_row(yf + t * ldf, nf), red);
    if (threadIdx.x == 0) tok[t] = sqrt(attn) + sqrt(ffn);
}

__global__ void __launch_bounds__(kMcapThreads) mcap_accumulate_kernel(const double *tok, int64_t m, double weight,
                                                                     double *score)
{
    __shared__ double red[kMcapThreads / 32];
    double acc = 0.0;
    for (int64_t t = threadIdx.x; t < m; t += kMcapThreads) acc += tok[t];
    const double s = cta_sum(acc, red);
    if (threadIdx.x == 0) *score += weight * s;
}

}  // namespace
}  // namespace mcapq

using namespace mcapq;

extern "C" {

size_t mcapq_mcap_workspace_bytes(int64_t m) { return m > 0 ? (size_t)m * sizeof(double) : 0; }

mcapq_status mcapq_mcap_accumulate(const uint16_t *yq, int64_t ldq, int64_t nq, const uint16_t *yv, int64_t ldv,
                                   int64_t nv, const uint16_t *yffn, int64_t ldf, int64_t nf, int64_t m,
                                   double weight, double *score, void *ws, size_t ws_bytes, void *stream)
{
    clear_error();
    MCAPQ_REQUIRE(yq && yv && yffn && score && ws, MCAPQ_EINVAL, "NULL pointer");
    MCAPQ_REQUIRE(m >= 1 && nq >= 1 && nv >= 1 && nf >= 1, MCAPQ_EINVAL, "bad shape m=%lld nq=%lld nv=%lld nf=%lld",
                  (long long)m, (long long)nq, (long long)nv, (long long)nf);
    MCAPQ_REQUIRE(ldq >= nq && ldv >= nv && ldf >= nf, MCAPQ_EINVAL, "leading dimension below the row length");
    MCAPQ_REQUIRE(m <= 0x7fffffff, MCAPQ_EINVAL, "m too large");
    MCAPQ_REQUIRE(ws_bytes >= mcapq_mcap_workspace_bytes(m), MCAPQ_ENOSPACE, "workspace %zu < %zu bytes", ws_bytes,
                  mcapq_mcap_workspace_bytes(m));
    MCAPQ_REQUIRE(std::isfinite(weight), MCAPQ_EINVAL, "weight is not finite");
    MCAPQ_REQUIRE((reinterpret_cast<uintptr_t>(ws) & 7u) == 0 && (reinterpret_cast<uintptr_t>(score) & 7u) == 0,
                  MCAPQ_EINVAL, "ws / score not 8-byte aligned");
    double *tok = reinterpret_cast<double *>(ws);
    cudaStream_t s = as_stream(stream);
    mcap_token_kernel<<<(unsigned)m, kMcapThreads, 0, s>>>(yq, ldq, nq, yv, ldv, nv, yffn, ldf, nf, tok);
    MCAPQ_CUDA_TRY(cudaGetLastError());
    mcap_accumulate_kernel<<<1, kMcapThreads, 0, s>>>(tok, m, weight, score);
    MCAPQ_CUDA_TRY(cudaGetLastError());
    return MCAPQ_OK;
}

}  // extern "C"
