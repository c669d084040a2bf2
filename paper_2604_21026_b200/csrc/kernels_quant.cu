// kernels_quant.cu -- load-time Q4_0 weight pack (row a1) and the per-token
// int8 activation quantiser (row a2) for sm_100a.
//
// Both are bit-exact with the CPU oracle: the same IEEE operations in the same
// order (IEEE division __fdiv_rn, roundf = half away from zero, cvt.rn.f16.f32),
// built without fast-math / FTZ.  Max reductions are exact in any order; the
// first-index tie-break of a1 is kept by a (|x| bits, 31 - j) key.
#include <cuda_fp16.h>

#include "internal.h"

namespace mcapq {
namespace {

__device__ __forceinline__ uint16_t f32_to_f16_bits(float f)
{
    uint16_t h;
    asm("cvt.rn.f16.f32 %0, %1;" : "=h"(h) : "f"(f));
    return h;
}

// a1 (readings A2-A5, A21).  One warp per 32-block,
// lane j owns element j: this keeps the ±a tie-break and every IEEE step
// identical to the serial definition while reading the block coalesced.
template <typename T>
__global__ void __launch_bounds__(256) pack_w4_kernel(const T *__restrict__ w, int64_t n, int64_t k, int64_t ldw,
                                                      uint8_t *__restrict__ nib, uint16_t *__restrict__ scale,
                                                      uint32_t *__restrict__ dev_err)
{
    const int lane = threadIdx.x & 31;
    const int64_t G = k / 32;
    const int64_t blk = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (blk >= n * G) return;
    const int64_t r = blk / G, g = blk % G;

    float x;
    if constexpr (sizeof(T) == 2)
        x = dev::bf16_bits_to_float(reinterpret_cast<const uint16_t *>(w)[r * ldw + g * 32 + lane]);
    else
        x = reinterpret_cast<const float *>(w)[r * ldw + g * 32 + lane];

    const bool finite = __all_sync(0xffffffffu, isfinite(x));
    // 1. m = x[argmax |x_j|], first index on ties: maximise (|x| bits, 31 - j).
    const uint32_t abits = __float_as_uint(fabsf(x));
    const uint64_t key = ((uint64_t)abits << 32) | (uint32_t)(31 - lane);
    uint64_t best = key;
    for (int off = 16; off > 0; off >>= 1) {
        const uint64_t o = __shfl_xor_sync(0xffffffffu, best, off);
        best = o > best ? o : best;
    }
    const int src = 31 - (int)(best & 0xffffffffu);
    const float m = __shfl_sync(0xffffffffu, x, src);

    uint16_t d16;
    int code;
    uint32_t err = 0;
    if (!finite) {                       // S:287 -> flag, store a zero block
        d16 = 0;
        code = 8;
        err = MCAPQ_PACK_NONFINITE;
    } else {
        // 2. d = fp16_rne(m / -8)
        d16 = f32_to_f16_bits(__fdiv_rn(m, -8.0f));
        if ((d16 & 0x7fffu) == 0x7c00u) {   // fp16 overflow (A4)
            code = 8;
            err = MCAPQ_PACK_OVERFLOW;
        } else {
            const float d = dev::half_bits_to_float(d16);
            if (d == 0.0f) {                  // zero block (also d underflow): +0, codes 8 (A21)
                d16 = 0;
                code = 8;
            } else {
                // 3. c = clamp(round_half_away(x / f32(d)), -8, 7) + 8
                float q = roundf(__fdiv_rn(x, d));
                q = fminf(fmaxf(q, -8.0f), 7.0f);
                code = (int)q + 8;
            }
        }
    }
    // 5. split layout: byte t = c_t | c_{t+16} << 4
    const int hi = __shfl_down_sync(0xffffffffu, code, 16);
    if (lane < 16) nib[r * (k / 2) + g * 16 + lane] = (uint8_t)(code | (hi << 4));
    if (lane == 0) {
        scale[r * G + g] = d16;
        if (err && dev_err) atomicOr(dev_err, err);
    }
}

// a2 (readings A6-A8, A21).  One warp per (token, 32-group),
// lane j owns element j; amax is an exact max, sum q an exact int sum.
__global__ void __launch_bounds__(256) quant_a8_kernel(const uint16_t *__restrict__ x, int64_t m, int64_t k,
                                                       int64_t ldx, int8_t *__restrict__ q,
                                                       float *__restrict__ sx, int32_t *__restrict__ sq)
{
    dev::griddep_launch();   // let the consuming GEMV start streaming weights now
    dev::griddep_wait();     // x may be written by the previous kernel
    const int lane = threadIdx.x & 31;
    const int64_t G = k / 32;
    const int64_t grp = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (grp >= m * G) return;
    const int64_t i = grp / G, g = grp % G;
    const float v = dev::bf16_bits_to_float(x[i * ldx + g * 32 + lane]);
    const bool finite = __all_sync(0xffffffffu, isfinite(v));
    // (1) amax: max over |x| bit patterns (monotone for non-negative floats)
    const float amax = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(fabsf(v))));
    // (2) s = amax / 127
    const float s = __fdiv_rn(amax, 127.0f);
    int code = 0;
    const bool live = finite && s != 0.0f;
    if (live) {
        // (3) q = clamp(round(x / s), -127, 127)
        float r = roundf(__fdiv_rn(v, s));
        r = fminf(fmaxf(r, -127.0f), 127.0f);
        code = (int)r;
    }
    q[i * k + g * 32 + lane] = (int8_t)code;
    const int sum = __reduce_add_sync(0xffffffffu, code);
    if (lane == 0) {
        sx[i * G + g] = live ? s : 0.0f;
        sq[i * G + g] = sum;
    }
}

}  // namespace

cudaError_t launch_pack_w4(const void *w, int wdt, int64_t n, int64_t k, int64_t ldw, uint8_t *nib,
                           uint16_t *scale, uint32_t *dev_err, cudaStream_t s)
{
    const int64_t blocks = n * (k / 32);
    const int64_t grid = (blocks + 7) / 8;
    if (grid == 0) return cudaSuccess;
    if (wdt == MCAPQ_BF16)
        pack_w4_kernel<uint16_t><<<(unsigned)grid, 256, 0, s>>>((const uint16_t *)w, n, k, ldw, nib, scale, dev_err);
    else
        pack_w4_kernel<float><<<(unsigned)grid, 256, 0, s>>>((const float *)w, n, k, ldw, nib, scale, dev_err);
    return cudaGetLastError();
}

cudaError_t launch_quant_a8(const uint16_t *x, int64_t m, int64_t k, int64_t ldx, int8_t *q, float *sx,
                            int32_t *sq, cudaStream_t s, bool pdl)
{
    const int64_t groups = m * (k / 32);
    const int64_t grid = (groups + 7) / 8;
    if (grid == 0) return cudaSuccess;
    return launch_pdl(quant_a8_kernel, dim3((unsigned)grid), dim3(256), 0, s, pdl, x, m, k, ldx, q, sx, sq);
}

}  // namespace mcapq
