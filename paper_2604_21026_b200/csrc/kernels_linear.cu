// kernels_linear.cu -- the decode linears of the MCAP/NVE hot path on sm_100a.
//
//   w4a8_gemv_dp4a : row a3, W4A8 at M = 1.  One warp
//                    per output row, lane l owns the 32-blocks g = l, l+32, ...
//                    of the row: one coalesced 128-bit nibble load per block,
//                    8 IDP.4A per block, deferred zero-point correction
//                    D = sumi - 8 sum_x, fp32 scale-and-accumulate, a fixed
//                    xor-butterfly warp reduction.
//   tc_linear<A8>  : rows a5 (W4A8, int8 IMMA m16n8k32) and a4/a6 (W4A16, bf16
//                    HMMA m16n8k16 on exact c-8 operands).  Swap-AB: the weight
//                    rows are the MMA's M = 16 side, tokens the N = 8 side.  A
//                    CTA owns a 16-row tile; its 8 warps split K (warp w takes
//                    blocks w, w+8, ...), and a fixed-order smem reduction
//                    combines them.  One MMA k32 (IMMA) / two k16 (HMMA) cover
//                    exactly one Q4_0 block, so the per-block scale is applied
//                    in fp32 right after the MMA (exact int32 D for W4A8,
//                    exact fp32 products for W4A16).
//
// Reduction order of every output depends on K only (never on N, M, the grid or
// the tile position), so column shards are bit-identical to the full matrix
// (reading A22).  All kernels read weights before griddepcontrol.wait so that,
// under programmatic dependent launch, the weight stream overlaps the previous
// kernel's tail; only the activations wait.
#include "internal.h"

namespace mcapq {
namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;

// ------------------------------------------------------------- integer stage
// One 16-byte Q4_0 nibble block against its 32 int8 activations:
// word u holds elements 4u..4u+3 in its low nibbles and 4u+16..4u+19 in its
// high nibbles (split layout), which line up with q words u and 4+u.
__device__ __forceinline__ int block_sumi_dp4a(uint4 w, int4 qa, int4 qb)
{
    int acc = 0;
    acc = __dp4a((int)(w.x & 0x0F0F0F0Fu), qa.x, acc);
    acc = __dp4a((int)((w.x >> 4) & 0x0F0F0F0Fu), qb.x, acc);
    acc = __dp4a((int)(w.y & 0x0F0F0F0Fu), qa.y, acc);
    acc = __dp4a((int)((w.y >> 4) & 0x0F0F0F0Fu), qb.y, acc);
    acc = __dp4a((int)(w.z & 0x0F0F0F0Fu), qa.z, acc);
    acc = __dp4a((int)((w.z >> 4) & 0x0F0F0F0Fu), qb.z, acc);
    acc = __dp4a((int)(w.w & 0x0F0F0F0Fu), qa.w, acc);
    acc = __dp4a((int)((w.w >> 4) & 0x0F0F0F0Fu), qb.w, acc);
    return acc;
}

// int8 tensor-core fragment of one block (m16n8k32, .row.col, s8 x s8 -> s32).
// Thread (gid = lane/4, t = lane%4) supplies word t of its two rows' blocks:
// A reg0/reg2 = row gid, k 4t..4t+3 / 4t+16..4t+19  (low / high nibbles of the word)
// A reg1/reg3 = row gid+8, same k.  B reg0/reg1 = q[token gid][4t..4t+3 | 4t+16..4t+19].
__device__ __forceinline__ void imma_block(uint32_t wa, uint32_t wb, uint32_t b0, uint32_t b1, int c[4])
{
    const uint32_t a0 = wa & 0x0F0F0F0Fu, a2 = (wa >> 4) & 0x0F0F0F0Fu;
    const uint32_t a1 = wb & 0x0F0F0F0Fu, a3 = (wb >> 4) & 0x0F0F0F0Fu;
    c[0] = c[1] = c[2] = c[3] = 0;
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// bf16 fragments of one block with exact c - 8 (m16n8k16 x2).  OR-ing a nibble
// into the mantissa of the bf16 magic 0x4300 (= 128) gives 128 + c exactly; one
// packed FMA (x 1, - 136) maps it to c - 8, exact in bf16.  Element order per
// thread t (the split layout puts element 4t+i in the low nibble of byte i and
// 4t+16+i in its high nibble):
//   p0 = (4t, 4t+2)  p1 = (4t+16, 4t+18)  p2 = (4t+1, 4t+3)  p3 = (4t+17, 4t+19)
// MMA0 uses k-slots {2t,2t+1 <- p0, 2t+8,2t+9 <- p2}; MMA1 the same with p1/p3.
// The activation B fragments are staged in exactly this order.
__device__ __forceinline__ void dequant_word_bf16(uint32_t w, uint32_t p[4])
{
    const uint32_t magic = 0x43004300u;      // bf16x2 (128, 128)
    const uint32_t lo0 = (w & 0x000F000Fu) | magic;
    const uint32_t hi0 = ((w >> 4) & 0x000F000Fu) | magic;
    const uint32_t lo1 = ((w >> 8) & 0x000F000Fu) | magic;
    const uint32_t hi1 = ((w >> 12) & 0x000F000Fu) | magic;
    const uint32_t m136 = 0xC308C308u;       // bf16x2 (-136, -136)
    const uint32_t one = 0x3F803F80u;        // bf16x2 (1, 1)
    asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(p[0]) : "r"(lo0), "r"(one), "r"(m136));
    asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(p[1]) : "r"(hi0), "r"(one), "r"(m136));
    asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(p[2]) : "r"(lo1), "r"(one), "r"(m136));
    asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(p[3]) : "r"(hi1), "r"(one), "r"(m136));
}

__device__ __forceinline__ void hmma16816(const uint32_t a[4], uint32_t b0, uint32_t b1, float c[4])
{
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// ------------------------------------------------------------- M = 1 W4A8
constexpr int kGemvChunk = 8;   // blocks per lane loaded ahead

__global__ void __launch_bounds__(kThreads) w4a8_gemv_dp4a(const uint8_t *__restrict__ nib,
                                                          const uint16_t *__restrict__ scale, int64_t n,
                                                          int64_t k, const int8_t *__restrict__ q,
                                                          const float *__restrict__ sx,
                                                          const int32_t *__restrict__ sq, void *__restrict__ y,
                                                          int ydt)
{
    extern __shared__ __align__(16) uint8_t smem[];
    const int G = (int)(k / 32);
    int8_t *q_s = reinterpret_cast<int8_t *>(smem);                  // [k]
    float *sx_s = reinterpret_cast<float *>(smem + k);                // [G]
    int32_t *sq_s = reinterpret_cast<int32_t *>(smem + k + 4 * G);     // [G]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * kWarps + warp;
    const bool live = row < n;
    const uint8_t *wrow = nib + (live ? row : 0) * (k / 2);
    const uint16_t *srow = scale + (live ? row : 0) * G;

    // prefetch the first chunk of weights (independent of the predecessor)
    uint4 wv[kGemvChunk];
    uint16_t dv[kGemvChunk];
#pragma unroll
    for (int j = 0; j < kGemvChunk; ++j) {
        const int g = lane + 32 * j;
        if (g < G) {
            wv[j] = dev::ld_stream_128(wrow + 16 * g);
            dv[j] = dev::ld_nc_16(srow + g);
        }
    }
    dev::griddep_wait();
    // stage the activation codes, scales and sums of token 0
    for (int i = threadIdx.x; i < (int)(k / 16); i += kThreads)
        reinterpret_cast<int4 *>(q_s)[i] = reinterpret_cast<const int4 *>(q)[i];
    for (int i = threadIdx.x; i < G; i += kThreads) {
        sx_s[i] = sx[i];
        sq_s[i] = sq[i];
    }
    __syncthreads();
    dev::griddep_launch();

    float acc = 0.0f;
    for (int j0 = 0; j0 < (G + 31) / 32; j0 += kGemvChunk) {
        if (j0 > 0) {
#pragma unroll
            for (int j = 0; j < kGemvChunk; ++j) {
                const int g = lane + 32 * (j0 + j);
                if (g < G) {
                    wv[j] = dev::ld_stream_128(wrow + 16 * g);
                    dv[j] = dev::ld_nc_16(srow + g);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < kGemvChunk; ++j) {
            const int g = lane + 32 * (j0 + j);
            if (g < G) {
                const int4 qa = reinterpret_cast<const int4 *>(q_s + 32 * g)[0];
                const int4 qb = reinterpret_cast<const int4 *>(q_s + 32 * g)[1];
                const int D = block_sumi_dp4a(wv[j], qa, qb) - 8 * sq_s[g];   // deferred correction
                const float ds = dev::half_bits_to_float(dv[j]) * sx_s[g];
                acc = fmaf(ds, (float)D, acc);
            }
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (live && lane == 0) dev::store_out(y, ydt, row, acc);
}

// ------------------------------------------------------------- tensor-core path
// Activation staging (shared memory), per pass of up to 8 tokens:
//  A8 : q_s [tok][k + 16] int8 (natural order; +16 B pad breaks bank conflicts),
//       sx_s [tok][G] fp32, sq_s [tok][G] int32
//  A16: x_s [tok][2k + 64] bytes, bf16 permuted per (block, t) into the 8-value
//       order of dequant_word_bf16: (4t,4t+2,4t+1,4t+3,4t+16,4t+18,4t+17,4t+19)
template <bool A8>
__host__ __device__ constexpr int64_t tok_stride(int64_t k)
{
    return A8 ? (k + 16) : (2 * k + 64);
}
template <bool A8>
__host__ __device__ constexpr int64_t act_bytes_per_token(int64_t k)
{
    return A8 ? (k + 16 + 8 * (k / 32)) : (2 * k + 64);
}
constexpr int kRedBytes = kWarps * 16 * 8 * 4;

struct TcArgs {
    const uint8_t *nib;
    const uint16_t *scale;
    int64_t n, k;
    const int8_t *q;      // A8
    const float *sx;      // A8
    const int32_t *sq;    // A8
    const uint16_t *x;    // A16
    int64_t ldx;          // A16
    int64_t m;
    int tokens_per_pass;  // tokens staged per pass (<= 8)
    void *y;
    int ydt;
    int64_t ldy;
};

template <bool A8>
__global__ void __launch_bounds__(kThreads) tc_linear(TcArgs a)
{
    extern __shared__ __align__(16) uint8_t smem[];
    const int64_t k = a.k;
    const int G = (int)(k / 32);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = lane >> 2, t = lane & 3;
    const int64_t row0 = (int64_t)blockIdx.x * 16;
    const int64_t rA = min(row0 + gid, a.n - 1), rB = min(row0 + gid + 8, a.n - 1);
    const uint8_t *wA = a.nib + rA * (k / 2) + 4 * t;
    const uint8_t *wB = a.nib + rB * (k / 2) + 4 * t;
    const uint16_t *sA = a.scale + rA * G;
    const uint16_t *sB = a.scale + rB * G;

    float *red = reinterpret_cast<float *>(smem);                       // [8 warps][16][8]
    uint8_t *act = smem + kRedBytes;

    // prefetch this warp's first blocks before waiting on the predecessor
    constexpr int U = 4;
    uint32_t pwa[U], pwb[U];
    uint16_t pda[U], pdb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int g = warp + kWarps * u;
        if (g < G) {
            pwa[u] = dev::ld_nc_32(wA + 16 * g);
            pwb[u] = dev::ld_nc_32(wB + 16 * g);
            pda[u] = dev::ld_nc_16(sA + g);
            pdb[u] = dev::ld_nc_16(sB + g);
        }
    }
    dev::griddep_wait();

    const int TP = a.tokens_per_pass;
    for (int64_t tok0 = 0; tok0 < a.m; tok0 += TP) {
        const int ntok = (int)((a.m - tok0) < TP ? (a.m - tok0) : TP);
        // ---- stage activations of tokens tok0 .. tok0+ntok-1
        if (tok0 > 0) __syncthreads();
        if constexpr (A8) {
            const int64_t ts = tok_stride<true>(k);
            float *sx_s = reinterpret_cast<float *>(act + TP * ts);
            int32_t *sq_s = reinterpret_cast<int32_t *>(act + TP * ts + 4 * TP * G);
            for (int i = threadIdx.x; i < ntok * (int)(k / 16); i += kThreads) {
                const int tk = i / (int)(k / 16), c = i % (int)(k / 16);
                reinterpret_cast<int4 *>(act + tk * ts)[c] =
                    reinterpret_cast<const int4 *>(a.q + (tok0 + tk) * k)[c];
            }
            for (int i = threadIdx.x; i < ntok * G; i += kThreads) {
                sx_s[i] = a.sx[tok0 * G + i];
                sq_s[i] = a.sq[tok0 * G + i];
            }
        } else {
            const int64_t ts = tok_stride<false>(k);
            // one thread per (token, block, t): 8 bf16 from two 8-byte runs
            for (int i = threadIdx.x; i < ntok * G * 4; i += kThreads) {
                const int tk = i / (G * 4), rem = i % (G * 4), g = rem >> 2, tt = rem & 3;
                const uint16_t *src = a.x + (tok0 + tk) * a.ldx + 32 * g + 4 * tt;
                const uint2 lo = *reinterpret_cast<const uint2 *>(src);        // x[4t..4t+3]
                const uint2 hi = *reinterpret_cast<const uint2 *>(src + 16);   // x[4t+16..4t+19]
                uint4 o;
                o.x = __byte_perm(lo.x, lo.y, 0x5410);   // (4t, 4t+2)
                o.y = __byte_perm(lo.x, lo.y, 0x7632);   // (4t+1, 4t+3)
                o.z = __byte_perm(hi.x, hi.y, 0x5410);   // (4t+16, 4t+18)
                o.w = __byte_perm(hi.x, hi.y, 0x7632);   // (4t+17, 4t+19)
                *reinterpret_cast<uint4 *>(act + tk * ts + 64 * g + 16 * tt) = o;
            }
        }
        __syncthreads();
        if (tok0 == 0) dev::griddep_launch();

        // ---- main loop: this warp's blocks g = warp, warp+8, ...
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        const bool tok_live = gid < ntok;                      // B fragment column gid
        const int tc0 = 2 * t, tc1 = 2 * t + 1;                // C fragment columns
        for (int gb = 0; gb * kWarps + warp < G; gb += U) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int g = warp + kWarps * (gb + u);
                if (g >= G) break;
                uint32_t wa, wb;
                uint16_t da16, db16;
                if (tok0 == 0 && gb == 0) {
                    wa = pwa[u]; wb = pwb[u]; da16 = pda[u]; db16 = pdb[u];
                } else {
                    wa = dev::ld_nc_32(wA + 16 * g);
                    wb = dev::ld_nc_32(wB + 16 * g);
                    da16 = dev::ld_nc_16(sA + g);
                    db16 = dev::ld_nc_16(sB + g);
                }
                const float da = dev::half_bits_to_float(da16), db = dev::half_bits_to_float(db16);
                if constexpr (A8) {
                    const int64_t ts = tok_stride<true>(k);
                    const float *sx_s = reinterpret_cast<const float *>(act + TP * ts);
                    const int32_t *sq_s = reinterpret_cast<const int32_t *>(act + TP * ts + 4 * TP * G);
                    uint32_t b0 = 0, b1 = 0;
                    if (tok_live) {
                        const uint8_t *qp = act + gid * ts + 32 * g + 4 * t;
                        b0 = *reinterpret_cast<const uint32_t *>(qp);
                        b1 = *reinterpret_cast<const uint32_t *>(qp + 16);
                    }
                    int c[4];
                    imma_block(wa, wb, b0, b1, c);
                    const float s0 = tc0 < ntok ? sx_s[tc0 * G + g] : 0.f;
                    const float s1 = tc1 < ntok ? sx_s[tc1 * G + g] : 0.f;
                    const int q0 = tc0 < ntok ? sq_s[tc0 * G + g] : 0;
                    const int q1 = tc1 < ntok ? sq_s[tc1 * G + g] : 0;
                    acc[0] = fmaf(da * s0, (float)(c[0] - 8 * q0), acc[0]);
                    acc[1] = fmaf(da * s1, (float)(c[1] - 8 * q1), acc[1]);
                    acc[2] = fmaf(db * s0, (float)(c[2] - 8 * q0), acc[2]);
                    acc[3] = fmaf(db * s1, (float)(c[3] - 8 * q1), acc[3]);
                } else {
                    const int64_t ts = tok_stride<false>(k);
                    uint4 bx = make_uint4(0, 0, 0, 0);
                    if (tok_live) bx = *reinterpret_cast<const uint4 *>(act + gid * ts + 64 * g + 16 * t);
                    uint32_t pa[4], pb[4];
                    dequant_word_bf16(wa, pa);
                    dequant_word_bf16(wb, pb);
                    const uint32_t A0[4] = {pa[0], pb[0], pa[2], pb[2]};
                    const uint32_t A1[4] = {pa[1], pb[1], pa[3], pb[3]};
                    float c[4] = {0.f, 0.f, 0.f, 0.f};
                    hmma16816(A0, bx.x, bx.y, c);
                    hmma16816(A1, bx.z, bx.w, c);
                    acc[0] = fmaf(da, c[0], acc[0]);
                    acc[1] = fmaf(da, c[1], acc[1]);
                    acc[2] = fmaf(db, c[2], acc[2]);
                    acc[3] = fmaf(db, c[3], acc[3]);
                }
            }
        }
        // ---- fixed-order cross-warp reduction and store
        float *rw = red + warp * 128;
        rw[gid * 8 + tc0] = acc[0];
        rw[gid * 8 + tc1] = acc[1];
        rw[(gid + 8) * 8 + tc0] = acc[2];
        rw[(gid + 8) * 8 + tc1] = acc[3];
        __syncthreads();
        if (threadIdx.x < 128) {
            const int r = threadIdx.x >> 3, tk = threadIdx.x & 7;
            float s = red[threadIdx.x];
#pragma unroll
            for (int w = 1; w < kWarps; ++w) s += red[w * 128 + threadIdx.x];
            const int64_t row = row0 + r;
            if (row < a.n && tk < ntok) dev::store_out(a.y, a.ydt, (tok0 + tk) * a.ldy + row, s);
        }
    }
}

// Test kernel: the integer stage D through either the dp4a block
// routine (mode 0) or the IMMA fragment routine (mode 1).
__global__ void group_dots_kernel(const uint8_t *__restrict__ nib, int64_t n, int64_t k,
                                  const int8_t *__restrict__ q, const int32_t *__restrict__ sq, int64_t m,
                                  int32_t *__restrict__ D, int mode)
{
    const int G = (int)(k / 32);
    const int lane = threadIdx.x & 31;
    if (mode == 0) {
        const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        if (idx >= m * n * G) return;
        const int64_t i = idx / (n * G), r = (idx / G) % n, g = idx % G;
        const uint4 w = *reinterpret_cast<const uint4 *>(nib + r * (k / 2) + 16 * g);
        const int4 qa = *reinterpret_cast<const int4 *>(q + i * k + 32 * g);
        const int4 qb = *reinterpret_cast<const int4 *>(q + i * k + 32 * g + 16);
        D[idx] = block_sumi_dp4a(w, qa, qb) - 8 * sq[i * G + g];
        return;
    }
    // mode 1: one warp per (16-row tile, 8-token tile, block)
    const int64_t tiles_r = (n + 15) / 16, tiles_t = (m + 7) / 8;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (wid >= tiles_r * tiles_t * G) return;
    const int64_t g = wid % G, tt = (wid / G) % tiles_t, tr = wid / (G * tiles_t);
    const int gid = lane >> 2, t = lane & 3;
    const int64_t rA = min(tr * 16 + gid, n - 1), rB = min(tr * 16 + gid + 8, n - 1);
    const uint32_t wa = *reinterpret_cast<const uint32_t *>(nib + rA * (k / 2) + 16 * g + 4 * t);
    const uint32_t wb = *reinterpret_cast<const uint32_t *>(nib + rB * (k / 2) + 16 * g + 4 * t);
    const int64_t tokB = tt * 8 + gid;
    uint32_t b0 = 0, b1 = 0;
    if (tokB < m) {
        b0 = *reinterpret_cast<const uint32_t *>(q + tokB * k + 32 * g + 4 * t);
        b1 = *reinterpret_cast<const uint32_t *>(q + tokB * k + 32 * g + 16 + 4 * t);
    }
    int c[4];
    imma_block(wa, wb, b0, b1, c);
    const int64_t rows[4] = {tr * 16 + gid, tr * 16 + gid, tr * 16 + gid + 8, tr * 16 + gid + 8};
    const int64_t toks[4] = {tt * 8 + 2 * t, tt * 8 + 2 * t + 1, tt * 8 + 2 * t, tt * 8 + 2 * t + 1};
#pragma unroll
    for (int e = 0; e < 4; ++e)
        if (rows[e] < n && toks[e] < m)
            D[(toks[e] * n + rows[e]) * G + g] = c[e] - 8 * sq[toks[e] * G + g];
}

constexpr size_t kMaxSmem = 227 * 1024;

template <bool A8>
int tokens_per_pass(int64_t m, int64_t k)
{
    const int64_t per = act_bytes_per_token<A8>(k);
    int64_t tp = (int64_t)(kMaxSmem - kRedBytes) / per;
    tp = tp > 8 ? 8 : tp;
    tp = tp > m ? m : tp;
    return (int)(tp < 1 ? 1 : tp);
}

template <bool A8>
cudaError_t launch_tc(const TcArgs &a0, cudaStream_t s, bool pdl)
{
    TcArgs a = a0;
    a.tokens_per_pass = tokens_per_pass<A8>(a.m, a.k);
    const size_t smem = kRedBytes + (size_t)a.tokens_per_pass * act_bytes_per_token<A8>(a.k);
    cudaError_t e = kernel_smem_attr(reinterpret_cast<const void *>(tc_linear<A8>), (int)kMaxSmem);
    if (e != cudaSuccess) return e;
    const unsigned grid = (unsigned)((a.n + 15) / 16);
    return launch_pdl(tc_linear<A8>, dim3(grid), dim3(kThreads), smem, s, pdl, a);
}

}  // namespace

cudaError_t launch_w4a8(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k, const int8_t *q,
                        const float *sx, const int32_t *sq, int64_t m, void *y, int ydt, int64_t ldy,
                        cudaStream_t s, bool pdl)
{
    if (m == 1) {
        const size_t smem = (size_t)k + 8 * (size_t)(k / 32);
        cudaError_t e = kernel_smem_attr(reinterpret_cast<const void *>(w4a8_gemv_dp4a), (int)kMaxSmem);
        if (e != cudaSuccess) return e;
        if (smem <= kMaxSmem) {
            const unsigned grid = (unsigned)((n + kWarps - 1) / kWarps);
            return launch_pdl(w4a8_gemv_dp4a, dim3(grid), dim3(kThreads), smem, s, pdl, nib, scale, n, k, q, sx, sq,
                              y, ydt);
        }
    }
    TcArgs a = {};
    a.nib = nib; a.scale = scale; a.n = n; a.k = k;
    a.q = q; a.sx = sx; a.sq = sq; a.m = m; a.y = y; a.ydt = ydt; a.ldy = ldy;
    return launch_tc<true>(a, s, pdl);
}

cudaError_t launch_w4a16(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k, const uint16_t *x,
                         int64_t m, int64_t ldx, void *y, int ydt, int64_t ldy, cudaStream_t s, bool pdl)
{
    TcArgs a = {};
    a.nib = nib; a.scale = scale; a.n = n; a.k = k;
    a.x = x; a.ldx = ldx; a.m = m; a.y = y; a.ydt = ydt; a.ldy = ldy;
    return launch_tc<false>(a, s, pdl);
}

cudaError_t launch_w4a8_group_dots(const uint8_t *nib, int64_t n, int64_t k, const int8_t *q, const int32_t *sq,
                                   int64_t m, int32_t *D, int mode, cudaStream_t s)
{
    const int64_t G = k / 32;
    int64_t threads = mode == 0 ? m * n * G : ((n + 15) / 16) * ((m + 7) / 8) * G * 32;
    const int64_t grid = (threads + 255) / 256;
    if (grid == 0) return cudaSuccess;
    group_dots_kernel<<<(unsigned)grid, 256, 0, s>>>(nib, n, k, q, sq, m, D, mode);
    return cudaGetLastError();
}

int kernels_per_linear(int route, int64_t m)
{
    (void)m;
    return route == MCAPQ_W4A8 ? 2 : 1;
}

}  // namespace mcapq
