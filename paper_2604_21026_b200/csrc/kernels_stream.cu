// kernels_stream.cu -- persistent, TMA-bulk-fed decode linears for sm_100a
// (rows a3-a6 at M <= 8 tokens per pass; the "stream" path).
//
// One CTA per SM (grid <= #SMs), warp-specialised:
//   warp 8 (producer, one elected lane): walks the CTA's work items (16-row
//     tile x 1 KiB K-chunk) and moves each into a shared-memory ring with
//     cp.async.bulk (the 1-D TMA engine, SASS UBLKCP) -- 16 row copies of the
//     nibble chunk + 16 row copies of its fp16 scales, completion counted on the
//     stage's mbarrier (complete_tx).  It reads only weights, so it never waits
//     on the predecessor kernel: under programmatic dependent launch the weight
//     stream of linear i+1 starts while linear i drains.
//   warps 0-7 (consumers): griddepcontrol.wait, then stage this pass's
//     activations in shared memory -- for W4A8 they QUANTISE x themselves (the
//     same warp-per-group code as quant_a8_kernel, so q/s/sum_q are bit-identical;
//     no separate launch), for W4A16 they stage x in MMA-fragment order -- and
//     then consume the ring.
// Engines (one template parameter):
//   DP4A : W4A8, 1 token.  warp w owns rows 2w, 2w+1 of the tile, lane l the
//          blocks l, l+32 of the chunk: LDS.128 nibbles, 8 IDP.4A per block,
//          deferred correction D = sumi - 8 sum_x, fp32 (d s) D.
//   IMMA : W4A8, 2..8 tokens.  warp w owns blocks w, w+8, .. of the chunk for all
//          16 rows: ldmatrix.x4 hands each lane (gid, t) word t of rows gid /
//          gid+8 of two blocks -- exactly the m16n8k32 s8 A fragment of the split
//          nibble layout -- one mma.sync per block (exact int32 D per block).
//   HMMA : W4A16, 1..8 tokens.  Same fragments; nibbles -> exact bf16 (c - 8)
//          (magic 0x4300 + packed FMA), two m16n8k16 bf16 MMAs per block, fp32
//          per-block scale (exact products, fp32 accumulation).
// Work: a "group" of up to 4 linears sharing the same input x (fused QKV,
// fused gate/up; P:977 nve_qkv_matvec_w4a16) -- their 16-row tiles are numbered
// consecutively and split into contiguous, balanced ranges per CTA.
// Determinism: chunk size and the block->lane/warp maps depend on K only, the
// cross-lane/cross-warp reductions have a fixed order: every output row is
// bit-identical whatever N, the group, the grid or the shard (reading A22).
#include "internal.h"
#include "stream.h"

namespace mcapq {
namespace {

constexpr int kConsumerWarps = 8;
constexpr int kThreads = (kConsumerWarps + 1) * 32;
constexpr int kTileRows = 16;
constexpr int kChunkBytes = 1024;              // nibble bytes per row per stage (2048 weights)
constexpr int kNibStride = kChunkBytes + 16;    // padded smem row: ldmatrix rows hit distinct banks
constexpr int kScaleStride = 144;               // 64 fp16 scales + pad (16-B multiple, 4-bank skew)
constexpr int kStageBytes = kTileRows * (kNibStride + kScaleStride);
constexpr int kRedBytes = kConsumerWarps * kTileRows * 8 * 4;

enum Engine { DP4A = 0, IMMA = 1, HMMA = 2 };

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                         uint64_t policy)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void ldmatrix_x4(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3)
{
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ float h2f(uint16_t h)
{
    float f;
    asm("cvt.f32.f16 %0, %1;" : "=f"(f) : "h"(h));
    return f;
}

// ------------------------------------------------------------------ fragments
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

__device__ __forceinline__ void imma(uint32_t wa, uint32_t wb, uint32_t b0, uint32_t b1, int c[4])
{
    const uint32_t a0 = wa & 0x0F0F0F0Fu, a2 = (wa >> 4) & 0x0F0F0F0Fu;
    const uint32_t a1 = wb & 0x0F0F0F0Fu, a3 = (wb >> 4) & 0x0F0F0F0Fu;
    c[0] = c[1] = c[2] = c[3] = 0;
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void dequant_bf16(uint32_t w, uint32_t p[4])
{
    const uint32_t magic = 0x43004300u;   // bf16x2 (128, 128); 128 + c is exact for c < 16
    const uint32_t lo0 = (w & 0x000F000Fu) | magic;           // elements (4t, 4t+2)
    const uint32_t hi0 = ((w >> 4) & 0x000F000Fu) | magic;    // (4t+16, 4t+18)
    const uint32_t lo1 = ((w >> 8) & 0x000F000Fu) | magic;    // (4t+1, 4t+3)
    const uint32_t hi1 = ((w >> 12) & 0x000F000Fu) | magic;   // (4t+17, 4t+19)
    const uint32_t m136 = 0xC308C308u, one = 0x3F803F80u;     // -136, 1
    asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(p[0]) : "r"(lo0), "r"(one), "r"(m136));
    asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(p[1]) : "r"(hi0), "r"(one), "r"(m136));
    asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(p[2]) : "r"(lo1), "r"(one), "r"(m136));
    asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(p[3]) : "r"(hi1), "r"(one), "r"(m136));
}

__device__ __forceinline__ void hmma(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1,
                                     float c[4])
{
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// ------------------------------------------------------------------ the kernel
struct Smem {
    // layout (dynamic shared memory, 128-B aligned pieces)
    uint8_t *ring;          // stages x kStageBytes
    uint64_t *full, *empty; // stages each
    uint8_t *act;           // activations of this pass
    float *red;             // kRedBytes
};

__device__ __forceinline__ int linear_of_tile(const StreamArgs &a, int tile)
{
    int l = 0;
#pragma unroll
    for (int i = 1; i < kMaxGroup; ++i)
        if (i < a.count && tile >= a.tile_start[i]) l = i;
    return l;
}

template <int E>
__global__ void __launch_bounds__(kThreads, 1) stream_linear(const StreamArgs a)
{
    extern __shared__ __align__(128) uint8_t smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t k = a.k;
    const int G = (int)(k / 32);
    const int nchunks = (int)((k / 2 + kChunkBytes - 1) / kChunkBytes);
    const int S = a.stages;

    uint8_t *ring = smem_raw;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem_raw + (size_t)S * kStageBytes);
    uint64_t *empty = full + S;
    uint8_t *act = reinterpret_cast<uint8_t *>(empty + S) + 0;
    act = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(act) + 127) & ~(uintptr_t)127);
    float *red = reinterpret_cast<float *>(act + a.act_bytes);

    // this CTA's contiguous tile range
    const int T = a.tile_start[a.count];
    const int t0 = (int)(((int64_t)T * blockIdx.x) / gridDim.x);
    const int t1 = (int)(((int64_t)T * (blockIdx.x + 1)) / gridDim.x);
    const int items = (t1 - t0) * nchunks;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    dev::griddep_launch();   // the next linear may launch now; it only touches weights until its own wait

    if (warp == kConsumerWarps) {
        // ================= producer =================
        if (lane == 0) {
            const uint64_t pol = evict_first_policy();
            for (int it = 0; it < items; ++it) {
                const int s = it % S;
                const uint32_t ph = (uint32_t)(it / S) & 1u;
                mbar_wait(&empty[s], ph ^ 1u);
                const int tile = t0 + it / nchunks, ch = it % nchunks;
                const int li = linear_of_tile(a, tile);
                const int64_t row0 = (int64_t)(tile - a.tile_start[li]) * kTileRows;
                const int rows = (int)imin64(kTileRows, a.n[li] - row0);
                const int64_t off = (int64_t)ch * kChunkBytes;
                const uint32_t cb = (uint32_t)imin64(kChunkBytes, k / 2 - off);
                const uint32_t sb = cb / 8;   // fp16 scale bytes: cb/16 blocks x 2 B
                uint8_t *st = ring + (size_t)s * kStageBytes;
                mbar_expect_tx(&full[s], (uint32_t)rows * (cb + sb));
                const uint8_t *nsrc = a.nib[li] + row0 * (k / 2) + off;
                const uint8_t *ssrc = reinterpret_cast<const uint8_t *>(a.scale[li]) + row0 * (k / 16) + off / 8;
                for (int r = 0; r < rows; ++r) {
                    bulk_g2s(st + r * kNibStride, nsrc + r * (k / 2), cb, &full[s], pol);
                    bulk_g2s(st + kTileRows * kNibStride + r * kScaleStride, ssrc + r * (k / 16), sb, &full[s], pol);
                }
            }
        }
        return;
    }

    // ================= consumers: stage activations =================
    dev::griddep_wait();
    const int ntok = a.ntok;
    if constexpr (E == DP4A || E == IMMA) {
        // fused per-token, per-32-group quantisation (identical arithmetic to quant_a8_kernel)
        const int64_t qs = k + 16;
        int8_t *q_s = reinterpret_cast<int8_t *>(act);
        float *sx_s = reinterpret_cast<float *>(act + a.ntok_cap * qs);
        int32_t *sq_s = reinterpret_cast<int32_t *>(act + a.ntok_cap * qs + 4 * a.ntok_cap * G);
        // 4 groups per warp in flight (independent chains), lane j = element j of a group
        for (int base = warp; base < ntok * G; base += 4 * kConsumerWarps) {
            float v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int grp = base + u * kConsumerWarps;
                v[u] = 0.f;
                if (grp < ntok * G) {
                    const int i = grp / G, g = grp % G;
                    v[u] = dev::bf16_bits_to_float(a.x[(a.tok0 + i) * a.ldx + 32 * g + lane]);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int grp = base + u * kConsumerWarps;
                if (grp >= ntok * G) break;
                const int i = grp / G, g = grp % G;
                const bool finite = __all_sync(0xffffffffu, isfinite(v[u]));
                const float amax = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(fabsf(v[u]))));
                const float s = __fdiv_rn(amax, 127.0f);
                int code = 0;
                const bool live = finite && s != 0.0f;
                if (live) {
                    float r = roundf(__fdiv_rn(v[u], s));
                    r = fminf(fmaxf(r, -127.0f), 127.0f);
                    code = (int)r;
                }
                q_s[i * qs + 32 * g + lane] = (int8_t)code;
                const int sum = __reduce_add_sync(0xffffffffu, code);
                if (lane == 0) {
                    sx_s[i * G + g] = live ? s : 0.0f;
                    sq_s[i * G + g] = sum;
                }
            }
        }
    } else {
        // x in fragment order per (token, block, t): (4t,4t+2) (4t+1,4t+3) (4t+16,4t+18) (4t+17,4t+19)
        const int64_t xs = 2 * k + 64;
        for (int idx = threadIdx.x; idx < ntok * G * 4; idx += kConsumerWarps * 32) {
            const int tk = idx / (G * 4), rem = idx % (G * 4), g = rem >> 2, tt = rem & 3;
            const uint16_t *src = a.x + (a.tok0 + tk) * a.ldx + 32 * g + 4 * tt;
            const uint2 lo = *reinterpret_cast<const uint2 *>(src);
            const uint2 hi = *reinterpret_cast<const uint2 *>(src + 16);
            uint4 o;
            o.x = __byte_perm(lo.x, lo.y, 0x5410);
            o.y = __byte_perm(lo.x, lo.y, 0x7632);
            o.z = __byte_perm(hi.x, hi.y, 0x5410);
            o.w = __byte_perm(hi.x, hi.y, 0x7632);
            *reinterpret_cast<uint4 *>(act + tk * xs + 64 * g + 16 * tt) = o;
        }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");   // consumers only

    // ================= consumers: main loop =================
    const int gid = lane >> 2, t = lane & 3;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int it = 0; it < items; ++it) {
        const int s = it % S;
        const uint32_t ph = (uint32_t)(it / S) & 1u;
        const int tile = t0 + it / nchunks, ch = it % nchunks;
        const int nblk = (int)(imin64(kChunkBytes, k / 2 - (int64_t)ch * kChunkBytes) / 16);
        const int blk0 = ch * (kChunkBytes / 16);   // first block of the chunk within the row
        if (ch == 0) acc[0] = acc[1] = acc[2] = acc[3] = 0.f;
        mbar_wait(&full[s], ph);
        const uint8_t *st = ring + (size_t)s * kStageBytes;
        const uint8_t *sc = st + kTileRows * kNibStride;

        if constexpr (E == DP4A) {
            const int8_t *q_s = reinterpret_cast<const int8_t *>(act);
            const float *sx_s = reinterpret_cast<const float *>(act + a.ntok_cap * (k + 16));
            const int32_t *sq_s = reinterpret_cast<const int32_t *>(act + a.ntok_cap * (k + 16) + 4 * a.ntok_cap * G);
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
                const int r = 2 * warp + rr;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int b = lane + 32 * h;
                    if (b < nblk) {
                        const uint4 w = *reinterpret_cast<const uint4 *>(st + r * kNibStride + 16 * b);
                        const uint16_t d16 = *reinterpret_cast<const uint16_t *>(sc + r * kScaleStride + 2 * b);
                        const int g = blk0 + b;
                        const int4 qa = *reinterpret_cast<const int4 *>(q_s + 32 * g);
                        const int4 qb = *reinterpret_cast<const int4 *>(q_s + 32 * g + 16);
                        const int D = block_sumi_dp4a(w, qa, qb) - 8 * sq_s[g];
                        acc[rr] = fmaf(h2f(d16) * sx_s[g], (float)D, acc[rr]);
                    }
                }
            }
        } else {
            // warp w: blocks w, w+8, ... of the chunk, two per ldmatrix.x4
            const uint32_t st_a = smem_addr(st);
            for (int b = warp; b < nblk; b += 2 * kConsumerWarps) {
                const int b2 = b + kConsumerWarps;
                const bool two = b2 < nblk;
                // lanes 0-7: rows 0-7 @ b, 8-15: rows 8-15 @ b, 16-23: rows 0-7 @ b2, 24-31: rows 8-15 @ b2
                const int mrow = (lane & 7) + ((lane >> 3) & 1) * 8;
                const int mblk = (lane >> 4) ? (two ? b2 : b) : b;
                uint32_t wa0, wb0, wa1, wb1;
                ldmatrix_x4(st_a + mrow * kNibStride + 16 * mblk, wa0, wb0, wa1, wb1);
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    if (u == 1 && !two) break;
                    const int bb = u ? b2 : b;
                    const uint32_t wa = u ? wa1 : wa0, wb = u ? wb1 : wb0;
                    const float da = h2f(*reinterpret_cast<const uint16_t *>(sc + gid * kScaleStride + 2 * bb));
                    const float db = h2f(*reinterpret_cast<const uint16_t *>(sc + (gid + 8) * kScaleStride + 2 * bb));
                    const int g = blk0 + bb;
                    if constexpr (E == IMMA) {
                        const int64_t qs = k + 16;
                        const int8_t *q_s = reinterpret_cast<const int8_t *>(act);
                        const float *sx_s = reinterpret_cast<const float *>(act + a.ntok_cap * qs);
                        const int32_t *sq_s =
                            reinterpret_cast<const int32_t *>(act + a.ntok_cap * qs + 4 * a.ntok_cap * G);
                        uint32_t b0 = 0, b1 = 0;
                        if (gid < ntok) {
                            b0 = *reinterpret_cast<const uint32_t *>(q_s + gid * qs + 32 * g + 4 * t);
                            b1 = *reinterpret_cast<const uint32_t *>(q_s + gid * qs + 32 * g + 16 + 4 * t);
                        }
                        int c[4];
                        imma(wa, wb, b0, b1, c);
                        const int c0 = 2 * t, c1 = 2 * t + 1;
                        const float s0 = c0 < ntok ? sx_s[c0 * G + g] : 0.f;
                        const float s1 = c1 < ntok ? sx_s[c1 * G + g] : 0.f;
                        const int q0 = c0 < ntok ? sq_s[c0 * G + g] : 0;
                        const int q1 = c1 < ntok ? sq_s[c1 * G + g] : 0;
                        acc[0] = fmaf(da * s0, (float)(c[0] - 8 * q0), acc[0]);
                        acc[1] = fmaf(da * s1, (float)(c[1] - 8 * q1), acc[1]);
                        acc[2] = fmaf(db * s0, (float)(c[2] - 8 * q0), acc[2]);
                        acc[3] = fmaf(db * s1, (float)(c[3] - 8 * q1), acc[3]);
                    } else {
                        uint4 bx = make_uint4(0, 0, 0, 0);
                        if (gid < ntok) bx = *reinterpret_cast<const uint4 *>(act + gid * (2 * k + 64) + 64 * g + 16 * t);
                        uint32_t pa[4], pb[4];
                        dequant_bf16(wa, pa);
                        dequant_bf16(wb, pb);
                        float c[4] = {0.f, 0.f, 0.f, 0.f};
                        hmma(pa[0], pb[0], pa[2], pb[2], bx.x, bx.y, c);
                        hmma(pa[1], pb[1], pa[3], pb[3], bx.z, bx.w, c);
                        acc[0] = fmaf(da, c[0], acc[0]);
                        acc[1] = fmaf(da, c[1], acc[1]);
                        acc[2] = fmaf(db, c[2], acc[2]);
                        acc[3] = fmaf(db, c[3], acc[3]);
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);

        if (ch == nchunks - 1) {
            // ---- tile epilogue: fixed-order reductions, store
            const int li = linear_of_tile(a, tile);
            const int64_t row0 = (int64_t)(tile - a.tile_start[li]) * kTileRows;
            const int64_t n = a.n[li];
            if constexpr (E == DP4A) {
#pragma unroll
                for (int rr = 0; rr < 2; ++rr)
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) acc[rr] += __shfl_xor_sync(0xffffffffu, acc[rr], off);
                if (lane < 2) {
                    const int64_t row = row0 + 2 * warp + lane;
                    if (row < n) dev::store_out(a.y[li], a.ydt, a.tok0 * a.ldy[li] + row, lane ? acc[1] : acc[0]);
                }
            } else {
                float *rw = red + warp * 128;
                const int c0 = 2 * t, c1 = 2 * t + 1;
                rw[gid * 8 + c0] = acc[0];
                rw[gid * 8 + c1] = acc[1];
                rw[(gid + 8) * 8 + c0] = acc[2];
                rw[(gid + 8) * 8 + c1] = acc[3];
                asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
                if (threadIdx.x < 128) {
                    const int r = threadIdx.x >> 3, tk = threadIdx.x & 7;
                    float sum = red[threadIdx.x];
#pragma unroll
                    for (int w = 1; w < kConsumerWarps; ++w) sum += red[w * 128 + threadIdx.x];
                    const int64_t row = row0 + r;
                    if (row < n && tk < ntok) dev::store_out(a.y[li], a.ydt, (a.tok0 + tk) * a.ldy[li] + row, sum);
                }
                asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
            }
        }
    }
}

}  // namespace

// activation bytes of one pass of `ntok` tokens
static size_t act_bytes(int engine, int64_t k, int ntok)
{
    const int64_t G = k / 32;
    if (engine == HMMA) return (size_t)ntok * (size_t)(2 * k + 64);
    return (size_t)ntok * (size_t)(k + 16) + (size_t)ntok * 8 * (size_t)G;
}

bool stream_supported(int64_t k) { return k >= 256 && k % 256 == 0; }

int stream_tokens_per_pass(int route, int64_t k)
{
    // keep activations + 3 ring stages within ~110 KB so two CTAs (this linear and the
    // next, PDL-overlapped) can share an SM
    const int engine = route == MCAPQ_W4A16 ? HMMA : IMMA;
    const size_t budget = 110 * 1024 - 3 * (size_t)kStageBytes - kRedBytes - 256;
    int tp = 8;
    while (tp > 1 && act_bytes(engine, k, tp) > budget) --tp;
    return tp;
}

template <int E>
static cudaError_t launch_one(StreamArgs a, cudaStream_t s, bool pdl, int sms)
{
    const size_t ab = (act_bytes(E, a.k, a.ntok_cap) + 127) & ~(size_t)127;
    a.act_bytes = (int)ab;
    // stages: as many as fit in ~110 KB (>= 2)
    const size_t fixed = ab + kRedBytes + 256;
    int S = (int)((110 * 1024 - (long)fixed) / (kStageBytes + 16));
    S = S < 2 ? 2 : (S > 6 ? 6 : S);
    a.stages = S;
    const size_t smem = (size_t)S * kStageBytes + 16 * (size_t)S + 128 + fixed;
    static int attr_done[3] = {0, 0, 0};
    if (!attr_done[E]) {
        cudaError_t e = cudaFuncSetAttribute(stream_linear<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        attr_done[E] = 1;
    }
    const int T = a.tile_start[a.count];
    const int grid = T < sms ? T : sms;
    if (grid == 0) return cudaSuccess;
    return launch_pdl(stream_linear<E>, dim3(grid), dim3(kThreads), smem, s, pdl, a);
}

cudaError_t launch_stream_group(int route, const StreamGroup &g, const uint16_t *x, int64_t m, int64_t ldx, int ydt,
                                cudaStream_t s, bool pdl)
{
    StreamArgs a = {};
    a.count = g.count;
    int tiles = 0;
    for (int i = 0; i < g.count; ++i) {
        a.nib[i] = g.nib[i];
        a.scale[i] = g.scale[i];
        a.n[i] = g.n[i];
        a.y[i] = g.y[i];
        a.ldy[i] = g.ldy[i];
        a.tile_start[i] = tiles;
        tiles += (int)((g.n[i] + kTileRows - 1) / kTileRows);
    }
    a.tile_start[g.count] = tiles;
    a.k = g.k;
    a.x = x;
    a.ldx = ldx;
    a.ydt = ydt;
    const int sms = device_sms();
    const int tp = stream_tokens_per_pass(route, g.k);
    for (int64_t tok0 = 0; tok0 < m; tok0 += tp) {
        a.tok0 = tok0;
        a.ntok = (int)((m - tok0) < tp ? (m - tok0) : tp);
        a.ntok_cap = a.ntok;
        cudaError_t e;
        if (route == MCAPQ_W4A16)
            e = launch_one<HMMA>(a, s, pdl, sms);
        else if (a.ntok == 1)
            e = launch_one<DP4A>(a, s, pdl, sms);
        else
            e = launch_one<IMMA>(a, s, pdl, sms);
        if (e != cudaSuccess) return e;
        pdl = true;
    }
    return cudaSuccess;
}

}  // namespace mcapq
