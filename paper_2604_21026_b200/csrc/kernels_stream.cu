// kernels_stream.cu -- persistent, TMA-fed decode linears for sm_100a
// (rows a3-a6 at <= 8 tokens per pass; the "stream" path, K % 256 == 0, K >= 2048).
//
// One CTA per SM (grid <= #SMs), warp-specialised:
//   warp 8 (producer, one elected lane): walks the CTA's work items (16-row
//     tile x 1 KiB K-chunk = 2048 weights per row) and moves each into a
//     shared-memory ring with 2-D TMA (cp.async.bulk.tensor, 128-B swizzle):
//     8 boxes of {128 B x 16 rows} of nibbles + 1 box of {64 fp16 x 16 rows} of
//     scales per stage, completion counted on the stage's mbarrier.  It reads
//     only weights and never waits on the predecessor kernel, so under
//     programmatic dependent launch the weight stream of linear i+1 starts
//     while linear i drains.  Rows past N are zero-filled by TMA (never stored).
//   warps 0-7 (consumers): griddepcontrol.wait, one bulk copy of this pass's x
//     into shared memory, then W4A8 consumers QUANTISE it themselves (the same
//     warp-per-group arithmetic as quant_a8_kernel -> bit-identical q / s / sum q,
//     no separate launch) and W4A16 consumers re-stage it in MMA-fragment order;
//     then they consume the ring.
// Engines (template parameter):
//   DP4A : W4A8, 1 token.  warp w owns rows 2w, 2w+1 of the tile, lane l the
//          blocks l, l+32 of the chunk: one conflict-free LDS.128 per block,
//          8 IDP.4A, deferred correction D = sumi - 8 sum_x,
//          fp32 (d s) D.
//   IMMA : W4A8, 2..8 tokens.  warp w owns blocks w, w+8, .. of the chunk for all
//          16 rows; ldmatrix.x4 hands lane (gid, t) word t of rows gid / gid+8 of
//          two blocks -- exactly the m16n8k32.s8 A fragment of the split nibble
//          layout; one mma.sync per block gives the exact int32 D.
//   HMMA : W4A16, 1..8 tokens.  Same fragments; nibbles -> exact bf16 (c - 8)
//          (OR into the 0x4300 mantissa + one packed FMA), two m16n8k16 bf16
//          MMAs per block, fp32 per-block scale (exact products, fp32 sums).
// Work: a group of up to 4 linears sharing x (fused QKV / gate-up):
// their 16-row tiles are numbered consecutively and split into contiguous,
// balanced ranges per CTA.
// Determinism: the chunking and the block->lane/warp maps depend on K only and
// all reductions have a fixed order, so an output row is bit-identical whatever
// N, the group, the grid or the column shard (reading A22).
#include <cmath>
#include <cstdlib>
#include <vector>

#include "internal.h"
#include "stream.h"

namespace mcapq {
namespace {

constexpr int kConsumerWarps = 16;   // one output row per warp per 16-row tile (DP4A); 4 warps / SMSP
constexpr int kThreads = (kConsumerWarps + 1) * 32;
constexpr int kTileRows = 16;
constexpr int kChunkBytes = 1024;                  // nibble bytes per row per stage
constexpr int kChunkBlocks = kChunkBytes / 16;     // 64 Q4_0 blocks
constexpr int kBox = 128 * kTileRows;              // one {128 B x 16 rows} TMA box
constexpr int kStageBytes = 8 * kBox + kBox;       // 8 nibble boxes + 1 scale box (18 KiB)
constexpr int kRedBytes = kConsumerWarps * kTileRows * 8 * 4;
constexpr int kMaxStages = 16;
constexpr int kHmma1Blocks = 1;                   // min CTAs per SM of stream_linear<HMMA1> (launch bounds)
constexpr int kRedSlots = 4;                      // HMMA1 lean path: tile slots of 1 KiB in the reduction area
static_assert(kRedSlots * 1024 <= kRedBytes, "HMMA1 tile slots fit the reduction area");
constexpr int kBarBytes = 512;                     // mbarriers: full[S] + empty[S] + done + go <= 16*16 + 16

// HMMA1: W4A16 with a single token (only MMA column 0 is computed);  NONE: bandwidth probe
// DUMP: the DP4A engine (same staging, same fused quantiser, same block_D) writing the
// staged activation codes and every block's exact int32 D instead of y (test entry)
enum Engine { DP4A = 0, IMMA = 1, HMMA = 2, NONE = 3, HMMA1 = 4, DUMP = 5 };

// ------------------------------------------------------------------ PTX helpers
// All shared-memory traffic uses explicit 32-bit shared-window addresses
// (ld.shared / st.shared): the 1024-B alignment of the dynamic smem base would
// otherwise turn the pointers generic (LD.E with 64-bit address math).
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap *map, int x, int y, uint32_t bar,
                                       uint64_t policy)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void tma_3d(uint32_t dst, const CUtensorMap *map, int x, int y, int z, uint32_t bar,
                                       uint64_t policy)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(bar), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
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
__device__ __forceinline__ uint4 lds128(uint32_t a)
{
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t a)
{
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a)
{
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint16_t lds16(uint32_t a)
{
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v)
{
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v)
{
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts8(uint32_t a, uint32_t v)
{
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ float h2f(uint16_t h)
{
    float f;
    asm("cvt.f32.f16 %0, %1;" : "=f"(f) : "h"(h));
    return f;
}
__device__ __forceinline__ uint4 ldg_nc_128(const void *p)
{
    uint4 v;
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ uint2 ldg_nc_64(const void *p)
{
    uint2 v;
    asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ unsigned long long globaltimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void bar_consumers() { asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory"); }

// 128-B swizzle of a {128 B x 16 rows} box: 16-B chunk c of row r sits at c ^ (r & 7).
__device__ __forceinline__ uint32_t nib_off(int r, int b)          // block b (0..63) of the chunk, row r
{
    return (uint32_t)((b >> 3) * kBox + r * 128 + (((b & 7) ^ (r & 7)) << 4));
}
__device__ __forceinline__ uint32_t scale_off(int r, int b)
{
    return (uint32_t)(8 * kBox + r * 128 + ((((b >> 3) ^ (r & 7))) << 4) + ((b & 7) << 1));
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

// W4A16 A fragment as 128 + c (exact bf16): one LOP3 (+ one shift) per pair, no
// per-element subtract -- the -136 (= -128 offset - 8 zero point) enters through
// the MMA accumulator init (kernel: corr = -136 * sum x).  Element order per
// thread t: p0 = (4t, 4t+2)  p1 = (4t+16, 4t+18)  p2 = (4t+1, 4t+3)  p3 = (4t+17, 4t+19).
__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t mask, uint32_t magic)
{
    // (a & mask) | magic in ONE LOP3 (the compiler splits it in two with two immediates)
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(mask), "r"(magic));
    return d;
}
__device__ __forceinline__ void magic_bf16(uint32_t w, uint32_t mask, uint32_t magic, uint32_t p[4])
{
    p[0] = lop3_and_or(w, mask, magic);
    p[1] = lop3_and_or(w >> 4, mask, magic);
    p[2] = lop3_and_or(w >> 8, mask, magic);
    p[3] = lop3_and_or(w >> 12, mask, magic);
}

// Exact per-token activation code q = clamp(round_half_away(fl(v / s)), -127, 127)
// from a per-group reciprocal: with inv within 1 ulp of 1/s, v * inv is within
// 3.1e-5 of fl(v/s) for |v/s| <= 127.01, so both round to the same integer unless
// v * inv lies within 1e-4 of a half-integer; those rare cases take the IEEE division.  Bit-identical to
// roundf(__fdiv_rn(v, s)) clamped (test_gpu_parity: quantiser bit-exact vs oracle).
__device__ __forceinline__ int quant_code(float v, float s, float inv)
{
    const float qa = v * inv;
    const float aq = fabsf(qa);
    const float fr = aq - truncf(aq);
    // off the half-integers rint (RNE) == round-half-away; the integer is read from the
    // bits of qa + 1.5 * 2^23 (no F2I on the quarter-rate conversion pipe)
    int code = __float_as_int(qa + 12582912.0f) - 0x4B400000;
    if (fabsf(fr - 0.5f) <= 1e-4f || !(aq <= 128.0f)) code = (int)roundf(__fdiv_rn(v, s));
    return code < -127 ? -127 : (code > 127 ? 127 : code);
}

// quant_code out of line (the rare slow path of the fused quantisers)
__device__ __noinline__ int quant_code_ool(float v, float s, float inv) { return quant_code(v, s, inv); }

// D = A.B + C with an explicit accumulator init (C may repeat registers).
__device__ __forceinline__ void hmma_c(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1,
                                       float c0, float c1, float c2, float c3, float d[4])
{
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%11,%12,%13};"
        : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "f"(c0), "f"(c1), "f"(c2), "f"(c3));
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
#include "stream_engines.cuh"
#include "stream_kernel.cuh"
#include "stack_kernel.cuh"
#include "gemm_kernel.cuh"
#include "tc05_kernel.cuh"

// ------------------------------------------------------------------ host side
}  // namespace

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn()
{
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

bool encode_maps(CUtensorMap *tn, CUtensorMap *ts, const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k)
{
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    // nibbles as a 3-D view {128 B column slice, row, 128-B column}: one box
    // {128, 16 rows, 8 columns} = one 16 KiB stage, landing in smem as [column][row][128 B]
    // with the 128-B swizzle keyed by the row (the layout nib_off() reads).
    const cuuint64_t nd[3] = {128, (cuuint64_t)n, (cuuint64_t)(k / 256)};
    const cuuint64_t ns[2] = {(cuuint64_t)(k / 2), 128};
    const cuuint32_t nbox[3] = {128, kTileRows, 8};
    const cuuint32_t es[3] = {1, 1, 1};
    if (fn(tn, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t *>(nib), nd, ns, nbox, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    const cuuint64_t sd[2] = {(cuuint64_t)(k / 32), (cuuint64_t)n};
    const cuuint64_t ss[1] = {(cuuint64_t)(k / 16)};
    const cuuint32_t sbox[2] = {kChunkBlocks, kTileRows};
    return fn(ts, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<uint16_t *>(scale), sd, ss, sbox, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

namespace {
size_t act_bytes(int engine, int64_t k, int ntok)
{
    const int64_t G = k / 32;
    if (engine == HMMA || engine == HMMA1 || engine == NONE) return (size_t)ntok * (size_t)(2 * k + 64) + 32 * (size_t)G;
    return (size_t)ntok * (size_t)(k + 16) + (size_t)ntok * 8 * (size_t)G;
}

size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Shared-memory plan: ring (S stages) | barriers | x raw | activations | reduction.
// Aim at <= ~113 KB so that this linear and the next (PDL) fit on one SM together.
// Launch-shape knobs, read once from the environment (benchmarking / tuning only;
// the defaults are the tuned values):
//   MCAPQ_STREAM_SMEM_KB   shared-memory plan per CTA (default 112: two CTAs per SM)
//   MCAPQ_STREAM_STAGES    max ring stages (default 12)
//   MCAPQ_STREAM_NOCOMPUTE 1 = consumers only drain the ring (bandwidth probe; outputs garbage)
//   MCAPQ_STREAM_PDL       1 = API calls also launch with programmatic dependent launch
struct Tune {
    // step_smem_kb 120: a ~5-stage ring keeps the HBM pipe busy while bounding the
    // per-SM queue of in-flight weight data that the chain's L2 accesses wait behind
    int smem_kb = 112, max_stages = 12, nocompute = 0, pdl = 0, trace = 0, step_smem_kb = 200, step = 1,
        step_flags = 0, step_spin_ns = 16, step_polls = 1, ctas_per_sm = 0, step_ep_log2 = 1, smem_kb_env = 0,
        step_hold = 2, step_rec_spin = 64, a8_tc05 = 1, a16_tc05 = 1;
};
const Tune &tune()
{
    static Tune t = [] {
        Tune v;
        if (const char *e = getenv("MCAPQ_STREAM_SMEM_KB")) {
            v.smem_kb = atoi(e);
            v.smem_kb_env = 1;
        }
        if (const char *e = getenv("MCAPQ_STREAM_STAGES")) v.max_stages = atoi(e);
        if (const char *e = getenv("MCAPQ_STREAM_NOCOMPUTE")) v.nocompute = atoi(e);
        if (const char *e = getenv("MCAPQ_STREAM_PDL")) v.pdl = atoi(e);
        if (const char *e = getenv("MCAPQ_STREAM_TRACE")) v.trace = atoi(e);
        if (const char *e = getenv("MCAPQ_STEP_SMEM_KB")) v.step_smem_kb = atoi(e);
        if (const char *e = getenv("MCAPQ_STEP_KERNEL")) v.step = atoi(e);
        if (const char *e = getenv("MCAPQ_STEP_FLAGS")) v.step_flags = atoi(e);
        if (const char *e = getenv("MCAPQ_STEP_SPIN_NS")) v.step_spin_ns = atoi(e);
        if (const char *e = getenv("MCAPQ_STEP_POLLS")) v.step_polls = atoi(e);
        if (const char *e = getenv("MCAPQ_STREAM_CTAS_PER_SM")) v.ctas_per_sm = atoi(e);
        if (const char *e = getenv("MCAPQ_STEP_EP_LOG2")) v.step_ep_log2 = atoi(e);
        if (const char *e = getenv("MCAPQ_STEP_HOLD")) v.step_hold = atoi(e);
        if (const char *e = getenv("MCAPQ_STEP_REC_SPIN")) v.step_rec_spin = atoi(e);
        if (const char *e = getenv("MCAPQ_GEMM_A8_TC05")) v.a8_tc05 = atoi(e);
        if (const char *e = getenv("MCAPQ_GEMM_A16_TC05")) v.a16_tc05 = atoi(e);
        if (v.step_ep_log2 < 1) v.step_ep_log2 = 1;
        if (v.step_ep_log2 > 3) v.step_ep_log2 = 3;
        if (v.ctas_per_sm < 0 || v.ctas_per_sm > 2) v.ctas_per_sm = 0;
        if (v.step_smem_kb < 60) v.step_smem_kb = 60;
        if (v.step_smem_kb > 226) v.step_smem_kb = 226;
        if (v.smem_kb < 40) v.smem_kb = 40;
        if (v.smem_kb > 226) v.smem_kb = 226;
        if (v.max_stages < 2) v.max_stages = 2;
        return v;
    }();
    return t;
}

unsigned long long *g_trace = nullptr;   // debug timeline buffer (MCAPQ_STREAM_TRACE)
size_t g_trace_used = 0;
int g_trace_launches = 0;

size_t plan_smem(int engine, int64_t k, int ntok, StreamArgs &a)
{
    const size_t xraw = 0;   // x is read from global directly (no smem staging copy)
    (void)ntok;
    const size_t act = round_up(act_bytes(engine, k, ntok), 128);
    const size_t fixed = kBarBytes + xraw + act + kRedBytes;
    const size_t budget = (size_t)(a.smem_kb ? a.smem_kb : tune().smem_kb) * 1024;
    int S = (int)(((long)budget - (long)fixed - 1024) / kStageBytes);
    S = S < 2 ? 2 : (S > tune().max_stages ? tune().max_stages : S);
    S = S > kMaxStages ? kMaxStages : S;
    a.stages = S;
    a.xraw_off = (int)((size_t)S * kStageBytes + kBarBytes);
    a.act_off = (int)(a.xraw_off + xraw);
    a.red_off = (int)(a.act_off + act);
    return 1024 + (size_t)a.red_off + kRedBytes;
}

template <int E>
cudaError_t launch_one(StreamArgs &a, cudaStream_t s, bool pdl, int sms)
{
    const size_t smem = plan_smem(E, a.k, a.ntok, a);
    // one L1/shared carveout for every linear: consecutive (PDL-overlapped) kernels
    // never force an SM to drain for a carveout change
    cudaError_t e = kernel_smem_attr(reinterpret_cast<const void *>(stream_linear<E>), 227 * 1024, 100);
    if (e != cudaSuccess) return e;
    const int T = a.tile_start[a.count];
    const int grid = T < sms ? T : sms;
    if (grid == 0) return cudaSuccess;
    a.trace = nullptr;
    if (tune().trace) {
        // debug timeline: one 8 x u64 record per CTA, bump-allocated per launch (wraps)
        constexpr size_t kCap = 1u << 20;
        if (!g_trace) {
            if (cudaMalloc(&g_trace, kCap * 64) != cudaSuccess) g_trace = nullptr;
            else cudaMemset(g_trace, 0, kCap * 64);
        }
        if (g_trace) {
            if (g_trace_used + (size_t)grid > kCap) g_trace_used = 0;
            a.trace = g_trace + 8 * g_trace_used;
            a.launch_id = g_trace_launches++;
            g_trace_used += (size_t)grid;
        }
    }
    return launch_pdl(stream_linear<E>, dim3(grid), dim3(kThreads), smem, s, pdl, a);
}

}  // namespace

// gemm maps: nibbles 2-D {K/2, N}, box {128 B, bn rows}, 128B swizzle (row r's 16-B
// chunk c at c ^ (r & 7)); scales 2-D {K/32, N}, box {8, bn rows}, no swizzle (16 B/row).
bool encode_gemm_maps(CUtensorMap *tn, CUtensorMap *ts, const uint8_t *nib, const uint16_t *scale, int64_t n,
                      int64_t k, int bn)
{
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t nd[2] = {(cuuint64_t)(k / 2), (cuuint64_t)n};
    const cuuint64_t ns[1] = {(cuuint64_t)(k / 2)};
    const cuuint32_t nbox[2] = {128, (cuuint32_t)bn};
    const cuuint32_t es[2] = {1, 1};
    if (fn(tn, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t *>(nib), nd, ns, nbox, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    const cuuint64_t sd[2] = {(cuuint64_t)(k / 32), (cuuint64_t)n};
    const cuuint64_t ss[1] = {(cuuint64_t)(k / 16)};
    const cuuint32_t sbox[2] = {8, (cuuint32_t)bn};
    return fn(ts, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<uint16_t *>(scale), sd, ss, sbox, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// gemm activation maps, boxes of mp token rows (rows past m read as zeros):
//   W4A8  q  [m][k] int8 as 3-D {128 B, m, k/128}, box {128, mp, 2} (= one 256-K slice),
//         128B swizzle -> smem [2][mp][128 B];  sx / sq [m][k/32] 2-D, box {8, mp} -> [mp][8]
//   W4A16 x  [m][ldx] bf16 as 3-D {64, m, k/64}, box {64, mp, 4}, 128B swizzle -> [4][mp][128 B]
bool encode_gemm_act_maps(CUtensorMap *h, bool a8, const void *x_or_q, const float *sx, const int32_t *sq, int64_t m,
                          int64_t k, int64_t ldx, int mp)
{
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    if (a8) {
        const cuuint64_t qd[3] = {128, (cuuint64_t)m, (cuuint64_t)(k / 128)};
        const cuuint64_t qs[2] = {(cuuint64_t)k, 128};
        const cuuint32_t qb[3] = {128, (cuuint32_t)mp, 2};
        const cuuint32_t e3[3] = {1, 1, 1};
        if (fn(&h[0], CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void *>(x_or_q), qd, qs, qb, e3,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
        const cuuint64_t sd[2] = {(cuuint64_t)(k / 32), (cuuint64_t)m};
        const cuuint64_t ss[1] = {(cuuint64_t)(k / 32) * 4};
        const cuuint32_t sb[2] = {8, (cuuint32_t)mp};
        const cuuint32_t e2[2] = {1, 1};
        if (fn(&h[1], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(sx), sd, ss, sb, e2,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
        return fn(&h[2], CU_TENSOR_MAP_DATA_TYPE_INT32, 2, const_cast<int32_t *>(sq), sd, ss, sb, e2,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    const cuuint64_t xd[3] = {64, (cuuint64_t)m, (cuuint64_t)(k / 64)};
    const cuuint64_t xs[2] = {(cuuint64_t)ldx * 2, 128};
    const cuuint32_t xb[3] = {64, (cuuint32_t)mp, 4};
    const cuuint32_t e3[3] = {1, 1, 1};
    return fn(&h[0], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(x_or_q), xd, xs, xb, e3,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ------------------------------------------------------------------ batched decode (gemm_w4)
bool gemm_supported(int64_t k) { return k >= 256 && k % 256 == 0 && encode_fn() != nullptr; }

namespace {
// Tile configurations per padded pass width Mp: (MT, NT, WT) -> BN = 16 MT (8 / WT), Mp = 8 NT WT.
struct GemmCfg {
    int mt, nt, wt;
    int bn() const { return 16 * mt * (kGemmWarps / wt); }
    int mp() const { return 8 * nt * wt; }
};
constexpr GemmCfg kCfg16[] = {{2, 1, 2}, {1, 1, 2}};
constexpr GemmCfg kCfg32[] = {{2, 2, 2}, {1, 2, 2}, {1, 1, 4}};
constexpr GemmCfg kCfg64[] = {{4, 2, 4}, {2, 2, 4}, {1, 2, 4}};
// W4A16 at Mp = 64: fewer token-warps (each weight dequantised by WT warps of the CTA)
constexpr GemmCfg kCfg64h[] = {{2, 4, 2}, {1, 4, 2}, {1, 2, 4}};

template <bool A8, int MT, int NT>
cudaError_t launch_gemm_cfg(GemmArgs &a, size_t smem, int grid, cudaStream_t s, bool pdl)
{
    cudaError_t e = kernel_smem_attr(reinterpret_cast<const void *>(gemm_w4<A8, MT, NT>), 227 * 1024);
    if (e != cudaSuccess) return e;
    return launch_pdl(gemm_w4<A8, MT, NT>, dim3(grid), dim3(kGemmThreads), smem, s, pdl, a);
}

template <bool A8>
cudaError_t dispatch_gemm(const GemmCfg &c, GemmArgs &a, size_t smem, int grid, cudaStream_t s, bool pdl)
{
    if (c.mt == 4 && c.nt == 2) return launch_gemm_cfg<A8, 4, 2>(a, smem, grid, s, pdl);
    if (c.mt == 2 && c.nt == 4) return launch_gemm_cfg<A8, 2, 4>(a, smem, grid, s, pdl);
    if (c.mt == 1 && c.nt == 4) return launch_gemm_cfg<A8, 1, 4>(a, smem, grid, s, pdl);
    if (c.mt == 2 && c.nt == 2) return launch_gemm_cfg<A8, 2, 2>(a, smem, grid, s, pdl);
    if (c.mt == 1 && c.nt == 2) return launch_gemm_cfg<A8, 1, 2>(a, smem, grid, s, pdl);
    if (c.mt == 2 && c.nt == 1) return launch_gemm_cfg<A8, 2, 1>(a, smem, grid, s, pdl);
    if (c.mt == 1 && c.nt == 1) return launch_gemm_cfg<A8, 1, 1>(a, smem, grid, s, pdl);
    return cudaErrorInvalidValue;
}
}  // namespace

// ------------------------------------------------------------------ batched W4A16 on tcgen05
namespace {
template <int MP>
cudaError_t launch_tc05_mp(GemmArgs &a, size_t smem, int grid, cudaStream_t s, bool pdl)
{
    cudaError_t e = kernel_smem_attr(reinterpret_cast<const void *>(tc05_w4a16<MP>), 227 * 1024);
    if (e != cudaSuccess) return e;
    return launch_pdl(tc05_w4a16<MP>, dim3(grid), dim3(tc05::kThreads), smem, s, pdl, a);
}
}  // namespace

// tc05_w4a16 (bf16-dequantised weights, tcgen05): 128-row CTA tiles, passes of <= 64
// tokens (MP = 16 / 32 / 64); K % 256 == 0.
cudaError_t launch_tc05(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k, const uint16_t *x,
                        int64_t ldx, int64_t m, void *y, int ydt, int64_t ldy, cudaStream_t s, bool pdl)
{
    const int sms = device_sms();
    for (int64_t tok0 = 0; tok0 < m; tok0 += 64) {
        const int ntok = (int)((m - tok0) < 64 ? (m - tok0) : 64);
        const int mp = ntok <= 16 ? 16 : (ntok <= 32 ? 32 : 64);
        GemmArgs a;
        memset(&a, 0, sizeof(a));
        if (!encode_gemm_maps(&a.maps[0], &a.maps[1], nib, scale, n, k, 128) || !encode_gemm_act_maps(a.amaps, false, x, nullptr, nullptr, m, k, ldx, mp))
            return cudaErrorInvalidValue;
        a.y = y;
        a.ldy = ldy;
        a.n = n;
        a.k = k;
        a.ydt = ydt;
        a.tok0 = tok0;
        a.ntok = ntok;
        a.mp = mp;
        a.bn = 128;
        a.row_tiles = (int)((n + 127) / 128);
        a.stage_bytes = tc05::kNibBytes + tc05::kScBytes + (uint32_t)mp * 512u;
        const size_t fixed = 1024 + (size_t)tc05::kNA * tc05::kAtomBytes + 256;
        int S = (int)((227 * 1024 - fixed) / a.stage_bytes);
        S = S > 8 ? 8 : S;   // weight ring: as deep as shared memory allows (<= 8 slices)
        if (S < 2) return cudaErrorInvalidValue;
        a.stages = S;
        const size_t smem = fixed + (size_t)S * a.stage_bytes;
        const int grid = a.row_tiles < sms ? a.row_tiles : sms;
        cudaError_t e = mp == 16 ? launch_tc05_mp<16>(a, smem, grid, s, pdl)
                                 : (mp == 32 ? launch_tc05_mp<32>(a, smem, grid, s, pdl)
                                             : launch_tc05_mp<64>(a, smem, grid, s, pdl));
        if (e != cudaSuccess) return e;
        pdl = true;
    }
    return cudaSuccess;
}

// ------------------------------------------------------------------ NEXT-4 prefill
cudaError_t launch_dequant_w4_bf16(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k, uint16_t *w,
                                   cudaStream_t s)
{
    const int64_t nb = n * (k / 32);
    dequant_w4_bf16_kernel<<<(unsigned)((nb + 255) / 256), 256, 0, s>>>(nib, scale, nb, w);
    return cudaGetLastError();
}

namespace {
bool encode_bf16_rows(CUtensorMap *m, const void *base, int64_t rows, int64_t k, int64_t ld, int box_rows)
{
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t d[2] = {(cuuint64_t)k, (cuuint64_t)rows};
    const cuuint64_t st[1] = {(cuuint64_t)ld * 2};
    const cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    const cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), d, st, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
template <int MP>
cudaError_t launch_prefill_mp(PrefillArgs &a, size_t smem, int grid, cudaStream_t s, bool pdl)
{
    cudaError_t e = kernel_smem_attr(reinterpret_cast<const void *>(tc05_prefill<MP>), 227 * 1024);
    if (e != cudaSuccess) return e;
    return launch_pdl(tc05_prefill<MP>, dim3(grid), dim3(192), smem, s, pdl, a);
}
}  // namespace

// y = X . W^T for a bf16 W^ [n][k] (k % 64 == 0), ONE launch: work units = (token pass of
// MP = 64 / 128 / 256 tokens, 128-row tile) pairs spread over the persistent CTAs.
cudaError_t launch_prefill(const uint16_t *w, int64_t n, int64_t k, const uint16_t *x, int64_t ldx, int64_t m, void *y,
                           int ydt, int64_t ldy, cudaStream_t s, bool pdl)
{
    const int sms = device_sms();
    const int mp = m <= 64 ? 64 : (m <= 128 ? 128 : 256);
    PrefillArgs a;
    memset(&a, 0, sizeof(a));
    if (!encode_bf16_rows(&a.amap, w, n, k, k, 128) || !encode_bf16_rows(&a.xmap, x, m, k, ldx, mp))
        return cudaErrorInvalidValue;
    a.y = y;
    a.ldy = ldy;
    a.n = n;
    a.k = k;
    a.ydt = ydt;
    a.m = m;
    a.passes = (int)((m + mp - 1) / mp);
    a.row_tiles = (int)((n + 127) / 128);
    if ((int64_t)a.row_tiles * a.passes > (1 << 20)) return cudaErrorInvalidValue;   // 32-bit unit partition
    a.stage_bytes = 128u * 128u + (uint32_t)mp * 128u;
    const size_t fixed = 1024 + 256;
    int S = (int)((227 * 1024 - fixed) / a.stage_bytes);
    S = S > 8 ? 8 : S;
    if (S < 2) return cudaErrorInvalidValue;
    a.stages = S;
    const size_t smem = fixed + (size_t)S * a.stage_bytes;
    const int units = a.row_tiles * a.passes;
    const int grid = units < sms ? units : sms;
    return mp == 64 ? launch_prefill_mp<64>(a, smem, grid, s, pdl)
                    : (mp == 128 ? launch_prefill_mp<128>(a, smem, grid, s, pdl) : launch_prefill_mp<256>(a, smem, grid, s, pdl));
}

namespace {
template <int MP>
cudaError_t launch_tc05_a8_mp(GemmArgs &a, size_t smem, int grid, cudaStream_t s, bool pdl)
{
    cudaError_t e = kernel_smem_attr(reinterpret_cast<const void *>(tc05_w4a8<MP>), 227 * 1024);
    if (e != cudaSuccess) return e;
    return launch_pdl(tc05_w4a8<MP>, dim3(grid), dim3(tc05::kA8Threads<MP>), smem, s, pdl, a);
}
}  // namespace

// tc05_w4a8 (a5 on tcgen05 kind::i8): 128-row CTA tiles, passes of <= 64 tokens
// (MP = 16 / 32 / 64), q / sx from the quant_a8 workspace; K % 256 == 0.
cudaError_t launch_tc05_a8(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k, const int8_t *q,
                           const float *sx, const int32_t *sq, int64_t m, void *y, int ydt, int64_t ldy, cudaStream_t s,
                           bool pdl)
{
    const int sms = device_sms();
    for (int64_t tok0 = 0; tok0 < m; tok0 += 64) {
        const int ntok = (int)((m - tok0) < 64 ? (m - tok0) : 64);
        const int mp = ntok <= 16 ? 16 : (ntok <= 32 ? 32 : 64);
        GemmArgs a;
        memset(&a, 0, sizeof(a));
        if (!encode_gemm_maps(&a.maps[0], &a.maps[1], nib, scale, n, k, 128) ||
            !encode_gemm_act_maps(a.amaps, true, q, sx, sq, m, k, k, mp))
            return cudaErrorInvalidValue;
        a.y = y;
        a.ldy = ldy;
        a.n = n;
        a.k = k;
        a.ydt = ydt;
        a.tok0 = tok0;
        a.ntok = ntok;
        a.mp = mp;
        a.bn = 128;
        a.row_tiles = (int)((n + 127) / 128);
        static const int dbg = getenv("MCAPQ_TC05_DBG") ? atoi(getenv("MCAPQ_TC05_DBG")) : 0;
        a.wt = dbg;   // debug flags (timing experiments only; outputs wrong when set)
        a.stage_bytes = (uint32_t)round_up(tc05::kNibBytes + tc05::kScBytes + (size_t)mp * 288, 1024);
        const int na = mp == 64 ? tc05::kA8NA<64> : tc05::kA8NA<16>;
        const int ne = mp == 64 ? tc05::kA8NE<64> : tc05::kA8NE<16>;
        const size_t fixed = 1024 + (size_t)na * tc05::kA8AtomBytes + (size_t)ne * (2048 + 32 * (size_t)mp) +
                             (mp == 16 ? 128 * (size_t)mp * 4 : 0) + 1024;
        int S = (int)((227 * 1024 - fixed) / a.stage_bytes);
        S = S > 8 ? 8 : S;
        if (S < 2) return cudaErrorInvalidValue;
        a.stages = S;
        const size_t smem = fixed + (size_t)S * a.stage_bytes;
        const int grid = a.row_tiles < sms ? a.row_tiles : sms;
        cudaError_t e = mp == 16 ? launch_tc05_a8_mp<16>(a, smem, grid, s, pdl)
                                 : (mp == 32 ? launch_tc05_a8_mp<32>(a, smem, grid, s, pdl)
                                             : launch_tc05_a8_mp<64>(a, smem, grid, s, pdl));
        if (e != cudaSuccess) return e;
        pdl = true;
    }
    return cudaSuccess;
}

namespace {
template <int MP, bool TS>
cudaError_t launch_tc05_a16x_mp(GemmArgs &a, size_t smem, int grid, cudaStream_t s, bool pdl)
{
    cudaError_t e = kernel_smem_attr(reinterpret_cast<const void *>(tc05_w4a16x<MP, TS>), 227 * 1024);
    if (e != cudaSuccess) return e;
    return launch_pdl(tc05_w4a16x<MP, TS>, dim3(grid), dim3(tc05::kXThreads<MP, TS>), smem, s, pdl, a);
}
}  // namespace

// tc05_w4a16x (exact W4A16 on tcgen05, one accumulator per Q4_0 block): 128-row CTA tiles,
// passes of <= 64 tokens; K % 256 == 0.
cudaError_t launch_tc05_a16x(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k, const uint16_t *x,
                             int64_t ldx, int64_t m, void *y, int ydt, int64_t ldy, cudaStream_t s, bool pdl)
{
    const int sms = device_sms();
    for (int64_t tok0 = 0; tok0 < m; tok0 += 64) {
        const int ntok = (int)((m - tok0) < 64 ? (m - tok0) : 64);
        const int mp = ntok <= 16 ? 16 : (ntok <= 32 ? 32 : 64);
        GemmArgs a;
        memset(&a, 0, sizeof(a));
        if (!encode_gemm_maps(&a.maps[0], &a.maps[1], nib, scale, n, k, 128) ||
            !encode_gemm_act_maps(a.amaps, false, x, nullptr, nullptr, m, k, ldx, mp))
            return cudaErrorInvalidValue;
        a.y = y;
        a.ldy = ldy;
        a.n = n;
        a.k = k;
        a.ydt = ydt;
        a.tok0 = tok0;
        a.ntok = ntok;
        a.mp = mp;
        a.bn = 128;
        a.row_tiles = (int)((n + 127) / 128);
        static const int dbg = getenv("MCAPQ_TC05_DBG") ? atoi(getenv("MCAPQ_TC05_DBG")) : 0;
        a.wt = dbg;   // debug flags (timing experiments only; outputs wrong when set)
        a.stage_bytes = tc05::kNibBytes + tc05::kScBytes + (uint32_t)mp * 512u;
        static const int na_env = getenv("MCAPQ_TC05_NA") ? atoi(getenv("MCAPQ_TC05_NA")) : 0;
        a.na = na_env >= 4 ? (na_env & ~3) : 4;   // A-atom ring slots (smem-A kernel; a multiple of 4)
        // A operand from tensor memory (tcgen05.st by the dequantise warps, no shared-memory
        // atoms): 8B lm_head M = 16 141 -> 128 us; at MP = 64 the 512 columns leave one
        // accumulator quad and the smem-A kernel is faster (177 vs 185 us).
        // MCAPQ_TC05_TS: 0 never, 1 always, default MP <= 32.
        static const int ts_env = getenv("MCAPQ_TC05_TS") ? atoi(getenv("MCAPQ_TC05_TS")) : -1;
        const bool ts = ts_env < 0 ? mp <= 32 : ts_env != 0;
        const size_t fixed = 1024 + (ts ? 0 : (size_t)a.na * tc05::kAtomBytes) + (size_t)tc05::kXNE * 2048 +
                             (mp == 16 ? 128 * (size_t)mp * 4 : 0) + 1024;
        int S = (int)((227 * 1024 - fixed) / a.stage_bytes);
        static const int scap = getenv("MCAPQ_TC05_STAGES") ? atoi(getenv("MCAPQ_TC05_STAGES")) : 8;
        S = S > scap ? scap : S;
        if (S < 2) return cudaErrorInvalidValue;
        a.stages = S;
        const size_t smem = fixed + (size_t)S * a.stage_bytes;
        const int grid = a.row_tiles < sms ? a.row_tiles : sms;
        cudaError_t e = ts ? (mp == 16 ? launch_tc05_a16x_mp<16, true>(a, smem, grid, s, pdl)
                                       : (mp == 32 ? launch_tc05_a16x_mp<32, true>(a, smem, grid, s, pdl)
                                                   : launch_tc05_a16x_mp<64, true>(a, smem, grid, s, pdl)))
                           : (mp == 16 ? launch_tc05_a16x_mp<16, false>(a, smem, grid, s, pdl)
                                       : (mp == 32 ? launch_tc05_a16x_mp<32, false>(a, smem, grid, s, pdl)
                                                   : launch_tc05_a16x_mp<64, false>(a, smem, grid, s, pdl)));
        if (e != cudaSuccess) return e;
        pdl = true;
    }
    return cudaSuccess;
}

cudaError_t launch_gemm(int route, const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k, const uint16_t *x,
                        int64_t ldx, const int8_t *q, const float *sx, const int32_t *sq, int64_t m, void *y, int ydt,
                        int64_t ldy, cudaStream_t s, bool pdl)
{
    const bool a8 = route == MCAPQ_W4A8;
    // W4A8 on tcgen05 kind::i8 for passes of more than 32 tokens over at least one 128-row
    // tile per SM (8B lm_head M = 64: 190 us vs 228 us on mma.sync); at M <= 32, or with
    // fewer tiles than SMs (3B q / up: 24 / 64 tiles), the IMMA kernel below is faster
    // (lm_head M = 16: 80 vs 103 us: the per-block MMA -> commit -> TMEM read-back chain,
    // not the FP work, bounds tcgen05 there).  MCAPQ_GEMM_A8_TC05: 0 never, 1 auto
    // (default), 2 always.
    if (a8 && (tune().a8_tc05 == 2 || (tune().a8_tc05 == 1 && m > 32 && (n + 127) / 128 >= device_sms())))
        return launch_tc05_a8(nib, scale, n, k, q, sx, sq, m, y, ydt, ldy, s, pdl);
    // exact W4A16 on tcgen05 (tc05_w4a16x) over at least one 128-row tile per SM: the 8B
    // lm_head M = 64 250 -> 140 us, M = 16 135 -> 112 us (narrower linears stay on mma.sync:
    // the 3B q / up at 24 / 64 tiles).  MCAPQ_GEMM_A16_TC05: 0 never, 1 auto, 2 always.
    if (!a8 && (tune().a16_tc05 == 2 || (tune().a16_tc05 == 1 && (n + 127) / 128 >= device_sms())))
        return launch_tc05_a16x(nib, scale, n, k, x, ldx, m, y, ydt, ldy, s, pdl);
    const int sms = device_sms();
    for (int64_t tok0 = 0; tok0 < m; tok0 += 64) {
        const int ntok = (int)((m - tok0) < 64 ? (m - tok0) : 64);
        const GemmCfg *cfgs = ntok <= 16 ? kCfg16 : (ntok <= 32 ? kCfg32 : (a8 ? kCfg64 : kCfg64h));
        const int ncfg = ntok <= 16 ? 2 : 3;
        // the largest tile that still fills ~the machine, else the smallest
        GemmCfg c = cfgs[ncfg - 1];
        for (int i = 0; i < ncfg; ++i)
            if ((n + cfgs[i].bn() - 1) / cfgs[i].bn() >= (sms * 4) / 5) {
                c = cfgs[i];
                break;
            }
        const int bn = c.bn(), mp = c.mp();
        GemmArgs a;
        memset(&a, 0, sizeof(a));
        if (!encode_gemm_maps(&a.maps[0], &a.maps[1], nib, scale, n, k, bn) || !encode_gemm_act_maps(a.amaps, a8, a8 ? (const void *)q : (const void *)x, sx, sq, m, k, ldx, mp))
            return cudaErrorInvalidValue;
        a.y = y;
        a.ldy = ldy;
        a.n = n;
        a.k = k;
        a.ydt = ydt;
        a.tok0 = tok0;
        a.ntok = ntok;
        a.mp = mp;
        a.bn = bn;
        a.wt = c.wt;
        a.row_tiles = (int)((n + bn - 1) / bn);
        // stage: nibbles | scales | activations (| W4A8 s, sq), swizzled boxes 1 KiB aligned
        a.nib_bytes = (uint32_t)bn * 128u;
        a.sc_off = (uint32_t)round_up(a.nib_bytes, 1024);
        a.act_off = (uint32_t)round_up(a.sc_off + (size_t)bn * 16, 1024);
        const size_t act = a8 ? (size_t)mp * 256 : (size_t)mp * 512;
        a.ss_off = (uint32_t)round_up(a.act_off + act, 128);
        a.sq_off = a.ss_off + (uint32_t)mp * 32u;
        a.stage_bytes = (uint32_t)round_up(a.ss_off + (a8 ? (size_t)mp * 64 : 0), 1024);
        int S = (int)((227 * 1024 - 1024 - 256) / a.stage_bytes);
        S = S > kGemmMaxStages ? kGemmMaxStages : S;
        if (S < 2) return cudaErrorInvalidValue;
        a.stages = S;
        const size_t smem = 1024 + (size_t)S * a.stage_bytes + 16 * (size_t)S;
        const int grid = a.row_tiles < sms ? a.row_tiles : sms;
        cudaError_t e = a8 ? dispatch_gemm<true>(c, a, smem, grid, s, pdl) : dispatch_gemm<false>(c, a, smem, grid, s, pdl);
        if (e != cudaSuccess) return e;
        pdl = true;
    }
    return cudaSuccess;
}

namespace {
thread_local bool t_api_pdl = false;
}
bool api_pdl() { return t_api_pdl; }
void set_api_pdl(bool on) { t_api_pdl = on; }

cudaError_t launch_linear_group(int route, const StreamGroup &g, const uint16_t *x, int64_t m, int64_t ldx, int ydt,
                                void *ws, cudaStream_t s, bool pdl)
{
    pdl = pdl || api_pdl();
    if (m >= kGemmMinTokens && gemm_supported(g.k)) {
        const int8_t *q = nullptr;
        const float *sx = nullptr;
        const int32_t *sq = nullptr;
        if (route == MCAPQ_W4A8) {
            // quantise once into the workspace, shared by every member of the group (A15)
            if (!ws) return cudaErrorInvalidValue;
            const A8Workspace w = a8_workspace(ws, m, g.k);
            cudaError_t e = launch_quant_a8(x, m, g.k, ldx, w.q, w.sx, w.sq, s, pdl);
            if (e != cudaSuccess) return e;
            q = w.q;
            sx = w.sx;
            sq = w.sq;
            pdl = true;
        }
        for (int i = 0; i < g.count; ++i) {
            cudaError_t e =
                launch_gemm(route, g.nib[i], g.scale[i], g.n[i], g.k, x, ldx, q, sx, sq, m, g.y[i], ydt, g.ldy[i], s, pdl);
            if (e != cudaSuccess) return e;
            pdl = true;
        }
        return cudaSuccess;
    }
    return launch_stream_group(route, g, x, m, ldx, ydt, s, pdl);
}

// ------------------------------------------------------------------ persistent step
size_t stack_op_bytes() { return sizeof(StackOp); }
bool stack_step_enabled() { return tune().step != 0 && encode_fn() != nullptr; }

bool stack_fill_op(void *host_op, int route, const StreamGroup &g, const uint16_t *x, int ydt, const StackDeps &d,
                   CUtensorMap *host_maps, const CUtensorMap *dev_maps)
{
    StackOp op;
    memset(&op, 0, sizeof(op));
    int tiles = 0;
    for (int i = 0; i < g.count; ++i) {
        memset(host_maps + 2 * i, 0, 2 * sizeof(CUtensorMap));
        if (!encode_maps(host_maps + 2 * i, host_maps + 2 * i + 1, g.nib[i], g.scale[i], g.n[i], g.k)) return false;
        op.maps[i] = dev_maps + 2 * i;
        op.y[i] = g.y[i];
        op.n[i] = (int)g.n[i];
        op.tile_start[i] = tiles;
        tiles += (int)((g.n[i] + kTileRows - 1) / kTileRows);
    }
    op.tile_start[g.count] = tiles;
    if (tiles > (1 << 20)) return false;   // the kernel's 32-bit tile partition (T * grid < 2^32)
    op.count = g.count;
    op.route = route;
    op.ydt = ydt;
    op.k = g.k;
    op.x = x;
    op.xt = d.xt;
    op.xt_op = d.xt_op;
    for (int i = 0; i < g.count; ++i) op.yt[i] = d.yt[i];
    op.wait_op = d.wait_op;
    op.publish = d.publish;
    // an op whose outputs feed producer-quantised records hands its tiles out in 32-row
    // pairs (quantisation groups; every member's N a multiple of 32, so a pair never
    // spans two members); the other ops keep the contiguous balanced split
    bool recs = false;
    for (int i = 0; i < g.count; ++i) recs = recs || d.yq[i] != nullptr;
    bool paired = recs && stack_clustered() && (tiles % 2 == 0);
    for (int i = 0; i < g.count; ++i) paired = paired && g.n[i] % 32 == 0;
    op.paired = paired ? 1 : 0;
    for (int i = 0; i < g.count; ++i) op.yq[i] = paired ? d.yq[i] : nullptr;
    op.xq = d.xq;
    memcpy(host_op, &op, sizeof(op));
    return true;
}

// Every CTA's tile range per op of a step program: [nops][grid] {t0, t1 | straddle << 31}.
// Paired ops of a clustered launch (producer-side records): 32-row pairs split over the
// clusters by weight -- a pair of a member whose epilogue also builds records weighs
// 1 + rec_r 2048 / K (the record work is fixed per group while a tile's compute grows
// with K; rec_r = 0.75, MCAPQ_STEP_REC_R), the others 1 -- and each cluster's range in
// halves over its two CTAs, so a quantisation group lies in one CTA or, at most once per
// op, straddles the pair (the straddle flag: rank 0's last tile is its first half, rank
// 1's first tile its second).  Otherwise contiguous balanced ranges.
void stack_partition(const void *ops_host, int nops, int grid, bool clustered, double rec_r, int2 *out)
{
    const StackOp *ops = reinterpret_cast<const StackOp *>(ops_host);
    for (int i = 0; i < nops; ++i) {
        const StackOp &op = ops[i];
        const int T = op.tile_start[op.count];
        if (clustered && op.paired) {
            const int C = grid / 2;
            const double wr = 1.0 + rec_r * (2048.0 / (double)op.k);
            std::vector<double> wm(op.count);
            double W = 0.0;
            for (int m = 0; m < op.count; ++m) {
                wm[m] = op.yq[m] ? wr : 1.0;
                W += (double)((op.tile_start[m + 1] - op.tile_start[m]) >> 1) * wm[m];
            }
            auto pair_at = [&](int c) {
                if (c >= C) return T >> 1;
                double t = W * c / C;
                int base = 0;
                for (int m = 0; m < op.count; ++m) {
                    const int np_m = (op.tile_start[m + 1] - op.tile_start[m]) >> 1;
                    if (t < np_m * wm[m]) return base + (int)std::floor(t / wm[m] + 1e-9);
                    t -= np_m * wm[m];
                    base += np_m;
                }
                return base;
            };
            for (int b = 0; b < grid; ++b) {
                const int c = b >> 1, r = b & 1;
                const int p0 = pair_at(c), p1 = pair_at(c + 1), np = p1 - p0;
                const int t0 = 2 * p0 + (r ? np : 0), t1 = r ? 2 * p1 : 2 * p0 + np;
                out[(size_t)i * grid + b] = make_int2(t0, t1 | ((np & 1) ? (int)0x80000000u : 0));
            }
        } else {
            for (int b = 0; b < grid; ++b)
                out[(size_t)i * grid + b] = make_int2((int)(((int64_t)T * b) / grid), (int)(((int64_t)T * (b + 1)) / grid));
        }
    }
}

double stack_rec_r()
{
    static const double v = [] {
        const char *e = getenv("MCAPQ_STEP_REC_R");
        return e ? atof(e) : 0.75;
    }();
    return v;
}

int64_t stack_rec_min_k()
{
    static const int64_t v = [] {
        const char *e = getenv("MCAPQ_STEP_REC_MINK");
        return e ? (int64_t)atoll(e) : (int64_t)4096;
    }();
    return v;
}

// One cluster of 2 per SM pair over the whole grid (1 CTA per SM: the step's shared
// memory), checked once with the occupancy API; otherwise the plain cooperative launch.
bool stack_clustered()
{
    static int v = -1;
    if (v >= 0) return v != 0;
    v = 0;
    if (getenv("MCAPQ_STEP_CLUSTER") && atoi(getenv("MCAPQ_STEP_CLUSTER")) == 0) return false;
    const void *f = reinterpret_cast<const void *>(stack_step<false, 2>);
    if (kernel_smem_attr(f, 227 * 1024) != cudaSuccess) return false;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(device_sms());
    cfg.blockDim = dim3(kStepThreads);
    cfg.dynamicSmemBytes = 200 * 1024;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, f, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    v = (2 * n >= device_sms() && device_sms() % 2 == 0) ? 1 : 0;
    return v != 0;
}

cudaError_t launch_stack_step(const void *ops_dev, const void *part_dev, int nops, unsigned int *counters_dev,
                              int64_t max_k, bool clustered, int route_kinds, cudaStream_t s)
{
    for (const void *f : {reinterpret_cast<const void *>(stack_step<false, 2>),
                          reinterpret_cast<const void *>(stack_step<true, 2>),
                          reinterpret_cast<const void *>(stack_step<false, 4>),
                          reinterpret_cast<const void *>(stack_step<true, 4>),
                          reinterpret_cast<const void *>(stack_step<false, 2, 1>),
                          reinterpret_cast<const void *>(stack_step<false, 2, 2>),
                          reinterpret_cast<const void *>(stack_step<false, 4, 1>),
                          reinterpret_cast<const void *>(stack_step<false, 4, 2>)}) {
        cudaError_t e = kernel_smem_attr(f, 227 * 1024);
        if (e != cudaSuccess) return e;
    }
    StackArgs a;
    memset(&a, 0, sizeof(a));
    a.ops = reinterpret_cast<const StackOp *>(ops_dev);
    a.nops = nops;
    a.counters = counters_dev;
    a.flags = tune().step_flags;
    a.spin_ns = tune().step_spin_ns;
    a.polls = tune().step_polls;
    a.ep_log2 = tune().step_ep_log2;
    a.hold = tune().step_hold;
    a.rec_spin = tune().step_rec_spin;
    // one CTA per SM: activations for the largest K under either route, the rest is ring
    const size_t act = round_up(act_bytes(HMMA1, max_k, 1) > act_bytes(DP4A, max_k, 1) ? act_bytes(HMMA1, max_k, 1)
                                                                                           : act_bytes(DP4A, max_k, 1),
                                128);
    const size_t budget = (size_t)tune().step_smem_kb * 1024;
    const size_t prog_ops = round_up(sizeof(StackOp) * (size_t)nops, 16);
    const size_t prog = round_up(prog_ops + sizeof(int2) * (size_t)nops, 128);   // ops + this CTA's ranges
    int S = (int)(((long)budget - 1024 - (long)kBarBytes - (long)prog - (long)act - kRedBytes) / kStageBytes);
    S = S < 2 ? 2 : (S > kMaxStages ? kMaxStages : S);
    S = S > 13 ? 13 : S;   // the step's barrier area: 16 S + 288 bytes <= kBarBytes
    a.stages = S;
    a.ops_off = S * kStageBytes + kBarBytes;
    a.part_off = (int)(a.ops_off + prog_ops);
    a.part = reinterpret_cast<const int2 *>(part_dev);
    a.act_off = (int)(a.ops_off + prog);
    a.red_off = (int)(a.act_off + act);
    const size_t smem = 1024 + (size_t)a.red_off + kRedBytes;
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    const int grid = device_sms();
    if (tune().trace) {
        // debug timeline: [op][cta] records at the start of the trace buffer
        constexpr size_t kCap = 1u << 20;
        if (!g_trace && cudaMalloc(&g_trace, kCap * 64) != cudaSuccess) g_trace = nullptr;
        if (g_trace && 2 * (size_t)nops * grid <= kCap) {
            a.trace = g_trace;
            g_trace_used = 2 * (size_t)nops * grid;   // + the epilogue records
        }
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kStepThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    a.clustered = (clustered && stack_clustered()) ? 1 : 0;
    if (a.clustered) {
        // clusters of 2 (paired tiles); all CTAs co-resident: one per SM, and the
        // occupancy check found room for every cluster
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
    } else {
        attr[0].id = cudaLaunchAttributeCooperative;   // all CTAs co-resident: the grid barrier is safe
        attr[0].val.cooperative = 1;
    }
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // route_kinds: bit 0 = some W4A8 linear, bit 1 = some W4A16 linear (a single-route
    // program takes the instantiation without the other engine)
    const int kinds = a.trace ? 3 : (route_kinds & 3);
    if (max_k <= 8192) {
        if (a.trace) return cudaLaunchKernelEx(&cfg, stack_step<true, 2>, a);
        if (kinds == 1) return cudaLaunchKernelEx(&cfg, stack_step<false, 2, 1>, a);
        if (kinds == 2) return cudaLaunchKernelEx(&cfg, stack_step<false, 2, 2>, a);
        return cudaLaunchKernelEx(&cfg, stack_step<false, 2>, a);
    }
    if (a.trace) return cudaLaunchKernelEx(&cfg, stack_step<true, 4>, a);
    if (kinds == 1) return cudaLaunchKernelEx(&cfg, stack_step<false, 4, 1>, a);
    if (kinds == 2) return cudaLaunchKernelEx(&cfg, stack_step<false, 4, 2>, a);
    return cudaLaunchKernelEx(&cfg, stack_step<false, 4>, a);
}

size_t stream_trace_read(unsigned long long *host_out, size_t max_records)
{
    if (!g_trace) return 0;
    const size_t n = g_trace_used < max_records ? g_trace_used : max_records;
    if (cudaDeviceSynchronize() != cudaSuccess) return 0;
    if (cudaMemcpy(host_out, g_trace, n * 64, cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
    return n;
}

// ------------------------------------------------------------------ NEXT-2 greedy decode
namespace {
// keys[i] = max_n argmax_key(logits[i][n], row_off + n): one CTA per token row
__global__ void argmax_rows_kernel(const float *__restrict__ logits, int64_t n, int64_t ld, int64_t row_off,
                                   unsigned long long *keys)
{
    __shared__ unsigned long long wbest[32];
    const float *row = logits + (int64_t)blockIdx.x * ld;
    unsigned long long best = 0ull;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
        const unsigned long long key = argmax_key(row[j], row_off + j);
        best = key > best ? key : best;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long v = __shfl_xor_sync(0xffffffffu, best, o);
        best = v > best ? v : best;
    }
    if ((threadIdx.x & 31) == 0) wbest[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x < 32) {
        best = threadIdx.x < blockDim.x / 32 ? wbest[threadIdx.x] : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long v = __shfl_xor_sync(0xffffffffu, best, o);
            best = v > best ? v : best;
        }
        if (threadIdx.x == 0) keys[blockIdx.x] = best;
    }
}

__global__ void argmax_combine_kernel(const unsigned long long *keys, int parts, int64_t m, int64_t *idx, float *val)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long best = 0ull;
        for (int p = 0; p < parts; ++p) {
            const unsigned long long v = keys[(int64_t)p * m + i];
            best = v > best ? v : best;
        }
        idx[i] = (int64_t)(0xffffffffu - (uint32_t)(best & 0xffffffffull));
        if (val) val[i] = argmax_key_value(best);
    }
}
}  // namespace

cudaError_t launch_argmax_rows(const float *logits, int64_t m, int64_t n, int64_t ld, int64_t row_off,
                               unsigned long long *keys, cudaStream_t s)
{
    argmax_rows_kernel<<<(unsigned)m, 512, 0, s>>>(logits, n, ld, row_off, keys);
    return cudaGetLastError();
}

cudaError_t launch_argmax_combine(const unsigned long long *keys, int parts, int64_t m, int64_t *idx, float *val,
                                  cudaStream_t s)
{
    argmax_combine_kernel<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(keys, parts, m, idx, val);
    return cudaGetLastError();
}

// M = 1 on the stream path: the linear's epilogue folds every row into the argmax key
cudaError_t launch_argmax_fused(int route, const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k,
                                const uint16_t *x, int64_t row_off, unsigned long long *key, cudaStream_t s)
{
    cudaError_t e = cudaMemsetAsync(key, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    StreamArgs a;
    memset(&a, 0, sizeof(a));
    a.count = 1;
    if (!encode_maps(&a.maps[0][0], &a.maps[0][1], nib, scale, n, k)) return cudaErrorInvalidValue;
    a.n[0] = n;
    a.ldy[0] = n;
    a.tile_start[0] = 0;
    a.tile_start[1] = (int)((n + kTileRows - 1) / kTileRows);
    a.k = k;
    a.x = x;
    a.ldx = k;
    a.ntok = 1;
    a.ydt = MCAPQ_F32;
    a.amax_key = key;
    a.amax_off = row_off;
    const bool one_cta = route == MCAPQ_W4A16 && kHmma1Blocks == 1;
    const int per_sm = tune().ctas_per_sm ? tune().ctas_per_sm
                                          : (one_cta ? 1 : (a.tile_start[1] >= 16 * device_sms() ? 2 : 1));
    a.smem_kb = (!tune().smem_kb_env && per_sm == 1 && k >= 8192) ? 130 : 0;
    const bool pdl = tune().pdl || api_pdl();
    return route == MCAPQ_W4A16 ? launch_one<HMMA1>(a, s, pdl, device_sms() * per_sm)
                                : launch_one<DP4A>(a, s, pdl, device_sms() * per_sm);
}

namespace {
// q [k] int8, sx / sq [G] from the DUMP engine's copy of the staged activations
__global__ void unpack_stream_dump(const uint32_t *act, int64_t k, int8_t *q, float *sx, int32_t *sq)
{
    const int G = (int)(k / 32);
    const uint8_t *b = reinterpret_cast<const uint8_t *>(act);
    const uint32_t *ssq = act + k / 4;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < k; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = j / 32, t = j % 32;
        q[j] = (int8_t)b[(t < 16 ? 0 : k / 2) + 16 * g + (t & 15)];
        if (t == 0) {
            sx[g] = __uint_as_float(ssq[2 * g]);
            sq[g] = (int32_t)ssq[2 * g + 1] / 8;
        }
    }
    (void)G;
}
}  // namespace

size_t stream_dump_workspace_bytes(int64_t k) { return (size_t)(k / 4 + 2 * (k / 32)) * 4; }

cudaError_t launch_stream_dump(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k, const uint16_t *x,
                               int8_t *q, float *sx, int32_t *sq, int32_t *D, void *ws, cudaStream_t s)
{
    StreamArgs a;
    memset(&a, 0, sizeof(a));
    a.count = 1;
    if (!encode_maps(&a.maps[0][0], &a.maps[0][1], nib, scale, n, k)) return cudaErrorInvalidValue;
    a.n[0] = n;
    a.y[0] = nullptr;
    a.ldy[0] = n;
    a.tile_start[0] = 0;
    a.tile_start[1] = (int)((n + kTileRows - 1) / kTileRows);
    a.k = k;
    a.x = x;
    a.ldx = k;
    a.ntok = 1;
    a.ydt = MCAPQ_F32;
    a.dump_d = D;
    a.dump_act = reinterpret_cast<uint32_t *>(ws);
    cudaError_t e = launch_one<DUMP>(a, s, false, device_sms());
    if (e != cudaSuccess) return e;
    unpack_stream_dump<<<(unsigned)((k + 255) / 256), 256, 0, s>>>(a.dump_act, k, q, sx, sq);
    return cudaGetLastError();
}

bool stream_supported(int64_t k) { return k >= 2048 && k % 256 == 0 && encode_fn() != nullptr; }

int stream_tokens_per_pass(int route, int64_t k)
{
    // activations of up to 8 tokens, as long as >= 2 ring stages fit the ~112 KB plan
    const int engine = route == MCAPQ_W4A16 ? HMMA : IMMA;
    int tp = 8;
    while (tp > 1) {
        const size_t need = 1024 + kBarBytes +
                            round_up(act_bytes(engine, k, tp), 128) + kRedBytes + 2 * (size_t)kStageBytes;
        if (need <= 112 * 1024) break;
        --tp;
    }
    return tp;
}

cudaError_t launch_stream_group(int route, const StreamGroup &g, const uint16_t *x, int64_t m, int64_t ldx, int ydt,
                                cudaStream_t s, bool pdl)
{
    StreamArgs a;
    memset(&a, 0, sizeof(a));
    a.count = g.count;
    int tiles = 0;
    for (int i = 0; i < g.count; ++i) {
        if (!encode_maps(&a.maps[i][0], &a.maps[i][1], g.nib[i], g.scale[i], g.n[i], g.k))
            return cudaErrorInvalidValue;
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
    a.npeers = (m == 1 && g.npeers > 0) ? (g.npeers < kMaxPeers ? g.npeers : kMaxPeers) : 0;
    for (int p = 0; p < a.npeers; ++p) a.peer_delta[p] = g.peer_delta[p];
    // grid: one CTA per SM leaves room for the next linear's CTA under PDL (hides the
    // ramp of back-to-back linears); a long linear (>= 16 tiles per SM) instead runs two
    // CTAs per SM -- twice the consumer warps per SM, and its ramp is amortised anyway
    // (8B lm_head: 6.08 -> 6.47 TB/s).  MCAPQ_STREAM_CTAS_PER_SM forces 1 or 2.
    // (the W4A16 M = 1 engine runs one CTA per SM: its lean loop keeps its lane offsets in
    // registers -- 86 of them -- instead of re-deriving them under the 56-register cap of
    // two CTAs per SM: 8B lm_head 80.9 -> 66.3 us, gate 13.4 -> 10.5 us)
    // (a mid-size grouped linear, 10-16 tiles per SM -- the 8B gate+up -- also runs two CTAs per
    // SM, at 96 KB each: 14.5 -> 13.3 us; a single 8B gate at 6 tiles per SM stays at one)
    const bool one_cta = route == MCAPQ_W4A16 && m == 1 && kHmma1Blocks == 1;
    const bool mid = tiles >= 10 * device_sms() && tiles < 16 * device_sms();
    const int per_sm = tune().ctas_per_sm ? tune().ctas_per_sm
                                          : (one_cta ? 1 : (tiles >= 16 * device_sms() || mid ? 2 : 1));
    const int sms = device_sms() * per_sm;
    // shared-memory plan: ~112 KB (two CTAs per SM: the next linear's CTA co-resides under
    // PDL); a wide input (K >= 8192: a 9-15 KB activation area) at one CTA per SM takes
    // 130 KB instead -- two more ring stages beat the PDL overlap there (1B down 6.2 ->
    // 4.8 us, 8B down 11.3 -> 10.6 us; 8B gate at K = 4096 stays faster at 112 KB).
    // MCAPQ_STREAM_SMEM_KB overrides both.
    a.smem_kb = tune().smem_kb_env ? 0 : (per_sm == 1 && g.k >= 8192 ? 130 : (per_sm == 2 && mid ? 96 : 0));
    const int tp = stream_tokens_per_pass(route, g.k);
    pdl = pdl || tune().pdl || api_pdl();
    for (int64_t tok0 = 0; tok0 < m; tok0 += tp) {
        a.tok0 = tok0;
        a.ntok = (int)((m - tok0) < tp ? (m - tok0) : tp);
        cudaError_t e;
        if (tune().nocompute)
            e = launch_one<NONE>(a, s, pdl, sms);
        else if (route == MCAPQ_W4A16)
            e = a.ntok == 1 ? launch_one<HMMA1>(a, s, pdl, sms) : launch_one<HMMA>(a, s, pdl, sms);
        else if (a.ntok == 1)
            e = launch_one<DP4A>(a, s, pdl, sms);
        else
            e = launch_one<IMMA>(a, s, pdl, sms);
        if (e != cudaSuccess) return e;
        pdl = true;
    }
    return cudaSuccess;
}

cudaError_t launch_linear_peers(int route, const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k,
                                const uint16_t *x, void *y, int ydt, const int64_t *delta, int npeers, cudaStream_t s)
{
    if (npeers < 1 || npeers > kMaxPeers) return cudaErrorInvalidValue;
    StreamGroup g = {};
    g.count = 1;
    g.k = k;
    g.nib[0] = nib;
    g.scale[0] = scale;
    g.n[0] = n;
    g.y[0] = y;
    g.ldy[0] = n;
    g.npeers = npeers;
    for (int p = 0; p < npeers; ++p) g.peer_delta[p] = delta[p];
    return launch_stream_group(route, g, x, 1, k, ydt, s, false);
}

}  // namespace mcapq
