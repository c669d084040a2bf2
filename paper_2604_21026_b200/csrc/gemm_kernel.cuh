// gemm_kernel.cuh -- batched decode, rows a5 (W4A8) / a6 (W4A16) for M = 9..64 tokens
// per pass (included by kernels_stream.cu after the PTX helpers and fragments).
//
// One pass streams every weight ONCE for all the pass's tokens (the M <= 8 stream
// kernel instead holds all of K's activations beside its ring, which caps a pass at
// 8 tokens).  A CTA owns a BN-row x Mp-token output tile and walks K in slices of
// 256 (8 Q4_0 blocks):
//   producer warp: per slice one TMA box of nibbles {128 B, BN rows} (128B swizzle),
//                  one TMA box of scales {8, BN}, and one bulk copy per token of the
//                  slice's activations (W4A8: q 256 B + s 32 B + sq 32 B from the
//                  quant_a8 workspace; W4A16: 512 B of bf16 x) into an mbarrier ring;
//   8 consumer warps (WR row-warps x WT token-warps): each owns MT m16 tiles x NT n8
//                  tiles; per block one MMA per (m, n) tile pair -- IMMA m16n8k32
//                  (exact int32 D = sum c q - 8 sq) or two HMMA m16n8k16 on
//                  the exact bf16 (c - 8) (A13) -- then the block's fp32 scale-
//                  accumulate, the order fixed by K only (A22).
// B fragments and per-token scalars are loaded once per (n-tile, block) and reused
// across the warp's MT m-tiles.
#pragma once

constexpr int kGemmWarps = 8;
constexpr int kGemmThreads = (kGemmWarps + 1) * 32;
constexpr int kGemmKS = 256;                 // K per slice (stage)
constexpr int kGemmMaxStages = 8;

struct GemmArgs {
    // activation maps as kernel parameters (encoded per launch; nothing cached per buffer):
    // W4A8 {q, sx, sq}, W4A16 {x} (encode_gemm_act_maps)
    alignas(64) CUtensorMap amaps[3];
    // weight maps, also kernel parameters (encoded per launch, never cached or allocated):
    // {nib box {128 B, bn}, scale box {8, bn}} (encode_gemm_maps)
    alignas(64) CUtensorMap maps[2];
    void *y;
    int64_t ldy;
    int64_t n, k;
    int ydt;
    int64_t tok0;              // first token of this pass
    int ntok;                  // tokens in this pass (<= 64)
    int mp;                    // padded tokens of the pass (activation box rows)
    int bn, wt;                // CTA rows; token-warps (row-warps = 8 / wt)
    int row_tiles;
    int stages;
    uint32_t nib_bytes, sc_off, act_off, ss_off, sq_off, stage_bytes;   // per-stage layout
    int na;                    // tc05_w4a16x: A-atom ring slots (even)
};

// IMMA m16n8k32 with an explicit int32 accumulator init (C may repeat registers)
__device__ __forceinline__ void imma_c(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1,
                                       int c0, int c1, int d[4])
{
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%11,%10,%11};"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "r"(c0), "r"(c1));
}

template <bool A8, int MT, int NT>
__global__ void __launch_bounds__(kGemmThreads, 1) gemm_w4(const __grid_constant__ GemmArgs a)
{
    extern __shared__ __align__(16) uint8_t smem_raw[];
    const uint32_t sb = (smem_addr(smem_raw) + 1023u) & ~1023u;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int S = a.stages;
    const uint32_t full = sb + (uint32_t)S * a.stage_bytes;
    const uint32_t empty = full + 8u * S;
    const int nslices = (int)(a.k / kGemmKS);
    const int G = (int)(a.k / 32);

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + 8u * s, 1);
            mbar_init(empty + 8u * s, kGemmWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    dev::griddep_launch();   // the next kernel may launch: it only touches weights until its own wait

    if (warp == kGemmWarps) {
        // ================= producer: one thread, TMA only =================
        if (lane == 0) {
            for (int j = 0; j < 2; ++j) {
                asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(a.maps + j)) : "memory");
                asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(a.amaps + j)) : "memory");
            }
            const uint64_t pol = evict_first_policy();
            const uint32_t act_tx = A8 ? (uint32_t)a.mp * (256u + 64u) : (uint32_t)a.mp * 512u;
            const uint32_t tx = a.nib_bytes + (uint32_t)a.bn * 16u + act_tx;
            const int y0 = (int)a.tok0;
            int s = 0;
            uint32_t ph = 0;
            bool waited = false;
            for (int tile = blockIdx.x; tile < a.row_tiles; tile += gridDim.x) {
                const int row0 = tile * a.bn;
                for (int sl = 0; sl < nslices; ++sl) {
                    mbar_wait(empty + 8u * s, ph ^ 1u);
                    const uint32_t st = sb + (uint32_t)s * a.stage_bytes;
                    const uint32_t fb = full + 8u * s;
                    mbar_expect_tx(fb, tx);
                    tma_2d(st, a.maps, sl * 128, row0, fb, pol);
                    tma_2d(st + a.sc_off, a.maps + 1, sl * 8, row0, fb, pol);
                    // activations only after the predecessor (PDL); weights above never wait
                    if (!waited) {
                        dev::griddep_wait();
                        waited = true;
                    }
                    if (A8) {
                        tma_3d(st + a.act_off, a.amaps, 0, y0, sl * 2, fb, 0);
                        tma_2d(st + a.ss_off, a.amaps + 1, sl * 8, y0, fb, 0);
                        tma_2d(st + a.sq_off, a.amaps + 2, sl * 8, y0, fb, 0);
                    } else {
                        tma_3d(st + a.act_off, a.amaps, 0, y0, sl * 4, fb, 0);
                    }
                    if (++s == S) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            }
        }
        return;
    }

    // ================= consumers =================
    const int wr = warp / a.wt, wtk = warp % a.wt;
    const int gid = lane >> 2, t = lane & 3;
    const int mrow = (lane & 7) + ((lane >> 3) & 1) * 8;   // ldmatrix row of this lane
    const int mhalf = lane >> 4;                            // lanes 16-31: the second block
    const int rbase = wr * MT * 16;                         // first row of this warp in the tile
    const int tbase = wtk * NT * 8;                         // first token of this warp in the pass
    int s = 0;
    uint32_t ph = 0;
    for (int tile = blockIdx.x; tile < a.row_tiles; tile += gridDim.x) {
        f2_t acc[MT][NT][2];   // [.][.][0]: row gid, tokens (2t, 2t+1); [1]: row gid + 8
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0ull;
        for (int sl = 0; sl < nslices; ++sl) {
            mbar_wait(full + 8u * s, ph);
            const uint32_t st = sb + (uint32_t)s * a.stage_bytes;
            const uint32_t sc = st + a.sc_off;
            const uint32_t act = st + a.act_off;
#pragma unroll
            for (int gp = 0; gp < 4; ++gp) {          // pairs of blocks: one ldmatrix.x4 per m-tile
                uint32_t wv[MT][4], scA[MT], scB[MT];   // scales: blocks 2gp, 2gp+1 of rows gid, gid + 8
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    scA[mt] = lds32(sc + 16u * (uint32_t)(rbase + mt * 16 + gid) + 4u * gp);
                    scB[mt] = lds32(sc + 16u * (uint32_t)(rbase + mt * 16 + gid + 8) + 4u * gp);
                    const int r = rbase + mt * 16 + mrow, b = 2 * gp + mhalf;
                    ldmatrix_x4(st + (uint32_t)(r * 128 + ((b ^ (r & 7)) << 4)), wv[mt][0], wv[mt][1], wv[mt][2],
                                wv[mt][3]);
                }
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int g = 2 * gp + j;         // block within the slice
                    if constexpr (A8) {
                        // A: the block's nibbles split once per m-tile (low = k 4t.., high = k 4t+16..)
                        uint32_t af[MT][4];
                        f2_t dA2[MT], dB2[MT];
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt) {
                            const uint32_t wa = wv[mt][2 * j], wb = wv[mt][2 * j + 1];
                            af[mt][0] = wa & 0x0F0F0F0Fu;
                            af[mt][1] = wb & 0x0F0F0F0Fu;
                            af[mt][2] = (wa >> 4) & 0x0F0F0F0Fu;
                            af[mt][3] = (wb >> 4) & 0x0F0F0F0Fu;
                            const float da = h2f((uint16_t)(scA[mt] >> (16 * j)));
                            const float db = h2f((uint16_t)(scB[mt] >> (16 * j)));
                            dA2[mt] = f2_pack(da, da);
                            dB2[mt] = f2_pack(db, db);
                        }
                        const f2_t magic2 = f2_pack(12582912.0f, 12582912.0f);
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt) {
                            const int tk = tbase + nt * 8;
                            // q of token tk + gid, bytes 32g + 4t (low half) and + 16 (high half):
                            // smem [2][mp][128 B], 16-B unit u of row r at u ^ (r & 7)
                            const uint32_t tok = (uint32_t)(tk + gid);
                            const uint32_t qrow = act + (uint32_t)(g >> 2) * (uint32_t)a.mp * 128u + tok * 128u + 4u * t;
                            const uint32_t u0 = 2u * (uint32_t)(g & 3);
                            const uint32_t b0 = lds32(qrow + ((u0 ^ (tok & 7u)) << 4));
                            const uint32_t b1 = lds32(qrow + (((u0 + 1u) ^ (tok & 7u)) << 4));
                            const uint32_t ss0 = st + a.ss_off + (uint32_t)(tk + 2 * t) * 32u + 4u * g;
                            const uint32_t sq0 = st + a.sq_off + (uint32_t)(tk + 2 * t) * 32u + 4u * g;
                            const f2_t s2 = f2_pack_bits(lds32(ss0), lds32(ss0 + 32u));   // (s of token 2t, 2t+1)
                            // accumulator init 1.5 * 2^23 - 8 sq: the int32 result is the bit
                            // pattern of the float 1.5 * 2^23 + D (|D| < 2^17), so one FADD2
                            // recovers D exactly (no I2F, no separate - 8 sq)
                            const int m0 = 0x4B400000 - 8 * (int)lds32(sq0);
                            const int m1 = 0x4B400000 - 8 * (int)lds32(sq0 + 32u);
#pragma unroll
                            for (int mt = 0; mt < MT; ++mt) {
                                int c[4];
                                imma_c(af[mt][0], af[mt][1], af[mt][2], af[mt][3], b0, b1, m0, m1, c);
                                const f2_t Da = f2_add(f2_pack_bits((uint32_t)c[0], (uint32_t)c[1]), magic2 ^ 0x8000000080000000ull);
                                const f2_t Db = f2_add(f2_pack_bits((uint32_t)c[2], (uint32_t)c[3]), magic2 ^ 0x8000000080000000ull);
                                acc[mt][nt][0] = f2_fma(f2_mul(dA2[mt], s2), Da, acc[mt][nt][0]);
                                acc[mt][nt][1] = f2_fma(f2_mul(dB2[mt], s2), Db, acc[mt][nt][1]);
                            }
                        }
                    } else {
                        // A = c - 8, exact in bf16 (A13): element order per thread t:
                        // p0 = (4t, 4t+2) p1 = (4t+16, 4t+18) p2 = (4t+1, 4t+3) p3 = (4t+17, 4t+19);
                        // B in the same order from x[4t..4t+3], x[4t+16..4t+19] (byte permutes)
                        uint32_t bx[NT][4];
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt) {
                            const int tk = tbase + nt * 8;
                            // x of token tk + gid, elements 32g + 4t.. (8 B) and + 16: smem
                            // [4][mp][128 B], 16-B unit u of row r at u ^ (r & 7)
                            const uint32_t tok = (uint32_t)(tk + gid);
                            const uint32_t xrow = act + (uint32_t)(g >> 1) * (uint32_t)a.mp * 128u + tok * 128u +
                                                  8u * (uint32_t)(t & 1);
                            const uint32_t u0 = 4u * (uint32_t)(g & 1) + (uint32_t)(t >> 1);
                            const uint2 lo = lds64(xrow + ((u0 ^ (tok & 7u)) << 4));
                            const uint2 hi = lds64(xrow + (((u0 + 2u) ^ (tok & 7u)) << 4));
                            bx[nt][0] = __byte_perm(lo.x, lo.y, 0x5410);
                            bx[nt][1] = __byte_perm(lo.x, lo.y, 0x7632);
                            bx[nt][2] = __byte_perm(hi.x, hi.y, 0x5410);
                            bx[nt][3] = __byte_perm(hi.x, hi.y, 0x7632);
                        }
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt) {
                            uint32_t pa[4], pb[4];
                            dequant_bf16(wv[mt][2 * j], pa);
                            dequant_bf16(wv[mt][2 * j + 1], pb);
                            const float da = h2f((uint16_t)(scA[mt] >> (16 * j)));
                            const float db = h2f((uint16_t)(scB[mt] >> (16 * j)));
#pragma unroll
                            for (int nt = 0; nt < NT; ++nt) {
                                float c[4];
                                hmma_c(pa[0], pb[0], pa[2], pb[2], bx[nt][0], bx[nt][1], 0.f, 0.f, 0.f, 0.f, c);
                                hmma(pa[1], pb[1], pa[3], pb[3], bx[nt][2], bx[nt][3], c);
                                acc[mt][nt][0] = f2_fma(f2_pack(da, da), f2_pack(c[0], c[1]), acc[mt][nt][0]);
                                acc[mt][nt][1] = f2_fma(f2_pack(db, db), f2_pack(c[2], c[3]), acc[mt][nt][1]);
                            }
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + 8u * s);
            if (++s == S) {
                s = 0;
                ph ^= 1u;
            }
        }
        // ---- store: thread holds rows (gid, gid + 8) x tokens (2t, 2t + 1) of each tile pair
        dev::griddep_wait();   // outputs are ordered after the predecessor (no-op once satisfied)
        const int64_t row0 = (int64_t)tile * a.bn + rbase;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const int tk = tbase + nt * 8 + 2 * t;
                const int64_t r0 = row0 + mt * 16 + gid, r1 = r0 + 8;
                const float2 va = f2_unpack(acc[mt][nt][0]), vb = f2_unpack(acc[mt][nt][1]);
                const float v[4] = {va.x, va.y, vb.x, vb.y};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int64_t row = (e < 2) ? r0 : r1;
                    const int tok = tk + (e & 1);
                    if (row < a.n && tok < a.ntok) dev::store_out(a.y, a.ydt, (a.tok0 + tok) * a.ldy + row, v[e]);
                }
            }
    }
}
