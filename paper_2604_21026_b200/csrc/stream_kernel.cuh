// stream_kernel.cuh -- the persistent TMA-fed decode-linear kernel (included by
// kernels_stream.cu, which holds the PTX helpers, fragments and host launch).
//
// Shared memory (dynamic, 1024-B aligned base sb; all offsets are 32-bit shared
// addresses):  ring [S x 18 KiB] | full[S] empty[S] xbar | x raw | activations | reduction
// Activation layouts (per token, tsz bytes apart):
//  W4A8 : q_lo [G][16] | q_hi [G][16] | 16 B pad   (q_lo = elements 0..15 of each
//         32-group, q_hi = 16..31: lane-per-block LDS.128 are consecutive), then
//         sx [ntok][G] fp32 and sq [ntok][G] int32 after all tokens.
//  W4A16: [G][4 t][8 bf16] in fragment order (4t,4t+2,4t+1,4t+3,4t+16,4t+18,4t+17,4t+19) | 64 B pad,
//         then corr [G][8 tokens] fp32 = -136 * sum_j x_j of the group (see HMMA below).
#pragma once

template <int E>
// 2 CTAs per SM (<= 60 registers, <= ~113 KB smem): under PDL the next linear's CTA
// becomes resident beside this one and starts its weight stream early.
__global__ void __launch_bounds__(kThreads, 2) stream_linear(const __grid_constant__ StreamArgs a)
{
    extern __shared__ __align__(16) uint8_t smem_raw[];
    const uint32_t sraw = smem_addr(smem_raw);
    const uint32_t sb = (sraw + 1023u) & ~1023u;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t k = a.k;
    const int G = (int)(k / 32);
    const int K2 = (int)(k / 2);
    const int nchunks = (K2 + kChunkBytes - 1) / kChunkBytes;
    const int S = a.stages;

    const uint32_t ring = sb;
    const uint32_t full = sb + (uint32_t)S * kStageBytes;       // S x 8 B
    const uint32_t empty = full + 8u * S;                        // S x 8 B
    const uint32_t xbar = empty + 8u * S;
    const uint32_t xraw = sb + a.xraw_off;
    const uint32_t act = sb + a.act_off;
    const uint32_t red = sb + a.red_off;

    const int T = a.tile_start[a.count];
    const int t0 = (int)(((int64_t)T * blockIdx.x) / gridDim.x);
    const int t1 = (int)(((int64_t)T * (blockIdx.x + 1)) / gridDim.x);

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + 8u * s, 1);
            mbar_init(empty + 8u * s, kConsumerWarps);
        }
        mbar_init(xbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    dev::griddep_launch();   // the next linear may launch: it only touches weights until its own wait
    unsigned long long tr_start = 0, tr_wait = 0, tr_ready = 0, tr_x = 0, tr_first = 0;
    if (a.trace) tr_start = globaltimer();

    if (warp == kConsumerWarps) {
        // ================= producer =================
        if (lane == 0) {
            for (int i = 0; i < a.count; ++i) {
                asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(a.maps[i])) : "memory");
                asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(a.maps[i] + 1)) : "memory");
            }
            const uint64_t pol = evict_first_policy();
            int s = 0;
            uint32_t ph = 0;
            int li = 0;
            for (int tile = t0; tile < t1; ++tile) {
                while (li + 1 < a.count && tile >= a.tile_start[li + 1]) ++li;
                const int row0 = (tile - a.tile_start[li]) * kTileRows;
                for (int ch = 0; ch < nchunks; ++ch) {
                    mbar_wait(empty + 8u * s, ph ^ 1u);
                    const uint32_t st = ring + (uint32_t)s * kStageBytes;
                    const uint32_t fb = full + 8u * s;
                    // full boxes always: TMA zero-fills rows past N / columns past K and counts them
                    mbar_expect_tx(fb, (uint32_t)kStageBytes);
                    tma_3d(st, a.maps[li], 0, row0, ch * 8, fb, pol);
                    tma_2d(st + 8 * kBox, a.maps[li] + 1, ch * kChunkBlocks, row0, fb, pol);
                    if (++s == S) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            }
        }
        return;
    }

    // ================= consumers: stage activations =================
    dev::griddep_wait();
    if (a.trace) tr_wait = globaltimer();
    const int ntok = a.ntok;
    // x is read straight from global (L2) by all consumer threads in parallel: one
    // memory round trip, no serial copy + barrier on the dependent-kernel chain
    const uint16_t *xg = a.x + a.tok0 * a.ldx;
    (void)xraw;
    (void)xbar;
    constexpr bool kA16 = (E == HMMA || E == HMMA1 || E == NONE);
    const uint32_t tsz = kA16 ? (uint32_t)(2 * k + 64) : (uint32_t)(k + 16);
    const uint32_t sx_s = act + (uint32_t)ntok * tsz;                    // W4A8: [ntok][G] fp32
    const uint32_t sq_s = sx_s + 4u * (uint32_t)(ntok * G);              // W4A8: [ntok][G] int32
    const uint32_t corr_s = act + (uint32_t)ntok * tsz;                  // W4A16: [G][8] fp32
    if constexpr (!kA16) {
        // Per-token, per-32-group quantisation, a quad of threads per
        // group (8 elements each): the same IEEE operations as quant_a8_kernel
        // (exact max, __fdiv_rn, roundf, clamp, exact int sum), so q / s / sum q are
        // bit-identical.  All lanes of a warp run the same trip count (quad shuffles).
        const int nq = ntok * G * 4;
        for (int base = 0; base < nq; base += kConsumerWarps * 32) {
            const int idx = base + threadIdx.x;
            const bool on = idx < nq;
            const int grp = on ? (idx >> 2) : 0, sub = idx & 3;
            const int i = grp / G, g = grp - i * G;
            const uint4 u = ldg_nc_128(xg + i * a.ldx + 32 * g + 8 * sub);
            const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
            float v[8];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                v[2 * e] = __uint_as_float(w4[e] << 16);
                v[2 * e + 1] = __uint_as_float(w4[e] & 0xffff0000u);
            }
            float amax = 0.0f;
            int fin = 1;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                fin &= isfinite(v[j]) ? 1 : 0;
                amax = fmaxf(amax, fabsf(v[j]));
            }
            if (a.trace && base == 0) tr_x = globaltimer();   // x of the first pass has arrived
            amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 1));
            amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 2));
            fin &= __shfl_xor_sync(0xffffffffu, fin, 1);
            fin &= __shfl_xor_sync(0xffffffffu, fin, 2);
            const float s = __fdiv_rn(amax, 127.0f);
            const bool live = fin && s != 0.0f;
            const float inv = __frcp_rn(s);
            uint32_t lo = 0, hi = 0;
            int sum = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int code = live ? quant_code(v[j], s, inv) : 0;
                sum += code;
                if (j < 4)
                    lo |= ((uint32_t)code & 0xffu) << (8 * j);
                else
                    hi |= ((uint32_t)code & 0xffu) << (8 * (j - 4));
            }
            sum += __shfl_xor_sync(0xffffffffu, sum, 1);
            sum += __shfl_xor_sync(0xffffffffu, sum, 2);
            if (on) {
                // elements 8sub..8sub+7: sub 0/1 -> q_lo, sub 2/3 -> q_hi
                const uint32_t qt = act + (uint32_t)i * tsz + (sub < 2 ? 0u : (uint32_t)K2) + 16u * g + 8u * (sub & 1);
                asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(qt), "r"(lo), "r"(hi) : "memory");
                if (sub == 0) {
                    sts32(sx_s + 4u * (uint32_t)(i * G + g), __float_as_uint(live ? s : 0.0f));
                    sts32(sq_s + 4u * (uint32_t)(i * G + g), (uint32_t)sum);
                }
            }
        }
    } else {
        // tokens >= ntok contribute a zero accumulator init
        for (int idx = threadIdx.x; idx < G * 8; idx += kConsumerWarps * 32)
            if ((idx & 7) >= ntok) sts32(corr_s + 4u * (uint32_t)idx, 0u);
        const int nq = ntok * G * 4;
        for (int base = 0; base < nq; base += kConsumerWarps * 32) {
            const int idx = base + threadIdx.x;
            const bool on = idx < nq;
            const int q = on ? idx : 0;
            const int tk = q / (G * 4), rem = q - tk * G * 4, g = rem >> 2, tt = rem & 3;
            const uint16_t *src = xg + tk * a.ldx + 32 * g + 4 * tt;
            const uint2 lo = ldg_nc_64(src);        // x[4t..4t+3]
            const uint2 hi = ldg_nc_64(src + 16);   // x[4t+16..4t+19]
            // corr[g][tok] = -136 * sum of the group's 32 x in fp32 (fixed order: this
            // thread's 8 in sequence, then the quad butterfly)
            float part = 0.0f;
            const uint32_t e8[4] = {lo.x, lo.y, hi.x, hi.y};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                part += __uint_as_float(e8[e] << 16);
                part += __uint_as_float(e8[e] & 0xffff0000u);
            }
            part += __shfl_xor_sync(0xffffffffu, part, 1);
            part += __shfl_xor_sync(0xffffffffu, part, 2);
            if (on) {
                uint4 o;
                o.x = __byte_perm(lo.x, lo.y, 0x5410);
                o.y = __byte_perm(lo.x, lo.y, 0x7632);
                o.z = __byte_perm(hi.x, hi.y, 0x5410);
                o.w = __byte_perm(hi.x, hi.y, 0x7632);
                sts128(act + (uint32_t)tk * tsz + 64u * g + 16u * tt, o);
                if (tt == 0) sts32(corr_s + 4u * (uint32_t)(g * 8 + tk), __float_as_uint(-136.0f * part));
            }
        }
    }
    bar_consumers();
    if (a.trace) tr_ready = globaltimer();

    // ================= consumers: main loop =================
    const int gid = lane >> 2, t = lane & 3;
    const int mrow = (lane & 7) + ((lane >> 3) & 1) * 8;    // ldmatrix row of this lane
    const int mhalf = lane >> 4;                             // ldmatrix: lanes 16-31 address the 2nd block
    uint32_t kNib2 = 0x000F000Fu, kMagic = 0x43004300u;      // in registers: one LOP3 per bf16 pair
    asm volatile("" : "+r"(kNib2), "+r"(kMagic));
    int s = 0;
    uint32_t ph = 0;
    int li = 0;
    for (int tile = t0; tile < t1; ++tile) {
        while (li + 1 < a.count && tile >= a.tile_start[li + 1]) ++li;
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        for (int ch = 0; ch < nchunks; ++ch) {
            const int rem = K2 - ch * kChunkBytes;
            const int nblk = (rem < kChunkBytes ? rem : kChunkBytes) / 16;
            const int blk0 = ch * kChunkBlocks;
            mbar_wait(full + 8u * s, ph);
            if (a.trace && tr_first == 0) tr_first = globaltimer();   // first weight stage available
            const uint32_t st = ring + (uint32_t)s * kStageBytes;

            if constexpr (E == NONE) {
                // bandwidth probe: drain the stage without computing
            } else if constexpr (E == DP4A) {
                // warp w: row w of the tile; lane l: blocks l and l+32 of the chunk (in that order)
                const int r = warp;
                if (nblk == kChunkBlocks) {
                    // full chunk: no predicates, both blocks' load/dp4a chains interleave
                    const int g0 = blk0 + lane, g1 = g0 + 32;
                    const uint4 w0 = lds128(st + nib_off(r, lane));
                    const uint4 w1 = lds128(st + nib_off(r, lane + 32));
                    const uint4 qa0 = lds128(act + 16u * g0), qb0 = lds128(act + (uint32_t)K2 + 16u * g0);
                    const uint4 qa1 = lds128(act + 16u * g1), qb1 = lds128(act + (uint32_t)K2 + 16u * g1);
                    const float d0 = h2f(lds16(st + scale_off(r, lane)));
                    const float d1 = h2f(lds16(st + scale_off(r, lane + 32)));
                    const float s0 = __uint_as_float(lds32(sx_s + 4u * g0));
                    const float s1 = __uint_as_float(lds32(sx_s + 4u * g1));
                    const int D0 = block_sumi_dp4a(w0, make_int4(qa0.x, qa0.y, qa0.z, qa0.w),
                                                   make_int4(qb0.x, qb0.y, qb0.z, qb0.w)) - 8 * (int)lds32(sq_s + 4u * g0);
                    const int D1 = block_sumi_dp4a(w1, make_int4(qa1.x, qa1.y, qa1.z, qa1.w),
                                                   make_int4(qb1.x, qb1.y, qb1.z, qb1.w)) - 8 * (int)lds32(sq_s + 4u * g1);
                    acc[0] = fmaf(d0 * s0, (float)D0, acc[0]);
                    acc[0] = fmaf(d1 * s1, (float)D1, acc[0]);
                } else {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int b = lane + 32 * h;
                        if (b < nblk) {
                            const int g = blk0 + b;
                            const uint4 qa = lds128(act + 16u * g), qb = lds128(act + (uint32_t)K2 + 16u * g);
                            const uint4 w = lds128(st + nib_off(r, b));
                            const int D = block_sumi_dp4a(w, make_int4(qa.x, qa.y, qa.z, qa.w),
                                                          make_int4(qb.x, qb.y, qb.z, qb.w)) - 8 * (int)lds32(sq_s + 4u * g);
                            acc[0] = fmaf(h2f(lds16(st + scale_off(r, b))) * __uint_as_float(lds32(sx_s + 4u * g)),
                                          (float)D, acc[0]);
                        }
                    }
                }
            } else {
                // warp w: blocks 4w .. 4w+3 of the chunk (contiguous; in that order) for all 16 rows
                const int bq = 4 * warp;
                if (bq < nblk) {
                    uint32_t wv[8];   // [block j][row half]: wa(j) = wv[2j], wb(j) = wv[2j+1]
                    ldmatrix_x4(st + nib_off(mrow, bq + mhalf), wv[0], wv[1], wv[2], wv[3]);
                    ldmatrix_x4(st + nib_off(mrow, bq + 2 + mhalf), wv[4], wv[5], wv[6], wv[7]);
                    // scales of rows gid / gid+8 for the 4 blocks: one 8-byte load each
                    const uint2 sa = lds64(st + scale_off(gid, bq));
                    const uint2 sbb = lds64(st + scale_off(gid + 8, bq));
                    const float dA[4] = {h2f((uint16_t)(sa.x & 0xffff)), h2f((uint16_t)(sa.x >> 16)),
                                         h2f((uint16_t)(sa.y & 0xffff)), h2f((uint16_t)(sa.y >> 16))};
                    const float dB[4] = {h2f((uint16_t)(sbb.x & 0xffff)), h2f((uint16_t)(sbb.x >> 16)),
                                         h2f((uint16_t)(sbb.y & 0xffff)), h2f((uint16_t)(sbb.y >> 16))};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t wa = wv[2 * j], wb = wv[2 * j + 1];
                        const int g = blk0 + bq + j;
                        if constexpr (E == IMMA) {
                            uint32_t b0 = 0, b1 = 0;
                            if (gid < ntok) {
                                const uint32_t qt = act + (uint32_t)gid * tsz;
                                b0 = lds32(qt + 16u * g + 4u * t);
                                b1 = lds32(qt + (uint32_t)K2 + 16u * g + 4u * t);
                            }
                            int c[4];
                            imma(wa, wb, b0, b1, c);
                            const int c0 = 2 * t, c1 = 2 * t + 1;
                            const float s0 = c0 < ntok ? __uint_as_float(lds32(sx_s + 4u * (c0 * G + g))) : 0.f;
                            const float s1 = c1 < ntok ? __uint_as_float(lds32(sx_s + 4u * (c1 * G + g))) : 0.f;
                            const int q0 = c0 < ntok ? (int)lds32(sq_s + 4u * (c0 * G + g)) : 0;
                            const int q1 = c1 < ntok ? (int)lds32(sq_s + 4u * (c1 * G + g)) : 0;
                            acc[0] = fmaf(dA[j] * s0, (float)(c[0] - 8 * q0), acc[0]);
                            acc[1] = fmaf(dA[j] * s1, (float)(c[1] - 8 * q1), acc[1]);
                            acc[2] = fmaf(dB[j] * s0, (float)(c[2] - 8 * q0), acc[2]);
                            acc[3] = fmaf(dB[j] * s1, (float)(c[3] - 8 * q1), acc[3]);
                        } else {
                            // A = 128 + c (exact bf16, one LOP3 per pair, no per-element
                            // subtract); D = sum_j (128 + c_j) x_j is exact per product, and
                            // corr = -136 * sum_j x_j restores sum_j (c_j - 8) x_j in fp32.
                            uint4 bx = make_uint4(0, 0, 0, 0);
                            if (gid < ntok) bx = lds128(act + (uint32_t)gid * tsz + 64u * g + 16u * t);
                            uint32_t pa[4], pb[4];
                            magic_bf16(wa, kNib2, kMagic, pa);
                            magic_bf16(wb, kNib2, kMagic, pb);
                            float c[4];
                            hmma_c(pa[0], pb[0], pa[2], pb[2], bx.x, bx.y, 0.f, 0.f, 0.f, 0.f, c);
                            hmma(pa[1], pb[1], pa[3], pb[3], bx.z, bx.w, c);
                            if constexpr (E == HMMA1) {
                                // one token: only column 0 (lanes t == 0) is live
                                const float crx = __uint_as_float(lds32(corr_s + 32u * g));
                                acc[0] = fmaf(dA[j], c[0] + crx, acc[0]);
                                acc[2] = fmaf(dB[j], c[2] + crx, acc[2]);
                            } else {
                                const uint2 cru = lds64(corr_s + 32u * g + 8u * t);
                                const float crx = __uint_as_float(cru.x), cry = __uint_as_float(cru.y);
                                acc[0] = fmaf(dA[j], c[0] + crx, acc[0]);
                                acc[1] = fmaf(dA[j], c[1] + cry, acc[1]);
                                acc[2] = fmaf(dB[j], c[2] + crx, acc[2]);
                                acc[3] = fmaf(dB[j], c[3] + cry, acc[3]);
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
        // ---- tile epilogue: fixed-order reductions, store
        const int64_t row0 = (int64_t)(tile - a.tile_start[li]) * kTileRows;
        const int64_t n = a.n[li];
        if constexpr (E == DP4A) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], off);
            if (lane == 0) {
                const int64_t row = row0 + warp;
                if (row < n) dev::store_out(a.y[li], a.ydt, a.tok0 * a.ldy[li] + row, acc[0]);
            }
        } else {
            const uint32_t rw = red + 512u * warp;
            const int c0 = 2 * t, c1 = 2 * t + 1;
            sts32(rw + 4u * (gid * 8 + c0), __float_as_uint(acc[0]));
            sts32(rw + 4u * (gid * 8 + c1), __float_as_uint(acc[1]));
            sts32(rw + 4u * ((gid + 8) * 8 + c0), __float_as_uint(acc[2]));
            sts32(rw + 4u * ((gid + 8) * 8 + c1), __float_as_uint(acc[3]));
            bar_consumers();
            if (threadIdx.x < 128) {
                const int r = threadIdx.x >> 3, tk = threadIdx.x & 7;
                float sum = __uint_as_float(lds32(red + 4u * threadIdx.x));
#pragma unroll
                for (int w = 1; w < kConsumerWarps; ++w) sum += __uint_as_float(lds32(red + 512u * w + 4u * threadIdx.x));
                const int64_t row = row0 + r;
                if (row < n && tk < ntok) dev::store_out(a.y[li], a.ydt, (a.tok0 + tk) * a.ldy[li] + row, sum);
            }
            bar_consumers();
        }
    }
    if (a.trace && threadIdx.x == 0) {
        unsigned long long *r = a.trace + 8ull * (unsigned long long)blockIdx.x;
        r[0] = (unsigned long long)a.launch_id;
        r[1] = blockIdx.x;
        r[2] = tr_start;
        r[3] = tr_wait;
        r[4] = tr_ready;
        r[5] = globaltimer();
        r[6] = tr_x;
        r[7] = tr_first;
    }
}
