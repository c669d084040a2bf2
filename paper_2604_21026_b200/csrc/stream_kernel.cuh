// stream_kernel.cuh -- the persistent TMA-fed kernel for ONE (grouped) linear
// (included by kernels_stream.cu after stream_engines.cuh).
//
// Shared memory (dynamic, 1024-B aligned base sb; 32-bit shared addresses):
//   ring [S x 18 KiB] | full[S] empty[S] | activations | reduction
#pragma once

// 2 CTAs per SM (<= 56 registers, <= ~113 KB smem): under PDL the next linear's CTA
// becomes resident beside this one and starts its weight stream early.  The W4A16 M = 1
// engine (HMMA1) instead runs one CTA per SM with up to 112 registers (kHmma1Blocks, see
// the launchers): its dequantise-MMA loop is instruction-bound, and at 56 registers it
// re-derived its lane offsets every stage.
template <int E>
__global__ void __launch_bounds__(kThreads, E == HMMA1 ? kHmma1Blocks : 2) stream_linear(const __grid_constant__ StreamArgs a)
{
    extern __shared__ __align__(16) uint8_t smem_raw[];
    const uint32_t sb = (smem_addr(smem_raw) + 1023u) & ~1023u;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t k = a.k;
    const int G = (int)(k / 32);
    const int K2 = (int)(k / 2);
    const int nchunks = (K2 + kChunkBytes - 1) / kChunkBytes;
    const int S = a.stages;

    const uint32_t ring = sb;
    const uint32_t full = sb + (uint32_t)S * kStageBytes;       // S x 8 B
    const uint32_t empty = full + 8u * S;                        // S x 8 B
    const uint32_t act = sb + a.act_off;
    const uint32_t red = sb + a.red_off;

    const int T = a.tile_start[a.count];
    const int t0 = (int)(((int64_t)T * blockIdx.x) / gridDim.x);
    const int t1 = (int)(((int64_t)T * (blockIdx.x + 1)) / gridDim.x);

    const uint32_t amax_slot = full + 480u;                      // greedy-decode mode: the CTA's best key
    // HMMA1 lean path: kRedSlots tile slots of 16 warps x 16 rows fp32 partials in `red`,
    // an arrival counter per slot (the 16th warp to arrive reduces the tile) and a
    // "slot consumed" mbarrier per slot (count 1: the reducing warp)
    const uint32_t rcnt = full + 256u, repe = full + 288u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + 8u * s, 1);
            mbar_init(empty + 8u * s, kConsumerWarps);
        }
        if constexpr (E == HMMA1)
            for (int j = 0; j < kRedSlots; ++j) {
                sts32(rcnt + 4u * j, 0u);
                mbar_init(repe + 8u * j, 1);
            }
        asm volatile("st.shared.u64 [%0], %1;" ::"r"(amax_slot), "l"(0ull) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    dev::griddep_launch();   // the next linear may launch: it only touches weights until its own wait
    unsigned long long tr_start = 0, tr_wait = 0, tr_ready = 0, tr_first = 0;
    if (a.trace) tr_start = globaltimer();

    if (warp == kConsumerWarps) {
        // ================= producer: weights only, never waits on the predecessor =================
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

    // ================= consumers: activations =================
    dev::griddep_wait();
    if (a.trace) tr_wait = globaltimer();
    const int ntok = a.ntok;
    constexpr bool kA16 = (E == HMMA || E == HMMA1 || E == NONE);
    const ActSmem L = act_layout(kA16, act, k, ntok);
    const uint16_t *xg = a.x + a.tok0 * a.ldx;
    if constexpr (kA16)
        stage_a16<false>(xg, a.ldx, ntok, k, L, threadIdx.x, kConsumerWarps * 32);
    else
        stage_a8<false>(xg, a.ldx, ntok, k, L, threadIdx.x, kConsumerWarps * 32);
    bar_consumers();
    if (a.trace) tr_ready = globaltimer();
    if constexpr (E == DUMP) {
        // test entry: CTA 0 copies the staged activations (q_lo | q_hi, then the {s, 8 sum q} pairs)
        if (blockIdx.x == 0) {
            const int nq = (int)(k / 4);   // q_lo | q_hi words of the one token
            for (int w = threadIdx.x; w < nq + 2 * G; w += kConsumerWarps * 32)
                a.dump_act[w] = w < nq ? lds32(L.act + 4u * (uint32_t)w) : lds32(L.ssq + 4u * (uint32_t)(w - nq));
        }
    }

    // ================= consumers: main loop =================
    uint32_t kNib2 = 0x000F000Fu, kMagic = 0x43004300u;      // in registers: one LOP3 per bf16 pair
    asm volatile("" : "+r"(kNib2), "+r"(kMagic));
    int s = 0;
    uint32_t ph = 0;
    int li = 0;
    unsigned long long best = 0ull;   // greedy-decode mode: this thread's running argmax key
    if constexpr (E == HMMA1) {
        if ((K2 & (kChunkBytes - 1)) == 0 && !a.trace) {
            // ---- lean W4A16 M = 1 loop (every chunk full: K % 2048 == 0).  No per-stage
            // predicates; the tile's cross-warp reduction is handed to whichever warp
            // arrives last at the tile's slot (no CTA-wide barrier per tile: the other
            // warps go straight on to the next tile's stages).  Same chunk_mma arithmetic
            // and the same fixed reduction order (warp 0 + warp 1 + .. + warp 15) as
            // epilogue_mma, so the outputs are bit-identical to the generic path.
            uint32_t st = ring + (uint32_t)s * kStageBytes;
            uint32_t ts = 0;
            const Hmma1Lane H = hmma1_lane(L, warp, lane);
            for (int tile = t0; tile < t1; ++tile, ++ts) {
                while (li + 1 < a.count && tile >= a.tile_start[li + 1]) ++li;
                float acc[4] = {0.f, 0.f, 0.f, 0.f};
                for (int ch = 0; ch < nchunks; ++ch) {
                    mbar_wait(full + 8u * s, ph);
                    chunk_hmma1(st, 4096u * (uint32_t)ch, 2048u * (uint32_t)ch, H, kNib2, kMagic, acc[0], acc[2]);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(empty + 8u * s);
                    if (++s == S) {
                        s = 0;
                        ph ^= 1u;
                        st = ring;
                    } else {
                        st += (uint32_t)kStageBytes;
                    }
                }
                const uint32_t slot = ts & (uint32_t)(kRedSlots - 1);
                if (ts >= (uint32_t)kRedSlots) mbar_wait(repe + 8u * slot, ((ts / kRedSlots) - 1u) & 1u);
                const uint32_t sl = red + 1024u * slot;
                // lanes t == 0 hold rows gid (acc[0]) and gid + 8 (acc[2]) of the token
                if ((lane & 3) == 0) {
                    sts32(sl + 64u * warp + 4u * (lane >> 2), __float_as_uint(acc[0]));
                    sts32(sl + 64u * warp + 4u * ((lane >> 2) + 8), __float_as_uint(acc[2]));
                }
                __syncwarp();
                uint32_t old = 0;
                if (lane == 0)
                    asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                                 : "=r"(old)
                                 : "r"(rcnt + 4u * slot)
                                 : "memory");
                old = __shfl_sync(0xffffffffu, old, 0);
                if ((old & (uint32_t)(kConsumerWarps - 1)) == (uint32_t)(kConsumerWarps - 1)) {
                    __syncwarp();   // lane 0's acquire orders the whole warp's reads
                    if (lane < kTileRows) {
                        float v = __uint_as_float(lds32(sl + 4u * lane));
#pragma unroll
                        for (int w = 1; w < kConsumerWarps; ++w) v += __uint_as_float(lds32(sl + 64u * w + 4u * lane));
                        const int64_t row = (int64_t)(tile - a.tile_start[li]) * kTileRows + lane;
                        if (row < a.n[li]) {
                            if (a.amax_key) {
                                const unsigned long long key = argmax_key(v, a.amax_off + row);
                                best = key > best ? key : best;
                            } else {
                                store_out_peers(a.y[li], a.ydt, a.tok0 * a.ldy[li] + row, v, a.peer_delta, a.npeers);
                            }
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(repe + 8u * slot);   // the slot is consumed
                }
            }
            goto consumers_done;
        }
    }
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
            if constexpr (E == DP4A)
                chunk_dp4a(st, nblk, blk0, (uint32_t)K2, L, warp, lane, acc[0]);
            else if constexpr (E == DUMP)
                chunk_dump(st, nblk, blk0, (uint32_t)K2, L, warp, lane,
                           (int64_t)(tile - a.tile_start[li]) * kTileRows, a.n[li], G, a.dump_d);
            else if constexpr (E != NONE)
                chunk_mma<E>(st, nblk, blk0, (uint32_t)K2, L, G, ntok, warp, lane, kNib2, kMagic, acc);
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + 8u * s);
            if (++s == S) {
                s = 0;
                ph ^= 1u;
            }
        }
        const int64_t row0 = (int64_t)(tile - a.tile_start[li]) * kTileRows;
        if constexpr (E == DUMP) {
            continue;
        } else if constexpr (E == DP4A) {
            if (a.amax_key)
                epilogue_dp4a_amax(acc[0], row0, a.n[li], a.amax_off, warp, lane, best);
            else
                epilogue_dp4a(acc[0], row0, a.n[li], a.y[li], a.ydt, a.tok0 * a.ldy[li], warp, lane, a.peer_delta,
                              a.npeers);
        } else {
            epilogue_mma(acc, red, row0, a.n[li], a.y[li], a.ydt, a.ldy[li], a.tok0, ntok, warp, lane,
                         a.amax_key ? &best : nullptr, a.amax_off, a.peer_delta, a.npeers);
        }
    }
consumers_done:
    if (a.amax_key) {
        // greedy decode: CTA maximum in shared memory, then one global atomic per CTA
        if (best) asm volatile("atom.shared.max.u64 %0, [%1], %2;" : "=l"(best) : "r"(amax_slot), "l"(best) : "memory");
        bar_consumers();
        if (threadIdx.x == 0) {
            unsigned long long v;
            asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(amax_slot) : "memory");
            if (v) atomicMax(a.amax_key, v);
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
        r[6] = 0;
        r[7] = tr_first;
    }
}
