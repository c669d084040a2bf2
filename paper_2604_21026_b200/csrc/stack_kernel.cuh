// stack_kernel.cuh -- the persistent decode-step kernel (row a9): every linear of a
// routed decode step (16 layers x {qkv, o, gate/up, down} for Llama-3.2-1B) in ONE
// cooperative launch, one CTA per SM (included by kernels_stream.cu).
//
//   producer warp : streams the weights of ALL the step's linears back to back
//                   through the TMA ring (3-D nibble box + scale box per stage).
//                   Weights never depend on activations, so the weight stream
//                   never stops at a linear boundary: the HBM pipe stays full
//                   while consumers wait for the previous linear's outputs.
//   consumers     : per linear i: grid barrier on linear i-1 (a global counter
//                   reaching gridDim: every CTA has stored its rows of y_{i-1}),
//                   stage x_i (W4A8: fused per-token quantiser; W4A16: fragment
//                   order), consume linear i's stages (DP4A / HMMA1 engines, the
//                   same code as stream_linear), store y_i, arrive on counter i.
// The dependency order is the decode chain: linear i reads its input only after
// linear i-1 completed everywhere (the whole decode step
// replayed as one graph; here as one kernel).  route(layer) from the MCAP
// dispatch table selects the engine per linear.
#pragma once

struct StackOp {
    const CUtensorMap *maps[kMaxGroup];
    void *y[kMaxGroup];
    int64_t n[kMaxGroup];
    int tile_start[kMaxGroup + 1];
    int count;
    int route;        // MCAPQ_W4A8 (DP4A engine) or MCAPQ_W4A16 (HMMA1 engine)
    int ydt;
    int64_t k;
    const uint16_t *x;
};
static_assert(sizeof(StackOp) % 16 == 0, "StackOp is copied to shared memory in 16-byte pieces");

struct StackArgs {
    const StackOp *ops;          // device array [nops]
    int nops;
    unsigned int *counters;      // [nops], zero at launch: CTAs done with linear i
    int stages;
    int ops_off, act_off, red_off;   // shared-memory offsets of the program copy, activations, reduction
    unsigned long long *trace;   // debug: [nops][grid][8] or null
    int flags;                   // debug (MCAPQ_STEP_FLAGS): 1 no compute, 2 no grid barrier, 4 no staging, 8 no chain
};

__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int *p)
{
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

constexpr int kStepThreads = (kConsumerWarps + 2) * 32;   // consumers + producer warp + sync warp

__global__ void __launch_bounds__(kStepThreads, 1) stack_step(const __grid_constant__ StackArgs a)
{
    extern __shared__ __align__(16) uint8_t smem_raw[];
    const uint32_t sb = (smem_addr(smem_raw) + 1023u) & ~1023u;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int S = a.stages;
    const uint32_t ring = sb;
    const uint32_t full = sb + (uint32_t)S * kStageBytes;
    const uint32_t empty = full + 8u * S;
    const uint32_t done = empty + 8u * S;   // phase i: every consumer warp finished linear i
    const uint32_t go = done + 8u;          // phase i: linear i finished in every CTA
    const uint32_t act = sb + a.act_off;
    const uint32_t red = sb + a.red_off;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + 8u * s, 1);
            mbar_init(empty + 8u * s, kConsumerWarps);
        }
        mbar_init(done, kConsumerWarps);
        mbar_init(go, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // the program (a few KB) into shared memory once: op records are read at every
    // linear boundary by the producer and the consumers, never from global again
    StackOp *ops = reinterpret_cast<StackOp *>(smem_raw + (sb - smem_addr(smem_raw)) + a.ops_off);
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(a.ops);
        uint4 *dst = reinterpret_cast<uint4 *>(ops);
        const int n16 = (int)(sizeof(StackOp) * a.nops / 16);
        for (int i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();

    if (warp == kConsumerWarps + 1) {
        // ================= sync warp: publish and await linears, off the consumers' path =====
        // done(i) -> release-add counters[i] (the CTA's y_i stores, ordered by the
        // consumers' mbarrier arrives, become visible at gpu scope first) -> poll until
        // every CTA published -> go(i) releases the consumers into linear i+1.
        if (lane == 0 && !(a.flags & 8)) {
            for (int i = 0; i < a.nops; ++i) {
                mbar_wait(done, (uint32_t)i & 1u);
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.counters + i) : "memory");
                if (i + 1 == a.nops) break;
                if (!(a.flags & 2))
                    while (ld_acquire_gpu(a.counters + i) < gridDim.x) __nanosleep(20);
                mbar_arrive(go);
            }
        }
        return;
    }

    if (warp == kConsumerWarps) {
        // ================= producer: the whole step's weights, in op order =================
        if (lane == 0) {
            const uint64_t pol = evict_first_policy();
            int s = 0;
            uint32_t ph = 0;
            auto prefetch_maps = [&](int j) {
                // TMA descriptors of linear j into the TMA unit's cache before first use
                if (j >= a.nops) return;
                for (int m = 0; m < ops[j].count; ++m) {
                    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(ops[j].maps[m]))
                                 : "memory");
                    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(ops[j].maps[m] + 1))
                                 : "memory");
                }
            };
            prefetch_maps(0);
            prefetch_maps(1);
            for (int i = 0; i < a.nops; ++i) {
                prefetch_maps(i + 2);
                const StackOp &op = ops[i];
                const int count = op.count;
                const int K2 = (int)(op.k / 2);
                const int nchunks = (K2 + kChunkBytes - 1) / kChunkBytes;
                const int T = op.tile_start[count];
                const int t0 = (int)(((int64_t)T * blockIdx.x) / gridDim.x);
                const int t1 = (int)(((int64_t)T * (blockIdx.x + 1)) / gridDim.x);
                // warm this linear's input in L2 (evict_last) while its weights stream: the
                // consumers read x on the dependent chain, an L2 hit instead of a DRAM trip
                // queued behind the weight stream.  A prefetch only fills L2, so it is safe
                // even when x is written by the previous linear later (L2 is coherent).
                const int xlines = (int)((op.k * 2 + 127) / 128);
                for (int ln = blockIdx.x; ln < xlines; ln += gridDim.x)
                    asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(op.x + 64 * ln) : "memory");
                int li = 0;
                for (int tile = t0; tile < t1; ++tile) {
                    while (li + 1 < count && tile >= op.tile_start[li + 1]) ++li;
                    const CUtensorMap *map = op.maps[li];
                    const int row0 = (tile - op.tile_start[li]) * kTileRows;
                    for (int ch = 0; ch < nchunks; ++ch) {
                        mbar_wait(empty + 8u * s, ph ^ 1u);
                        const uint32_t st = ring + (uint32_t)s * kStageBytes;
                        const uint32_t fb = full + 8u * s;
                        mbar_expect_tx(fb, (uint32_t)kStageBytes);
                        tma_3d(st, map, 0, row0, ch * 8, fb, pol);
                        tma_2d(st + 8 * kBox, map + 1, ch * kChunkBlocks, row0, fb, pol);
                        if (++s == S) {
                            s = 0;
                            ph ^= 1u;
                        }
                    }
                }
            }
        }
        return;
    }

    // ================= consumers =================
    uint32_t kNib2 = 0x000F000Fu, kMagic = 0x43004300u;
    asm volatile("" : "+r"(kNib2), "+r"(kMagic));
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < a.nops; ++i) {
        const StackOp &op = ops[i];
        const int count = op.count, route = op.route;
        const int64_t k = op.k;
        const int G = (int)(k / 32);
        const int K2 = (int)(k / 2);
        const int nchunks = (K2 + kChunkBytes - 1) / kChunkBytes;
        const int T = op.tile_start[count];
        const int t0 = (int)(((int64_t)T * blockIdx.x) / gridDim.x);
        const int t1 = (int)(((int64_t)T * (blockIdx.x + 1)) / gridDim.x);
        unsigned long long tr0 = 0, tr1 = 0, tr2 = 0;
        if (a.trace) tr0 = globaltimer();

        // ---- wait for linear i-1 everywhere (its outputs may be this linear's input)
        if (i > 0 && !(a.flags & 8)) mbar_wait(go, (uint32_t)(i - 1) & 1u);
        if (a.trace) tr1 = globaltimer();
        const bool a16 = route == MCAPQ_W4A16;
        const ActSmem L = act_layout(a16, act, k, 1);
        if (!(a.flags & 4)) {
            if (a16)
                stage_a16<true>(op.x, k, 1, k, L, threadIdx.x, kConsumerWarps * 32);
            else
                stage_a8<true>(op.x, k, 1, k, L, threadIdx.x, kConsumerWarps * 32);
        }
        bar_consumers();
        if (a.trace) tr2 = globaltimer();

        int li = 0;
        for (int tile = t0; tile < t1; ++tile) {
            while (li + 1 < count && tile >= op.tile_start[li + 1]) ++li;
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            for (int ch = 0; ch < nchunks; ++ch) {
                const int rem = K2 - ch * kChunkBytes;
                const int nblk = (rem < kChunkBytes ? rem : kChunkBytes) / 16;
                const int blk0 = ch * kChunkBlocks;
                mbar_wait(full + 8u * s, ph);
                const uint32_t st = ring + (uint32_t)s * kStageBytes;
                if (a.flags & 1) {
                    // debug: drain only
                } else if (a16) {
                    chunk_mma<HMMA1>(st, nblk, blk0, (uint32_t)K2, L, G, 1, warp, lane, kNib2, kMagic, acc);
                } else {
                    chunk_dp4a(st, nblk, blk0, (uint32_t)K2, L, warp, lane, acc[0]);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(empty + 8u * s);
                if (++s == S) {
                    s = 0;
                    ph ^= 1u;
                }
            }
            const int64_t row0 = (int64_t)(tile - op.tile_start[li]) * kTileRows;
            if (a16)
                epilogue_mma(acc, red, row0, op.n[li], op.y[li], op.ydt, op.n[li], 0, 1, warp, lane);
            else
                epilogue_dp4a(acc[0], row0, op.n[li], op.y[li], op.ydt, 0, warp, lane);
        }
        // ---- this warp's rows of linear i are stored: tell the sync warp (no CTA-wide wait)
        __syncwarp();
        if (lane == 0) mbar_arrive(done);
        if (a.trace && threadIdx.x == 0) {
            unsigned long long *r = a.trace + 8ull * ((unsigned long long)i * gridDim.x + blockIdx.x);
            r[0] = (unsigned long long)i;
            r[1] = blockIdx.x;
            r[2] = tr0;
            r[3] = tr1;
            r[4] = tr2;
            r[5] = globaltimer();
            r[6] = 0;
            r[7] = 0;
        }
    }
}
