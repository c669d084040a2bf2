// stack_kernel.cuh -- the persistent decode-step kernel (row a9): every linear of a
// routed decode step (16 layers x {qkv, o, gate/up, down} for Llama-3.2-1B) in ONE
// cooperative launch, one CTA per SM (included by kernels_stream.cu).
//
//   producer warp : streams the weights of ALL the step's linears back to back
//                   through the TMA ring (3-D nibble box + scale box per stage).
//                   Weights never depend on activations, so the weight stream
//                   never stops at a linear boundary: the HBM pipe stays full
//                   while consumers wait for the previous linear's outputs.
//   consumers     : per linear i: stage x_i (W4A8: fused per-token quantiser;
//                   W4A16: fragment order), consume linear i's stages (DP4A / HMMA1
//                   engines, the same code as stream_linear), store y_i.
//   sync warp     : publishes linears other linears wait on (global counters) and
//                   releases consumers into a linear whose wait is a barrier.
//
// Dependencies are the data's own (the program builder, stack.cu, derives them
// from the registered buffers):
//   * dataflow (x_i is exactly y_j of an earlier linear j, bf16): linear j also
//     stores y_j as tagged words {bf16 | tag << 16} (tag = this launch's epoch);
//     linear i reads those words and re-reads any whose tag is stale.  The load IS
//     the wait: one L2 round trip instead of publish + poll + load.
//   * barrier (any other overlap: partial aliasing, WAR, WAW): linear i waits
//     until every CTA published linear j (counter j == gridDim).
//   * none (x_i is a step input): linear i starts as soon as its CTA gets there.
// The dependency order is the decode chain (the whole decode
// step replayed as one graph; here as one kernel).  route(layer) from the MCAP
// dispatch table selects the engine per linear.
#pragma once

struct StackOp {
    const CUtensorMap *maps[kMaxGroup];
    void *y[kMaxGroup];
    uint32_t *yt[kMaxGroup];   // tagged copy of y[m] read by a later linear of the step, or null
    int n[kMaxGroup];
    int tile_start[kMaxGroup + 1];
    int count;
    int route;        // MCAPQ_W4A8 (DP4A engine) or MCAPQ_W4A16 (HMMA1 engine)
    int ydt;
    int64_t k;
    const uint16_t *x;
    const uint32_t *xt;   // dataflow source: tagged y of the producing linear (then x is not read)
    int xt_op;            // the producing linear (its counter is the slow-path wait), or -1
    int wait_op;          // barrier dependency: linear index, or -1
    int publish;          // a later linear waits on this one's counter: 2 release (barrier), 1 relaxed (hint)
    int paired;           // tiles are handed out in 32-row pairs per CTA pair (cluster), see cta_tiles
    // producer-side quantisation (W4A8 consumers): the epilogue quantises every 32-row
    // group of y[m] once and stores its record (6 tagged u64 words: 32 codes, fp32 s,
    // int16 8 sum q) to yq[m]; a consumer with xq != null stages those records instead
    // of quantising the bf16 words itself (148 times)
    unsigned long long *yq[kMaxGroup];
    const unsigned long long *xq;
    int pad_[4];
};
static_assert(sizeof(StackOp) % 16 == 0, "StackOp is copied to shared memory in 16-byte pieces");

struct StackArgs {
    const StackOp *ops;          // device array [nops]
    int nops;
    unsigned int *counters;      // [nops] CTAs done with linear i, [nops] exit count, [nops + 1] epoch;
                                 // zero-initialised once, reset by the last CTA to leave
    int stages;
    int ops_off, act_off, red_off;   // shared-memory offsets (program copy, activations, tile slots)
    unsigned long long *trace;   // debug: [nops][grid][8] or null
    int flags;                   // debug (MCAPQ_STEP_FLAGS): 1 no compute, 2 no barrier polls, 4 no staging,
                                 // 8 no waits at all (barriers skipped, tags not checked),
                                 // 16 no publishing (only with 8), 32 no epilogue stores, 128 no W4A8 quantiser (loads only),
                                 // 256 no weight loads (the chain alone on stale ring data), 512 no epilogue work (handshake only)
    int spin_ns;                 // first back-off between re-reads of stale tagged words (doubles, <= 1 us)
    int polls;                   // CTA-wide re-read rounds before waiting on the producer's counter
    int ep_log2;                 // log2 of the tile slots between the consumers and the epilogue warp (1..3)
    int hold;                    // 1: the producer holds ring refills while this CTA stages an input (see `hold`)
    int clustered;               // launched as clusters of 2 CTAs: paired ops split their tiles per cluster
    int rec_spin;                // > 0: record consumers spin per thread (back-off cap, ns); 0: counter scheme
    // [nops][gridDim] {t0, t1 | straddle << 31}: every CTA's tile range per op, computed on the
    // host with the program (stack_partition) -- no partition arithmetic in the kernel
    const int2 *part;
    int part_off;                // shared-memory offset of this CTA's column of `part`
};

__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int *p)
{
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint4 ld_relaxed_128(const void *p)
{
    uint4 v;
    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}
__device__ __forceinline__ uint32_t lds32_volatile(uint32_t addr)
{
    uint32_t v;
    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
// The refill-hold flag is a lock-free flag between a consumer thread (writer) and the
// producer thread (poller): atomic accesses on both sides, so it is not a data race
// (compute-sanitizer racecheck) and every poll sees the latest write.
__device__ __forceinline__ void hold_write(uint32_t addr, uint32_t v)
{
    asm volatile("atom.shared.exch.b32 _, [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t hold_read(uint32_t addr)
{
    uint32_t v;
    asm volatile("atom.shared.or.b32 %0, [%1], 0;" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ bool tags_ok(uint4 a, uint32_t t16)
{
    return (((a.x ^ t16) | (a.y ^ t16) | (a.z ^ t16) | (a.w ^ t16)) >> 16) == 0u;
}
// tagged words -> packed bf16 pairs
__device__ __forceinline__ uint2 untag(uint4 a)
{
    return make_uint2(__byte_perm(a.x, a.y, 0x5410), __byte_perm(a.z, a.w, 0x5410));
}

// ---- producer-side quantisation records and the CTA-pair exchange (clusters of 2)
constexpr int kRecWords = 6;   // u64 per 32-group: 7 payload bytes + 1 tag byte each
__device__ __forceinline__ uint32_t cluster_rank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa_peer(uint32_t addr, uint32_t rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync_all()
{
    asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITC_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_bar)
{
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote_relaxed(uint32_t cluster_bar)
{
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ void st_async_u32(uint32_t cluster_addr, uint32_t v, uint32_t cluster_bar)
{
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u32 [%0], %1, [%2];" ::"r"(cluster_addr),
                 "r"(v), "r"(cluster_bar)
                 : "memory");
}
__device__ __forceinline__ void ld_relaxed_2x64(const unsigned long long *p, unsigned long long &a, unsigned long long &b)
{
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ bool rec_ok(unsigned long long w, uint32_t t8) { return (uint32_t)(w >> 56) == t8; }

// Quantise one 32-row group held one bf16 value per lane (lane j = element j of the
// group) and store its record: codes, s = fl(amax / 127) and 8 sum q,
// bit-identical to quant_a8_kernel (same fast path and IEEE fallback as a8_*_store).
// All 32 lanes call it.
// scr: 48 B of this warp's shared scratch (6 x u64, 8-aligned): the record is assembled
// there byte by byte (lane j's code at byte 7 (j / 7) + j % 7 of the payload stream) and
// read back as six tagged words
__device__ __forceinline__ void quant_group_record(uint32_t xb, unsigned long long *rec, uint32_t t8, int lane,
                                                   uint32_t scr)
{
    const uint32_t m = __reduce_max_sync(0xffffffffu, xb & 0x7fffu);
    const float s = div127_rn(__uint_as_float(m << 16));
    const bool live = m < 0x7f80u && s != 0.0f;
    const float inv = rcp_group(s);
    const float v = __uint_as_float(xb << 16);
    const float qa = __fmul_rn(v, inv);
    const float t = __fadd_rn(qa, 12582912.0f);
    const float r = __fsub_rn(qa, __fsub_rn(t, 12582912.0f));
    int c = __float_as_int(t) - 0x4B400000;
    // a NaN residual (inv = inf) counts as bad: !(|r| < 0.4999)
    if (__any_sync(0xffffffffu, !(fabsf(r) < 0.4999f)) && live) c = quant_code_ool(v, s, inv);
    if (!live) c = 0;
    const int sum = __reduce_add_sync(0xffffffffu, c);
    const uint32_t cb = (uint32_t)c & 0xffu;
    const uint32_t sbits = __float_as_uint(live ? s : 0.0f);
    const uint32_t sq16 = (uint32_t)(8 * sum) & 0xffffu;
    // payload stream: codes 0..31, s (4 bytes LE), 8 sum q (2 bytes LE), 4 zero bytes; stream
    // byte i sits in word i / 7, byte i % 7; byte 7 of every word is the tag
    if (lane < kRecWords)
        asm volatile("st.shared.u64 [%0], %1;" ::"r"(scr + 8u * (uint32_t)lane), "l"((unsigned long long)t8 << 56)
                     : "memory");
    __syncwarp();
    auto put = [&](int i, uint32_t byte) {
        asm volatile("st.shared.u8 [%0], %1;" ::"r"(scr + 8u * (uint32_t)(i / 7) + (uint32_t)(i % 7)), "r"(byte)
                     : "memory");
    };
    put(lane, cb);
    if (lane < 4) put(32 + lane, (sbits >> (8 * lane)) & 0xffu);
    else if (lane < 6) put(32 + lane, (sq16 >> (8 * (lane - 4))) & 0xffu);
    __syncwarp();
    if (lane < kRecWords) {
        unsigned long long word;
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(word) : "r"(scr + 8u * (uint32_t)lane) : "memory");
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(rec + lane), "l"(word) : "memory");
    }
    __syncwarp();   // the scratch is free again for the next record
}

// A record's payload into the engine's activation layout: q_lo (codes 0..15), q_hi
// (codes 16..31), {s, 8 sum q}.
__device__ __forceinline__ void rec_unpack_store(const unsigned long long w[kRecWords], int g, uint32_t K2,
                                                 const ActSmem &L)
{
    const unsigned long long M56 = 0x00ffffffffffffffull;
    const unsigned long long a = w[0] & M56, b = w[1] & M56, c = w[2] & M56, d = w[3] & M56, e = w[4] & M56,
                             f = w[5] & M56;
    const unsigned long long lo0 = a | (b << 56), lo1 = (b >> 8) | (c << 48);
    const unsigned long long hi0 = (c >> 16) | (d << 40), hi1 = (d >> 24) | (e << 32);
    const uint32_t sbits = (uint32_t)((e >> 32) | (f << 24));
    const int sq8 = (int)(int16_t)(uint16_t)((f >> 8) & 0xffffu);
    asm volatile("st.shared.v2.u64 [%0], {%1,%2};" ::"r"(L.act + 16u * (uint32_t)g), "l"(lo0), "l"(lo1) : "memory");
    asm volatile("st.shared.v2.u64 [%0], {%1,%2};" ::"r"(L.act + K2 + 16u * (uint32_t)g), "l"(hi0), "l"(hi1)
                 : "memory");
    asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(L.ssq + 8u * (uint32_t)g), "r"(sbits), "r"((uint32_t)sq8)
                 : "memory");
}

constexpr int kStepThreads = (kConsumerWarps + 2) * 32;   // consumers + producer warp + sync warp
constexpr int kStepMaxRounds = 4;                         // K <= 16384: G*4 quads over 512 consumer threads

__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity)
{
    uint32_t r;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(r)
        : "r"(bar), "r"(parity)
        : "memory");
    return r != 0;
}

// AND of a predicate over the consumer threads (also a consumer barrier).
__device__ __forceinline__ bool bar_consumers_and(bool v)
{
    uint32_t r;
    asm volatile(
        "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 q, %1, 0;\n\tbar.red.and.pred p, 1, %2, q;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(r)
        : "r"((uint32_t)v), "n"(kConsumerWarps * 32)
        : "memory");
    return r != 0;
}

// Stage one linear's input (M = 1) into shared memory: all loads of this thread are
// issued first (up to kStepMaxRounds x 32 B).  A dataflow input is then checked:
// if every tagged word is current (the producing linear finished everywhere before
// this CTA got here: the load was the only round trip) staging goes on; otherwise
// one thread waits for the producer's counter (low-traffic polling, no storm of
// data re-reads) and the stale words are re-read once.
// W4A8 with K <= 2048: one group per 8 threads (all 512 consumer threads busy at
// K = 2048, half the per-thread quantiser work of the quad layout).
__device__ __forceinline__ void stage_step_a8_oct(unsigned long long *tmid, const StackOp &op, const ActSmem &L, int tid, uint32_t t16,
                                                  bool check, int spin_ns, int polls, const unsigned int *counters,
                                                  bool quant)
{
    const int G = (int)(op.k / 32);
    const uint32_t K2 = (uint32_t)(op.k / 2);
    const bool tagged = op.xt != nullptr;
    const bool on = tid < G * 8;
    const int g = on ? tid >> 3 : 0, sub8 = tid & 7;
    const int e0 = 32 * g + 4 * sub8;
    uint4 ra = make_uint4(0, 0, 0, 0);
    if (on) {
        if (tagged) {
            ra = ld_relaxed_128(op.xt + e0);
        } else {
            const uint2 p = ldg_x64<true>(op.x + e0);
            ra = make_uint4(p.x, p.y, 0, 0);
        }
    }
    if (tagged && check && polls < 0) {
        // per-thread re-reads of this thread's 16 B until current, back-off capped at -polls ns
        int backoff = spin_ns;
        while (on && !tags_ok(ra, t16)) {
            __nanosleep(backoff);
            ra = ld_relaxed_128(op.xt + e0);
            backoff = backoff < -polls ? 2 * backoff : -polls;
        }
    } else if (tagged && check) {
        int backoff = spin_ns;
        for (int p = 0;; ++p) {
            const bool ok = !on || tags_ok(ra, t16);
            if (bar_consumers_and(ok)) break;
            if (p >= polls) {
                if (tid == 0)
                    while (ld_acquire_gpu(counters + op.xt_op) < gridDim.x) __nanosleep(spin_ns);
                bar_consumers();
                if (!ok) {
                    ra = ld_relaxed_128(op.xt + e0);
                    while (!tags_ok(ra, t16)) {   // the producer published (a hint): re-read until current
                        __nanosleep(spin_ns);
                        ra = ld_relaxed_128(op.xt + e0);
                    }
                }
                break;
            }
            if (!ok) {
                __nanosleep(backoff);
                ra = ld_relaxed_128(op.xt + e0);
            }
            backoff = backoff < 1024 ? 2 * backoff : 1024;
        }
    }
    if (tmid) *tmid = globaltimer();
    uint2 w2;
    if (tagged) w2 = untag(ra);
    else w2 = make_uint2(ra.x, ra.y);
    if (quant) a8_oct_store(w2, on, g, sub8, K2, L);
}

// Stage a W4A8 input whose producer quantised it (records, see quant_group_record): one
// thread per 32-group loads its 6 tagged words (48 B instead of the 128 B of tagged
// bf16 words), the same current-tag protocol as the bf16 staging (CTA-wide re-read
// rounds, then the producer's counter, then per-thread re-reads), and unpacks codes and
// {s, 8 sum q} into the engine's layout -- no quantiser on the consumer side.
__device__ __forceinline__ void stage_step_rec(unsigned long long *tmid, const StackOp &op, const ActSmem &L, int tid,
                                               uint32_t t8, bool check, int spin_ns, int polls,
                                               const unsigned int *counters, int rec_spin)
{
    const int G = (int)(op.k / 32);
    const uint32_t K2 = (uint32_t)(op.k / 2);
    const bool on = tid < G;
    const unsigned long long *src = op.xq + (size_t)(on ? tid : 0) * kRecWords;
    unsigned long long w[kRecWords] = {0, 0, 0, 0, 0, 0};
    if (on) {
        ld_relaxed_2x64(src, w[0], w[1]);
        ld_relaxed_2x64(src + 2, w[2], w[3]);
        ld_relaxed_2x64(src + 4, w[4], w[5]);
    }
    if (check && rec_spin > 0) {
        // records are small (48 B per group): every thread re-reads its own until current,
        // back-off capped at rec_spin ns -- no CTA-wide rounds, no counter round trip
        int backoff = spin_ns;
        while (on && !(rec_ok(w[0], t8) && rec_ok(w[1], t8) && rec_ok(w[2], t8) && rec_ok(w[3], t8) &&
                       rec_ok(w[4], t8) && rec_ok(w[5], t8))) {
            __nanosleep(backoff);
            ld_relaxed_2x64(src, w[0], w[1]);
            ld_relaxed_2x64(src + 2, w[2], w[3]);
            ld_relaxed_2x64(src + 4, w[4], w[5]);
            backoff = backoff < rec_spin ? 2 * backoff : rec_spin;
        }
    } else if (check) {
        int backoff = spin_ns;
        for (int p = 0;; ++p) {
            const bool ok = !on || (rec_ok(w[0], t8) && rec_ok(w[1], t8) && rec_ok(w[2], t8) && rec_ok(w[3], t8) &&
                                    rec_ok(w[4], t8) && rec_ok(w[5], t8));
            if (bar_consumers_and(ok)) break;
            if (p >= polls) {
                if (tid == 0)
                    while (ld_acquire_gpu(counters + op.xt_op) < gridDim.x) __nanosleep(spin_ns);
                bar_consumers();
                // the producer published (a hint): re-read until current
                while (on && !(rec_ok(w[0], t8) && rec_ok(w[1], t8) && rec_ok(w[2], t8) && rec_ok(w[3], t8) &&
                               rec_ok(w[4], t8) && rec_ok(w[5], t8))) {
                    __nanosleep(spin_ns);
                    ld_relaxed_2x64(src, w[0], w[1]);
                    ld_relaxed_2x64(src + 2, w[2], w[3]);
                    ld_relaxed_2x64(src + 4, w[4], w[5]);
                }
                break;
            }
            if (!ok) {
                __nanosleep(backoff);
                ld_relaxed_2x64(src, w[0], w[1]);
                ld_relaxed_2x64(src + 2, w[2], w[3]);
                ld_relaxed_2x64(src + 4, w[4], w[5]);
            }
            backoff = backoff < 1024 ? 2 * backoff : 1024;
        }
    }
    if (tmid) *tmid = globaltimer();
    if (on) rec_unpack_store(w, tid, K2, L);
}

// Rounds q0 / NT .. q0 / NT + kRounds - 1 of the quad staging (one phase; see stage_step).
template <int kRounds>
__device__ __forceinline__ void stage_step_phase(unsigned long long *tmid, const StackOp &op, bool a16, const ActSmem &L,
                                                 int tid, uint32_t t16, bool check, int spin_ns, int polls,
                                                 const unsigned int *counters, bool quant, int q0)
{
    const int G = (int)(op.k / 32);
    const uint32_t K2 = (uint32_t)(op.k / 2);
    const int nq = G * 4;
    const bool tagged = op.xt != nullptr;
    constexpr int NT = kConsumerWarps * 32;
    uint4 ra[kRounds], rb[kRounds];
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const int idx = q0 + r * NT + tid;
        if (q0 + r * NT < nq && idx < nq) {
            const int g = idx >> 2, sub = idx & 3;
            // element offsets: W4A8 quad member sub holds 8 sub .. 8 sub + 7; W4A16 4t..4t+3, 4t+16..4t+19
            const int e0 = 32 * g + (a16 ? 4 * sub : 8 * sub);
            const int e1 = a16 ? e0 + 16 : e0 + 4;
            if (tagged) {
                ra[r] = ld_relaxed_128(op.xt + e0);
                rb[r] = ld_relaxed_128(op.xt + e1);
            } else if (a16) {
                const uint2 lo = ldg_x64<true>(op.x + e0), hi = ldg_x64<true>(op.x + e1);
                ra[r] = make_uint4(lo.x, lo.y, hi.x, hi.y);
            } else {
                ra[r] = ldg_x128<true>(op.x + e0);
            }
        }
    }
    if (tagged && check) {
        // re-read only this thread's stale words, with exponential back-off; after
        // `polls` CTA-wide rounds fall back to the producer's counter
        auto reload_stale = [&]() {
#pragma unroll
            for (int r = 0; r < kRounds; ++r) {
                const int idx = q0 + r * NT + tid;
                if (q0 + r * NT < nq && idx < nq && !(tags_ok(ra[r], t16) && tags_ok(rb[r], t16))) {
                    const int g = idx >> 2, sub = idx & 3;
                    const int e0 = 32 * g + (a16 ? 4 * sub : 8 * sub);
                    const int e1 = a16 ? e0 + 16 : e0 + 4;
                    ra[r] = ld_relaxed_128(op.xt + e0);
                    rb[r] = ld_relaxed_128(op.xt + e1);
                }
            }
        };
        int backoff = spin_ns;
        if (polls < 0) {
            // independent per-thread spin on this thread's stale words (back-off capped at
            // -polls ns), no CTA-wide rounds
            const int cap = -polls;
            for (;;) {
                bool ok = true;
#pragma unroll
                for (int r = 0; r < kRounds; ++r)
                    if (q0 + r * NT + tid < nq) ok = ok && tags_ok(ra[r], t16) && tags_ok(rb[r], t16);
                if (ok) break;
                __nanosleep(backoff);
                reload_stale();
                backoff = backoff < cap ? 2 * backoff : cap;
            }
        }
        for (int p = 0; polls >= 0; ++p) {
            bool ok = true;
#pragma unroll
            for (int r = 0; r < kRounds; ++r)
                if (q0 + r * NT + tid < nq) ok = ok && tags_ok(ra[r], t16) && tags_ok(rb[r], t16);
            if (bar_consumers_and(ok)) break;
            if (p >= polls) {
                if (tid == 0)
                    while (ld_acquire_gpu(counters + op.xt_op) < gridDim.x) __nanosleep(spin_ns);
                bar_consumers();
                if (!ok) reload_stale();
                break;
            }
            if (!ok) {
                __nanosleep(backoff);
                reload_stale();
            }
            backoff = backoff < 1024 ? 2 * backoff : 1024;
        }
    }
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        if (r == 0 && q0 == 0 && tmid) *tmid = globaltimer();
        if (q0 + r * NT >= nq) break;   // CTA-uniform
        const int idx = q0 + r * NT + tid;
        const bool on = idx < nq;
        const int q = on ? idx : 0;
        const int g = q >> 2, sub = q & 3;
        uint32_t w4[4];
        if (tagged) {
            if (on && check) {
                // the producer published: current now (guards the relaxed re-read)
                const int e0 = 32 * g + (a16 ? 4 * sub : 8 * sub);
                const int e1 = a16 ? e0 + 16 : e0 + 4;
                while (!(tags_ok(ra[r], t16) && tags_ok(rb[r], t16))) {
                    __nanosleep(spin_ns);
                    ra[r] = ld_relaxed_128(op.xt + e0);
                    rb[r] = ld_relaxed_128(op.xt + e1);
                }
            }
            const uint2 lo = untag(ra[r]), hi = untag(rb[r]);
            w4[0] = lo.x; w4[1] = lo.y; w4[2] = hi.x; w4[3] = hi.y;
        } else {
            w4[0] = ra[r].x; w4[1] = ra[r].y; w4[2] = ra[r].z; w4[3] = ra[r].w;
        }
        if (a16) {
            a16_quad_store(make_uint2(w4[0], w4[1]), make_uint2(w4[2], w4[3]), on, 0, g, sub, L);
        } else {
            if (quant) a8_quad_store(w4, on, 0, g, sub, G, K2, L);
        }
    }
}

// Stage one linear's input (M = 1) into shared memory, quads of threads per 32-group.
// At most two rounds of 512 quads are held in registers at a time: a K > 8192 input
// (kRounds = 4) is staged in two phases, so the K = 14336 variant of the step kernel has
// the register profile of the K <= 8192 one (the whole kernel shares the 96-register cap).
template <int kRounds>
__device__ __forceinline__ void stage_step(unsigned long long *tmid, const StackOp &op, bool a16, const ActSmem &L, int tid, uint32_t t16,
                                           bool check, int spin_ns, int polls, const unsigned int *counters,
                                           bool quant, uint32_t t8, int rec_spin)
{
    if (!a16 && op.xq) {
        stage_step_rec(tmid, op, L, tid, t8, check, spin_ns, polls, counters, rec_spin);
        return;
    }
    if (!a16 && op.k <= 2048) {
        stage_step_a8_oct(tmid, op, L, tid, t16, check, spin_ns, polls, counters, quant);
        return;
    }
    constexpr int NT = kConsumerWarps * 32;
    const int G = (int)(op.k / 32);
    if (a16)
        for (int idx = tid; idx < G * 8; idx += NT)     // tokens 1..7 of corr: zero
            if ((idx & 7) != 0) sts32(L.corr + 4u * (uint32_t)idx, 0u);
    if constexpr (kRounds <= 2) {
        stage_step_phase<kRounds>(tmid, op, a16, L, tid, t16, check, spin_ns, polls, counters, quant, 0);
    } else {
#pragma unroll 1
        for (int q0 = 0; q0 < kRounds * NT; q0 += 2 * NT) {
            if (q0 >= G * 4) break;   // CTA-uniform
            stage_step_phase<2>(tmid, op, a16, L, tid, t16, check, spin_ns, polls, counters, quant, q0);
        }
    }
}

// Store one output element: the caller's y and, when a later linear reads it in
// this step, its tagged copy.
__device__ __forceinline__ void store_step(const StackOp &op, int m, int64_t row, float v, uint32_t t16)
{
    dev::store_out(op.y[m], op.ydt, row, v);
    if (op.yt[m]) {
        const uint32_t w = (uint32_t)dev::float_to_bf16_bits(v) | t16;
        asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(op.yt[m] + row), "r"(w) : "memory");
    }
}

// kRounds: staging rounds of 512 quads (2: K <= 8192, 4: K <= 16384) -- fewer rounds,
// fewer live registers under the 96-register cap of 18 warps per SM
// kRoutes: 3 = a mixed program (both engines), 1 = W4A8 only, 2 = W4A16 only -- a
// single-route program runs an instantiation without the other engine's code (a
// smaller kernel: the mixed one regressed untouched W4A16 loops by ~8 % as it grew)
template <bool kTrace, int kRounds, int kRoutes = 3>
__global__ void __launch_bounds__(kStepThreads, 1) stack_step(const __grid_constant__ StackArgs a)
{
    extern __shared__ __align__(16) uint8_t smem_raw[];
    const uint32_t sb = (smem_addr(smem_raw) + 1023u) & ~1023u;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int S = a.stages;
    const uint32_t ring = sb;
    const uint32_t full = sb + (uint32_t)S * kStageBytes;
    const uint32_t empty = full + 8u * S;
    const uint32_t go = empty + 8u * S;   // phase j: the j-th barrier-waiting linear may start
    const int EL = a.ep_log2;
    const uint32_t EN = 1u << EL;         // tile slots (<= 8)
    const uint32_t epf = go + 8u;         // [EN] tile slot written by every consumer warp
    const uint32_t epe = go + 72u;        // [EN] tile slot stored out by the epilogue warp
    // refill hold: set by the consumers from the last stage of a linear until the next
    // linear's input is staged; the producer issues no ring refill meanwhile, so the
    // latency-critical activation loads do not queue behind this SM's in-flight weight
    // data (the refills it holds are for later linears: the current one is resident)
    const uint32_t hold = go + 136u;
    const uint32_t act = sb + a.act_off;
    const uint32_t red = sb + a.red_off;  // [EN] tile slots: [16 warps][16 rows] fp32
    // this launch's tag (epoch + 1, never 0): the epoch only changes after every CTA left
    const uint32_t epoch = *reinterpret_cast<volatile unsigned int *>(a.counters + a.nops + 1);
    const uint32_t t16 = ((epoch % 65535u) + 1u) << 16;
    const uint32_t t8 = (epoch % 255u) + 1u;   // record tag (consecutive launches differ)
    // CTA-pair exchange of a group's first 16 rows when its two tiles sit on the two CTAs
    // of a cluster: xfull[2] (st.async complete_tx), xempty[2] (the reader's release), xbuf[2][32 B]
    const uint32_t xfull = go + 144u, xempty = go + 160u, xbuf = go + 176u;
    const uint32_t rscr = go + 240u;   // the epilogue warp's 48-B record scratch (quant_group_record)

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + 8u * s, 1);
            mbar_init(empty + 8u * s, kConsumerWarps);
        }
        mbar_init(go, 1);
        sts32(hold, 0u);
        for (int j = 0; j < (int)EN; ++j) {
            mbar_init(epf + 8u * j, kConsumerWarps);
            mbar_init(epe + 8u * j, 1);
        }
        for (int j = 0; j < 2; ++j) {
            mbar_init(xfull + 8u * j, 1);
            mbar_init(xempty + 8u * j, 1);
        }
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
    int2 *part_s = reinterpret_cast<int2 *>(smem_raw + (sb - smem_addr(smem_raw)) + a.part_off);
    for (int i = threadIdx.x; i < a.nops; i += blockDim.x) part_s[i] = a.part[(size_t)i * gridDim.x + blockIdx.x];
    __syncthreads();
    if (a.clustered) cluster_sync_all();   // the peer's exchange barriers are initialised

    // This CTA's tiles [t0, t1) of an op.  Paired ops (clusters of 2): 32-row pairs are
    // split evenly over the clusters and each cluster's range in halves over its two
    // CTAs, so a quantisation group (two tiles) lies in one CTA or, at most once per op,
    // straddles the cluster's two CTAs (`straddle`: rank 0's last tile is its first
    // half, rank 1's first tile its second half).  Otherwise contiguous balanced ranges.
    // (the ranges come from the host's partition table, see StackArgs::part / stack_partition)
    auto cta_tiles = [&](int i, int &t0, int &t1, bool &straddle) {
        const int2 v = part_s[i];
        t0 = v.x;
        t1 = v.y & 0x7fffffff;
        straddle = v.y < 0;
    };
    // The order a CTA works through its tiles (the producer's stages, the epilogue's
    // slots; the consumers just follow the ring): rank 0 of a straddling pair takes the
    // shared group's first half FIRST, so both halves are done at the same time and the
    // exchange never waits for the rest of rank 0's range.
    auto tile_seq = [&](int j, int t0, int t1, bool straddle) {
        return (straddle && (blockIdx.x & 1u) == 0) ? (j == 0 ? t1 - 1 : t0 + j - 1) : t0 + j;
    };

    if (warp == kConsumerWarps + 1) {
        // ================= epilogue / sync warp =================
        // Per tile (in the consumers' order): wait until the 16 consumer warps left
        // their partial row sums in the tile slot, reduce them in a fixed order
        // (W4A16: 16 warp partials per row; W4A8: one value per row), store the 16 rows
        // (caller's y + tagged copy) in one instruction, release the slot.  Per linear:
        // barrier waits (poll counter[wait_op], then `go`) and publishing (its own
        // stores, then release-add counter[i]).  Last: the exit count; the last CTA out
        // resets the counters and advances the epoch for the next launch.
        const bool nowait = (a.flags & 10) != 0;
        uint32_t ts = 0;   // tile sequence number of this CTA
        uint32_t held = 0, xsend = 0, xrecv = 0;   // producer-side quantisation state
        for (int i = 0; i < a.nops; ++i) {
            const StackOp &op = ops[i];
            int t0, t1;
            bool straddle;
            cta_tiles(i, t0, t1, straddle);
            if (op.wait_op >= 0 && t1 > t0) {
                if (lane == 0) {
                    if (!nowait)
                        while (ld_acquire_gpu(a.counters + op.wait_op) < gridDim.x) __nanosleep(20);
                    // one go phase in flight at a time: the consumers passed every earlier
                    // one (this warp already stored every earlier tile they computed)
                    mbar_arrive(go);
                }
                __syncwarp();
            }
            const bool a16 = kRoutes == 2 ? true : (kRoutes == 1 ? false : op.route == MCAPQ_W4A16);
            // the tile loop in two instantiations: ops whose outputs feed records carry the
            // producer-side quantiser; the others keep the plain loop (the record code in a
            // shared loop slowed W4A16 tiles by ~3.5 % although it never ran for them)
            auto ep_tiles = [&](auto rec_c) {
                constexpr bool kRec = decltype(rec_c)::value;
                // member li of the group and its first tile, advanced incrementally (the
                // reordered rank-0 range of a straddling pair restarts the walk once)
                int li = 0, li_start = 0, li_next = op.count > 1 ? op.tile_start[1] : 0x7fffffff;
                for (int j = 0; j < t1 - t0; ++j, ++ts) {
                    const int tile = tile_seq(j, t0, t1, straddle);
                    if (j <= 1 && straddle) {
                        li = 0;
                        li_start = 0;
                        li_next = op.count > 1 ? op.tile_start[1] : 0x7fffffff;
                    }
                    while (tile >= li_next) {
                        ++li;
                        li_start = li_next;
                        li_next = li + 1 < op.count ? op.tile_start[li + 1] : 0x7fffffff;
                    }
                    const uint32_t slot = ts & (EN - 1u);
                    mbar_wait(epf + 8u * slot, (ts >> EL) & 1u);
                    unsigned long long te0 = 0;
                    if (kTrace && lane == 0 && j == t1 - t0 - 1) te0 = globaltimer();
                    const uint32_t sl = red + 1024u * slot;
                    float v = 0.0f;
                    const int tl = tile - li_start;
                    if (lane < kTileRows && !(a.flags & 512)) {
                        float x[kConsumerWarps];
    #pragma unroll
                        for (int w = 0; w < kConsumerWarps; ++w) x[w] = __uint_as_float(lds32(sl + 64u * w + 4u * lane));
                        if (a16) {
                            // HMMA1 partials: the stream kernel's linear order over the warps
                            v = x[0];
    #pragma unroll
                            for (int w = 1; w < kConsumerWarps; ++w) v += x[w];
                        } else {
                            // row-lane DP4A: warp w holds level 1 of stream_linear's butterfly
                            // (lanes w, w + 16); levels 2..5 pair w with w + 8, + 4, + 2, + 1
    #pragma unroll
                            for (int h = kConsumerWarps / 2; h > 0; h >>= 1)
    #pragma unroll
                                for (int w = 0; w < h; ++w) x[w] += x[w + h];
                            v = x[0];
                        }
                    }
                    if (lane < kTileRows && !(a.flags & 512)) {
                        const int64_t row = (int64_t)tl * kTileRows + lane;
                        if (row < op.n[li] && !(a.flags & 32)) store_step(op, li, row, v, t16);
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(epe + 8u * slot);   // the slot is consumed: release it
                    if (kRec && op.yq[li] && !(a.flags & 512)) {
                        // producer-side quantisation of group tl / 2 (rows 32 (tl/2) ..): this
                        // tile's 16 bf16 values (exactly what y holds) in lanes 0..15
                        const uint32_t b = lane < kTileRows ? (uint32_t)dev::float_to_bf16_bits(v) : 0u;
                        if ((tl & 1) == 0) {
                            if (straddle && tile == t1 - 1) {
                                // first half of the group the peer (rank 1) completes: push the 16
                                // values into its exchange slot (st.async + complete_tx)
                                const uint32_t xs = xsend & 1u;
                                if (lane == 0) mbar_wait_cluster(xempty + 8u * xs, ((xsend >> 1) & 1u) ^ 1u);
                                __syncwarp();
                                const uint32_t lo = __shfl_sync(0xffffffffu, b, (2 * lane) & 31);
                                const uint32_t hi = __shfl_sync(0xffffffffu, b, (2 * lane + 1) & 31);
                                if (lane < 8)
                                    st_async_u32(mapa_peer(xbuf + 32u * xs + 4u * lane, 1u), lo | (hi << 16),
                                                 mapa_peer(xfull + 8u * xs, 1u));
                                ++xsend;
                            } else {
                                held = b;
                            }
                        } else {
                            uint32_t first = held;
                            if (straddle && tile == t0) {
                                // second half here, first half from the peer (rank 0)
                                const uint32_t xs = xrecv & 1u;
                                if (lane == 0) mbar_expect_tx(xfull + 8u * xs, 32u);
                                mbar_wait(xfull + 8u * xs, (xrecv >> 1) & 1u);
                                first = lane < kTileRows ? lds16(xbuf + 32u * xs + 2u * lane) : 0u;
                            }
                            const uint32_t second = __shfl_sync(0xffffffffu, b, lane & 15);
                            quant_group_record(lane < kTileRows ? first : second, op.yq[li] + (size_t)(tl >> 1) * kRecWords,
                                               t8, lane, rscr);
                            if (straddle && tile == t0) {
                                // the exchange slot is free again: every lane consumed its value
                                // (the record is built from it), so a relaxed arrive suffices
                                __syncwarp();
                                if (lane == 0) mbar_arrive_remote_relaxed(mapa_peer(xempty + 8u * (xrecv & 1u), 0u));
                                ++xrecv;
                            }
                        }
                    }
                    if (kTrace && lane == 0 && j == t1 - t0 - 1) {
                        // debug: the op's last tile in this epilogue (start, stores issued)
                        unsigned long long *r = a.trace + 8ull * ((unsigned long long)(a.nops + i) * gridDim.x + blockIdx.x);
                        r[0] = te0;
                        r[1] = globaltimer();
                    }
                }
            };
            // (a W4A16-only program has no W4A8 consumer, hence no records)
            bool rec_op = false;
            for (int m = 0; m < op.count; ++m) rec_op = rec_op || op.yq[m] != nullptr;
            if constexpr (kRoutes == 2) rec_op = false;
            if constexpr (kRoutes == 2) {
                ep_tiles(std::false_type{});
            } else {
                if (rec_op)
                    ep_tiles(std::true_type{});
                else
                    ep_tiles(std::false_type{});
            }
            // publish: 2 = release (a barrier dependency reads through this counter),
            // 1 = relaxed (dataflow consumers only take it as a hint to re-read their tags;
            // a release here would hold this warp in a GPU-scope fence behind the SM's
            // in-flight weight traffic, 0.2 us per linear)
            if (op.publish && lane == 0 && !(a.flags & 16)) {
                if (op.publish == 2)
                    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.counters + i) : "memory");
                else
                    asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(a.counters + i) : "memory");
            }
        }
        if (lane == 0) {
            unsigned int prev;
            asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                         : "=r"(prev)
                         : "l"(a.counters + a.nops)
                         : "memory");
            if (prev == gridDim.x - 1) {
                for (int i = 0; i < a.nops; ++i) a.counters[i] = 0u;
                a.counters[a.nops] = 0u;
                a.counters[a.nops + 1] = epoch + 1u;
                __threadfence();
            }
        }
        if (a.clustered) cluster_sync_all();   // no CTA leaves while its peer may still address it
        return;
    }

    if (warp == kConsumerWarps) {
        // ================= producer: the whole step's weights, in op order =================
        if (lane == 0) {
            const uint64_t pol = evict_first_policy();
            int s = 0;
            uint32_t ph = 0;
            const bool noload = (a.flags & 256) != 0;
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
                int t0, t1;
                bool straddle_;
                cta_tiles(i, t0, t1, straddle_);
                if (!op.xt && !op.xq) {
                    // a step input: warm it in L2 (evict_last) while the weights stream
                    const int xlines = (int)((op.k * 2 + 127) / 128);
                    for (int ln = blockIdx.x; ln < xlines; ln += gridDim.x)
                        asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(op.x + 64 * ln) : "memory");
                }
#ifdef MCAPQ_ABL_PROD
                int li = 0;
                for (int tile = t0; tile < t1; ++tile) {
                    while (li + 1 < count && tile >= op.tile_start[li + 1]) ++li;
                    const CUtensorMap *map = op.maps[li];
                    const int row0 = (tile - op.tile_start[li]) * kTileRows;
                    for (int ch = 0; ch < nchunks; ++ch) {
                        mbar_wait(empty + 8u * s, ph ^ 1u);
                        if (a.hold)
                            while (lds32_volatile(hold) != 0u) __nanosleep(32);
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
                (void)noload;
                (void)straddle_;
#else
                int li = 0, li_start = 0, li_next = count > 1 ? op.tile_start[1] : 0x7fffffff;
                for (int j = 0; j < t1 - t0; ++j) {
                    const int tile = tile_seq(j, t0, t1, straddle_);
                    if (j <= 1 && straddle_) {
                        li = 0;
                        li_start = 0;
                        li_next = count > 1 ? op.tile_start[1] : 0x7fffffff;
                    }
                    while (tile >= li_next) {
                        ++li;
                        li_start = li_next;
                        li_next = li + 1 < count ? op.tile_start[li + 1] : 0x7fffffff;
                    }
                    const CUtensorMap *map = op.maps[li];
                    const int row0 = (tile - li_start) * kTileRows;
                    for (int ch = 0; ch < nchunks; ++ch) {
                        mbar_wait(empty + 8u * s, ph ^ 1u);
                        if (a.hold)
                            while (lds32_volatile(hold) != 0u) __nanosleep(32);
                        const uint32_t st = ring + (uint32_t)s * kStageBytes;
                        const uint32_t fb = full + 8u * s;
                        if (noload) {
                            mbar_arrive(fb);   // debug: no weight traffic (the chain alone, garbage results)
                        } else {
                            mbar_expect_tx(fb, (uint32_t)kStageBytes);
                            tma_3d(st, map, 0, row0, ch * 8, fb, pol);
                            tma_2d(st + 8 * kBox, map + 1, ch * kChunkBlocks, row0, fb, pol);
                        }
                        if (++s == S) {
                            s = 0;
                            ph ^= 1u;
                        }
                    }
                }
#endif
            }
        }
        if (a.clustered) cluster_sync_all();
        return;
    }

    // ================= consumers =================
    uint32_t kNib2 = 0x000F000Fu, kMagic = 0x43004300u;
    asm volatile("" : "+r"(kNib2), "+r"(kMagic));
    int s = 0;
    uint32_t ph = 0, goph = 0, ts = 0;
    // hold modes: 1 always, 2 only while a tagged-bf16 input is staged (not records), 3 only
    // for W4A16 inputs -- decided per linear from the linear about to be staged
    bool hold_on = false;
    auto hold_for = [&](int j) {
        if (j >= a.nops || a.hold == 0) return false;
        const StackOp &nx = ops[j];
        if (a.hold == 2) return nx.xt != nullptr;
        if (a.hold == 3) return nx.route == MCAPQ_W4A16;
        return true;
    };
    auto hold_set = [&](uint32_t v) {
        if (a.hold && threadIdx.x == 0 && (v == 0u || hold_on)) hold_write(hold, v);
    };
    for (int i = 0; i < a.nops; ++i) {
        const StackOp &op = ops[i];
        const int count = op.count, route = op.route;
        const int64_t k = op.k;
        const int G = (int)(k / 32);
        const int K2 = (int)(k / 2);
        const int nchunks = (K2 + kChunkBytes - 1) / kChunkBytes;
        int t0, t1;
        bool straddle_;
        cta_tiles(i, t0, t1, straddle_);
        unsigned long long tr0 = 0, tr1 = 0, tr2 = 0, tr3 = 0, tr4 = 0, trm = 0;
        unsigned int stalls = 0, nstages = 0;
        if (kTrace) tr0 = globaltimer();
        if (t1 > t0) {
            // ---- barrier dependency: wait for the sync warp's release
            if (op.wait_op >= 0) {
                mbar_wait(go, goph);
                goph ^= 1u;
            }
            if (kTrace) tr1 = globaltimer();
            const bool a16 = kRoutes == 2 ? true : (kRoutes == 1 ? false : route == MCAPQ_W4A16);
            const ActSmem L = act_layout(a16, act, k, 1);
            hold_on = hold_for(i);
            hold_set(1u);
            bar_consumers();   // every warp is done reading the previous linear's activations
            if (!(a.flags & 4)) stage_step<kRounds>(kTrace ? &trm : nullptr, op, a16, L, threadIdx.x, t16, !(a.flags & 8), a.spin_ns, a.polls, a.counters,
                                                         !(a.flags & 128), t8, a.rec_spin);
            bar_consumers();
            hold_set(0u);
            hold_on = hold_for(i + 1);   // the in-loop set below is for the next linear's staging
            if (kTrace) tr2 = globaltimer();

            if (!a16) {
                // ---- W4A8, row-lane DP4A: lane -> row r = lane & 15 of the tile, and
                // lambda = warp + 16 (lane >> 4) -> blocks lambda and lambda + 32 of every
                // chunk.  The (warp, half) slots are exactly the 32 lanes of stream_linear's
                // warp-per-row engine (lane lambda holds blocks lambda, lambda + 32, same
                // fmaf order over chunks); one shuffle (xor 16) makes that engine's first
                // butterfly level and the epilogue warp finishes its tree over the 16
                // warps -- bit-identical outputs, one shuffle per tile instead of five.
                const int r = lane & 15, lam = warp + 16 * (lane >> 4);
                const uint32_t o0 = nib_off(r, lam), o1 = nib_off(r, lam + 32);
                const uint32_t os0 = scale_off(r, lam), os1 = scale_off(r, lam + 32);
                // K = 2048 (one chunk): the lane's two activation blocks are the same in
                // every tile: registers (2-round variant only: the 96-register cap)
                const bool reg_act = kRounds == 2 && K2 == kChunkBytes;
                Dp4aAct A;
                if (reg_act) A = dp4a_act_load_pair(L, lam, lam + 32, (uint32_t)K2);
                if ((K2 & (kChunkBytes - 1)) == 0) {
                    // lean path (every chunk full: K % 2048 == 0, all the configs' step
                    // linears): no per-stage predicates, the stage address advanced
                    // incrementally, the activation mode a compile-time branch; the same
                    // loads, block order and fmaf chain as below, so the outputs are
                    // bit-identical
                    auto lean = [&](auto reg_c) {
                        constexpr bool kReg = decltype(reg_c)::value;
                        uint32_t st = ring + (uint32_t)s * kStageBytes;
                        uint32_t xa = L.act + 16u * (uint32_t)lam, xs = L.ssq + 8u * (uint32_t)lam;
                        for (int tile = t0; tile < t1; ++tile, ++ts) {
                            float acc = 0.f;
                            const int hold_ch = tile == t1 - 1 ? nchunks - 1 : -1;
                            for (int ch = 0; ch < nchunks; ++ch) {
                                if (kTrace) {
                                    ++nstages;
                                    if (!mbar_test(full + 8u * s, ph)) ++stalls;
                                }
                                mbar_wait(full + 8u * s, ph);
                                if (kTrace && tile == t0 && ch == 0) tr3 = globaltimer();
                                const uint4 w0 = lds128(st + o0), w1 = lds128(st + o1);
                                const uint32_t h0 = lds16(st + os0), h1 = lds16(st + os1);
                                if constexpr (!kReg) {
                                    const uint32_t xo = 16u * kChunkBlocks * (uint32_t)ch;
                                    A.qa0 = lds128(xa + xo);
                                    A.qb0 = lds128(xa + xo + (uint32_t)K2);
                                    A.qa1 = lds128(xa + xo + 512u);
                                    A.qb1 = lds128(xa + xo + 512u + (uint32_t)K2);
                                    A.p0 = lds64(xs + xo / 2u);
                                    A.p1 = lds64(xs + xo / 2u + 256u);
                                }
                                __syncwarp();
                                if (lane == 0) mbar_arrive(empty + 8u * s);
                                if (ch == hold_ch) hold_set(1u);   // the linear's last stage is resident
                                if (++s == S) {
                                    s = 0;
                                    ph ^= 1u;
                                    st = ring;
                                } else {
                                    st += (uint32_t)kStageBytes;
                                }
                                const int D0 = block_D(w0, A.qa0, A.qb0, (int)A.p0.y);
                                const int D1 = block_D(w1, A.qa1, A.qb1, (int)A.p1.y);
                                acc = fmaf(h2f((uint16_t)h0) * __uint_as_float(A.p0.x), (float)D0, acc);
                                acc = fmaf(h2f((uint16_t)h1) * __uint_as_float(A.p1.x), (float)D1, acc);
                            }
                            if (kTrace) tr4 = globaltimer();
                            acc += __shfl_xor_sync(0xffffffffu, acc, 16);
                            const uint32_t slot = ts & (EN - 1u);
                            if (ts >= EN) mbar_wait(epe + 8u * slot, ((ts >> EL) - 1u) & 1u);
                            if (lane < 16) sts32(red + 1024u * slot + 64u * warp + 4u * lane, __float_as_uint(acc));
                            __syncwarp();
                            if (lane == 0) mbar_arrive(epf + 8u * slot);
                        }
                    };
                    if (reg_act)
                        lean(std::true_type{});
                    else
                        lean(std::false_type{});
                } else
                for (int tile = t0; tile < t1; ++tile, ++ts) {
                    float acc = 0.f;
                    for (int ch = 0; ch < nchunks; ++ch) {
                        const int rem = K2 - ch * kChunkBytes;
                        const int nblk = (rem < kChunkBytes ? rem : kChunkBytes) / 16;
                        const int blk0 = ch * kChunkBlocks;
                        if (kTrace) {
                            ++nstages;
                            if (!mbar_test(full + 8u * s, ph)) ++stalls;   // stage not resident yet
                        }
                        mbar_wait(full + 8u * s, ph);
                        if (tile == t1 - 1 && ch == nchunks - 1) hold_set(1u);   // the linear's last stage is resident
                        if (kTrace && tile == t0 && ch == 0) tr3 = globaltimer();
                        const uint32_t st = ring + (uint32_t)s * kStageBytes;
                        const bool on0 = lam < nblk, on1 = lam + 32 < nblk;
                        uint4 w0 = make_uint4(0, 0, 0, 0), w1 = w0;
                        uint32_t h0 = 0, h1 = 0;
                        if (on0) {
                            w0 = lds128(st + o0);
                            h0 = lds16(st + os0);
                        }
                        if (on1) {
                            w1 = lds128(st + o1);
                            h1 = lds16(st + os1);
                        }
                        if (!reg_act) A = dp4a_act_load_pair(L, blk0 + lam, blk0 + lam + 32, (uint32_t)K2);
                        const Dp4aAct &X = A;
                        __syncwarp();
                        if (lane == 0) mbar_arrive(empty + 8u * s);   // release: the stage's reads are done
                        if (++s == S) {
                            s = 0;
                            ph ^= 1u;
                        }
                        if (!(a.flags & 1)) {
                            if (on0) acc = fmaf(h2f((uint16_t)h0) * __uint_as_float(X.p0.x),
                                                (float)block_D(w0, X.qa0, X.qb0, (int)X.p0.y), acc);
                            if (on1) acc = fmaf(h2f((uint16_t)h1) * __uint_as_float(X.p1.x),
                                                (float)block_D(w1, X.qa1, X.qb1, (int)X.p1.y), acc);
                        }
                    }
                    if (kTrace) tr4 = globaltimer();
                    acc += __shfl_xor_sync(0xffffffffu, acc, 16);
                    const uint32_t slot = ts & (EN - 1u);
                    if (ts >= EN) mbar_wait(epe + 8u * slot, ((ts >> EL) - 1u) & 1u);
                    if (lane < 16) sts32(red + 1024u * slot + 64u * warp + 4u * lane, __float_as_uint(acc));
                    __syncwarp();
                    if (lane == 0) mbar_arrive(epf + 8u * slot);
                }
            } else {
                // ---- W4A16, HMMA1 engine (warp w owns blocks 4w..4w+3 for all 16 rows)
                // every chunk full (K % 2048 == 0): chunk_hmma1 with the lane offsets computed
                // once per linear (bit-identical to chunk_mma<HMMA1>) -- W4A16-only programs
                // (in the mixed kernel the extra live registers spill in the W4A8 staging)
                const bool full_chunks = kRoutes == 2 && (K2 & (kChunkBytes - 1)) == 0;
                const Hmma1Lane H = hmma1_lane(L, warp, lane);

                for (int tile = t0; tile < t1; ++tile, ++ts) {
                    float acc[4] = {0.f, 0.f, 0.f, 0.f};
                    for (int ch = 0; ch < nchunks; ++ch) {
                        const int rem = K2 - ch * kChunkBytes;
                        const int nblk = (rem < kChunkBytes ? rem : kChunkBytes) / 16;
                        const int blk0 = ch * kChunkBlocks;
                        if (kTrace) {
                            ++nstages;
                            if (!mbar_test(full + 8u * s, ph)) ++stalls;   // stage not resident yet
                        }
                        mbar_wait(full + 8u * s, ph);
                        if (tile == t1 - 1 && ch == nchunks - 1) hold_set(1u);   // the linear's last stage is resident
                        if (kTrace && tile == t0 && ch == 0) tr3 = globaltimer();
                        const uint32_t st = ring + (uint32_t)s * kStageBytes;
                        if (full_chunks && !(a.flags & 1))
                            chunk_hmma1(st, 4096u * (uint32_t)ch, 2048u * (uint32_t)ch, H, kNib2, kMagic, acc[0], acc[2]);
                        else if (!(a.flags & 1))
                            chunk_mma<HMMA1>(st, nblk, blk0, (uint32_t)K2, L, G, 1, warp, lane, kNib2, kMagic, acc);
                        __syncwarp();
                        if (lane == 0) mbar_arrive(empty + 8u * s);
                        if (++s == S) {
                            s = 0;
                            ph ^= 1u;
                        }
                    }
                    if (kTrace) tr4 = globaltimer();
                    // ---- hand the tile's partials to the epilogue warp (slot ts mod EN)
                    const uint32_t slot = ts & (EN - 1u);
                    if (ts >= EN) mbar_wait(epe + 8u * slot, ((ts >> EL) - 1u) & 1u);
                    const uint32_t sl = red + 1024u * slot;
                    // HMMA1: lanes t == 0 hold rows gid (acc[0]) and gid + 8 (acc[2]) of token 0
                    if ((lane & 3) == 0) {
                        sts32(sl + 64u * warp + 4u * (lane >> 2), __float_as_uint(acc[0]));
                        sts32(sl + 64u * warp + 4u * ((lane >> 2) + 8), __float_as_uint(acc[2]));
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(epf + 8u * slot);
                }
            }
        }
        if (kTrace && threadIdx.x == 0) {
            unsigned long long *r = a.trace + 8ull * ((unsigned long long)i * gridDim.x + blockIdx.x);
            r[0] = (unsigned long long)i;
            // CTA | staging split (ns from the go point to loads checked, 16 bits) | stalls | stages
            const unsigned long long mid = trm > tr1 ? (trm - tr1 < 65535ull ? trm - tr1 : 65535ull) : 0ull;
            r[1] = ((unsigned long long)blockIdx.x << 48) | (mid << 32) | ((unsigned long long)stalls << 16) | nstages;
            r[2] = tr0;
            r[3] = tr1;
            r[4] = tr2;
            r[5] = globaltimer();
            r[6] = tr3;
            r[7] = tr4;
        }
    }
    hold_set(0u);   // never leave the producer held
    if (a.clustered) cluster_sync_all();
}
