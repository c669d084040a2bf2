// stream.h -- the persistent TMA-fed decode-linear path (kernels_stream.cu).
#pragma once
#include <cuda.h>

#include "internal.h"

namespace mcapq {

constexpr int kMaxGroup = 4;   // linears sharing one input per launch (q/k/v, gate/up)
constexpr int kMaxPeers = 8;   // a8 fused column shard: one NVSwitch node

// Host description of a group of linears that share the same input x.
struct StreamGroup {
    int count;
    int64_t k;
    const uint8_t *nib[kMaxGroup];
    const uint16_t *scale[kMaxGroup];
    int64_t n[kMaxGroup];
    void *y[kMaxGroup];
    int64_t ldy[kMaxGroup];
    // a8 fused epilogue (M = 1): every output element is also stored at byte offset
    // peer_delta[p] from its local address, p < npeers (the LSA peers' replicas of y_full,
    // NVLink stores); npeers = 0: local stores only
    int64_t peer_delta[kMaxPeers];
    int npeers;
};

// Kernel parameters.  The TMA descriptors travel IN the parameter block
// (__grid_constant__), encoded on the host per launch: a hot-path call never
// allocates, never uploads and holds no per-weight cache, so it is capturable at any
// time (maps[i] = {nib map, scale map} of linear i of the group):
//   nib  : uint8 3-D view {128 B, N rows, K/256 columns}, box {128, 16, 8}, 128B swizzle
//   scale: uint16 [N][K/32], box {64, 16 rows}, 128B swizzle
struct StreamArgs {
    alignas(64) CUtensorMap maps[kMaxGroup][2];
    void *y[kMaxGroup];
    int64_t n[kMaxGroup];
    int64_t ldy[kMaxGroup];
    int tile_start[kMaxGroup + 1];
    int count;
    int64_t k;
    const uint16_t *x;
    int64_t ldx;
    int64_t tok0;
    int ntok;
    int ydt;
    int stages;
    int act_off;     // byte offset of the activation area in dynamic smem
    int red_off;     // byte offset of the reduction area
    int xraw_off;    // byte offset of the raw x staging area
    unsigned long long *trace;   // debug timeline (MCAPQ_STREAM_TRACE): 8 u64 per CTA, or null
    int launch_id;
    int smem_kb;     // host side: shared-memory plan of this launch (plan_smem)
    int32_t *dump_d;     // DUMP engine: D [n][k/32] int32
    uint32_t *dump_act;  // DUMP engine: CTA 0's staged activations (q_lo|q_hi bytes, then {s, 8 sum q} pairs)
    // NEXT-2 greedy-decode mode (one linear, one token): no y is stored; each row's fp32
    // output y_n becomes the key argmax_key(y_n, amax_off + n) and the largest key of
    // the launch is atomicMax-ed into *amax_key (zeroed by the launcher first)
    unsigned long long *amax_key;
    int64_t amax_off;
    int64_t peer_delta[kMaxPeers];   // see StreamGroup
    int npeers;
};

// Debug timeline (MCAPQ_STREAM_TRACE=1): per CTA {launch, block, t_start, t_wait,
// t_ready, t_end, 0, 0} from %globaltimer (ns).  Returns the number of records
// copied into host_out (<= max_records).
size_t stream_trace_read(unsigned long long *host_out, size_t max_records);

// K % 256 == 0 (16-B aligned scale rows for the tensor maps) and 16-B aligned planes.
bool stream_supported(int64_t k);
// Persistent decode-step kernel (stack_kernel.cuh): a program of ops, one per
// grouped linear, executed in order in ONE cooperative launch (M = 1 tokens).
size_t stack_op_bytes();
bool stack_step_enabled();   // MCAPQ_STEP_KERNEL (default 1)
// Dependencies of one op inside the step (stack.cu derives them from the buffers).
struct StackDeps {
    const uint32_t *xt;           // x is the tagged output of an earlier op (dataflow), or null
    int xt_op;                    // that op
    uint32_t *yt[kMaxGroup];      // tagged copies of this op's outputs read later, or null
    int wait_op;                  // barrier: wait until every CTA finished op wait_op, or -1
    int publish;                  // some later op waits on this one
    // producer-side quantisation: quantised records of this op's outputs read later by a
    // W4A8 op (6 u64 per 32-group), and the records this op's x comes from
    unsigned long long *yq[kMaxGroup];
    const unsigned long long *xq;
};
// The step kernel runs as clusters of 2 CTAs (paired tiles, producer-side quantisation):
// the device co-schedules one cluster per SM pair for the whole grid.
bool stack_clustered();
constexpr size_t kStackRecBytes = 48;   // one 32-group record
// Smallest consumer K that takes producer-side quantised records (MCAPQ_STEP_REC_MINK):
// below it the consumer quantises the tagged bf16 words itself.
int64_t stack_rec_min_k();
// Largest K the step kernel stages (4 rounds of 512 quad threads).
constexpr int64_t kStepMaxK = 16384;
// Fill one op (host memory, stack_op_bytes() bytes) for `route` over group g with
// input x [k] bf16 and outputs g.y (ydt); encodes/uploads descriptors on `s`.
// The op's TMA descriptors are encoded into host_maps[2 * count] (copied by the caller
// to dev_maps, the stack's own device array; op.maps point there).
bool stack_fill_op(void *host_op, int route, const StreamGroup &g, const uint16_t *x, int ydt, const StackDeps &d,
                   CUtensorMap *host_maps, const CUtensorMap *dev_maps);
// Launch the step: ops_dev = nops filled ops in device memory; counters_dev = nops + 2
// uint32 (zeroed once at allocation; the kernel's last CTA resets them and advances
// the epoch at [nops + 1]); max_k = the largest K of the program; clustered = the
// program uses producer-quantised records (clusters of 2, requires stack_clustered());
// route_kinds = bit 0 some W4A8 op, bit 1 some W4A16 op.
cudaError_t launch_stack_step(const void *ops_dev, const void *part_dev, int nops, unsigned int *counters_dev,
                              int64_t max_k, bool clustered, int route_kinds, cudaStream_t s);
// [nops][grid] int2 tile ranges of a step program (host; see kernels_stream.cu)
void stack_partition(const void *ops_host, int nops, int grid, bool clustered, double rec_r, int2 *out);
double stack_rec_r();

// Encode the {nib, scale} tensor-map pair of a packed weight for the stream / step
// kernels (host only; false if the driver entry point is missing or encoding fails).
bool encode_maps(CUtensorMap *tn, CUtensorMap *ts, const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k);
int stream_tokens_per_pass(int route, int64_t k);
// NEXT-2: per-token argmax keys of a routed linear's fp32 outputs, row indices offset by
// row_off: keys[i] = max_n argmax_key(y[i][n], row_off + n).  M = 1 on the stream path:
// fused into the linear's epilogue (the logits never reach memory); otherwise the fp32
// logits go to ws (argmax_logits_bytes) and a row-reduction kernel takes the keys.
cudaError_t launch_argmax_fused(int route, const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k,
                                const uint16_t *x, int64_t row_off, unsigned long long *key, cudaStream_t s);
cudaError_t launch_argmax_rows(const float *logits, int64_t m, int64_t n, int64_t ld, int64_t row_off,
                               unsigned long long *keys, cudaStream_t s);
// idx[i] / val[i] from the largest of keys[p][i] over p < parts (any order: max is exact)
cudaError_t launch_argmax_combine(const unsigned long long *keys, int parts, int64_t m, int64_t *idx, float *val,
                                  cudaStream_t s);
// TEST ENTRY (DUMP engine, one token, W4A8): the stream kernel's fused quantiser output
// (q [k] int8, sx/sq [k/32]) and every block's exact D [n][k/32] -- the production staging
// and block_D code, with the fp32 scale-accumulate replaced by stores.
size_t stream_dump_workspace_bytes(int64_t k);
cudaError_t launch_stream_dump(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k, const uint16_t *x,
                               int8_t *q, float *sx, int32_t *sq, int32_t *D, void *ws, cudaStream_t s);

// Batched decode (rows a5/a6): one weight pass per 64 tokens (gemm_kernel.cuh).
// Used for m >= kGemmMinTokens when K % 256 == 0.  W4A8 reads the quant_a8
// workspace (q [m][k], sx/sq [m][k/32]); W4A16 reads x [m][ldx] directly.
constexpr int64_t kGemmMinTokens = 9;
bool gemm_supported(int64_t k);
cudaError_t launch_tc05(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k, const uint16_t *x,
                        int64_t ldx, int64_t m, void *y, int ydt, int64_t ldy, cudaStream_t s, bool pdl);
cudaError_t launch_dequant_w4_bf16(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k, uint16_t *w,
                                   cudaStream_t s);
cudaError_t launch_prefill(const uint16_t *w, int64_t n, int64_t k, const uint16_t *x, int64_t ldx, int64_t m, void *y,
                           int ydt, int64_t ldy, cudaStream_t s, bool pdl);
cudaError_t launch_gemm(int route, const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k, const uint16_t *x,
                        int64_t ldx, const int8_t *q, const float *sx, const int32_t *sq, int64_t m, void *y, int ydt,
                        int64_t ldy, cudaStream_t s, bool pdl);
// A group of linears sharing x: the gemm path for m >= kGemmMinTokens (W4A8 quantises
// into ws first: a8_workspace_bytes(m, k) bytes), else the stream kernels.
cudaError_t launch_linear_group(int route, const StreamGroup &g, const uint16_t *x, int64_t m, int64_t ldx, int ydt,
                                void *ws, cudaStream_t s, bool pdl);
cudaError_t launch_stream_group(int route, const StreamGroup &g, const uint16_t *x, int64_t m, int64_t ldx,
                                int ydt, cudaStream_t s, bool pdl);
// a8 fused epilogue: one routed linear (M = 1, stream path: K % 256 == 0, K >= 2048) whose
// epilogue stores every output element at y + row and at the npeers byte offsets delta[p]
// from it (the LSA peers' replicas of y_full; the local one is delta 0)
cudaError_t launch_linear_peers(int route, const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k,
                                const uint16_t *x, void *y, int ydt, const int64_t *delta, int npeers, cudaStream_t s);

}  // namespace mcapq
