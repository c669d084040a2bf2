/*
 * mcapq.h -- C ABI of the B200-native MCAP/NVE mixed-precision decode linear
 * (arXiv 2604.21026).  Library: paper_2604_21026_b200/lib/libmcapq.so (sm_100a).
 *
 * The hot path: per layer i, route(i) = W4A16 if s^_i >= tau else W4A8
 * (Alg. 1 line 13 P:557, tau = 0.7 P:643-645), where
 *   W4A8  = Q4_0 int4 weights x per-token, per-32-group int8 activations, exact
 *           int32 group dot products, fp32 scale-and-accumulate (P:925-943,
 *           Appendix A);
 *   W4A16 = the same Q4_0 weights dequantised in register against bf16
 *           activations, fp32 accumulation.
 * Citations: "P:n" = PAPER.md line n, "S:n" = SPEC.md line n; "A<n>" = reading
 * n in DESIGN.md ("Readings of the paper").
 *
 * CONVENTIONS (apply to every call unless a call says otherwise)
 *  - Pointers: caller-owned DEVICE memory, except where a parameter says "host".
 *    The library never allocates device memory on a hot-path call and never
 *    frees caller memory.  Opaque objects (mcapq_profile, mcapq_comm,
 *    mcapq_stack) are library-owned and released by their *_free / *_destroy.
 *  - Streams: `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Every device call is stream-ordered, asynchronous, never
 *    synchronises and is CUDA-graph capturable (exceptions are marked).
 *  - Status: every call returns mcapq_status; nothing aborts or throws across
 *    the ABI.  Arguments are validated before anything is launched; on a non-OK
 *    status nothing was launched.  mcapq_last_error() gives a thread-local
 *    message for the last non-OK status on the calling thread.  Asynchronous
 *    device faults surface at the caller's next synchronisation.
 *  - Shapes: N = output features, K = input features (nn.Linear.weight is
 *    [N, K], row-major), M = tokens.  K % 32 == 0 (one Q4_0 block / activation
 *    group = 32 consecutive k, reading A1).  N >= 1, M >= 1.
 *  - Alignment: weights / activations / outputs 16-byte aligned; leading
 *    dimensions (ld*) in elements, multiples of 8, >= the row length.
 *  - Dtypes: activations are bf16 (uint16 bit patterns); outputs are bf16
 *    (RNE from fp32) or fp32, selected by mcapq_dtype (reading A11).
 *  - Hot-path calls do NOT check for non-finite inputs: outputs are then
 *    unspecified (never a fault).  mcapq_pack_w4 does check (dev_err).
 *
 * DATA LAYOUT of a packed weight ("Q4_0 SoA", reading A1/A2/A18):
 *    nib   : uint8  [N][K/2]; block g of row n = bytes 16g..16g+15 of the row,
 *            byte t = c[32g+t] | c[32g+t+16] << 4 (llama.cpp split nibble
 *            format); codes c in [0,15], value = d (c - 8)
 *            (zero point 8).
 *    scale : uint16 [N][K/32]: the block's d as IEEE binary16 bits (P:932:
 *            18 bytes per 32 elements = 16 nibble bytes + 2-byte fp16 d).
 *  The nibble bytes are byte-identical to the Q4_0 block's nibble field; only
 *  the d's are split into their own plane (structure-of-arrays).
 */
#ifndef MCAPQ_H
#define MCAPQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MCAPQ_ABI_VERSION 1

typedef enum {
    MCAPQ_OK = 0,
    MCAPQ_EINVAL = 1,  /* null pointer, bad shape (K % 32, M/N < 1), alignment, ld */
    MCAPQ_EDTYPE = 2,  /* unsupported dtype value */
    MCAPQ_ERANGE = 3,  /* value out of range (tau, world/rank, ...) */
    MCAPQ_EPARSE = 4,  /* malformed profile JSON */
    MCAPQ_ECUDA = 5,   /* CUDA runtime error (message in mcapq_last_error) */
    MCAPQ_ENCCL = 6,   /* NCCL error */
    MCAPQ_EUNSUP = 7,  /* valid request this build does not support */
    MCAPQ_ENOSPACE = 8 /* caller-provided workspace too small */
} mcapq_status;

typedef enum { MCAPQ_BF16 = 0, MCAPQ_F32 = 1 } mcapq_dtype;
typedef enum { MCAPQ_W4A8 = 0, MCAPQ_W4A16 = 1 } mcapq_route;

/* dev_err bits written by mcapq_pack_w4 (atomic OR into a caller uint32). */
#define MCAPQ_PACK_NONFINITE 0x1u /* a block contained inf/nan: stored as a zero block */
#define MCAPQ_PACK_OVERFLOW 0x2u  /* |m|/8 rounds to fp16 inf (A4): d stored as inf, codes 8 */

/* ---------------------------------------------------------------- library */
int mcapq_abi_version(void);
/* Thread-local text for the last non-OK status of this thread ("" if none). */
const char *mcapq_last_error(void);
const char *mcapq_status_string(int status);
/* Number of streaming multiprocessors of the current device (0 on error). */
int mcapq_device_sms(void);
/*
 * Launch the linears this host thread issues from now on with programmatic
 * dependent launch (enable = 1) or plainly (0, the default).  Under PDL a
 * linear's weight stream starts while the previous kernel on the stream is
 * still running (activations and outputs still wait for it), which hides the
 * launch and pipeline ramp of back-to-back decode linears.  The caller
 * guarantees that no kernel still in flight on the stream writes the packed
 * weights (true for weights packed and synchronised at load time).
 * Thread-local; returns the previous setting.
 */
int mcapq_set_pdl(int enable);

/* --------------------------------------------------------- packed weights */
/* Bytes of the nibble plane (N*K/2) and of the scale plane (N*(K/32)*2). */
size_t mcapq_w4_nib_bytes(int64_t n, int64_t k);
size_t mcapq_w4_scale_bytes(int64_t n, int64_t k);

/*
 * a1. Q4_0 weight pack (load time).  P:932-933; S:283-299;
 * readings A2-A5, A21.  Per row n, per 32-block g:
 *   m = x[argmax_j |x_j|] (first index on ties, A3); d = fp16_rne(m / -8) (A2);
 *   c_j = clamp(round_half_away(x_j / f32(d)), -8, 7) + 8 with IEEE division on
 *   the stored fp16 d (A4, A5); d == 0 -> all codes 8 and d stored +0 (A21).
 * w       : [n][ldw] of dtype wdt (MCAPQ_BF16 or MCAPQ_F32), ldw >= k.
 * nib     : out, [n][k/2] uint8.   scale: out, [n][k/32] fp16 bits.
 * dev_err : nullable device uint32; MCAPQ_PACK_* bits are OR-ed in (never
 *           cleared).  A non-finite block is stored as a zero block; an fp16
 *           overflow stores d = +-inf with all codes 8.
 * Bit-exact with the oracle (tests/test_gpu_parity.py).
 */
mcapq_status mcapq_pack_w4(const void *w, int wdt, int64_t n, int64_t k, int64_t ldw, uint8_t *nib,
                           uint16_t *scale, uint32_t *dev_err, void *stream);

/*
 * a2. Per-token, per-32-group int8 activation quantisation.  P:929-931,
 * Appendix A.1; readings A6-A8, A21.  Per row i, group g:
 *   a = max |x|; s = a / 127.0f (IEEE); q = clamp(round_half_away(x / s), -127,
 *   127); sq = sum q (int32, the paper's sum_x).  a == 0 (or s == 0) -> s = +0,
 *   q = 0.
 * x : [m][ldx] bf16.  q: out [m][k] int8.  sx: out [m][k/32] fp32.
 * sq: out [m][k/32] int32.  Bit-exact with the oracle.
 */
mcapq_status mcapq_quant_a8(const uint16_t *x, int64_t m, int64_t k, int64_t ldx, int8_t *q, float *sx,
                            int32_t *sq, void *stream);

/*
 * a3/a5. W4A8 linear on pre-quantised activations.
 * (deferred bias correction), reading A9:
 *   D[i][n][g] = sum_j c_{n,32g+j} q_{i,32g+j} - 8 sq[i][g]   (exact int32)
 *   y[i][n]    = sum_g (f32(d_{n,g}) * sx[i][g]) * f32(D)      (fp32 accumulate)
 * nib/scale: packed weight [n, k].  q/sx/sq: as written by mcapq_quant_a8 for m
 * tokens (row strides k, k/32, k/32).  y: out [m][ldy] of dtype ydt.
 * m == 1 runs the batch-1 GEMV (dp4a), m > 1 the int8 tensor-core kernel; for
 * m >= 9 with K % 256 == 0 (and sx, sq 16-byte aligned) the batched kernel
 * streams each weight once per 64 tokens (rows a5: mma.sync IMMA m16n8k32 per
 * block; for m > 32 with at least one 128-row tile per SM, tcgen05 kind::i8 with
 * the per-block D read back from TMEM).  Within one kernel the fp32 summation
 * order depends on K only (never on N, M or the grid), so a column shard of the
 * weight gives bit-identical rows (A22) whenever shard and whole run the same
 * kernel; the two batched kernels differ by fp32 rounding (within reading T).
 */
mcapq_status mcapq_w4a8(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k, const int8_t *q,
                        const float *sx, const int32_t *sq, int64_t m, void *y, int ydt, int64_t ldy,
                        void *stream);

/*
 * Workspace (device bytes) a fused-quantise call needs for m tokens of k:
 * q + sx + sq, 256-byte aligned pieces.  Route W4A16 needs 0.
 */
size_t mcapq_workspace_bytes(int route, int64_t m, int64_t n, int64_t k);

/*
 * a2+a3/a5. W4A8 from bf16 activations: quantise x into the workspace
 * (mcapq_quant_a8), then mcapq_w4a8; the two launches are chained with
 * programmatic dependent launch so the GEMV's weight stream starts while the
 * quantiser runs.  ws: device workspace of >= mcapq_workspace_bytes(W4A8,...).
 */
mcapq_status mcapq_w4a8_x(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k, const uint16_t *x,
                          int64_t m, int64_t ldx, void *y, int ydt, int64_t ldy, void *ws, size_t ws_bytes,
                          void *stream);

/*
 * a4/a6. W4A16 linear: exact dequantisation (reading A10/A13):
 *   y[i][n] = sum_k (f32(d_{n,k/32}) (c_{n,k} - 8)) x_{i,k}, fp32 accumulation.
 * Each term is exact in fp32; the inner per-group sums run on bf16 tensor cores
 * (c - 8 is exact in bf16) with fp32 accumulation, the scale d is applied per
 * group in fp32.  x: [m][ldx] bf16.  y: out [m][ldy].  m >= 9 with K % 256 == 0
 * runs the batched kernel (row a6: one weight pass per 64 tokens; mma.sync HMMA on
 * c - 8, or -- with at least one 128-row tile per SM -- tcgen05 kind::f16 with one
 * TMEM accumulator per Q4_0 block, the same semantics within reading T).
 */
mcapq_status mcapq_w4a16(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k, const uint16_t *x,
                         int64_t m, int64_t ldx, void *y, int ydt, int64_t ldy, void *stream);

/*
 * a6 (bf16-dequant semantics, reading A13): W4A16 as "dequantise to 16-bit, then a
 * dense GEMM" (the paper's prefill path, "materializes F16 for cuBLAS"):
 *   W^[n][k] = bf16_rne(f32(d_{n,k/32}) (c_{n,k} - 8)),  y[i][n] = sum_k W^[n][k] x[i][k]
 * with fp32 accumulation over all of K.  Unlike mcapq_w4a16 each weight is rounded
 * once to bf16 (|W^ - d (c - 8)| <= 2^-9 |d (c - 8)|), which lets the whole K
 * reduction stay in the tensor core: tcgen05.mma kind::f16, accumulator in TMEM,
 * 128 weight rows x <= 64 tokens per CTA, one weight pass per 64 tokens.  Meant for
 * batched decode / prefill (m >= 9); any m >= 1 is accepted.
 * Layout/ownership as mcapq_w4a16 (x [m][ldx] bf16, y [m][ldy], caller-owned device
 * memory, stream-ordered, graph-capturable).  Errors: MCAPQ_EUNSUP unless k % 256 == 0;
 * MCAPQ_EINVAL for a scale plane not 16-byte aligned, ldx % 8 != 0, or the checks of
 * mcapq_w4a16.
 */
mcapq_status mcapq_w4a16_bf16deq(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k,
                                 const uint16_t *x, int64_t m, int64_t ldx, void *y, int ydt, int64_t ldy,
                                 void *stream);

/*
 * NEXT-4 (prefill / large M; the paper's "dequantise to 16-bit, then GEMM"): the
 * bf16-dequant semantics of mcapq_w4a16_bf16deq with the weights materialised ONCE:
 *   mcapq_dequant_w4_bf16: W^[n][k] = bf16_rne(f32(d) (c - 8)), bf16 row-major, caller's w
 *     (16-byte aligned, n*k*2 bytes; = mcapq_prefill_workspace_bytes(n, k)); load time or per
 *     prefill; bandwidth-bound (0.5625 B read + 2 B written per weight).
 *   mcapq_bf16w_gemm: y[i][n] = sum_k W^[n][k] x[i][k], fp32 accumulation: tcgen05.mma
 *     kind::f16 with the accumulator in TMEM, 128 weight rows x <= 256 tokens per CTA,
 *     W^ and x by TMA; K % 64 == 0 (else MCAPQ_EUNSUP), ldx % 8 == 0.
 *   mcapq_w4a16_bf16deq_prefill: both, W^ in ws (>= mcapq_prefill_workspace_bytes).
 * Layouts/ownership as mcapq_w4a16; stream-ordered, graph-capturable, no allocation.
 */
size_t mcapq_prefill_workspace_bytes(int64_t n, int64_t k);
mcapq_status mcapq_dequant_w4_bf16(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k, uint16_t *w,
                                   void *stream);
mcapq_status mcapq_bf16w_gemm(const uint16_t *w, int64_t n, int64_t k, const uint16_t *x, int64_t m, int64_t ldx,
                              void *y, int ydt, int64_t ldy, void *stream);
mcapq_status mcapq_w4a16_bf16deq_prefill(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k,
                                         const uint16_t *x, int64_t m, int64_t ldx, void *y, int ydt, int64_t ldy,
                                         void *ws, size_t ws_bytes, void *stream);

/*
 * NEXT-2: greedy decode on the lm_head ("decode uses greedy (argmax) sampling
 * throughout").  idx[i] = argmax_n y[i][n] of the routed linear's fp32
 * outputs (exactly the values mcapq_linear writes with ydt = MCAPQ_F32), ties -> the
 * lowest n (-0.0 == +0.0); val[i] = y[i][idx[i]] (val nullable).  idx: device [m] int64.
 * M = 1 with K % 256 == 0, K >= 2048 fuses the reduction into the linear's epilogue (the
 * logits never reach memory); otherwise the fp32 logits go to ws and a row reduction
 * follows.  Non-finite logits give an unspecified index.  ws: >=
 * mcapq_argmax_workspace_bytes(route, m, n, k, 1) device bytes, 16-byte aligned.
 *
 * mcapq_argmax_keys: the building block -- keys[i] (device uint64, [m], 8-byte aligned)
 * = the largest of key(y[i][n], row_offset + n) over the n rows of this (shard of the)
 * weight, key(v, j) = (the IEEE bits of v in unsigned total order) << 32 |
 * (0xffffffff - j): unsigned max of keys = larger value, then smaller index, so shards
 * combine in any order.  row_offset + n <= 2^32 - 1.  ws as above (unused on the fused
 * path).  mcapq_argmax_combine: idx / val of the largest key over keys[p][i], p < parts.
 */
size_t mcapq_argmax_workspace_bytes(int route, int64_t m, int64_t n, int64_t k, int parts);
mcapq_status mcapq_linear_argmax(int route, const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k,
                                 const uint16_t *x, int64_t m, int64_t ldx, int64_t *idx, float *val, void *ws,
                                 size_t ws_bytes, void *stream);
mcapq_status mcapq_argmax_keys(int route, const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k,
                               const uint16_t *x, int64_t m, int64_t ldx, int64_t row_offset, uint64_t *keys,
                               void *ws, size_t ws_bytes, void *stream);
mcapq_status mcapq_argmax_combine(const uint64_t *keys, int parts, int64_t m, int64_t *idx, float *val, void *stream);

/* Routed linear: route MCAPQ_W4A8 -> mcapq_w4a8_x, MCAPQ_W4A16 -> mcapq_w4a16. */
mcapq_status mcapq_linear(int route, const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k,
                          const uint16_t *x, int64_t m, int64_t ldx, void *y, int ydt, int64_t ldy, void *ws,
                          size_t ws_bytes, void *stream);

/*
 * Grouped routed linear: `count` (1..4) linears that share the same input x
 * (q/k/v, gate/up; the paper's fused QKV kernel P:977) in ONE launch.  Host
 * arrays nibs/scales/ns/ys/ldys give each linear's packed weight, N, output and
 * its leading dimension; k, x, m, ldx, ydt are shared.  Results are identical
 * to `count` separate mcapq_linear calls (bit-for-bit).  ws: as mcapq_linear
 * (route W4A8 needs it when a linear falls off the K % 256 == 0 fast path, and
 * for m >= 9, where x is quantised once into ws for the batched kernel; else
 * MCAPQ_ENOSPACE / MCAPQ_EINVAL).
 */
mcapq_status mcapq_linear_group(int route, int count, const uint8_t *const *nibs, const uint16_t *const *scales,
                                const int64_t *ns, int64_t k, const uint16_t *x, int64_t m, int64_t ldx,
                                void *const *ys, int ydt, const int64_t *ldys, void *ws, size_t ws_bytes,
                                void *stream);

/*
 * End-to-end routed linear from HOST activations: copies x_host (pinned host,
 * [m][k] bf16) into the workspace, runs mcapq_linear, copies y back into y_host
 * (pinned host, [m][n] of ydt); all on `stream`, asynchronous (the caller
 * synchronises before reading y_host).  ws must hold
 * mcapq_host_workspace_bytes(route, m, n, k) bytes.
 */
size_t mcapq_host_workspace_bytes(int route, int64_t m, int64_t n, int64_t k);
mcapq_status mcapq_linear_host(int route, const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k,
                               const uint16_t *x_host, int64_t m, void *y_host, int ydt, void *ws,
                               size_t ws_bytes, void *stream);

/*
 * TEST ENTRY: the bit-exact integer stage of W4A8, D[i][n][g] (int32,
 * [m][n][k/32]) computed by the same fragment code as the tensor-core kernel
 * (mode 1) or the dp4a GEMV (mode 0).  P:937-942.
 */
mcapq_status mcapq_w4a8_group_dots(const uint8_t *nib, int64_t n, int64_t k, const int8_t *q, const int32_t *sq,
                                   int64_t m, int32_t *D, int mode, void *stream);

/*
 * TEST ENTRY: the persistent TMA stream kernel's W4A8 engine (the batch-1 DP4A path of
 * mcapq_linear, K % 256 == 0, K >= 2048) with its outputs replaced by its integer
 * stages: the fused in-kernel quantiser's codes for the one token x [k] bf16 (q [k]
 * int8, sx [k/32] fp32, sq [k/32] int32 -- a2's definition) and every
 * block's exact D [n][k/32] int32 = sum_j c q - 8 sq, computed by the
 * production staging and block_D code.  ws: >= mcapq_debug_stream_dump_workspace_bytes(k)
 * device bytes.  MCAPQ_EUNSUP off the stream path.
 */
size_t mcapq_debug_stream_dump_workspace_bytes(int64_t k);
mcapq_status mcapq_debug_stream_w4a8_dump(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k,
                                          const uint16_t *x, int8_t *q, float *sx, int32_t *sq, int32_t *D,
                                          void *ws, size_t ws_bytes, void *stream);

/*
 * DEBUG: per-CTA timeline of the stream kernels, recorded only when the
 * environment has MCAPQ_STREAM_TRACE=1 at library load.  Copies up to
 * max_records records of 8 uint64 into host memory (%globaltimer ns) and
 * synchronises the device; returns the number of records.
 *   per-linear kernels: {launch id, block, t_start, t_after_wait,
 *                        t_activations_ready, t_end, 0, t_first_stage}
 *   persistent step   : one record per (linear, CTA): {linear, block << 32 |
 *                        stalled stages << 16 | stages, t_start, t_after_go,
 *                        t_staged, t_end, t_first_stage, t_last_compute}
 */
size_t mcapq_debug_stream_trace(uint64_t *host_out, size_t max_records);

/*
 * DIAGNOSTIC (measurement only, never on the hot path): one streaming read of `bytes`
 * bytes of device memory at `buf` (16-B aligned, >= 16 bytes; the tail below 16 bytes
 * is skipped), LDG.128 with L1 no-allocate, 4 CTAs x 512 threads per
 * SM -- the pure-read HBM ceiling SURVEY 8(d) D.2 (iii) reports the GEMV beside.  `sink`
 * (device, 8 bytes) is written only to keep the loads live.  Stream-ordered; the caller
 * times it (CUDA events).  MCAPQ_EINVAL on a NULL / misaligned pointer.
 */
mcapq_status mcapq_debug_read_bw(const void *buf, size_t bytes, unsigned long long *sink, void *stream);

/* ------------------------------------------------------ dispatch table (a7) */
/*
 * MCAP profile -> per-layer routes.  Alg. 1 lines 8-13, P:840-846,
 * the 338-byte JSON profile.  Host-only, not graph-related.
 * JSON object (<= 64 KiB): "scores" (alias "normalized_scores") numeric array in
 * [0, 1], or "raw_scores" (min-max normalised; max - min < epsilon -> all 0,
 * P:550-552); optional "tau" (alias "threshold", default 0.7), "epsilon"
 * (default 1e-9, A14), "num_layers" (alias "layers", must equal the array
 * length); other keys ignored.  tau_override: NaN = use the file's / default.
 * route[i] = MCAPQ_W4A16 iff s^_i >= tau (ties -> W4A16).
 * Errors: MCAPQ_EPARSE (syntax, missing array, value outside [0,1], length
 * mismatch), MCAPQ_ERANGE (tau < 0 or non-finite).
 */
typedef struct mcapq_profile mcapq_profile;
mcapq_status mcapq_profile_parse(const char *json, size_t len, double tau_override, mcapq_profile **out);
int mcapq_profile_layers(const mcapq_profile *p);
double mcapq_profile_tau(const mcapq_profile *p);
mcapq_status mcapq_profile_scores(const mcapq_profile *p, double *scores_host, int n);
mcapq_status mcapq_profile_routes(const mcapq_profile *p, uint8_t *routes_host, int n);
void mcapq_profile_free(mcapq_profile *p);

/*
 * NEXT-3: the MCAP profile artifact from raw per-layer scores s_i (Alg. 1 line 10,
 * P:547-549): writes {"epsilon":1e-09,"format_version":1,"num_layers":L,"prompt_count":k,
 * "raw_scores":[...],"tau":tau} (NUL-terminated; keys sorted, every double in its shortest
 * round-trip form, so writing what mcapq_profile_parse read back gives the same bytes) into
 * buf (host, cap bytes); *len = length without the NUL.  mcapq_profile_parse of it min-max
 * normalises (lines 11-15) and routes (line 16); parse rejects epsilon <= 0 and negative raw
 * scores (sums of norms).  MCAPQ_ENOSPACE if cap < *len + 1; MCAPQ_EINVAL for NULL,
 * non-finite or negative input.
 */
mcapq_status mcapq_profile_write_json(const double *raw_scores_host, int layers, int prompts, double tau, char *buf,
                                      size_t cap, size_t *len);

/*
 * NEXT-3: MCAP profiling on the GPU (Alg. 1 lines 3-10).  For one layer and one
 * prompt of m tokens, given that layer's linear outputs as bf16 rows (Q x_t in yq [m][ldq],
 * first nq used; V x_t in yv; FFN(x_t) in yffn):
 *   a_t = || [Q x_t, V x_t] ||_2 + || FFN(x_t) ||_2      (fp64 from the exact bf16 values)
 *   *score += weight * sum_t a_t                          (fixed order: deterministic)
 * score: one device fp64 accumulator per layer (caller-owned, caller-initialised);
 * weight = 1 / (k m) gives Alg. 1's mean over prompts and tokens.  ws: device workspace of
 * >= mcapq_mcap_workspace_bytes(m) bytes.  Stream-ordered, no allocation, graph-capturable.
 * Errors: MCAPQ_EINVAL (NULL, m/n < 1, ld < n, non-finite weight), MCAPQ_ENOSPACE.
 */
size_t mcapq_mcap_workspace_bytes(int64_t m);
mcapq_status mcapq_mcap_accumulate(const uint16_t *yq, int64_t ldq, int64_t nq, const uint16_t *yv, int64_t ldv,
                                   int64_t nv, const uint16_t *yffn, int64_t ldf, int64_t nf, int64_t m,
                                   double weight, double *score, void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------ decode linear stack (a9) */
/*
 * A routed stack of decode linears: L layers x S slots, each slot a packed
 * weight, executed in (layer, slot) order with each layer's route from the
 * dispatch table (all slots of layer i share route[i], A12).  Slots that share
 * an input (same `input_id` within a layer, e.g. q/k/v) quantise it once
 * (A15).  The library owns a workspace and, after mcapq_stack_capture, a CUDA
 * graph that replays the whole step.
 *
 * Chaining: a slot's x may be an earlier slot's y (the decode chain, e.g. the
 * o input = the q output).  Ordering follows the buffers: a slot reads its x
 * only after every earlier writer of those bytes stored it, and writes its y
 * only after earlier readers/writers of those bytes are done.  At m = 1 an x
 * that is exactly an earlier bf16 y is passed by dataflow inside the
 * persistent step kernel (no grid barrier).  A slot's y must not overlap its
 * own x.
 *
 * mcapq_stack_create   : L layers, routes_host[L] (0/1), max_m tokens.
 * mcapq_stack_set      : register slot s of layer l: weight (device), the
 *                        device input x [m][k] bf16 and output y [m][n] (ydt),
 *                        input_id groups slots sharing x within the layer.
 * mcapq_stack_run      : launch every linear in order on `stream` (m tokens).
 * mcapq_stack_capture  : capture mcapq_stack_run into a graph (m tokens).
 * mcapq_stack_replay   : launch the captured graph on `stream`.
 * mcapq_stack_weight_bytes : total packed weight bytes (nib + scale).
 * mcapq_stack_launches : kernels one run launches.
 * mcapq_stack_host_bytes : bytes of one step's inputs (which = 0: every distinct
 *                        (layer, input_id) x that is a step input -- not written
 *                        by an earlier slot's y -- in that order, [m][k] bf16 each)
 *                        or outputs (which = 1: every slot's y in (layer, slot)
 *                        order, [m][n] of its ydt), packed back to back.
 * mcapq_stack_step_host : one end-to-end step from HOST memory: copy x_host
 *                        (pinned, the packed inputs) into the registered device
 *                        inputs, replay the captured graph (or run, if none was
 *                        captured for m), copy every output into y_host (pinned,
 *                        packed).  Asynchronous on `stream`.  Copies are merged
 *                        wherever consecutive slots are contiguous in device
 *                        memory (inputs placed in one arena in (layer, input_id)
 *                        order and outputs in (layer, slot) order => one H2D and
 *                        one D2H per step).
 */
typedef struct mcapq_stack mcapq_stack;
mcapq_status mcapq_stack_create(int layers, const uint8_t *routes_host, int64_t max_m, mcapq_stack **out);
mcapq_status mcapq_stack_set(mcapq_stack *st, int layer, int slot, int input_id, const uint8_t *nib,
                             const uint16_t *scale, int64_t n, int64_t k, const uint16_t *x, void *y, int ydt);
mcapq_status mcapq_stack_run(mcapq_stack *st, int64_t m, void *stream);
mcapq_status mcapq_stack_capture(mcapq_stack *st, int64_t m, void *stream);
mcapq_status mcapq_stack_replay(mcapq_stack *st, void *stream);
size_t mcapq_stack_weight_bytes(const mcapq_stack *st);
int mcapq_stack_launches(const mcapq_stack *st, int64_t m);
size_t mcapq_stack_host_bytes(const mcapq_stack *st, int64_t m, int which);
mcapq_status mcapq_stack_step_host(mcapq_stack *st, int64_t m, const void *x_host, void *y_host, void *stream);
void mcapq_stack_destroy(mcapq_stack *st);

/* ------------------------------------------- multi-GPU column shard (a8) */
/*
 * Column (output-feature) sharded linear across P GPUs of one node (north_star;
 * the paper is single-GPU).  Rank r owns rows [r N/P, (r+1) N/P)
 * of the packed weight (A22), computes its slice with the routed linear on the
 * replicated x, and all-gathers over NCCL (NVLink/NVSwitch) into y_full
 * [m][n_full] (bf16 or fp32), row-major.  Per-row arithmetic is identical to
 * the unsharded call, so y_full is bit-identical to a 1-GPU run.
 * mcapq_comm_unique_id (host): id[128] to broadcast (the caller uses a torch
 * process group); mcapq_comm_init: collective over the `world` ranks, binds the
 * communicator to the current CUDA device.  Not graph-capturable: init/destroy.
 * ws: >= mcapq_colshard_workspace_bytes(route, m, n_full, k, world).
 * Data path: M == 1 -- the local rows are written straight into y_full + r N/P and
 * the all-gather runs in place; M > 1 -- they go to slot r of a rank-major
 * [P][M][N/P] workspace, the all-gather fills it in place, and
 * mcapq_colshard_assemble writes y_full.
 *
 * mcapq_colshard_assemble: y_full[i][r N/P + j] = rank_major[r][i][j] for a rank-major
 * [world][m][n_full/world] buffer of ydt elements (device, caller-owned, no overlap).
 * The M > 1 assembly step of mcapq_linear_colshard; also a test entry (P shards
 * computed by mcapq_linear on one GPU, assembled, compared with the unsharded call).
 */
typedef struct mcapq_comm mcapq_comm;
mcapq_status mcapq_comm_unique_id(uint8_t *id_host_128);
mcapq_status mcapq_comm_init(const uint8_t *id_host_128, int world, int rank, mcapq_comm **out);
int mcapq_comm_world(const mcapq_comm *c);
int mcapq_comm_rank(const mcapq_comm *c);
size_t mcapq_colshard_workspace_bytes(int route, int64_t m, int64_t n_full, int64_t k, int world);
mcapq_status mcapq_linear_colshard(const mcapq_comm *c, int route, const uint8_t *nib_shard,
                                   const uint16_t *scale_shard, int64_t n_full, int64_t k, const uint16_t *x,
                                   int64_t m, void *y_full, int ydt, void *ws, size_t ws_bytes, int fused_epilogue,
                                   void *stream);
/*
 * fused_epilogue (SURVEY 8(e) "Collective: fused"; a8): with fused_epilogue != 0, m == 1
 * and a stream-path K (k % 256 == 0, k >= 2048), y_full must lie in a symmetric window from
 * mcapq_comm_window_alloc: the GEMV epilogue stores each of this rank's rows into EVERY
 * rank's replica of y_full directly over NVLink (NCCL symmetric window, LSA load/store
 * pointers; P stores per element), then one NCCL LSA barrier kernel orders them -- no
 * all-gather kernel, no separate copy.  Otherwise (fused_epilogue == 0, m > 1, or another
 * K) the NCCL all-gather path above runs.  Errors: MCAPQ_EINVAL if fused and y_full is not
 * in this communicator's window.
 *
 * mcapq_comm_window_alloc: COLLECTIVE over the communicator (every rank calls it with the
 * same bytes, in the same order): ncclMemAlloc + ncclCommWindowRegister(symmetric), and on
 * first use an ncclDevComm with one LSA barrier; *y_full = this rank's replica (device,
 * library-owned, 4 KiB-aligned size).  MCAPQ_EUNSUP when the ranks do not share one NVLink
 * (LSA) domain of <= 8 GPUs.  mcapq_comm_window_free: collective; frees it (synchronises
 * the device).  Not graph-capturable; the fused colshard call itself is.
 */
mcapq_status mcapq_comm_window_alloc(mcapq_comm *c, size_t bytes, void **y_full);
mcapq_status mcapq_comm_window_free(mcapq_comm *c, void *y_full);
/*
 * TEST ENTRY (a8 fused epilogue on one GPU): the routed linear (m = 1, stream-path K)
 * writing its n rows at y and, for every p < npeers, at y + peer_delta_host[p] bytes --
 * the per-peer stores of the fused epilogue with P emulated replicas in one allocation.
 * 1 <= npeers <= 8; peer_delta_host is host memory.
 */
mcapq_status mcapq_debug_linear_peers(int route, const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k,
                                      const uint16_t *x, void *y, int ydt, const int64_t *peer_delta_host, int npeers,
                                      void *stream);
mcapq_status mcapq_colshard_assemble(const void *rank_major, void *y_full, int64_t m, int64_t n_full, int world,
                                     int ydt, void *stream);
/*
 * a8 + NEXT-2: the column-sharded lm_head with a LOCAL argmax (greedy decode): rank r
 * reduces its N/P rows to m argmax keys (global row indices, mcapq_argmax_keys), an
 * all-gather moves P x m 8-byte keys instead of the m x N logits (M = 64, 8B lm_head:
 * 4 KB instead of 16.4 MB), and every rank combines them: idx / val exactly as
 * mcapq_linear_argmax on the unsharded weight.  ws: >= mcapq_argmax_workspace_bytes(route,
 * m, n_full / world, k, world).
 */
mcapq_status mcapq_linear_colshard_argmax(const mcapq_comm *c, int route, const uint8_t *nib_shard,
                                          const uint16_t *scale_shard, int64_t n_full, int64_t k, const uint16_t *x,
                                          int64_t m, int64_t *idx, float *val, void *ws, size_t ws_bytes,
                                          void *stream);
/*
 * NEXT-2 row-parallel (K-sharded) linear -- the Megatron partner of the column shard
 * ("row-parallel o/down with reduce-scatter or all-reduce instead of
 * gathering activations").  Rank r owns the K-slice [r K/P, (r+1) K/P) of the packed
 * weight (all n rows: nib_shard [n][k_shard/2], scale_shard [n][k_shard/32]) and of x
 * (x_shard [m][k_shard], row stride ldx elements) -- e.g. the output rows a column-sharded
 * up / q projection produced locally.  k_shard % 32 == 0, so every Q4_0 block and every
 * per-token int8 quantisation group lies in one rank: the codes and the
 * per-group int32 dot products are exactly the unsharded linear's; only the fp32
 * scale-and-accumulate over groups is split into P partial sums y_r[m][n]
 * (fp32), which the call sums over the ranks into y [m][n] (ydt bf16 or fp32, row stride
 * n) on every rank.  The sum order differs from the unsharded call: y equals it within
 * the north-star tolerance, not bit-for-bit.
 *   fused_epilogue == 0: y_r into ws (fp32; into y itself when ydt is fp32), NCCL sum
 *     all-reduce in place, conversion to ydt.  ws >= mcapq_rowshard_workspace_bytes().
 *   fused_epilogue != 0 (m == 1, stream-path k_shard): ws must be a window from
 *     mcapq_comm_window_alloc of >= P * n * 4 bytes ([P][n] fp32 slots).  LSA barrier
 *     (no peer still reads its slots), the GEMV epilogue stores y_r into slot r of EVERY
 *     rank's window over NVLink, LSA barrier, then every rank sums the P slots in rank
 *     order (mcapq_rowshard_reduce): one NVLink all-reduce, identical y on all ranks.
 * Errors: MCAPQ_EINVAL (k_shard not whole groups, NULL/misaligned buffers, fused ws not a
 * window), MCAPQ_EUNSUP (fused with m > 1 or a non-stream k_shard), MCAPQ_ENOSPACE.
 *
 * mcapq_rowshard_reduce: y[i][j] = sum_{r = 0 .. world-1} partials[r][i][j] in rank order
 * (fp32), written as ydt -- the fused path's reduction, the non-fused path's conversion
 * (world = 1), and a test entry (P shards computed by mcapq_linear on one GPU).
 * partials: device [world][m][n] fp32; y: device [m][n]; no overlap.
 */
size_t mcapq_rowshard_workspace_bytes(int route, int64_t m, int64_t n, int64_t k_shard, int world);
mcapq_status mcapq_linear_rowshard(const mcapq_comm *c, int route, const uint8_t *nib_shard,
                                   const uint16_t *scale_shard, int64_t n, int64_t k_shard, const uint16_t *x_shard,
                                   int64_t m, int64_t ldx, void *y, int ydt, void *ws, size_t ws_bytes,
                                   int fused_epilogue, void *stream);
mcapq_status mcapq_rowshard_reduce(const float *partials, int world, int64_t m, int64_t n, void *y, int ydt,
                                   void *stream);
void mcapq_comm_destroy(mcapq_comm *c);

#ifdef __cplusplus
}
#endif
#endif /* MCAPQ_H */
