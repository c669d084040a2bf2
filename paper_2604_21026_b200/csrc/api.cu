// api.cu -- the extern "C" boundary of libmcapq (include/mcapq.h): argument
// validation, status codes, workspace carve-up and route dispatch.  Every
// arithmetic step runs in the kernels of kernels_*.cu.
#include <cmath>
#include <cstring>
#include <mutex>
#include <set>
#include <utility>

#include "internal.h"
#include "stream.h"

namespace mcapq {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}
void clear_error() { g_err[0] = '\0'; }

int device_sms()
{
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    return sms;
}

cudaError_t kernel_smem_attr(const void *kernel, int smem_bytes, int carveout)
{
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> done;   // (kernel, device ordinal)
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    if (done.count({kernel, dev})) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (e == cudaSuccess && carveout >= 0)
        e = cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
    if (e == cudaSuccess) done.insert({kernel, dev});
    return e;
}

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

size_t a8_workspace_bytes(int64_t m, int64_t k)
{
    const int64_t G = k / 32;
    return align256((size_t)(m * k)) + align256((size_t)(m * G) * 4) + align256((size_t)(m * G) * 4);
}

A8Workspace a8_workspace(void *ws, int64_t m, int64_t k)
{
    const int64_t G = k / 32;
    uint8_t *p = reinterpret_cast<uint8_t *>(ws);
    A8Workspace w;
    w.q = reinterpret_cast<int8_t *>(p);
    p += align256((size_t)(m * k));
    w.sx = reinterpret_cast<float *>(p);
    p += align256((size_t)(m * G) * 4);
    w.sq = reinterpret_cast<int32_t *>(p);
    return w;
}

}  // namespace mcapq

using namespace mcapq;

#define CHECK_SHAPE(n, k, m)                                                                                  \
    MCAPQ_REQUIRE((n) >= 1 && (k) >= 32 && (k) % 32 == 0 && (m) >= 1, MCAPQ_EINVAL,                          \
                  "bad shape n=%lld k=%lld m=%lld (need n>=1, m>=1, k>=32, k%%32==0)", (long long)(n),      \
                  (long long)(k), (long long)(m))
#define CHECK_PTR(p, name) MCAPQ_REQUIRE((p) != nullptr, MCAPQ_EINVAL, "%s is NULL", name)
#define CHECK_AL16(p, name) MCAPQ_REQUIRE(aligned16(p), MCAPQ_EINVAL, "%s is not 16-byte aligned", name)
#define CHECK_LD(ld, minv, name)                                                                              \
    MCAPQ_REQUIRE((ld) >= (minv) && (ld) % 8 == 0, MCAPQ_EINVAL, "%s=%lld must be >= %lld and a multiple of 8", \
                  name, (long long)(ld), (long long)(minv))
#define CHECK_YDT(d) MCAPQ_REQUIRE((d) == MCAPQ_BF16 || (d) == MCAPQ_F32, MCAPQ_EDTYPE, "bad output dtype %d", (d))
#define LAUNCH_TRY(expr)                                                                                      \
    do {                                                                                                      \
        cudaError_t e_ = (expr);                                                                              \
        if (e_ != cudaSuccess) {                                                                              \
            set_error("kernel launch failed: %s", cudaGetErrorString(e_));                                  \
            return MCAPQ_ECUDA;                                                                               \
        }                                                                                                     \
    } while (0)

static mcapq_status check_weight(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k)
{
    CHECK_PTR(nib, "nib");
    CHECK_PTR(scale, "scale");
    CHECK_AL16(nib, "nib");
    MCAPQ_REQUIRE((reinterpret_cast<uintptr_t>(scale) & 1u) == 0, MCAPQ_EINVAL, "scale is not 2-byte aligned");
    (void)n;
    (void)k;
    return MCAPQ_OK;
}

extern "C" {

int mcapq_abi_version(void) { return MCAPQ_ABI_VERSION; }
const char *mcapq_last_error(void) { return g_err; }

const char *mcapq_status_string(int s)
{
    switch (s) {
    case MCAPQ_OK: return "ok";
    case MCAPQ_EINVAL: return "invalid argument";
    case MCAPQ_EDTYPE: return "unsupported dtype";
    case MCAPQ_ERANGE: return "value out of range";
    case MCAPQ_EPARSE: return "profile parse error";
    case MCAPQ_ECUDA: return "CUDA error";
    case MCAPQ_ENCCL: return "NCCL error";
    case MCAPQ_EUNSUP: return "unsupported";
    case MCAPQ_ENOSPACE: return "workspace too small";
    default: return "unknown status";
    }
}

int mcapq_device_sms(void) { return device_sms(); }

int mcapq_set_pdl(int enable)
{
    const int prev = api_pdl() ? 1 : 0;
    set_api_pdl(enable != 0);
    return prev;
}

size_t mcapq_debug_stream_trace(uint64_t *host_out, size_t max_records)
{
    if (!host_out) return 0;
    return stream_trace_read(reinterpret_cast<unsigned long long *>(host_out), max_records);
}

mcapq_status mcapq_debug_linear_peers(int route, const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k,
                                      const uint16_t *x, void *y, int ydt, const int64_t *peer_delta_host, int npeers,
                                      void *stream)
{
    clear_error();
    CHECK_SHAPE(n, k, 1);
    mcapq_status st = check_weight(nib, scale, n, k);
    if (st != MCAPQ_OK) return st;
    CHECK_PTR(x, "x");
    CHECK_PTR(y, "y");
    CHECK_YDT(ydt);
    MCAPQ_REQUIRE(peer_delta_host && npeers >= 1 && npeers <= kMaxPeers, MCAPQ_EINVAL, "bad peers");
    MCAPQ_REQUIRE(route == MCAPQ_W4A8 || route == MCAPQ_W4A16, MCAPQ_EINVAL, "bad route");
    MCAPQ_REQUIRE(stream_supported(k) && aligned16(scale), MCAPQ_EUNSUP, "stream-path K only (k %% 256 == 0, >= 2048)");
    LAUNCH_TRY(launch_linear_peers(route, nib, scale, n, k, x, y, ydt, peer_delta_host, npeers, as_stream(stream)));
    return MCAPQ_OK;
}

size_t mcapq_w4_nib_bytes(int64_t n, int64_t k) { return (n > 0 && k > 0) ? (size_t)(n * (k / 2)) : 0; }
size_t mcapq_w4_scale_bytes(int64_t n, int64_t k) { return (n > 0 && k > 0) ? (size_t)(n * (k / 32) * 2) : 0; }

mcapq_status mcapq_pack_w4(const void *w, int wdt, int64_t n, int64_t k, int64_t ldw, uint8_t *nib,
                           uint16_t *scale, uint32_t *dev_err, void *stream)
{
    clear_error();
    CHECK_SHAPE(n, k, 1);
    CHECK_PTR(w, "w");
    CHECK_PTR(nib, "nib");
    CHECK_PTR(scale, "scale");
    MCAPQ_REQUIRE(wdt == MCAPQ_BF16 || wdt == MCAPQ_F32, MCAPQ_EDTYPE, "bad weight dtype %d", wdt);
    MCAPQ_REQUIRE(ldw >= k, MCAPQ_EINVAL, "ldw=%lld < k=%lld", (long long)ldw, (long long)k);
    MCAPQ_REQUIRE((reinterpret_cast<uintptr_t>(w) & 3u) == 0 && (reinterpret_cast<uintptr_t>(scale) & 1u) == 0,
                  MCAPQ_EINVAL, "misaligned w/scale");
    LAUNCH_TRY(launch_pack_w4(w, wdt, n, k, ldw, nib, scale, dev_err, as_stream(stream)));
    return MCAPQ_OK;
}

mcapq_status mcapq_quant_a8(const uint16_t *x, int64_t m, int64_t k, int64_t ldx, int8_t *q, float *sx,
                            int32_t *sq, void *stream)
{
    clear_error();
    CHECK_SHAPE(1, k, m);
    CHECK_PTR(x, "x");
    CHECK_PTR(q, "q");
    CHECK_PTR(sx, "sx");
    CHECK_PTR(sq, "sq");
    MCAPQ_REQUIRE(ldx >= k, MCAPQ_EINVAL, "ldx=%lld < k", (long long)ldx);
    MCAPQ_REQUIRE((reinterpret_cast<uintptr_t>(x) & 1u) == 0, MCAPQ_EINVAL, "x misaligned");
    LAUNCH_TRY(launch_quant_a8(x, m, k, ldx, q, sx, sq, as_stream(stream), false));
    return MCAPQ_OK;
}

mcapq_status mcapq_w4a8(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k, const int8_t *q,
                        const float *sx, const int32_t *sq, int64_t m, void *y, int ydt, int64_t ldy, void *stream)
{
    clear_error();
    CHECK_SHAPE(n, k, m);
    mcapq_status st = check_weight(nib, scale, n, k);
    if (st != MCAPQ_OK) return st;
    CHECK_PTR(q, "q");
    CHECK_PTR(sx, "sx");
    CHECK_PTR(sq, "sq");
    CHECK_PTR(y, "y");
    CHECK_AL16(q, "q");
    CHECK_AL16(y, "y");
    CHECK_YDT(ydt);
    CHECK_LD(ldy, n, "ldy");
    if (m >= kGemmMinTokens && gemm_supported(k) && aligned16(scale) && aligned16(sx) && aligned16(sq)) {
        LAUNCH_TRY(launch_gemm(MCAPQ_W4A8, nib, scale, n, k, nullptr, 0, q, sx, sq, m, y, ydt, ldy, as_stream(stream),
                               false));
        return MCAPQ_OK;
    }
    LAUNCH_TRY(launch_w4a8(nib, scale, n, k, q, sx, sq, m, y, ydt, ldy, as_stream(stream), false));
    return MCAPQ_OK;
}

size_t mcapq_workspace_bytes(int route, int64_t m, int64_t n, int64_t k)
{
    (void)n;
    if (route != MCAPQ_W4A8 || m < 1 || k < 32) return 0;
    return a8_workspace_bytes(m, k);
}

mcapq_status mcapq_w4a8_x(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k, const uint16_t *x,
                          int64_t m, int64_t ldx, void *y, int ydt, int64_t ldy, void *ws, size_t ws_bytes,
                          void *stream)
{
    clear_error();
    CHECK_SHAPE(n, k, m);
    mcapq_status st = check_weight(nib, scale, n, k);
    if (st != MCAPQ_OK) return st;
    CHECK_PTR(x, "x");
    CHECK_PTR(y, "y");
    CHECK_PTR(ws, "ws");
    CHECK_AL16(x, "x");
    CHECK_AL16(y, "y");
    CHECK_AL16(ws, "ws");
    CHECK_YDT(ydt);
    CHECK_LD(ldx, k, "ldx");
    CHECK_LD(ldy, n, "ldy");
    MCAPQ_REQUIRE(ws_bytes >= a8_workspace_bytes(m, k), MCAPQ_ENOSPACE, "workspace %zu < %zu", ws_bytes,
                  a8_workspace_bytes(m, k));
    cudaStream_t s = as_stream(stream);
    if (stream_supported(k) && aligned16(scale)) {
        // persistent TMA-fed kernel with the quantiser fused into its prologue
        StreamGroup g = {};
        g.count = 1;
        g.k = k;
        g.nib[0] = nib;
        g.scale[0] = scale;
        g.n[0] = n;
        g.y[0] = y;
        g.ldy[0] = ldy;
        LAUNCH_TRY(launch_linear_group(MCAPQ_W4A8, g, x, m, ldx, ydt, ws, s, false));
        return MCAPQ_OK;
    }
    const A8Workspace w = a8_workspace(ws, m, k);
    LAUNCH_TRY(launch_quant_a8(x, m, k, ldx, w.q, w.sx, w.sq, s, false));
    LAUNCH_TRY(launch_w4a8(nib, scale, n, k, w.q, w.sx, w.sq, m, y, ydt, ldy, s, true));
    return MCAPQ_OK;
}

mcapq_status mcapq_w4a16(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k, const uint16_t *x,
                         int64_t m, int64_t ldx, void *y, int ydt, int64_t ldy, void *stream)
{
    clear_error();
    CHECK_SHAPE(n, k, m);
    mcapq_status st = check_weight(nib, scale, n, k);
    if (st != MCAPQ_OK) return st;
    CHECK_PTR(x, "x");
    CHECK_PTR(y, "y");
    CHECK_AL16(x, "x");
    CHECK_AL16(y, "y");
    CHECK_YDT(ydt);
    CHECK_LD(ldx, k, "ldx");
    CHECK_LD(ldy, n, "ldy");
    if (stream_supported(k) && aligned16(scale)) {
        StreamGroup g = {};
        g.count = 1;
        g.k = k;
        g.nib[0] = nib;
        g.scale[0] = scale;
        g.n[0] = n;
        g.y[0] = y;
        g.ldy[0] = ldy;
        LAUNCH_TRY(launch_linear_group(MCAPQ_W4A16, g, x, m, ldx, ydt, nullptr, as_stream(stream), false));
        return MCAPQ_OK;
    }
    LAUNCH_TRY(launch_w4a16(nib, scale, n, k, x, m, ldx, y, ydt, ldy, as_stream(stream), false));
    return MCAPQ_OK;
}

mcapq_status mcapq_w4a16_bf16deq(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k,
                                 const uint16_t *x, int64_t m, int64_t ldx, void *y, int ydt, int64_t ldy,
                                 void *stream)
{
    clear_error();
    CHECK_SHAPE(n, k, m);
    mcapq_status st = check_weight(nib, scale, n, k);
    if (st != MCAPQ_OK) return st;
    CHECK_PTR(x, "x");
    CHECK_PTR(y, "y");
    CHECK_AL16(x, "x");
    CHECK_AL16(y, "y");
    CHECK_YDT(ydt);
    CHECK_LD(ldx, k, "ldx");
    CHECK_LD(ldy, n, "ldy");
    MCAPQ_REQUIRE(k % 256 == 0 && gemm_supported(k), MCAPQ_EUNSUP, "w4a16_bf16deq needs K %% 256 == 0 (K = %lld)",
                  (long long)k);
    MCAPQ_REQUIRE(aligned16(scale) && ldx % 8 == 0, MCAPQ_EINVAL,
                  "w4a16_bf16deq needs a 16-byte aligned scale plane and ldx %% 8 == 0");
    LAUNCH_TRY(launch_tc05(nib, scale, n, k, x, ldx, m, y, ydt, ldy, as_stream(stream), api_pdl()));
    return MCAPQ_OK;
}

size_t mcapq_prefill_workspace_bytes(int64_t n, int64_t k) { return n > 0 && k > 0 ? (size_t)(2 * n * k) : 0; }

mcapq_status mcapq_dequant_w4_bf16(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k, uint16_t *w,
                                   void *stream)
{
    clear_error();
    CHECK_SHAPE(n, k, 1);
    mcapq_status st = check_weight(nib, scale, n, k);
    if (st != MCAPQ_OK) return st;
    CHECK_PTR(w, "w");
    CHECK_AL16(w, "w");
    CHECK_AL16(nib, "nib");
    LAUNCH_TRY(launch_dequant_w4_bf16(nib, scale, n, k, w, as_stream(stream)));
    return MCAPQ_OK;
}

mcapq_status mcapq_bf16w_gemm(const uint16_t *w, int64_t n, int64_t k, const uint16_t *x, int64_t m, int64_t ldx,
                              void *y, int ydt, int64_t ldy, void *stream)
{
    clear_error();
    CHECK_SHAPE(n, k, m);
    CHECK_PTR(w, "w");
    CHECK_PTR(x, "x");
    CHECK_PTR(y, "y");
    CHECK_AL16(w, "w");
    CHECK_AL16(x, "x");
    CHECK_AL16(y, "y");
    CHECK_YDT(ydt);
    CHECK_LD(ldx, k, "ldx");
    CHECK_LD(ldy, n, "ldy");
    MCAPQ_REQUIRE(k % 64 == 0, MCAPQ_EUNSUP, "bf16w_gemm needs K %% 64 == 0 (K = %lld)", (long long)k);
    MCAPQ_REQUIRE(ldx % 8 == 0, MCAPQ_EINVAL, "ldx %% 8 != 0");
    LAUNCH_TRY(launch_prefill(w, n, k, x, ldx, m, y, ydt, ldy, as_stream(stream), api_pdl()));
    return MCAPQ_OK;
}

mcapq_status mcapq_w4a16_bf16deq_prefill(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k,
                                         const uint16_t *x, int64_t m, int64_t ldx, void *y, int ydt, int64_t ldy,
                                         void *ws, size_t ws_bytes, void *stream)
{
    clear_error();
    MCAPQ_REQUIRE(ws && ws_bytes >= mcapq_prefill_workspace_bytes(n, k), MCAPQ_ENOSPACE,
                  "prefill workspace %zu < %zu bytes", ws_bytes, mcapq_prefill_workspace_bytes(n, k));
    mcapq_status st = mcapq_dequant_w4_bf16(nib, scale, n, k, reinterpret_cast<uint16_t *>(ws), stream);
    if (st != MCAPQ_OK) return st;
    return mcapq_bf16w_gemm(reinterpret_cast<const uint16_t *>(ws), n, k, x, m, ldx, y, ydt, ldy, stream);
}

mcapq_status mcapq_linear(int route, const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k,
                          const uint16_t *x, int64_t m, int64_t ldx, void *y, int ydt, int64_t ldy, void *ws,
                          size_t ws_bytes, void *stream)
{
    if (route == MCAPQ_W4A8) return mcapq_w4a8_x(nib, scale, n, k, x, m, ldx, y, ydt, ldy, ws, ws_bytes, stream);
    if (route == MCAPQ_W4A16) return mcapq_w4a16(nib, scale, n, k, x, m, ldx, y, ydt, ldy, stream);
    clear_error();
    set_error("bad route %d", route);
    return MCAPQ_EINVAL;
}

mcapq_status mcapq_linear_group(int route, int count, const uint8_t *const *nibs, const uint16_t *const *scales,
                                const int64_t *ns, int64_t k, const uint16_t *x, int64_t m, int64_t ldx,
                                void *const *ys, int ydt, const int64_t *ldys, void *ws, size_t ws_bytes,
                                void *stream)
{
    clear_error();
    MCAPQ_REQUIRE(count >= 1 && count <= kMaxGroup, MCAPQ_EINVAL, "group count %d not in [1, %d]", count, kMaxGroup);
    MCAPQ_REQUIRE(nibs && scales && ns && ys && ldys, MCAPQ_EINVAL, "NULL host array");
    MCAPQ_REQUIRE(route == MCAPQ_W4A8 || route == MCAPQ_W4A16, MCAPQ_EINVAL, "bad route %d", route);
    bool fast = stream_supported(k);
    for (int i = 0; i < count; ++i) {
        CHECK_SHAPE(ns[i], k, m);
        mcapq_status st = check_weight(nibs[i], scales[i], ns[i], k);
        if (st != MCAPQ_OK) return st;
        CHECK_PTR(ys[i], "y");
        CHECK_AL16(ys[i], "y");
        CHECK_LD(ldys[i], ns[i], "ldy");
        fast = fast && aligned16(scales[i]);
    }
    CHECK_PTR(x, "x");
    CHECK_AL16(x, "x");
    CHECK_YDT(ydt);
    CHECK_LD(ldx, k, "ldx");
    if (fast) {
        StreamGroup g = {};
        g.count = count;
        g.k = k;
        for (int i = 0; i < count; ++i) {
            g.nib[i] = nibs[i];
            g.scale[i] = scales[i];
            g.n[i] = ns[i];
            g.y[i] = ys[i];
            g.ldy[i] = ldys[i];
        }
        if (route == MCAPQ_W4A8 && m >= kGemmMinTokens && gemm_supported(k)) {
            CHECK_PTR(ws, "ws");
            CHECK_AL16(ws, "ws");
            MCAPQ_REQUIRE(ws_bytes >= a8_workspace_bytes(m, k), MCAPQ_ENOSPACE, "workspace %zu < %zu", ws_bytes,
                          a8_workspace_bytes(m, k));
        }
        LAUNCH_TRY(launch_linear_group(route, g, x, m, ldx, ydt, ws, as_stream(stream), false));
        return MCAPQ_OK;
    }
    for (int i = 0; i < count; ++i) {
        mcapq_status st = mcapq_linear(route, nibs[i], scales[i], ns[i], k, x, m, ldx, ys[i], ydt, ldys[i], ws,
                                       ws_bytes, stream);
        if (st != MCAPQ_OK) return st;
    }
    return MCAPQ_OK;
}

// ------------------------------------------------------------------ NEXT-2 greedy decode
static bool argmax_fused_path(int64_t m, int64_t k, const uint16_t *scale)
{
    return m == 1 && stream_supported(k) && aligned16(scale);
}

size_t mcapq_argmax_workspace_bytes(int route, int64_t m, int64_t n, int64_t k, int parts)
{
    if (m < 1 || n < 1 || k < 32 || parts < 1) return 0;
    // keys [parts][m] | fp32 logits [m][n] (off the fused path) | the routed linear's workspace
    return align256((size_t)(parts * m) * 8) + align256((size_t)(m * n) * 4) + mcapq_workspace_bytes(route, m, n, k);
}

mcapq_status mcapq_argmax_keys(int route, const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k,
                               const uint16_t *x, int64_t m, int64_t ldx, int64_t row_offset, uint64_t *keys,
                               void *ws, size_t ws_bytes, void *stream)
{
    clear_error();
    CHECK_SHAPE(n, k, m);
    mcapq_status st = check_weight(nib, scale, n, k);
    if (st != MCAPQ_OK) return st;
    CHECK_PTR(x, "x");
    CHECK_PTR(keys, "keys");
    CHECK_AL16(x, "x");
    CHECK_LD(ldx, k, "ldx");
    MCAPQ_REQUIRE(route == MCAPQ_W4A8 || route == MCAPQ_W4A16, MCAPQ_EINVAL, "bad route %d", route);
    MCAPQ_REQUIRE(row_offset >= 0 && row_offset + n <= 0xffffffffll, MCAPQ_ERANGE, "row indices must fit 32 bits");
    MCAPQ_REQUIRE((reinterpret_cast<uintptr_t>(keys) & 7u) == 0, MCAPQ_EINVAL, "keys is not 8-byte aligned");
    cudaStream_t s = as_stream(stream);
    unsigned long long *k64 = reinterpret_cast<unsigned long long *>(keys);
    if (argmax_fused_path(m, k, scale) && ldx == k) {
        LAUNCH_TRY(launch_argmax_fused(route, nib, scale, n, k, x, row_offset, k64, s));
        return MCAPQ_OK;
    }
    CHECK_PTR(ws, "ws");
    CHECK_AL16(ws, "ws");
    const size_t lb = align256((size_t)(m * n) * 4);
    MCAPQ_REQUIRE(ws_bytes >= lb + mcapq_workspace_bytes(route, m, n, k), MCAPQ_ENOSPACE, "workspace too small");
    float *logits = reinterpret_cast<float *>(ws);
    st = mcapq_linear(route, nib, scale, n, k, x, m, ldx, logits, MCAPQ_F32, n, reinterpret_cast<uint8_t *>(ws) + lb,
                      ws_bytes - lb, stream);
    if (st != MCAPQ_OK) return st;
    LAUNCH_TRY(launch_argmax_rows(logits, m, n, n, row_offset, k64, s));
    return MCAPQ_OK;
}

mcapq_status mcapq_argmax_combine(const uint64_t *keys, int parts, int64_t m, int64_t *idx, float *val, void *stream)
{
    clear_error();
    MCAPQ_REQUIRE(keys && idx && parts >= 1 && m >= 1, MCAPQ_EINVAL, "bad argmax_combine arguments");
    LAUNCH_TRY(launch_argmax_combine(reinterpret_cast<const unsigned long long *>(keys), parts, m, idx, val,
                                     as_stream(stream)));
    return MCAPQ_OK;
}

mcapq_status mcapq_linear_argmax(int route, const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k,
                                 const uint16_t *x, int64_t m, int64_t ldx, int64_t *idx, float *val, void *ws,
                                 size_t ws_bytes, void *stream)
{
    clear_error();
    CHECK_PTR(ws, "ws");
    CHECK_AL16(ws, "ws");
    MCAPQ_REQUIRE(ws_bytes >= mcapq_argmax_workspace_bytes(route, m, n, k, 1), MCAPQ_ENOSPACE, "workspace too small");
    uint64_t *keys = reinterpret_cast<uint64_t *>(ws);
    const size_t kb = align256((size_t)m * 8);
    mcapq_status st = mcapq_argmax_keys(route, nib, scale, n, k, x, m, ldx, 0, keys, reinterpret_cast<uint8_t *>(ws) + kb,
                                        ws_bytes - kb, stream);
    if (st != MCAPQ_OK) return st;
    return mcapq_argmax_combine(keys, 1, m, idx, val, stream);
}

size_t mcapq_host_workspace_bytes(int route, int64_t m, int64_t n, int64_t k)
{
    if (m < 1 || n < 1 || k < 32) return 0;
    const size_t xb = align256((size_t)(m * k) * 2), yb = align256((size_t)(m * n) * 4);
    return xb + yb + mcapq_workspace_bytes(route, m, n, k);
}

mcapq_status mcapq_linear_host(int route, const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k,
                               const uint16_t *x_host, int64_t m, void *y_host, int ydt, void *ws, size_t ws_bytes,
                               void *stream)
{
    clear_error();
    CHECK_SHAPE(n, k, m);
    CHECK_PTR(x_host, "x_host");
    CHECK_PTR(y_host, "y_host");
    CHECK_PTR(ws, "ws");
    CHECK_AL16(ws, "ws");
    CHECK_YDT(ydt);
    MCAPQ_REQUIRE(route == MCAPQ_W4A8 || route == MCAPQ_W4A16, MCAPQ_EINVAL, "bad route %d", route);
    MCAPQ_REQUIRE(ws_bytes >= mcapq_host_workspace_bytes(route, m, n, k), MCAPQ_ENOSPACE, "workspace too small");
    const size_t xb = align256((size_t)(m * k) * 2), yb = align256((size_t)(m * n) * 4);
    uint8_t *p = reinterpret_cast<uint8_t *>(ws);
    uint16_t *xd = reinterpret_cast<uint16_t *>(p);
    void *yd = p + xb;
    void *rest = p + xb + yb;
    cudaStream_t s = as_stream(stream);
    MCAPQ_CUDA_TRY(cudaMemcpyAsync(xd, x_host, (size_t)(m * k) * 2, cudaMemcpyHostToDevice, s));
    mcapq_status st = mcapq_linear(route, nib, scale, n, k, xd, m, k, yd, ydt, n, rest,
                                   ws_bytes - xb - yb, stream);
    if (st != MCAPQ_OK) return st;
    MCAPQ_CUDA_TRY(cudaMemcpyAsync(y_host, yd, (size_t)(m * n) * (ydt == MCAPQ_F32 ? 4 : 2),
                                   cudaMemcpyDeviceToHost, s));
    return MCAPQ_OK;
}

size_t mcapq_debug_stream_dump_workspace_bytes(int64_t k) { return k >= 32 ? stream_dump_workspace_bytes(k) : 0; }

mcapq_status mcapq_debug_stream_w4a8_dump(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k,
                                          const uint16_t *x, int8_t *q, float *sx, int32_t *sq, int32_t *D,
                                          void *ws, size_t ws_bytes, void *stream)
{
    clear_error();
    CHECK_SHAPE(n, k, 1);
    mcapq_status st = check_weight(nib, scale, n, k);
    if (st != MCAPQ_OK) return st;
    CHECK_PTR(x, "x");
    CHECK_PTR(q, "q");
    CHECK_PTR(sx, "sx");
    CHECK_PTR(sq, "sq");
    CHECK_PTR(D, "D");
    CHECK_PTR(ws, "ws");
    CHECK_AL16(x, "x");
    CHECK_AL16(ws, "ws");
    MCAPQ_REQUIRE(stream_supported(k) && aligned16(scale), MCAPQ_EUNSUP, "not on the stream path (K=%lld)",
                  (long long)k);
    MCAPQ_REQUIRE(ws_bytes >= stream_dump_workspace_bytes(k), MCAPQ_ENOSPACE, "workspace too small");
    LAUNCH_TRY(launch_stream_dump(nib, scale, n, k, x, q, sx, sq, D, ws, as_stream(stream)));
    return MCAPQ_OK;
}

mcapq_status mcapq_w4a8_group_dots(const uint8_t *nib, int64_t n, int64_t k, const int8_t *q, const int32_t *sq,
                                   int64_t m, int32_t *D, int mode, void *stream)
{
    clear_error();
    CHECK_SHAPE(n, k, m);
    CHECK_PTR(nib, "nib");
    CHECK_PTR(q, "q");
    CHECK_PTR(sq, "sq");
    CHECK_PTR(D, "D");
    CHECK_AL16(nib, "nib");
    CHECK_AL16(q, "q");
    MCAPQ_REQUIRE(mode == 0 || mode == 1, MCAPQ_EINVAL, "mode must be 0 (dp4a) or 1 (imma)");
    LAUNCH_TRY(launch_w4a8_group_dots(nib, n, k, q, sq, m, D, mode, as_stream(stream)));
    return MCAPQ_OK;
}

}  // extern "C"
