// comm.cu -- column (output-feature) sharded decode linear over NCCL (row a8).
//
// north_star: large linears (MLP, lm_head) are column-sharded across the GPUs
// of one 8xB200 node with an NCCL all-gather over NVLink/NVSwitch.  The paper
// itself is single-GPU.  Rank r owns rows [r N/P, (r+1) N/P) of
// the packed weight (reading A22); every rank holds the full x.  Each rank runs
// the routed linear on its shard; the per-row arithmetic depends on K only, so
// the gathered y is bit-identical to the single-GPU result.
//   M == 1 : the rank-major gather is already the row order of y: the linear writes
//            its rows straight into y_full + r N/P and the all-gather runs in place.
//   M  > 1 : the linear writes slot r of a rank-major [P][M][N/P] workspace, the
//            all-gather fills the other slots in place, and one assemble (permute)
//            kernel writes y_full[m][r N/P + j] (mcapq_colshard_assemble, also a test
//            entry: P-way shard emulation on one GPU).
#include <nccl.h>
#include <nccl_device.h>

#include <vector>

#include "internal.h"
#include "stream.h"

// A symmetric NCCL window holding one y_full replica per rank (a8 fused epilogue): the
// byte offsets from this rank's replica to every LSA peer's (NVLink load/store mapping).
struct McapqWindow {
    void *ptr = nullptr;
    size_t bytes = 0;
    ncclWindow_t win = nullptr;
    int npeers = 0;
    int64_t delta[mcapq::kMaxPeers] = {};
};

struct mcapq_comm {
    ncclComm_t comm = nullptr;
    int world = 1, rank = 0;
    bool dev_ok = false;        // ncclDevComm with one LSA barrier, created with the first window
    ncclDevComm dev = {};
    std::vector<McapqWindow> wins;
};

using namespace mcapq;

namespace {

__global__ void permute_rank_major(const uint8_t *__restrict__ src, uint8_t *__restrict__ dst, int64_t m,
                                   int64_t n_full, int world, int es)
{
    const int64_t per = n_full / world;
    const int64_t total = m * n_full;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = idx / n_full, c = idx % n_full;
        const int64_t r = c / per, j = c % per;
        const int64_t s = (r * m + i) * per + j;
        if (es == 4)
            reinterpret_cast<float *>(dst)[idx] = reinterpret_cast<const float *>(src)[s];
        else
            reinterpret_cast<uint16_t *>(dst)[idx] = reinterpret_cast<const uint16_t *>(src)[s];
    }
}

size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

// byte offsets from this rank's replica to each LSA peer's (ncclGetLsaPointer is device-side)
__global__ void lsa_peer_deltas(ncclWindow_t w, int npeers, int64_t *out)
{
    const int p = threadIdx.x;
    if (p < npeers)
        out[p] = reinterpret_cast<const char *>(ncclGetLsaPointer(w, 0, p)) -
                 reinterpret_cast<const char *>(ncclGetLocalPointer(w, 0));
}

// every LSA peer arrives, then waits: orders all peers' NVLink stores into the replicas
// (issued by the preceding kernel on each rank's stream) before anyone reads y_full
__global__ void lsa_barrier_kernel(ncclDevComm dev)
{
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dev, ncclTeamTagLsa(), 0);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

// NEXT-2 row-parallel reduction: y[i][j] = sum over r = 0 .. P-1 (rank order, fp32) of
// partials[r][i][j]; every rank sums the same slots in the same order, so y is identical
// on all ranks (the fused all-reduce), and P = 1 is the fp32 -> ydt conversion
__global__ void rowshard_sum(const float *__restrict__ partials, int world, int64_t total, void *__restrict__ y,
                             int ydt)
{
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        float v = partials[idx];
        for (int r = 1; r < world; ++r) v += partials[(int64_t)r * total + idx];
        if (ydt == MCAPQ_F32)
            reinterpret_cast<float *>(y)[idx] = v;
        else
            reinterpret_cast<uint16_t *>(y)[idx] = dev::float_to_bf16_bits(v);
    }
}

const McapqWindow *find_window(const mcapq_comm *c, const void *p, size_t bytes)
{
    for (const auto &v : c->wins)
        if (reinterpret_cast<const uint8_t *>(p) >= reinterpret_cast<const uint8_t *>(v.ptr) &&
            reinterpret_cast<const uint8_t *>(p) + bytes <= reinterpret_cast<const uint8_t *>(v.ptr) + v.bytes)
            return &v;
    return nullptr;
}

}  // namespace

#define NCCL_TRY(expr)                                                                                        \
    do {                                                                                                      \
        ncclResult_t r_ = (expr);                                                                             \
        if (r_ != ncclSuccess) {                                                                              \
            set_error("%s: %s", #expr, ncclGetErrorString(r_));                                              \
            return MCAPQ_ENCCL;                                                                               \
        }                                                                                                     \
    } while (0)

extern "C" {

mcapq_status mcapq_comm_unique_id(uint8_t *id_host_128)
{
    clear_error();
    MCAPQ_REQUIRE(id_host_128, MCAPQ_EINVAL, "id is NULL");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
    ncclUniqueId id;
    NCCL_TRY(ncclGetUniqueId(&id));
    memcpy(id_host_128, &id, 128);
    return MCAPQ_OK;
}

mcapq_status mcapq_comm_init(const uint8_t *id_host_128, int world, int rank, mcapq_comm **out)
{
    clear_error();
    MCAPQ_REQUIRE(id_host_128 && out, MCAPQ_EINVAL, "NULL argument");
    MCAPQ_REQUIRE(world >= 1 && rank >= 0 && rank < world, MCAPQ_ERANGE, "bad world=%d rank=%d", world, rank);
    ncclUniqueId id;
    memcpy(&id, id_host_128, 128);
    mcapq_comm *c = new (std::nothrow) mcapq_comm;
    MCAPQ_REQUIRE(c, MCAPQ_ECUDA, "out of host memory");
    ncclResult_t r = ncclCommInitRank(&c->comm, world, id, rank);
    if (r != ncclSuccess) {
        set_error("ncclCommInitRank: %s", ncclGetErrorString(r));
        delete c;
        return MCAPQ_ENCCL;
    }
    c->world = world;
    c->rank = rank;
    *out = c;
    return MCAPQ_OK;
}

int mcapq_comm_world(const mcapq_comm *c) { return c ? c->world : 0; }
int mcapq_comm_rank(const mcapq_comm *c) { return c ? c->rank : -1; }

size_t mcapq_colshard_workspace_bytes(int route, int64_t m, int64_t n_full, int64_t k, int world)
{
    if (world < 1 || m < 1 || n_full < 1 || k < 32 || n_full % world) return 0;
    size_t b = 256;
    if (m > 1) b += align256((size_t)(m * n_full) * 4);        // rank-major gather (fp32 worst case)
    if (route == MCAPQ_W4A8) b += a8_workspace_bytes(m, k);
    return b;
}

mcapq_status mcapq_colshard_assemble(const void *rank_major, void *y_full, int64_t m, int64_t n_full, int world,
                                     int ydt, void *stream)
{
    clear_error();
    MCAPQ_REQUIRE(rank_major && y_full && m >= 1 && n_full >= 1 && world >= 1 && n_full % world == 0, MCAPQ_EINVAL,
                  "bad colshard_assemble arguments");
    MCAPQ_REQUIRE(ydt == MCAPQ_BF16 || ydt == MCAPQ_F32, MCAPQ_EDTYPE, "bad ydt");
    const int64_t total = m * n_full;
    const int grid = (int)((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
    permute_rank_major<<<grid, 256, 0, as_stream(stream)>>>(reinterpret_cast<const uint8_t *>(rank_major),
                                                            reinterpret_cast<uint8_t *>(y_full), m, n_full, world,
                                                            ydt == MCAPQ_F32 ? 4 : 2);
    MCAPQ_CUDA_TRY(cudaGetLastError());
    return MCAPQ_OK;
}

mcapq_status mcapq_linear_colshard(const mcapq_comm *c, int route, const uint8_t *nib_shard,
                                   const uint16_t *scale_shard, int64_t n_full, int64_t k, const uint16_t *x,
                                   int64_t m, void *y_full, int ydt, void *ws, size_t ws_bytes, int fused_epilogue,
                                   void *stream)
{
    clear_error();
    MCAPQ_REQUIRE(c && c->comm, MCAPQ_EINVAL, "communicator is NULL");
    MCAPQ_REQUIRE(n_full % c->world == 0, MCAPQ_EINVAL, "N=%lld not divisible by P=%d", (long long)n_full, c->world);
    MCAPQ_REQUIRE(ydt == MCAPQ_BF16 || ydt == MCAPQ_F32, MCAPQ_EDTYPE, "bad ydt");
    MCAPQ_REQUIRE(route == MCAPQ_W4A8 || route == MCAPQ_W4A16, MCAPQ_EINVAL, "bad route");
    MCAPQ_REQUIRE(ws && aligned16(ws) && y_full && aligned16(y_full), MCAPQ_EINVAL, "NULL/misaligned ws or y");
    MCAPQ_REQUIRE(ws_bytes >= mcapq_colshard_workspace_bytes(route, m, n_full, k, c->world), MCAPQ_ENOSPACE,
                  "workspace too small");
    const int64_t per = n_full / c->world;
    MCAPQ_REQUIRE(per % 8 == 0, MCAPQ_EINVAL, "N/P=%lld must be a multiple of 8", (long long)per);
    const int es = ydt == MCAPQ_F32 ? 4 : 2;
    if (fused_epilogue && m == 1 && stream_supported(k) && aligned16(scale_shard)) {
        // a8 fused: the GEMV epilogue stores each of this rank's rows into every LSA
        // peer's replica of y_full (NVLink stores), then one LSA barrier -- no all-gather
        const McapqWindow *w = nullptr;
        for (const auto &v : c->wins)
            if (reinterpret_cast<uint8_t *>(y_full) >= reinterpret_cast<uint8_t *>(v.ptr) &&
                reinterpret_cast<uint8_t *>(y_full) + (size_t)n_full * es <= reinterpret_cast<uint8_t *>(v.ptr) + v.bytes)
                w = &v;
        MCAPQ_REQUIRE(w, MCAPQ_EINVAL, "fused_epilogue: y_full is not in a window from mcapq_comm_window_alloc");
        uint8_t *mine = reinterpret_cast<uint8_t *>(y_full) + (size_t)c->rank * (size_t)per * es;
        cudaStream_t s = as_stream(stream);
        cudaError_t e = launch_linear_peers(route, nib_shard, scale_shard, per, k, x, mine, ydt, w->delta, w->npeers, s);
        MCAPQ_REQUIRE(e == cudaSuccess, MCAPQ_ECUDA, "fused colshard launch: %s", cudaGetErrorString(e));
        lsa_barrier_kernel<<<1, 32, 0, s>>>(c->dev);
        MCAPQ_CUDA_TRY(cudaGetLastError());
        return MCAPQ_OK;
    }
    uint8_t *p = reinterpret_cast<uint8_t *>(ws) + 256;
    uint8_t *gathered = nullptr;
    if (m > 1) {
        gathered = p;
        p += align256((size_t)(m * n_full) * 4);
    }
    void *rest = p;
    const size_t rest_bytes = ws_bytes - (size_t)(p - reinterpret_cast<uint8_t *>(ws));
    cudaStream_t s = as_stream(stream);
    const ncclDataType_t dt = ydt == MCAPQ_F32 ? ncclFloat32 : ncclBfloat16;
    // the local rows go straight to their place in the gather buffer (in-place all-gather:
    // sendbuff = recvbuff + rank * count)
    uint8_t *dst = m == 1 ? reinterpret_cast<uint8_t *>(y_full) : gathered;
    uint8_t *mine = dst + (size_t)c->rank * (size_t)(m * per) * es;
    mcapq_status st = mcapq_linear(route, nib_shard, scale_shard, per, k, x, m, k, mine, ydt, per, rest, rest_bytes,
                                   stream);
    if (st != MCAPQ_OK) return st;
    NCCL_TRY(ncclAllGather(mine, dst, (size_t)(m * per), dt, c->comm, s));
    if (m > 1) return mcapq_colshard_assemble(gathered, y_full, m, n_full, c->world, ydt, stream);
    return MCAPQ_OK;
}

mcapq_status mcapq_linear_colshard_argmax(const mcapq_comm *c, int route, const uint8_t *nib_shard,
                                          const uint16_t *scale_shard, int64_t n_full, int64_t k, const uint16_t *x,
                                          int64_t m, int64_t *idx, float *val, void *ws, size_t ws_bytes, void *stream)
{
    clear_error();
    MCAPQ_REQUIRE(c && c->comm, MCAPQ_EINVAL, "communicator is NULL");
    MCAPQ_REQUIRE(n_full % c->world == 0, MCAPQ_EINVAL, "N=%lld not divisible by P=%d", (long long)n_full, c->world);
    MCAPQ_REQUIRE(ws && aligned16(ws), MCAPQ_EINVAL, "NULL/misaligned ws");
    const int64_t per = n_full / c->world;
    MCAPQ_REQUIRE(ws_bytes >= mcapq_argmax_workspace_bytes(route, m, per, k, c->world), MCAPQ_ENOSPACE,
                  "workspace too small");
    // rank r's keys (global row indices r N/P + n) into slot r of [P][m]; the all-gather of
    // P x m 8-byte keys replaces the m x N logit gather; every rank combines the same keys
    uint64_t *keys = reinterpret_cast<uint64_t *>(ws);
    const size_t kb = align256((size_t)(c->world * m) * 8);
    mcapq_status st = mcapq_argmax_keys(route, nib_shard, scale_shard, per, k, x, m, k, (int64_t)c->rank * per,
                                        keys + (size_t)c->rank * m, reinterpret_cast<uint8_t *>(ws) + kb, ws_bytes - kb,
                                        stream);
    if (st != MCAPQ_OK) return st;
    NCCL_TRY(ncclAllGather(keys + (size_t)c->rank * m, keys, (size_t)m, ncclUint64, c->comm, as_stream(stream)));
    return mcapq_argmax_combine(keys, c->world, m, idx, val, stream);
}

// ---- NEXT-2: row-parallel (K-sharded) linear, the Megatron partner of the column shard
size_t mcapq_rowshard_workspace_bytes(int route, int64_t m, int64_t n, int64_t k_shard, int world)
{
    if (world < 1 || m < 1 || n < 1 || k_shard < 32 || k_shard % 32) return 0;
    size_t b = 256 + align256((size_t)(m * n) * 4);   // this rank's fp32 partial (all-reduced in place)
    if (route == MCAPQ_W4A8) b += a8_workspace_bytes(m, k_shard);
    return b;
}

mcapq_status mcapq_rowshard_reduce(const float *partials, int world, int64_t m, int64_t n, void *y, int ydt,
                                   void *stream)
{
    clear_error();
    MCAPQ_REQUIRE(partials && y && world >= 1 && m >= 1 && n >= 1, MCAPQ_EINVAL, "bad rowshard_reduce arguments");
    MCAPQ_REQUIRE(ydt == MCAPQ_BF16 || ydt == MCAPQ_F32, MCAPQ_EDTYPE, "bad ydt");
    const int64_t total = m * n;
    const int grid = (int)((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
    rowshard_sum<<<grid, 256, 0, as_stream(stream)>>>(partials, world, total, y, ydt);
    MCAPQ_CUDA_TRY(cudaGetLastError());
    return MCAPQ_OK;
}

mcapq_status mcapq_linear_rowshard(const mcapq_comm *c, int route, const uint8_t *nib_shard,
                                   const uint16_t *scale_shard, int64_t n, int64_t k_shard, const uint16_t *x_shard,
                                   int64_t m, int64_t ldx, void *y, int ydt, void *ws, size_t ws_bytes,
                                   int fused_epilogue, void *stream)
{
    clear_error();
    MCAPQ_REQUIRE(c && c->comm, MCAPQ_EINVAL, "communicator is NULL");
    MCAPQ_REQUIRE(ydt == MCAPQ_BF16 || ydt == MCAPQ_F32, MCAPQ_EDTYPE, "bad ydt");
    MCAPQ_REQUIRE(route == MCAPQ_W4A8 || route == MCAPQ_W4A16, MCAPQ_EINVAL, "bad route");
    MCAPQ_REQUIRE(k_shard >= 32 && k_shard % 32 == 0, MCAPQ_EINVAL,
                  "K/P=%lld must be whole 32-groups (the W4A8 quantiser stays rank-local)", (long long)k_shard);
    MCAPQ_REQUIRE(m >= 1 && n >= 1 && ldx >= k_shard && x_shard && y && aligned16(y), MCAPQ_EINVAL,
                  "bad rowshard arguments");
    MCAPQ_REQUIRE(ws && aligned16(ws), MCAPQ_EINVAL, "NULL/misaligned ws");
    cudaStream_t s = as_stream(stream);
    if (fused_epilogue) {
        // fused all-reduce over NVLink: ws is a window from mcapq_comm_window_alloc holding
        // [P][m][n] fp32 slots.  The GEMV epilogue stores this rank's partial into slot
        // `rank` of every LSA peer's window; after the LSA barrier every rank sums the P
        // slots in rank order (rowshard_sum) -- identical y everywhere, no NCCL collective.
        // A barrier first: no peer is still reading its slots from the previous call.
        MCAPQ_REQUIRE(m == 1 && stream_supported(k_shard) && aligned16(scale_shard), MCAPQ_EUNSUP,
                      "fused rowshard: M = 1 and a stream-path K/P (K %% 256 == 0, >= 2048)");
        const size_t slot = (size_t)n * 4;
        const McapqWindow *w = find_window(c, ws, slot * (size_t)c->world);
        MCAPQ_REQUIRE(w, MCAPQ_EINVAL, "fused_epilogue: ws is not a window from mcapq_comm_window_alloc");
        MCAPQ_REQUIRE(ws_bytes >= slot * (size_t)c->world, MCAPQ_ENOSPACE, "window too small for P x N fp32");
        lsa_barrier_kernel<<<1, 32, 0, s>>>(c->dev);
        MCAPQ_CUDA_TRY(cudaGetLastError());
        uint8_t *mine = reinterpret_cast<uint8_t *>(ws) + (size_t)c->rank * slot;
        cudaError_t e = launch_linear_peers(route, nib_shard, scale_shard, n, k_shard, x_shard, mine, MCAPQ_F32,
                                            w->delta, w->npeers, s);
        MCAPQ_REQUIRE(e == cudaSuccess, MCAPQ_ECUDA, "fused rowshard launch: %s", cudaGetErrorString(e));
        lsa_barrier_kernel<<<1, 32, 0, s>>>(c->dev);
        MCAPQ_CUDA_TRY(cudaGetLastError());
        return mcapq_rowshard_reduce(reinterpret_cast<const float *>(ws), c->world, 1, n, y, ydt, stream);
    }
    MCAPQ_REQUIRE(ws_bytes >= mcapq_rowshard_workspace_bytes(route, m, n, k_shard, c->world), MCAPQ_ENOSPACE,
                  "workspace too small");
    // this rank's fp32 partial over its K-slice (its groups: codes and int32 dots exactly
    // those of the unsharded linear), then an in-place NCCL sum all-reduce
    float *part = ydt == MCAPQ_F32 ? reinterpret_cast<float *>(y)
                                   : reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(ws) + 256);
    uint8_t *rest = reinterpret_cast<uint8_t *>(ws) + 256 + align256((size_t)(m * n) * 4);
    const size_t rest_bytes = ws_bytes - (size_t)(rest - reinterpret_cast<uint8_t *>(ws));
    mcapq_status st = mcapq_linear(route, nib_shard, scale_shard, n, k_shard, x_shard, m, ldx, part, MCAPQ_F32, n,
                                   rest, rest_bytes, stream);
    if (st != MCAPQ_OK) return st;
    NCCL_TRY(ncclAllReduce(part, part, (size_t)(m * n), ncclFloat32, ncclSum, c->comm, s));
    if (ydt == MCAPQ_F32) return MCAPQ_OK;
    return mcapq_rowshard_reduce(part, 1, m, n, y, ydt, stream);
}

mcapq_status mcapq_comm_window_alloc(mcapq_comm *c, size_t bytes, void **y_full)
{
    clear_error();
    MCAPQ_REQUIRE(c && c->comm && y_full && bytes > 0, MCAPQ_EINVAL, "bad window_alloc arguments");
    McapqWindow w;
    w.bytes = (bytes + NCCL_WIN_REQUIRED_ALIGNMENT - 1) / NCCL_WIN_REQUIRED_ALIGNMENT * NCCL_WIN_REQUIRED_ALIGNMENT;
    NCCL_TRY(ncclMemAlloc(&w.ptr, w.bytes));
    ncclResult_t r = ncclCommWindowRegister(c->comm, w.ptr, w.bytes, &w.win, NCCL_WIN_COLL_SYMMETRIC);
    if (r != ncclSuccess) {
        ncclMemFree(w.ptr);
        set_error("ncclCommWindowRegister: %s", ncclGetErrorString(r));
        return MCAPQ_ENCCL;
    }
    if (!c->dev_ok) {
        ncclDevCommRequirements reqs = {};
        reqs.lsaBarrierCount = 1;
        NCCL_TRY(ncclDevCommCreate(c->comm, &reqs, &c->dev));
        c->dev_ok = true;
    }
    w.npeers = c->dev.lsaSize < kMaxPeers ? c->dev.lsaSize : kMaxPeers;
    MCAPQ_REQUIRE(c->dev.lsaSize == c->world && c->world <= kMaxPeers, MCAPQ_EUNSUP,
                  "fused epilogue needs every rank in one NVLink (LSA) domain of <= %d GPUs (lsa %d, world %d)",
                  kMaxPeers, c->dev.lsaSize, c->world);
    int64_t *d = nullptr;
    MCAPQ_CUDA_TRY(cudaMalloc(&d, sizeof(int64_t) * kMaxPeers));
    lsa_peer_deltas<<<1, 32>>>(w.win, w.npeers, d);
    cudaError_t e = cudaMemcpy(w.delta, d, sizeof(int64_t) * w.npeers, cudaMemcpyDeviceToHost);
    cudaFree(d);
    MCAPQ_CUDA_TRY(e);
    c->wins.push_back(w);
    *y_full = w.ptr;
    return MCAPQ_OK;
}

mcapq_status mcapq_comm_window_free(mcapq_comm *c, void *y_full)
{
    clear_error();
    MCAPQ_REQUIRE(c && c->comm, MCAPQ_EINVAL, "communicator is NULL");
    for (size_t i = 0; i < c->wins.size(); ++i)
        if (c->wins[i].ptr == y_full) {
            MCAPQ_CUDA_TRY(cudaDeviceSynchronize());
            NCCL_TRY(ncclCommWindowDeregister(c->comm, c->wins[i].win));
            NCCL_TRY(ncclMemFree(c->wins[i].ptr));
            c->wins.erase(c->wins.begin() + (long)i);
            return MCAPQ_OK;
        }
    MCAPQ_REQUIRE(false, MCAPQ_EINVAL, "not a window of this communicator");
}

void mcapq_comm_destroy(mcapq_comm *c)
{
    if (!c) return;
    if (c->comm) {
        cudaDeviceSynchronize();
        for (auto &w : c->wins) {
            ncclCommWindowDeregister(c->comm, w.win);
            ncclMemFree(w.ptr);
        }
        if (c->dev_ok) ncclDevCommDestroy(c->comm, &c->dev);
        ncclCommDestroy(c->comm);
    }
    delete c;
}

}  // extern "C"
