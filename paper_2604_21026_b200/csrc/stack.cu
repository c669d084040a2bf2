// stack.cu -- the routed decode-linear stack (row a9): L layers x S slots under
// the MCAP dispatch table, replayed as one CUDA graph per decode step
// ("CUDA graph capture for decode"; routing P:840-846).
//
// Each layer follows route[i] (all its slots, reading A12).  W4A8 layers
// quantise each distinct input once (slots with the same input_id, e.g. q/k/v,
// share it: reading A15) into one library-owned workspace.  Every
// kernel is launched with programmatic dependent launch: a GEMV starts
// streaming its weights while its predecessor drains and waits
// (griddepcontrol.wait) only before reading activations, so the step's
// 100+ launches overlap their ramps.  Data order stays total: each kernel waits
// for its predecessor's completion before touching activations.
#include <vector>

#include <cuda.h>

#include "internal.h"
#include "stream.h"

namespace {
constexpr int kMaxSlots = 16;
struct Slot {
    bool set = false;
    int input_id = 0;
    const uint8_t *nib = nullptr;
    const uint16_t *scale = nullptr;
    int64_t n = 0, k = 0;
    const uint16_t *x = nullptr;
    void *y = nullptr;
    int ydt = 0;
};
}  // namespace

struct mcapq_stack {
    int layers = 0;
    std::vector<uint8_t> routes;
    int64_t max_m = 1;
    std::vector<Slot> slots;   // [layers][kMaxSlots]
    void *ws = nullptr;
    size_t ws_bytes = 0;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int64_t graph_m = 0;
    // persistent step program (M = 1): one op per launch group, executed by stack_step
    bool prog_dirty = true, prog_ok = false;
    void *ops_dev = nullptr, *ops_host = nullptr;
    unsigned int *counters = nullptr;   // [nops] + exit count + epoch
    CUtensorMap *descs = nullptr;       // [nops][kMaxGroup][2] TMA descriptors the ops point at
    int2 *part = nullptr;               // [nops][grid] tile ranges per CTA (stack_partition)
    uint32_t *tags = nullptr;           // tagged copies of outputs consumed inside the step
    int nops = 0;
    int64_t max_k = 0;
    bool has_records = false;   // some op stages producer-quantised records: clustered launch
    int route_kinds = 3;        // bit 0: some W4A8 op, bit 1: some W4A16 op
};

using namespace mcapq;

static void free_program(mcapq_stack *st)
{
    if (st->ops_dev) cudaFree(st->ops_dev);
    if (st->ops_host) cudaFreeHost(st->ops_host);
    if (st->counters) cudaFree(st->counters);
    if (st->tags) cudaFree(st->tags);
    if (st->descs) cudaFree(st->descs);
    st->descs = nullptr;
    if (st->part) cudaFree(st->part);
    st->part = nullptr;
    st->ops_dev = st->ops_host = nullptr;
    st->counters = nullptr;
    st->tags = nullptr;
    st->nops = 0;
    st->prog_ok = false;
}

// A registration change invalidates the captured graph (it points at the old
// program / workspace): destroy it; replay then refuses until the next capture.
static void drop_graph(mcapq_stack *st)
{
    if (st->exec) cudaGraphExecDestroy(st->exec);
    if (st->graph) cudaGraphDestroy(st->graph);
    st->exec = nullptr;
    st->graph = nullptr;
    st->graph_m = 0;
}

static mcapq_status ensure_ws(mcapq_stack *st, int64_t k)
{
    const size_t need = a8_workspace_bytes(st->max_m, k);
    if (need <= st->ws_bytes) return MCAPQ_OK;
    if (st->ws) cudaFree(st->ws);
    st->ws = nullptr;
    st->ws_bytes = 0;
    MCAPQ_CUDA_TRY(cudaMalloc(&st->ws, need));
    st->ws_bytes = need;
    return MCAPQ_OK;
}

extern "C" {

mcapq_status mcapq_stack_create(int layers, const uint8_t *routes_host, int64_t max_m, mcapq_stack **out)
{
    clear_error();
    MCAPQ_REQUIRE(out && routes_host && layers >= 1 && max_m >= 1, MCAPQ_EINVAL, "bad stack_create arguments");
    for (int i = 0; i < layers; ++i)
        MCAPQ_REQUIRE(routes_host[i] <= 1, MCAPQ_EINVAL, "route[%d]=%d is not 0/1", i, routes_host[i]);
    mcapq_stack *st = new (std::nothrow) mcapq_stack;
    MCAPQ_REQUIRE(st, MCAPQ_ECUDA, "out of host memory");
    st->layers = layers;
    st->routes.assign(routes_host, routes_host + layers);
    st->max_m = max_m;
    st->slots.resize((size_t)layers * kMaxSlots);
    *out = st;
    return MCAPQ_OK;
}

mcapq_status mcapq_stack_set(mcapq_stack *st, int layer, int slot, int input_id, const uint8_t *nib,
                             const uint16_t *scale, int64_t n, int64_t k, const uint16_t *x, void *y, int ydt)
{
    clear_error();
    MCAPQ_REQUIRE(st, MCAPQ_EINVAL, "stack is NULL");
    MCAPQ_REQUIRE(layer >= 0 && layer < st->layers && slot >= 0 && slot < kMaxSlots, MCAPQ_EINVAL,
                  "layer/slot out of range");
    MCAPQ_REQUIRE(nib && scale && x && y && aligned16(nib) && aligned16(x) && aligned16(y), MCAPQ_EINVAL,
                  "NULL or misaligned pointer");
    MCAPQ_REQUIRE(n >= 1 && k >= 32 && k % 32 == 0 && n % 8 == 0, MCAPQ_EINVAL, "bad shape n=%lld k=%lld",
                  (long long)n, (long long)k);
    MCAPQ_REQUIRE(ydt == MCAPQ_BF16 || ydt == MCAPQ_F32, MCAPQ_EDTYPE, "bad ydt");
    Slot &s = st->slots[(size_t)layer * kMaxSlots + slot];
    s.set = true;
    s.input_id = input_id;
    s.nib = nib;
    s.scale = scale;
    s.n = n;
    s.k = k;
    s.x = x;
    s.y = y;
    s.ydt = ydt;
    st->prog_dirty = true;
    drop_graph(st);
    if (st->routes[layer] == MCAPQ_W4A8) return ensure_ws(st, k);
    return MCAPQ_OK;
}

}  // extern "C"

// Consecutive set slots of a layer with the same input_id form a launch group
// (<= kMaxGroup linears, same K, fast-path eligible).  Calls f(first, count).
template <typename F>
static mcapq_status for_each_group(const mcapq_stack *st, int l, F f)
{
    int sl = 0;
    while (sl < kMaxSlots) {
        const Slot &a = st->slots[(size_t)l * kMaxSlots + sl];
        if (!a.set) { ++sl; continue; }
        int cnt = 1;
        const bool fast = stream_supported(a.k) && aligned16(a.scale);
        while (fast && sl + cnt < kMaxSlots && cnt < kMaxGroup) {
            const Slot &b = st->slots[(size_t)l * kMaxSlots + sl + cnt];
            if (!b.set || b.input_id != a.input_id || b.k != a.k || b.x != a.x || b.ydt != a.ydt ||
                !aligned16(b.scale))
                break;
            ++cnt;
        }
        mcapq_status r = f(sl, cnt, fast);
        if (r != MCAPQ_OK) return r;
        sl += cnt;
    }
    return MCAPQ_OK;
}

static StreamGroup group_of(const mcapq_stack *st, int l, int first, int cnt)
{
    StreamGroup g = {};
    g.count = cnt;
    g.k = st->slots[(size_t)l * kMaxSlots + first].k;
    for (int i = 0; i < cnt; ++i) {
        const Slot &b = st->slots[(size_t)l * kMaxSlots + first + i];
        g.nib[i] = b.nib;
        g.scale[i] = b.scale;
        g.n[i] = b.n;
        g.y[i] = b.y;
        g.ldy[i] = b.n;
    }
    return g;
}

// Byte range [lo, hi) of a buffer.
struct Range {
    uintptr_t lo, hi;
    bool overlaps(const Range &o) const { return lo < o.hi && o.lo < hi; }
};

// Build the persistent-step program (one op per launch group, in decode order) in
// device memory.  Host-synchronous: call outside graph capture.  prog_ok stays
// false when a group is off the TMA fast path (then the per-linear path runs).
//
// Dependencies between ops come from the registered buffers (M = 1):
//   x_i == y_j (latest writer of any byte of x_i, whole buffer, bf16) -> dataflow:
//       op j also writes a tagged copy of y_j, op i reads it (no barrier);
//   any other overlap of x_i with an earlier y, or of y_i with an earlier plain-read
//       x or an earlier y (WAR / WAW)  -> barrier on the latest such op;
//   otherwise none: x_i is an input of the step.
static mcapq_status build_program(mcapq_stack *st)
{
    free_program(st);
    st->prog_dirty = false;
    if (!stack_step_enabled()) return MCAPQ_OK;
    std::vector<std::pair<int, std::pair<int, int>>> groups;   // (layer, (first, count))
    bool all_fast = true;
    for (int l = 0; l < st->layers; ++l)
        for_each_group(st, l, [&](int first, int cnt, bool fast) -> mcapq_status {
            all_fast = all_fast && fast;
            groups.push_back({l, {first, cnt}});
            return MCAPQ_OK;
        });
    if (!all_fast || groups.empty()) return MCAPQ_OK;
    const int nops = (int)groups.size();
    std::vector<StreamGroup> gs(nops);
    std::vector<const Slot *> heads(nops);
    st->max_k = 0;
    for (int i = 0; i < nops; ++i) {
        const int l = groups[i].first, first = groups[i].second.first, cnt = groups[i].second.second;
        gs[i] = group_of(st, l, first, cnt);
        heads[i] = &st->slots[(size_t)l * kMaxSlots + first];
        st->max_k = gs[i].k > st->max_k ? gs[i].k : st->max_k;
    }
    if (st->max_k > kStepMaxK) return MCAPQ_OK;

    // ---- dependencies
    auto xr = [&](int i) {
        const uintptr_t p = reinterpret_cast<uintptr_t>(heads[i]->x);
        return Range{p, p + (uintptr_t)(2 * gs[i].k)};
    };
    auto yr = [&](int i, int m) {
        const uintptr_t p = reinterpret_cast<uintptr_t>(gs[i].y[m]);
        return Range{p, p + (uintptr_t)(gs[i].n[m] * (heads[i]->ydt == MCAPQ_F32 ? 4 : 2))};
    };
    std::vector<StackDeps> deps(nops);
    std::vector<int> src_op(nops, -1), src_m(nops, -1);
    for (int i = 0; i < nops; ++i) {
        StackDeps &d = deps[i];
        d.xt = nullptr;
        d.xt_op = -1;
        for (int m = 0; m < kMaxGroup; ++m) d.yt[m] = nullptr;
        for (int m = 0; m < kMaxGroup; ++m) d.yq[m] = nullptr;
        d.xq = nullptr;
        d.wait_op = -1;
        d.publish = 0;
        // RAW on x_i: the latest earlier writer of any byte of x_i
        const Range x = xr(i);
        for (int j = i - 1; j >= 0 && src_op[i] < 0 && d.wait_op < 0; --j)
            for (int m = 0; m < gs[j].count; ++m) {
                const Range y = yr(j, m);
                if (!y.overlaps(x)) continue;
                if (y.lo == x.lo && y.hi == x.hi && heads[j]->ydt == MCAPQ_BF16) {
                    src_op[i] = j;
                    src_m[i] = m;
                } else {
                    d.wait_op = j;
                }
                break;
            }
        // WAR / WAW on y_i
        for (int j = i - 1; j > d.wait_op; --j) {
            bool hit = false;
            for (int m = 0; m < gs[i].count && !hit; ++m) {
                const Range y = yr(i, m);
                // an earlier op reads its x from memory unless it is a dataflow consumer
                if (src_op[j] < 0 && xr(j).overlaps(y)) hit = true;
                for (int mm = 0; mm < gs[j].count && !hit; ++mm)
                    if (yr(j, mm).overlaps(y)) hit = true;
            }
            if (hit) {
                d.wait_op = j;
                break;
            }
        }
    }
    // per (producer op, member) feeding a dataflow consumer: a tagged bf16 copy for W4A16
    // consumers, or -- in the clustered step, every member N a multiple of 32 -- quantised
    // records for W4A8 consumers (the producer's epilogue quantises each group once)
    auto rec_ok = [&](int j) {
        if (!stack_clustered()) return false;
        for (int m = 0; m < gs[j].count; ++m)
            if (gs[j].n[m] % 32) return false;
        return true;
    };
    std::vector<std::vector<size_t>> tag_off(nops, std::vector<size_t>(kMaxGroup, (size_t)-1));
    std::vector<std::vector<size_t>> rec_off(nops, std::vector<size_t>(kMaxGroup, (size_t)-1));
    std::vector<char> use_rec(nops, 0);
    size_t tag_words = 0, rec_words = 0;
    for (int i = 0; i < nops; ++i) {
        if (src_op[i] < 0) continue;
        const int j = src_op[i], m = src_m[i];
        if (st->routes[groups[i].first] == MCAPQ_W4A8 && rec_ok(j) && gs[i].k >= stack_rec_min_k()) {
            use_rec[i] = 1;
            if (rec_off[j][m] == (size_t)-1) {
                rec_off[j][m] = rec_words;
                rec_words += (size_t)(gs[j].n[m] / 32) * (kStackRecBytes / 8);
            }
        } else if (tag_off[j][m] == (size_t)-1) {
            tag_off[j][m] = tag_words;
            tag_words += (size_t)((gs[j].n[m] + 3) / 4 * 4);
        }
    }
    // one allocation: tagged words, then the 16-B aligned records (both zero: tag 0 is
    // never current)
    const size_t tag_bytes = (tag_words * 4 + 15) / 16 * 16;
    st->has_records = rec_words > 0;
    if (tag_words + rec_words) {
        MCAPQ_CUDA_TRY(cudaMalloc(&st->tags, tag_bytes + rec_words * 8));
        MCAPQ_CUDA_TRY(cudaMemset(st->tags, 0, tag_bytes + rec_words * 8));
    }
    unsigned long long *recs =
        reinterpret_cast<unsigned long long *>(reinterpret_cast<uint8_t *>(st->tags) + tag_bytes);
    for (int i = 0; i < nops; ++i) {
        for (int m = 0; m < gs[i].count; ++m) {
            if (tag_off[i][m] != (size_t)-1) deps[i].yt[m] = st->tags + tag_off[i][m];
            if (rec_off[i][m] != (size_t)-1) deps[i].yq[m] = recs + rec_off[i][m];
        }
        if (src_op[i] >= 0) {
            if (use_rec[i])
                deps[i].xq = recs + rec_off[src_op[i]][src_m[i]];
            else
                deps[i].xt = st->tags + tag_off[src_op[i]][src_m[i]];
            deps[i].xt_op = src_op[i];
            // the consumer's slow path waits on its counter only as a hint (the tags
            // decide): a relaxed add, no release fence on the epilogue warp's path
            if (deps[src_op[i]].publish < 1) deps[src_op[i]].publish = 1;
        }
        // a barrier dependency orders memory through the counter: release
        if (deps[i].wait_op >= 0) deps[deps[i].wait_op].publish = 2;
    }

    st->route_kinds = 0;
    for (int i = 0; i < nops; ++i) st->route_kinds |= st->routes[groups[i].first] == MCAPQ_W4A16 ? 2 : 1;
    const size_t ob = stack_op_bytes();
    st->nops = nops;
    MCAPQ_CUDA_TRY(cudaMallocHost(&st->ops_host, ob * nops));
    MCAPQ_CUDA_TRY(cudaMalloc(&st->ops_dev, ob * nops));
    MCAPQ_CUDA_TRY(cudaMalloc(&st->counters, sizeof(unsigned int) * (nops + 2)));
    MCAPQ_CUDA_TRY(cudaMemset(st->counters, 0, sizeof(unsigned int) * (nops + 2)));
    // the program's TMA descriptors: library-owned, uploaded once here (host-synchronous,
    // outside any capture), freed with the program
    const size_t nmaps = (size_t)nops * kMaxGroup * 2;
    std::vector<CUtensorMap> hmaps(nmaps);
    MCAPQ_CUDA_TRY(cudaMalloc(&st->descs, nmaps * sizeof(CUtensorMap)));
    for (int i = 0; i < nops; ++i) {
        const int l = groups[i].first;
        const size_t off = (size_t)i * kMaxGroup * 2;
        MCAPQ_REQUIRE(stack_fill_op(reinterpret_cast<uint8_t *>(st->ops_host) + ob * i, st->routes[l], gs[i],
                                    heads[i]->x, heads[i]->ydt, deps[i], hmaps.data() + off, st->descs + off),
                      MCAPQ_ECUDA, "stack op %d: TMA descriptor encode failed", i);
    }
    MCAPQ_CUDA_TRY(cudaMemcpy(st->descs, hmaps.data(), nmaps * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
    MCAPQ_CUDA_TRY(cudaMemcpy(st->ops_dev, st->ops_host, ob * nops, cudaMemcpyHostToDevice));
    // every CTA's tile range per op, for the grid and cluster shape launch_stack_step uses
    {
        const int grid = device_sms();
        std::vector<int2> part((size_t)nops * grid);
        stack_partition(st->ops_host, nops, grid, st->has_records && stack_clustered(), stack_rec_r(), part.data());
        MCAPQ_CUDA_TRY(cudaMalloc(&st->part, part.size() * sizeof(int2)));
        MCAPQ_CUDA_TRY(cudaMemcpy(st->part, part.data(), part.size() * sizeof(int2), cudaMemcpyHostToDevice));
    }
    st->prog_ok = true;
    return MCAPQ_OK;
}

extern "C" {

mcapq_status mcapq_stack_run(mcapq_stack *st, int64_t m, void *stream)
{
    clear_error();
    MCAPQ_REQUIRE(st && m >= 1 && m <= st->max_m, MCAPQ_EINVAL, "bad stack_run arguments");
    cudaStream_t s = as_stream(stream);
    if (m == 1 && st->prog_dirty) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(s, &cs);
        if (cs == cudaStreamCaptureStatusNone) {
            mcapq_status r = build_program(st);
            if (r != MCAPQ_OK) return r;
        }
    }
    if (m == 1 && !st->prog_dirty && st->prog_ok) {
        // the whole step in one persistent cooperative kernel
        cudaError_t e = launch_stack_step(st->ops_dev, st->part, st->nops, st->counters, st->max_k, st->has_records,
                                          st->route_kinds, s);
        MCAPQ_REQUIRE(e == cudaSuccess, MCAPQ_ECUDA, "stack_step launch: %s", cudaGetErrorString(e));
        return MCAPQ_OK;
    }
    for (int l = 0; l < st->layers; ++l) {
        const int route = st->routes[l];
        int last_input = -1 << 30;
        A8Workspace w = {};
        mcapq_status r = for_each_group(st, l, [&](int first, int cnt, bool fast) -> mcapq_status {
            const Slot &a = st->slots[(size_t)l * kMaxSlots + first];
            if (fast) {
                StreamGroup g = {};
                g.count = cnt;
                g.k = a.k;
                for (int i = 0; i < cnt; ++i) {
                    const Slot &b = st->slots[(size_t)l * kMaxSlots + first + i];
                    g.nib[i] = b.nib;
                    g.scale[i] = b.scale;
                    g.n[i] = b.n;
                    g.y[i] = b.y;
                    g.ldy[i] = b.n;
                }
                cudaError_t e = launch_linear_group(route, g, a.x, m, a.k, a.ydt, route == MCAPQ_W4A8 ? st->ws : nullptr,
                                                    s, true);
                MCAPQ_REQUIRE(e == cudaSuccess, MCAPQ_ECUDA, "stream launch: %s", cudaGetErrorString(e));
                return MCAPQ_OK;
            }
            // generic path (K % 256 != 0): separate quantiser + GEMV
            if (route == MCAPQ_W4A8) {
                if (a.input_id != last_input) {
                    w = a8_workspace(st->ws, m, a.k);
                    cudaError_t e = launch_quant_a8(a.x, m, a.k, a.k, w.q, w.sx, w.sq, s, true);
                    MCAPQ_REQUIRE(e == cudaSuccess, MCAPQ_ECUDA, "quant launch: %s", cudaGetErrorString(e));
                    last_input = a.input_id;
                }
                cudaError_t e = launch_w4a8(a.nib, a.scale, a.n, a.k, w.q, w.sx, w.sq, m, a.y, a.ydt, a.n, s, true);
                MCAPQ_REQUIRE(e == cudaSuccess, MCAPQ_ECUDA, "w4a8 launch: %s", cudaGetErrorString(e));
            } else {
                cudaError_t e = launch_w4a16(a.nib, a.scale, a.n, a.k, a.x, m, a.k, a.y, a.ydt, a.n, s, true);
                MCAPQ_REQUIRE(e == cudaSuccess, MCAPQ_ECUDA, "w4a16 launch: %s", cudaGetErrorString(e));
            }
            return MCAPQ_OK;
        });
        if (r != MCAPQ_OK) return r;
    }
    return MCAPQ_OK;
}

mcapq_status mcapq_stack_capture(mcapq_stack *st, int64_t m, void *stream)
{
    clear_error();
    MCAPQ_REQUIRE(st, MCAPQ_EINVAL, "stack is NULL");
    cudaStream_t s = as_stream(stream);
    MCAPQ_REQUIRE(s != nullptr, MCAPQ_EINVAL, "graph capture needs a non-default stream");
    if (m == 1 && st->prog_dirty) {
        mcapq_status r = build_program(st);   // allocations happen before the capture
        if (r != MCAPQ_OK) return r;
    }
    drop_graph(st);
    MCAPQ_CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    mcapq_status r = mcapq_stack_run(st, m, stream);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(s, &g);
    if (r != MCAPQ_OK) {
        if (g) cudaGraphDestroy(g);
        return r;
    }
    MCAPQ_CUDA_TRY(e);
    st->graph = g;
    MCAPQ_CUDA_TRY(cudaGraphInstantiate(&st->exec, g, 0));
    st->graph_m = m;
    return MCAPQ_OK;
}

mcapq_status mcapq_stack_replay(mcapq_stack *st, void *stream)
{
    clear_error();
    MCAPQ_REQUIRE(st && st->exec, MCAPQ_EINVAL, "no captured graph");
    MCAPQ_CUDA_TRY(cudaGraphLaunch(st->exec, as_stream(stream)));
    return MCAPQ_OK;
}

size_t mcapq_stack_weight_bytes(const mcapq_stack *st)
{
    if (!st) return 0;
    size_t b = 0;
    for (const Slot &s : st->slots)
        if (s.set) b += (size_t)(s.n * (s.k / 2)) + (size_t)(s.n * (s.k / 32) * 2);
    return b;
}

int mcapq_stack_launches(const mcapq_stack *st, int64_t m)
{
    if (!st || m < 1) return 0;
    if (m == 1 && !st->prog_dirty && st->prog_ok) return 1;   // the persistent step kernel
    int c = 0;
    for (int l = 0; l < st->layers; ++l) {
        int last = -1 << 30;
        for_each_group(st, l, [&](int first, int cnt, bool fast) -> mcapq_status {
            const Slot &a = st->slots[(size_t)l * kMaxSlots + first];
            if (fast) {
                const int tp = stream_tokens_per_pass(st->routes[l], a.k);
                c += (int)((m + tp - 1) / tp);
            } else {
                if (st->routes[l] == MCAPQ_W4A8 && a.input_id != last) {
                    ++c;
                    last = a.input_id;
                }
                c += 1;
            }
            (void)cnt;
            return MCAPQ_OK;
        });
    }
    return c;
}

}  // extern "C"

// Is the input of slot (l, sl) a step input, i.e. not written by an earlier slot's
// output (decode order)?  Only step inputs travel from the host in step_host.
static bool step_input(const mcapq_stack *st, int l, int sl, int64_t m)
{
    const Slot &a = st->slots[(size_t)l * kMaxSlots + sl];
    const uintptr_t x0 = reinterpret_cast<uintptr_t>(a.x), x1 = x0 + (uintptr_t)(m * a.k * 2);
    for (int l2 = 0; l2 <= l; ++l2)
        for (int s2 = 0; s2 < kMaxSlots; ++s2) {
            if (l2 == l && s2 >= sl) break;
            const Slot &b = st->slots[(size_t)l2 * kMaxSlots + s2];
            if (!b.set || (l2 == l && b.input_id == a.input_id)) continue;
            const uintptr_t y0 = reinterpret_cast<uintptr_t>(b.y);
            const uintptr_t y1 = y0 + (uintptr_t)(m * b.n * (b.ydt == MCAPQ_F32 ? 4 : 2));
            if (y0 < x1 && x0 < y1) return false;
        }
    return true;
}

extern "C" {

size_t mcapq_stack_host_bytes(const mcapq_stack *st, int64_t m, int which)
{
    if (!st || m < 1) return 0;
    size_t b = 0;
    for (int l = 0; l < st->layers; ++l) {
        int last = -1 << 30;
        for (int sl = 0; sl < kMaxSlots; ++sl) {
            const Slot &s = st->slots[(size_t)l * kMaxSlots + sl];
            if (!s.set) continue;
            if (which == 0) {
                if (s.input_id != last && step_input(st, l, sl, m)) b += (size_t)(m * s.k) * 2;
                last = s.input_id;
            } else {
                b += (size_t)(m * s.n) * (s.ydt == MCAPQ_F32 ? 4 : 2);
            }
        }
    }
    return b;
}

mcapq_status mcapq_stack_step_host(mcapq_stack *st, int64_t m, const void *x_host, void *y_host, void *stream)
{
    clear_error();
    MCAPQ_REQUIRE(st && x_host && y_host && m >= 1 && m <= st->max_m, MCAPQ_EINVAL, "bad stack_step_host arguments");
    cudaStream_t s = as_stream(stream);
    // One copy per maximal run that is contiguous on both sides: callers that place
    // the step's inputs (and outputs) in one device arena in slot order get a single
    // H2D and a single D2H per step instead of one per slot.
    struct Run {
        char *dev;
        char *host;
        size_t bytes;
    };
    auto push = [](std::vector<Run> &runs, char *dev, char *host, size_t b) {
        if (!runs.empty() && runs.back().dev + runs.back().bytes == dev && runs.back().host + runs.back().bytes == host)
            runs.back().bytes += b;
        else
            runs.push_back({dev, host, b});
    };
    std::vector<Run> xin, yout;
    char *xp = reinterpret_cast<char *>(const_cast<void *>(x_host));
    for (int l = 0; l < st->layers; ++l) {
        int last = -1 << 30;
        for (int sl = 0; sl < kMaxSlots; ++sl) {
            const Slot &s_ = st->slots[(size_t)l * kMaxSlots + sl];
            if (!s_.set || s_.input_id == last) continue;
            last = s_.input_id;
            if (!step_input(st, l, sl, m)) continue;   // produced inside the step
            const size_t b = (size_t)(m * s_.k) * 2;
            push(xin, reinterpret_cast<char *>(const_cast<uint16_t *>(s_.x)), xp, b);
            xp += b;
        }
    }
    char *yp = reinterpret_cast<char *>(y_host);
    for (size_t i = 0; i < st->slots.size(); ++i) {
        const Slot &s_ = st->slots[i];
        if (!s_.set) continue;
        const size_t b = (size_t)(m * s_.n) * (s_.ydt == MCAPQ_F32 ? 4 : 2);
        push(yout, reinterpret_cast<char *>(s_.y), yp, b);
        yp += b;
    }
    for (const Run &r : xin) MCAPQ_CUDA_TRY(cudaMemcpyAsync(r.dev, r.host, r.bytes, cudaMemcpyHostToDevice, s));
    if (st->exec && st->graph_m == m) {
        MCAPQ_CUDA_TRY(cudaGraphLaunch(st->exec, s));
    } else {
        mcapq_status r = mcapq_stack_run(st, m, stream);
        if (r != MCAPQ_OK) return r;
    }
    for (const Run &r : yout) MCAPQ_CUDA_TRY(cudaMemcpyAsync(r.host, r.dev, r.bytes, cudaMemcpyDeviceToHost, s));
    return MCAPQ_OK;
}

void mcapq_stack_destroy(mcapq_stack *st)
{
    if (!st) return;
    drop_graph(st);
    if (st->ws) cudaFree(st->ws);
    free_program(st);
    delete st;
}

}  // extern "C"
