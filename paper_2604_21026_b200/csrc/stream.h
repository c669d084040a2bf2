// stream.h -- the persistent TMA-bulk-fed decode-linear path (kernels_stream.cu).
#pragma once
#include "internal.h"

namespace mcapq {

constexpr int kMaxGroup = 4;   // linears sharing one input per launch (q/k/v, gate/up)

// Host description of a group of linears that share the same input x.
struct StreamGroup {
    int count;
    int64_t k;
    const uint8_t *nib[kMaxGroup];
    const uint16_t *scale[kMaxGroup];
    int64_t n[kMaxGroup];
    void *y[kMaxGroup];
    int64_t ldy[kMaxGroup];
};

// Kernel parameters (by value).
struct StreamArgs {
    int count;
    const uint8_t *nib[kMaxGroup];
    const uint16_t *scale[kMaxGroup];
    int64_t n[kMaxGroup];
    void *y[kMaxGroup];
    int64_t ldy[kMaxGroup];
    int tile_start[kMaxGroup + 1];
    int64_t k;
    const uint16_t *x;
    int64_t ldx;
    int64_t tok0;
    int ntok, ntok_cap;
    int ydt;
    int stages;
    int act_bytes;
};

// K % 256 == 0 (16-B aligned scale rows for the bulk copies) and 16-B aligned planes.
bool stream_supported(int64_t k);
int stream_tokens_per_pass(int route, int64_t k);
cudaError_t launch_stream_group(int route, const StreamGroup &g, const uint16_t *x, int64_t m, int64_t ldx,
                                int ydt, cudaStream_t s, bool pdl);

}  // namespace mcapq
