// Throughput probe: legacy mma.sync (HMMA bf16 m16n8k16, IMMA s8 m16n8k32) on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu && ./mma_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int KIND>
__global__ void probe(float *out, int iters)
{
    uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    float c[8][4] = {};
    int ci[8][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (KIND == 0) {
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                             : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
            } else {
                asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+r"(ci[j][0]), "+r"(ci[j][1]), "+r"(ci[j][2]), "+r"(ci[j][3])
                             : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
            }
        }
    }
    float s = 0;
    for (int j = 0; j < 8; ++j)
        for (int e = 0; e < 4; ++e) s += c[j][e] + (float)ci[j][e];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out;
    cudaMalloc(&out, sizeof(float) * sms * 4 * 1024);
    for (int kind = 0; kind < 2; ++kind)
        for (int warps : {4, 8, 16}) {
            const int iters = 4096, grid = sms * 2;
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            auto launch = [&]() {
                if (kind == 0) probe<0><<<grid, warps * 32>>>(out, iters);
                else probe<1><<<grid, warps * 32>>>(out, iters);
            };
            launch();
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double mmas = (double)grid * warps * iters * 8;
            const double flop = mmas * (kind == 0 ? 2.0 * 16 * 8 * 16 : 2.0 * 16 * 8 * 32);
            printf("{\"kind\": \"%s\", \"warps_per_cta\": %d, \"ctas_per_sm\": 2, \"T(FL)OP/s\": %.1f, \"mma_per_sm_per_clk_at_1.965GHz\": %.3f}\n",
                   kind == 0 ? "hmma.m16n8k16.bf16" : "imma.m16n8k32.s8", warps, flop / (ms * 1e-3) / 1e12,
                   mmas / (ms * 1e-3) / sms / 1.965e9);
        }
    return 0;
}
