// Throughput probe: TMEM read-back (tcgen05.ld) per SM on sm_100a -- the quantity that
// decides whether W4A8 batched decode can live on tcgen05 (kind::i8): Q4_0 needs one
// fp32 scale per 32-K block, so every block's int32 MMA result (128 rows x N tokens)
// must be read back from TMEM and scaled before the next block accumulates.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_ld tmem_ld.cu && ./tmem_ld
// Prints bytes per SM clock for tcgen05.ld.32x32b.{x16,x32,x64} with 4 / 8 / 16 warps,
// loads only, and with the Q4_0 epilogue arithmetic a W4A8 block needs per element
// (int32 -> fp32 via the magic add, (d s) product, fma into the fp32 accumulator).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int X>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, uint32_t (&r)[X])
{
    if constexpr (X == 16) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
    } else if constexpr (X == 32) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
              "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(taddr));
    }
}

template <int X, bool kEpi>
__global__ void probe(unsigned long long *cyc, float *sink, int iters)
{
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&tslot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t base = tslot + ((uint32_t)(32 * (warp & 3)) << 16);   // this warp's lane quarter
    const int nwarps = blockDim.x >> 5;
    float acc[X];
#pragma unroll
    for (int j = 0; j < X; ++j) acc[j] = 0.f;
    const float ds = 1.0f + threadIdx.x * 1e-7f;
    uint32_t x = 0;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        // each warp walks its own column window (the 4 lane quarters x 512 columns)
        const uint32_t col = (uint32_t)(((it * (nwarps / 4 > 0 ? nwarps / 4 : 1) + (warp >> 2)) * X) & 511);
        uint32_t r[X];
        tmem_ld<X>(base + col, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if constexpr (kEpi) {
#pragma unroll
            for (int j = 0; j < X; ++j) {
                const float D = __int_as_float((int)r[j]) - 12582912.0f;   // magic-biased int32 -> fp32
                acc[j] = fmaf(ds, D, acc[j]);
            }
        } else {
#pragma unroll
            for (int j = 0; j < X; ++j) x ^= r[j];
        }
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    float s = (float)x;
#pragma unroll
    for (int j = 0; j < X; ++j) s += acc[j];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tslot) : "memory");
}

template <int X, bool kEpi>
void run(int warps, int sms)
{
    const int iters = 4096;
    unsigned long long *cyc;
    float *sink;
    cudaMalloc(&cyc, sizeof(unsigned long long) * sms);
    cudaMalloc(&sink, sizeof(float) * sms * warps * 32);
    probe<X, kEpi><<<sms, warps * 32>>>(cyc, sink, 16);   // warm-up
    probe<X, kEpi><<<sms, warps * 32>>>(cyc, sink, iters);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return;
    }
    unsigned long long h[1024];
    cudaMemcpy(h, cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < sms; ++i) mean += (double)h[i] / sms;
    const double bytes = (double)warps * iters * 32 * X * 4;   // per CTA (one CTA per SM)
    printf("{\"probe\": \"tmem_ld\", \"x\": %d, \"epilogue\": %s, \"warps\": %d, \"cycles\": %.0f, "
           "\"bytes_per_clk_per_sm\": %.1f}\n",
           X, kEpi ? "true" : "false", warps, mean, bytes / mean);
    cudaFree(cyc);
    cudaFree(sink);
}

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int w : {4, 8, 16}) {
        run<16, false>(w, sms);
        run<32, false>(w, sms);
        run<16, true>(w, sms);
        run<32, true>(w, sms);
    }
    return 0;
}
