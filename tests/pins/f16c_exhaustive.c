/* Exhaustive pin of the oracle's fp32 -> fp16 (RNE) conversion against the x86
 * F16C hardware converter (VCVTPS2PH, round-to-nearest-even), over all 2^32
 * fp32 bit patterns.  NaN payloads are excluded (not part of the contract).
 * Independent of the oracle: F16C is the hardware's own IEEE implementation.
 * Usage: f16c_exhaustive  -> prints the mismatch count, exit 0 iff zero.      */
#include <immintrin.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

uint16_t oracle_f32_to_f16(float f);
float oracle_f16_to_f32(uint16_t h);

int main(void)
{
    long long bad = 0, bad_back = 0;
#pragma omp parallel for reduction(+ : bad, bad_back) schedule(static)
    for (long long hi = 0; hi < 65536; ++hi) {
        for (uint32_t lo = 0; lo < 65536; ++lo) {
            uint32_t u = ((uint32_t)hi << 16) | lo;
            float f;
            memcpy(&f, &u, 4);
            uint16_t ref = (uint16_t)_cvtss_sh(f, _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC);
            uint16_t got = oracle_f32_to_f16(f);
            int nan_r = ((ref & 0x7C00u) == 0x7C00u) && (ref & 0x3FFu);
            int nan_g = ((got & 0x7C00u) == 0x7C00u) && (got & 0x3FFu);
            if (nan_r && nan_g) continue;
            if (ref != got) ++bad;
        }
        if (hi == 0) {
            /* fp16 -> fp32 for all 65536 halves vs F16C VCVTPH2PS */
            for (uint32_t h = 0; h < 65536; ++h) {
                float r = _cvtsh_ss((unsigned short)h);
                float g = oracle_f16_to_f32((uint16_t)h);
                uint32_t ur, ug;
                memcpy(&ur, &r, 4);
                memcpy(&ug, &g, 4);
                if (r != r && g != g) continue;
                if (ur != ug) ++bad_back;
            }
        }
    }
    printf("%lld %lld\n", bad, bad_back);
    return (bad || bad_back) ? 1 : 0;
}
