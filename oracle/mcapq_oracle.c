/*
 * mcapq_oracle.c -- plain, slow, obviously-correct CPU oracle for the MCAP/NVE
 * mixed-precision decode linear (arXiv 2604.21026).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this file.  The product path
 * (paper_2604_21026_b200/) never links, imports or calls it, and this file shares
 * no source, header, table or helper with the CUDA path.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (LaTeX source), "S:n" =
 * SPEC.md line n.  Every reading of an ambiguous passage is listed in DESIGN.md
 * ("Readings") under the label given here (A1..A22, T).
 *
 * Build: gcc -O2 -std=c99 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC
 * (no FMA contraction, IEEE fp32 via SSE; the arithmetic below is written in the
 * order the paper / the readings state it, one term at a time).
 *
 * Layout conventions, identical to the ABI's:
 *   W      : [n][k] row-major float (bf16 or fp32 values), k % 32 == 0
 *   nib    : [n][k/2] bytes.  Block g of row r = bytes 16g..16g+15 of the row;
 *            byte t of a block = c[32g+t] | c[32g+t+16] << 4   ("llama.cpp
 *            split format")
 *   scale  : [n][k/32] IEEE binary16 bit patterns (the Q4_0 block's d; P:932
 *            "18 bytes per 32 elements" => 16 B nibbles + 2 B fp16 scale)
 *   q      : [m][k] int8, sx: [m][k/32] float, sq: [m][k/32] int32
 *   y      : [m][n]
 *
 * Parity pins: every function below is pinned by tests/test_oracle_*.py against
 * paper values, closed forms, brute force (exact rationals) or hardware
 * conversions.  See DESIGN.md "Oracle pins".
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL 1
#define OR_ERANGE 3

/* ------------------------------------------------------------------------- */
/* IEEE conversions written out bit by bit (pinned exhaustively vs F16C / torch) */
/* ------------------------------------------------------------------------- */

static uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

/* fp32 -> binary16, round to nearest, ties to even (IEEE 754 default). */
uint16_t oracle_f32_to_f16(float f)
{
    uint32_t u = f2u(f);
    uint16_t sign = (uint16_t)((u >> 16) & 0x8000u);
    uint32_t exp = (u >> 23) & 0xFFu;
    uint32_t man = u & 0x7FFFFFu;

    if (exp == 0xFFu) {                       /* inf / nan */
        if (man == 0) return (uint16_t)(sign | 0x7C00u);
        return (uint16_t)(sign | 0x7E00u | (man >> 13));  /* quiet nan, keep payload top bits */
    }
    int32_t e = (int32_t)exp - 127;           /* unbiased exponent */
    if (exp == 0) {                            /* fp32 zero / subnormal: far below fp16 range */
        return sign;                           /* |f| < 2^-126 rounds to 0 in fp16 */
    }
    uint32_t sig = man | 0x800000u;            /* 24-bit significand, value = sig * 2^(e-23) */
    if (e > 15) return (uint16_t)(sign | 0x7C00u);    /* overflow -> inf */
    if (e >= -14) {                            /* normal fp16: keep 11 bits of sig */
        uint32_t keep = sig >> 13;             /* 11 bits incl. hidden */
        uint32_t rem = sig & 0x1FFFu;          /* 13 dropped bits */
        uint32_t half = 0x1000u;
        if (rem > half || (rem == half && (keep & 1u))) keep += 1u;
        /* keep may now be 0x800 (2^11): carries into the exponent, handled by add below */
        uint32_t h = ((uint32_t)(e + 15) << 10) + (keep - 0x400u);
        if (keep == 0x800u) h = ((uint32_t)(e + 16) << 10);  /* exact power of two after carry */
        if (h >= 0x7C00u) return (uint16_t)(sign | 0x7C00u);
        return (uint16_t)(sign | h);
    }
    /* subnormal fp16: value = m * 2^-24, m < 1024 */
    int32_t shift = -14 - e + 13;              /* bits to drop from sig to land on 2^-24 units */
    if (shift > 24) return sign;               /* < 2^-25 (strictly below half the smallest subnormal) */
    uint32_t keep = sig >> shift;
    uint32_t rem = sig & ((1u << shift) - 1u);
    uint32_t half = 1u << (shift - 1);
    if (rem > half || (rem == half && (keep & 1u))) keep += 1u;
    return (uint16_t)(sign | keep);            /* keep == 0x400 becomes the smallest normal: correct */
}

/* binary16 -> fp32 (exact). */
float oracle_f16_to_f32(uint16_t h)
{
    uint32_t sign = ((uint32_t)h & 0x8000u) << 16;
    uint32_t exp = ((uint32_t)h >> 10) & 0x1Fu;
    uint32_t man = (uint32_t)h & 0x3FFu;
    if (exp == 0x1Fu) return u2f(sign | 0x7F800000u | (man << 13));
    if (exp == 0) {
        /* zero or subnormal: value = man * 2^-24, exactly representable in fp32 */
        float v = (float)man * (1.0f / 16777216.0f);
        return sign ? -v : v;
    }
    return u2f(sign | ((exp - 15u + 127u) << 23) | (man << 13));
}

/* bfloat16 -> fp32 (exact: bf16 is the top half of an fp32). */
float oracle_bf16_to_f32(uint16_t b) { return u2f((uint32_t)b << 16); }

/* fp32 -> bfloat16, round to nearest even; nan stays (quiet) nan. */
uint16_t oracle_f32_to_bf16(float f)
{
    uint32_t u = f2u(f);
    if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x7FFFFFu)) return (uint16_t)((u >> 16) | 0x40u);
    uint32_t keep = u >> 16;
    uint32_t rem = u & 0xFFFFu;
    if (rem > 0x8000u || (rem == 0x8000u && (keep & 1u))) keep += 1u;
    return (uint16_t)keep;
}

/* round half away from zero (S:344 reading A5).  C99 roundf has exactly this
 * contract; written out so the reader does not have to trust that.            */
static float round_half_away(float v)
{
    float a = fabsf(v);
    float t = floorf(a);
    float r = (a - t >= 0.5f) ? t + 1.0f : t;   /* a - t is exact for |a| < 2^23 */
    if (a >= 8388608.0f) r = a;                 /* already an integer */
    return (v < 0.0f) ? -r : r;
}

/* ------------------------------------------------------------------------- */
/* a1: Q4_0 weight pack (readings A2-A5, A21) */
/* ------------------------------------------------------------------------- */

/* Quantise one 32-element block x[0..31].  Writes 16 nibble bytes + fp16 scale.
 * Returns OR_OK, or OR_ERANGE for non-finite input / fp16 scale overflow.     */
int oracle_q4_0_block(const float *x, uint8_t *nib16, uint16_t *scale)
{
    /* 1. m = the element of maximum magnitude, first index on ties (A3) */
    float m = 0.0f, amax = 0.0f;
    for (int j = 0; j < 32; ++j) {
        if (!isfinite(x[j])) {                 /* non-finite input is an error */
            memset(nib16, 0x88, 16);
            *scale = 0x0000u;
            return OR_ERANGE;
        }
        if (fabsf(x[j]) > amax) { amax = fabsf(x[j]); m = x[j]; }
    }
    uint8_t c[32];
    /* 2. d = fp16_rne(m / -8)   (A2: llama.cpp convention, extreme maps to code 0) */
    float dq = m / -8.0f;
    uint16_t d16 = oracle_f32_to_f16(dq);
    if ((d16 & 0x7FFFu) == 0x7C00u) {          /* |d| rounds to inf: fp16 overflow (A4) */
        *scale = d16;
        memset(nib16, 0x88, 16);
        return OR_ERANGE;
    }
    float d = oracle_f16_to_f32(d16);
    if (d == 0.0f) {
        /* 4. zero block (also d underflowing to 0): codes 8, d = +0 (A4, A21) */
        for (int j = 0; j < 32; ++j) c[j] = 8;
        d16 = 0x0000u;
    } else {
        /* 3. c_j = clamp(round_half_away(x_j / f32(d)), -8, 7) + 8  (A4, A5) */
        for (int j = 0; j < 32; ++j) {
            float r = round_half_away(x[j] / d);
            if (r < -8.0f) r = -8.0f;
            if (r > 7.0f) r = 7.0f;
            c[j] = (uint8_t)((int)r + 8);
        }
    }
    /* 5. split nibble layout: byte t = c_t | c_{t+16} << 4 */
    for (int t = 0; t < 16; ++t) nib16[t] = (uint8_t)(c[t] | (c[t + 16] << 4));
    *scale = d16;
    return OR_OK;
}

/* Pack W[n][k] (fp32 values; a bf16 matrix is passed widened, which is exact).
 * Returns the first non-OK block status (every block is still written).       */
int oracle_pack_w4(const float *w, int64_t n, int64_t k, uint8_t *nib, uint16_t *scale)
{
    if (n < 0 || k <= 0 || k % 32) return OR_EINVAL;
    int64_t G = k / 32;
    int status = OR_OK;
    for (int64_t r = 0; r < n; ++r)
        for (int64_t g = 0; g < G; ++g) {
            int s = oracle_q4_0_block(w + r * k + g * 32, nib + r * (k / 2) + g * 16, scale + r * G + g);
            if (s != OR_OK && status == OR_OK) status = s;
        }
    return status;
}

/* Nibble code of element (r, j): undo the split layout.  Returns 0..15. */
static int code_at(const uint8_t *nib, int64_t k, int64_t r, int64_t j)
{
    int64_t g = j / 32, t = j % 32;
    uint8_t byte = nib[r * (k / 2) + g * 16 + (t % 16)];
    return (t < 16) ? (byte & 0x0F) : (byte >> 4);
}

/* Dequantise: W~[r][j] = f32(d) * (c - 8), in fp32 (the product is exact). */
void oracle_dequant_w4(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k, float *w)
{
    int64_t G = k / 32;
    for (int64_t r = 0; r < n; ++r)
        for (int64_t j = 0; j < k; ++j)
            w[r * k + j] = oracle_f16_to_f32(scale[r * G + j / 32]) * (float)(code_at(nib, k, r, j) - 8);
}

/* AoS export of one row: 18-byte blocks [d_f16 little endian][16 nibble bytes]
 * (the Q4_0 block itself).                                  */
void oracle_export_q4_0_aos(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k, uint8_t *out)
{
    int64_t G = k / 32;
    for (int64_t r = 0; r < n; ++r)
        for (int64_t g = 0; g < G; ++g) {
            uint8_t *b = out + (r * G + g) * 18;
            uint16_t d = scale[r * G + g];
            b[0] = (uint8_t)(d & 0xFF);
            b[1] = (uint8_t)(d >> 8);
            memcpy(b + 2, nib + r * (k / 2) + g * 16, 16);
        }
}

/* ------------------------------------------------------------------------- */
/* a2: per-token, per-32-group int8 activation quantisation                    */
/*     (readings A6, A7, A8, A21)           */
/* ------------------------------------------------------------------------- */
int oracle_quant_a8(const float *x, int64_t m, int64_t k, int8_t *q, float *sx, int32_t *sq)
{
    if (m < 0 || k <= 0 || k % 32) return OR_EINVAL;
    int64_t G = k / 32;
    int status = OR_OK;
    for (int64_t i = 0; i < m; ++i)
        for (int64_t g = 0; g < G; ++g) {
            const float *xg = x + i * k + g * 32;
            /* (1) amax */
            float amax = 0.0f;
            int finite = 1;
            for (int j = 0; j < 32; ++j) {
                if (!isfinite(xg[j])) finite = 0;
                if (fabsf(xg[j]) > amax) amax = fabsf(xg[j]);
            }
            if (!finite) status = OR_ERANGE;
            /* (2) s = amax / 127.0.  s == 0 (amax == 0, or an fp32 amax
             * below 127 * 2^-149 whose quotient underflows) is the zero group (A21). */
            float s = amax / 127.0f;
            int32_t sum = 0;
            for (int j = 0; j < 32; ++j) {
                int code = 0;
                if (s != 0.0f && finite) {
                    /* (3) q = round(x / s), clamped to [-127, 127] */
                    float r = round_half_away(xg[j] / s);
                    if (r < -127.0f) r = -127.0f;
                    if (r > 127.0f) r = 127.0f;
                    code = (int)r;
                }
                q[i * k + g * 32 + j] = (int8_t)code;
                sum += code;
            }
            sx[i * G + g] = (s != 0.0f && finite) ? s : 0.0f;   /* +0 for a zero group (A21) */
            sq[i * G + g] = sum;                          /* sum_x (A8) */
        }
    return status;
}

/* ------------------------------------------------------------------------- */
/* a3 / a5: W4A8 linear (readings A9, A1)             */
/* ------------------------------------------------------------------------- */

/* Integer stage: D[i][r][g] = sumi - 8 * sum_x with sumi = sum_j c_j * q_j over
 * the unsigned nibbles.  Exact int32.                              */
int oracle_w4a8_group_dots(const uint8_t *nib, int64_t n, int64_t k, const int8_t *q, const int32_t *sq,
                           int64_t m, int32_t *D)
{
    if (n < 0 || m < 0 || k <= 0 || k % 32) return OR_EINVAL;
    int64_t G = k / 32;
    for (int64_t i = 0; i < m; ++i)
        for (int64_t r = 0; r < n; ++r)
            for (int64_t g = 0; g < G; ++g) {
                int32_t sumi = 0;
                for (int j = 0; j < 32; ++j)
                    sumi += code_at(nib, k, r, g * 32 + j) * (int32_t)q[i * k + g * 32 + j];
                D[(i * n + r) * G + g] = sumi - 8 * sq[i * G + g];
            }
    return OR_OK;
}

/* Outputs: y32[i][r] = sum_g (f32(d) * s) * f32(D)   in fp32, increasing g,
 *          y64[i][r] = sum_g (double)d * (double)s * (double)D   (each term exact;
 * the north star's "int64 exact dot times scales" reference).
 * Either output pointer may be NULL.  Rows are independent (OpenMP over rows
 * changes nothing: the per-row order is fixed).                                */
int oracle_w4a8(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k,
                const int8_t *q, const float *sx, const int32_t *sq, int64_t m, float *y32, double *y64)
{
    if (n < 0 || m < 0 || k <= 0 || k % 32) return OR_EINVAL;
    int64_t G = k / 32;
    for (int64_t i = 0; i < m; ++i) {
#pragma omp parallel for schedule(static)
        for (int64_t r = 0; r < n; ++r) {
            float acc32 = 0.0f;
            double acc64 = 0.0;
            for (int64_t g = 0; g < G; ++g) {
                int32_t sumi = 0;
                for (int j = 0; j < 32; ++j)
                    sumi += code_at(nib, k, r, g * 32 + j) * (int32_t)q[i * k + g * 32 + j];
                int32_t Dg = sumi - 8 * sq[i * G + g];
                float d = oracle_f16_to_f32(scale[r * G + g]);
                float s = sx[i * G + g];
                float ds = d * s;
                float term = ds * (float)Dg;
                acc32 = acc32 + term;
                acc64 = acc64 + ((double)d * (double)s) * (double)Dg;
            }
            if (y32) y32[i * n + r] = acc32;
            if (y64) y64[i * n + r] = acc64;
        }
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* a4: W4A16 linear, exact dequant (reading A10)  */
/* ------------------------------------------------------------------------- */
/* y32[i][r] = sum_j (f32(d) * (c - 8)) * x_j in fp32, increasing j;
 * y64[i][r] = the same in fp64 (= fp64 matmul of the dequantised weights).
 * x is [m][k] fp32 (bf16 activations widened, which is exact).                 */
int oracle_w4a16(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k,
                 const float *x, int64_t m, float *y32, double *y64)
{
    if (n < 0 || m < 0 || k <= 0 || k % 32) return OR_EINVAL;
    int64_t G = k / 32;
    for (int64_t i = 0; i < m; ++i) {
#pragma omp parallel for schedule(static)
        for (int64_t r = 0; r < n; ++r) {
            float acc32 = 0.0f;
            double acc64 = 0.0;
            for (int64_t j = 0; j < k; ++j) {
                float d = oracle_f16_to_f32(scale[r * G + j / 32]);
                float wdq = d * (float)(code_at(nib, k, r, j) - 8);
                float xj = x[i * k + j];
                acc32 = acc32 + wdq * xj;
                acc64 = acc64 + (double)wdq * (double)xj;
            }
            if (y32) y32[i * n + r] = acc32;
            if (y64) y64[i * n + r] = acc64;
        }
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* a6: W4A16 batched semantics, dequantise-to-bf16 then GEMM (P:982 precedent; */
/*     reading A13): W^ = bf16_rne(f32(d) * (c - 8)); y = X . W^T, fp32 accum.  */
/* ------------------------------------------------------------------------- */
int oracle_w4a16_bf16deq(const uint8_t *nib, const uint16_t *scale, int64_t n, int64_t k,
                         const float *x, int64_t m, float *y32, double *y64)
{
    if (n < 0 || m < 0 || k <= 0 || k % 32) return OR_EINVAL;
    int64_t G = k / 32;
    for (int64_t i = 0; i < m; ++i) {
#pragma omp parallel for schedule(static)
        for (int64_t r = 0; r < n; ++r) {
            float acc32 = 0.0f;
            double acc64 = 0.0;
            for (int64_t j = 0; j < k; ++j) {
                float d = oracle_f16_to_f32(scale[r * G + j / 32]);
                float wdq = oracle_bf16_to_f32(oracle_f32_to_bf16(d * (float)(code_at(nib, k, r, j) - 8)));
                float xj = x[i * k + j];
                acc32 = acc32 + wdq * xj;
                acc64 = acc64 + (double)wdq * (double)xj;
            }
            if (y32) y32[i * n + r] = acc32;
            if (y64) y64[i * n + r] = acc64;
        }
    }
    return OR_OK;
}

/* Vectorised helpers for the Python wrapper (array-wide conversions). */
void oracle_f32_to_f16_array(const float *x, int64_t n, uint16_t *out)
{
    for (int64_t i = 0; i < n; ++i) out[i] = oracle_f32_to_f16(x[i]);
}
void oracle_f16_to_f32_array(const uint16_t *h, int64_t n, float *out)
{
    for (int64_t i = 0; i < n; ++i) out[i] = oracle_f16_to_f32(h[i]);
}
void oracle_f32_to_bf16_array(const float *x, int64_t n, uint16_t *out)
{
    for (int64_t i = 0; i < n; ++i) out[i] = oracle_f32_to_bf16(x[i]);
}

/* Exhaustive self-check helper used by the fp16 pin: counts the fp32 bit
 * patterns in [lo, hi) whose conversion differs from the table `ref` written by
 * an independent converter (F16C in tests/pins/f16c_ref.c).                    */
int64_t oracle_count_f16_mismatch(uint32_t lo, uint32_t hi, const uint16_t *ref)
{
    int64_t bad = 0;
    for (uint64_t u = lo; u < hi; ++u) {
        uint16_t h = oracle_f32_to_f16(u2f((uint32_t)u));
        uint16_t e = ref[u - lo];
        int nan_h = ((h & 0x7C00u) == 0x7C00u) && (h & 0x3FFu);
        int nan_e = ((e & 0x7C00u) == 0x7C00u) && (e & 0x3FFu);
        if (nan_h && nan_e) continue;          /* nan payloads are not part of the contract */
        if (h != e) ++bad;
    }
    return bad;
}
