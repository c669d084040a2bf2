// stream_engines.cuh -- the per-stage compute of the TMA-fed decode linears,
// shared by the per-linear kernel (stream_kernel.cuh) and the persistent
// decode-step kernel (stack_kernel.cuh).  Included by kernels_stream.cu after
// its PTX helpers and fragment routines.
//
// Activation layouts in shared memory (per token, tsz bytes apart):
//  W4A8 : q_lo [G][16] | q_hi [G][16] | 16 B pad   (q_lo = elements 0..15 of each
//         32-group, q_hi = 16..31: lane-per-block LDS.128 reads are consecutive),
//         then sx [ntok][G] fp32 and sq [ntok][G] int32 after all tokens.
//  W4A16: [G][4 t][8 bf16] in fragment order (4t,4t+2,4t+1,4t+3,4t+16,4t+18,4t+17,4t+19) | 64 B pad,
//         then corr [G][8 tokens] fp32 = -136 * sum_j x_j of the group.
#pragma once

// fp32 pairs in one 64-bit register (FFMA2 / FADD2 / FMUL2: two independent IEEE ops)
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t f2_pack(float a, float b)
{
    f2_t r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ f2_t f2_pack_bits(uint32_t a, uint32_t b)
{
    f2_t r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ float2 f2_unpack(f2_t r)
{
    float2 v;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
    return v;
}
__device__ __forceinline__ f2_t f2_fma(f2_t a, f2_t b, f2_t c)
{
    f2_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f2_t f2_add(f2_t a, f2_t b)
{
    f2_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2_t f2_mul(f2_t a, f2_t b)
{
    f2_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
struct ActSmem {
    uint32_t act, tsz, ssq, corr;
};

// W4A8 per-group scalars are stored as pairs ssq[tok][g] = {s (fp32 bits), 8 * sum q}.
__device__ __forceinline__ ActSmem act_layout(bool a16, uint32_t act, int64_t k, int ntok)
{
    ActSmem L;
    L.act = act;
    L.tsz = a16 ? (uint32_t)(2 * k + 64) : (uint32_t)(k + 16);
    L.ssq = act + (uint32_t)ntok * L.tsz;         // W4A8: [ntok][G] x {fp32 s, int32 8 sum q}
    L.corr = act + (uint32_t)ntok * L.tsz;        // W4A16: [G][8] fp32
    return L;
}

// u8 x s8 dot of 4 bytes (the high nibbles kept in place: 16 c_hi as u8)
__device__ __forceinline__ int dp4a_us(uint32_t a, int b, int c)
{
    int d;
    asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// D = sum_j c_j q_j - 8 sum q over one block, exact int32: the low
// nibbles (elements 4u..4u+3 of word u) against q words u, the high nibbles left in
// place (16 c, elements 4u+16..) against q words 4+u, then >> 4 (exact: a multiple of 16).
__device__ __forceinline__ int block_D(uint4 w, uint4 qa, uint4 qb, int sq8)
{
    int lo = 0, hi = 0;
    lo = __dp4a((int)(w.x & 0x0F0F0F0Fu), (int)qa.x, lo);
    hi = dp4a_us(w.x & 0xF0F0F0F0u, (int)qb.x, hi);
    lo = __dp4a((int)(w.y & 0x0F0F0F0Fu), (int)qa.y, lo);
    hi = dp4a_us(w.y & 0xF0F0F0F0u, (int)qb.y, hi);
    lo = __dp4a((int)(w.z & 0x0F0F0F0Fu), (int)qa.z, lo);
    hi = dp4a_us(w.z & 0xF0F0F0F0u, (int)qb.z, hi);
    lo = __dp4a((int)(w.w & 0x0F0F0F0Fu), (int)qa.w, lo);
    hi = dp4a_us(w.w & 0xF0F0F0F0u, (int)qb.w, hi);
    return lo + (hi >> 4) - sq8;
}

// ---------------------------------------------------------------- activation staging
// W4A8: per-token, per-32-group quantisation, a quad of threads per
// group (8 elements each), x read straight from global (L2): exact max,
// s = amax / 127 (IEEE), q = clamp(round_half_away(x / s)) via quant_code (exact),
// exact int sum -- bit-identical to quant_a8_kernel.  Warp-uniform trip counts
// (quad shuffles).  Called by all nthreads consumer threads (tid in [0, nthreads)).
// kCoherent: x may have been written by other CTAs of the same kernel (persistent
// step kernel) -> ld.global.cg (L2) instead of the read-only .nc path.
template <bool kCoherent>
__device__ __forceinline__ uint4 ldg_x128(const void *p)
{
    if constexpr (kCoherent) {
        uint4 v;
        asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
        return v;
    } else {
        return ldg_nc_128(p);
    }
}
template <bool kCoherent>
__device__ __forceinline__ uint2 ldg_x64(const void *p)
{
    if constexpr (kCoherent) {
        uint2 v;
        asm volatile("ld.global.cg.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
        return v;
    } else {
        return ldg_nc_64(p);
    }
}

// The 8 bf16 values (4 packed words) one quad member holds, as fp32 (exact).
__device__ __forceinline__ void bf16x8_to_f32(const uint32_t w4[4], float v[8])
{
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        v[2 * e] = __uint_as_float(w4[e] << 16);
        v[2 * e + 1] = __uint_as_float(w4[e] & 0xffff0000u);
    }
}

// s = fl(a / 127) (IEEE round-to-nearest) without the division: one
// correction step from r = fl(1/127) (q0 = a r, e = a - 127 q0 exactly by FMA,
// s = q0 + e r).  Exact for every finite bf16 magnitude a -- checked exhaustively
// against rational arithmetic by tests/test_quant_identities.py.
__device__ __forceinline__ float div127_rn(float a)
{
    const float r = 0x1.020408p-7f;
    const float q0 = __fmul_rn(a, r);
    const float e = __fmaf_rn(-q0, 127.0f, a);
    return __fmaf_rn(e, r, q0);
}

// 1/s for quant_code: MUFU.RCP (<= 1 ulp), inside quant_code's half-integer margin;
// a subnormal s (amax < 127 * 2^-126) takes the IEEE reciprocal.
__device__ __forceinline__ float rcp_group(float s)
{
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(s));
    if (s < 1.17549435e-38f) r = __frcp_rn(s);
    return r;
}

// max |x| over packed bf16 words as the bits of a bf16 magnitude (integer max of
// the sign-cleared bits == fp max for finite values; >= 0x7f80 <=> some x is inf/NaN)
__device__ __forceinline__ uint32_t absmax_bits(uint32_t acc, uint32_t w)
{
    return __vmaxu2(acc, w & 0x7fff7fffu);
}
__device__ __forceinline__ uint32_t absmax_fold(uint32_t m)
{
    return max(m & 0xffffu, m >> 16);
}

// Codes of N elements of one group, branch-free: q = rint(v * inv) read from the bits
// of fl(v * inv) + 1.5 * 2^23.  Off the half-integers rint == round_half_away(fl(v / s))
// (quant_code's margin argument); |fl(v / s)| <= 127.00003 for every element of a live
// group (|v| <= amax, s = fl(amax / 127)), so no clamp is needed.  Returns false when
// some element lies within 1e-4 of a half-integer or is not finite after the multiply
// (inv = inf for a subnormal s): the caller then recomputes the whole group with
// quant_code (IEEE division), so the codes are bit-identical to quant_a8_kernel.
template <int N>
__device__ __forceinline__ bool quant_codes_fast(const float *v, float inv, int *c)
{
    bool ok = true;
#pragma unroll
    for (int j = 0; j < N; ++j) {
        const float qa = __fmul_rn(v[j], inv);
        const float t = __fadd_rn(qa, 12582912.0f);
        const float r = __fsub_rn(qa, __fsub_rn(t, 12582912.0f));
        ok = ok && fabsf(r) < 0.4999f;
        c[j] = __float_as_int(t) - 0x4B400000;
    }
    return ok;
}

// Codes of the elements of packed bf16 words w[0..NW) (element 2e = low half of w[e]),
// packed four per word in element order into out[0..NW/2), branch-free on the f32x2
// pipe: q = rint(v * inv) is the low byte of fl(fl(v * inv) + 1.5 * 2^23) (the magic
// sum is M + rint exactly for |v * inv| < 2^22), packed by three PRMTs per four codes.
// Off the half-integers rint == round_half_away(fl(v / s)) (quant_code's margin
// argument; |fl(v / s)| <= 127.00003 in a live group, so no clamp).  Returns false when
// some element lies within 1e-4 of a half-integer: the caller then takes quant_code
// (IEEE division) for every element, so the codes stay bit-identical to quant_a8_kernel.
// For a live group with a finite inv every v * inv is finite (|v| <= amax), so the
// NaN-ignoring max below never hides a non-finite residual.
template <int NW>
__device__ __forceinline__ bool quant_words_fast(const uint32_t *w, float inv, uint32_t *out)
{
    const f2_t I = f2_pack(inv, inv), Mp = f2_pack(12582912.0f, 12582912.0f), Mn = f2_pack(-12582912.0f, -12582912.0f),
               N1 = f2_pack(-1.0f, -1.0f);
    uint32_t tb[2 * NW];
    float worst = 0.0f;
#pragma unroll
    for (int e = 0; e < NW; ++e) {
        const f2_t v = f2_pack_bits(w[e] << 16, w[e] & 0xffff0000u);
        const f2_t qa = f2_mul(v, I);
        const f2_t t = f2_add(qa, Mp);
        const f2_t d = f2_fma(f2_add(t, Mn), N1, qa);   // qa - rint(qa), exact
        const float2 dd = f2_unpack(d), tt = f2_unpack(t);
        worst = fmaxf(worst, fmaxf(fabsf(dd.x), fabsf(dd.y)));
        tb[2 * e] = __float_as_uint(tt.x);
        tb[2 * e + 1] = __float_as_uint(tt.y);
    }
#pragma unroll
    for (int o = 0; o < NW / 2; ++o)
        out[o] = __byte_perm(__byte_perm(tb[4 * o], tb[4 * o + 1], 0x0040), __byte_perm(tb[4 * o + 2], tb[4 * o + 3], 0x0040),
                             0x5410);
    // inv = inf (a live group with s < 2^-128: 1/s overflows) makes residuals NaN, which
    // fmaxf drops: such groups always take the IEEE path
    return worst < 0.4999f && inv < __int_as_float(0x7f800000);
}

// Slow path of quant_words_fast (a group with an element near a half-integer): four
// codes by quant_code (IEEE division), packed.  Out of line and register-only (scalar
// arguments, a scalar result): the rare path costs no instruction-cache space in the
// callers and no local memory.
__device__ __noinline__ uint32_t quant4_ieee(uint32_t w0, uint32_t w1, float s, float inv)
{
    uint32_t p = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t b = (j >> 1) ? w1 : w0;
        const float v = __uint_as_float((j & 1) ? (b & 0xffff0000u) : (b << 16));
        p |= ((uint32_t)quant_code(v, s, inv) & 0xffu) << (8 * j);
    }
    return p;
}
template <int NW>
__device__ __forceinline__ void quant_words_ieee(const uint32_t *w, float s, float inv, uint32_t *out)
{
#pragma unroll
    for (int o = 0; o < NW / 2; ++o) out[o] = quant4_ieee(w[2 * o], w[2 * o + 1], s, inv);
}

// Codes of NW packed bf16 words of a group whose abs-max bits are m (reduced over the
// group): s = fl(amax / 127), codes packed four per word, sum of the codes (dp4a
// against 0x01010101) -- the per-thread part of the per-token quantiser.
template <int NW>
__device__ __forceinline__ float quant_group_part(const uint32_t *w, uint32_t m, uint32_t *out, int &sum)
{
    const float s = div127_rn(__uint_as_float(m << 16));
    const bool live = m < 0x7f80u && s != 0.0f;
    const float inv = rcp_group(s);
    if (!quant_words_fast<NW>(w, inv, out) && live) quant_words_ieee<NW>(w, s, inv, out);
    sum = 0;
#pragma unroll
    for (int o = 0; o < NW / 2; ++o) {
        if (!live) out[o] = 0u;
        sum = __dp4a((int)out[o], 0x01010101, sum);
    }
    return live ? s : 0.0f;
}

// Quantise group (i, g): quad member `sub` holds elements 8 sub .. 8 sub + 7 as the
// packed bf16 words w4.  Stores its 8 codes and (sub 0) the group's {s, 8 sum q}.
// All 32 lanes call it (quad shuffles); `on` masks the stores of lanes past the end.
// q = clamp(round_half_away(fl(x / s)), -127, 127) with s = fl(amax / 127),
// bit-identical to quant_a8_kernel.
__device__ __forceinline__ void a8_quad_store(const uint32_t w4[4], bool on, int i, int g, int sub, int G,
                                              uint32_t K2, const ActSmem &L)
{
    uint32_t m = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) m = absmax_bits(m, w4[e]);
    m = absmax_fold(m);
    m = max(m, __shfl_xor_sync(0xffffffffu, m, 1));
    m = max(m, __shfl_xor_sync(0xffffffffu, m, 2));
    uint32_t q[2];
    int sum;
    const float s = quant_group_part<4>(w4, m, q, sum);
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    if (on) {
        // elements 8sub..8sub+7: sub 0/1 -> q_lo, sub 2/3 -> q_hi
        const uint32_t qt = L.act + (uint32_t)i * L.tsz + (sub < 2 ? 0u : K2) + 16u * g + 8u * (sub & 1);
        asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(qt), "r"(q[0]), "r"(q[1]) : "memory");
        if (sub == 0)
            asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(L.ssq + 8u * (uint32_t)(i * G + g)),
                         "r"(__float_as_uint(s)), "r"((uint32_t)(8 * sum))
                         : "memory");
    }
}

// Octet variant (one token): 8 threads per group, 4 elements each (elements 4 sub8 ..
// 4 sub8 + 3, packed bf16 words w2); the same per-element arithmetic as a8_quad_store,
// so the codes, s and sum q are bit-identical -- only the reduction tree spans 8 lanes.
__device__ __forceinline__ void a8_oct_store(uint2 w2, bool on, int g, int sub8, uint32_t K2, const ActSmem &L)
{
    uint32_t m = absmax_fold(absmax_bits(w2.x & 0x7fff7fffu, w2.y));
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    const uint32_t w[2] = {w2.x, w2.y};
    uint32_t q[1];
    int sum;
    const float s = quant_group_part<2>(w, m, q, sum);
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (on) {
        sts32(L.act + (sub8 < 4 ? 0u : K2) + 16u * g + 4u * (sub8 & 3), q[0]);
        if (sub8 == 0)
            asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(L.ssq + 8u * (uint32_t)g),
                         "r"(__float_as_uint(s)), "r"((uint32_t)(8 * sum))
                         : "memory");
    }
}

template <bool kCoherent>
__device__ __forceinline__ void stage_a8(const uint16_t *xg, int64_t ldx, int ntok, int64_t k, const ActSmem &L,
                                         int tid, int nthreads)
{
    const int G = (int)(k / 32);
    const uint32_t K2 = (uint32_t)(k / 2);
    const int nq = ntok * G * 4;
    for (int base = 0; base < nq; base += nthreads) {
        const int idx = base + tid;
        const bool on = idx < nq;
        const int grp = on ? (idx >> 2) : 0, sub = idx & 3;
        const int i = grp / G, g = grp - i * G;
        const uint4 u = ldg_x128<kCoherent>(xg + i * ldx + 32 * g + 8 * sub);
        const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
        a8_quad_store(w4, on, i, g, sub, G, K2, L);
    }
}

// W4A16 fragment-order store of x[4t..4t+3] (lo) and x[4t+16..4t+19] (hi) of group
// (tk, g) + corr[g][tk] = -136 * sum of the group (quad butterfly; all lanes call).
__device__ __forceinline__ void a16_quad_store(uint2 lo, uint2 hi, bool on, int tk, int g, int tt, const ActSmem &L)
{
    float part = 0.0f;
    const uint32_t e8[4] = {lo.x, lo.y, hi.x, hi.y};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        part += __uint_as_float(e8[e] << 16);
        part += __uint_as_float(e8[e] & 0xffff0000u);
    }
    part += __shfl_xor_sync(0xffffffffu, part, 1);
    part += __shfl_xor_sync(0xffffffffu, part, 2);
    if (on) {
        uint4 o;
        o.x = __byte_perm(lo.x, lo.y, 0x5410);
        o.y = __byte_perm(lo.x, lo.y, 0x7632);
        o.z = __byte_perm(hi.x, hi.y, 0x5410);
        o.w = __byte_perm(hi.x, hi.y, 0x7632);
        sts128(L.act + (uint32_t)tk * L.tsz + 64u * g + 16u * tt, o);
        if (tt == 0) sts32(L.corr + 4u * (uint32_t)(g * 8 + tk), __float_as_uint(-136.0f * part));
    }
}

// W4A16: x re-staged in MMA-fragment order + corr[g][tok] = -136 * sum of the group
// (fp32; this thread's 8 values in sequence, then the quad butterfly).
template <bool kCoherent>
__device__ __forceinline__ void stage_a16(const uint16_t *xg, int64_t ldx, int ntok, int64_t k, const ActSmem &L,
                                          int tid, int nthreads)
{
    const int G = (int)(k / 32);
    for (int idx = tid; idx < G * 8; idx += nthreads)     // tokens >= ntok: zero init
        if ((idx & 7) >= ntok) sts32(L.corr + 4u * (uint32_t)idx, 0u);
    const int nq = ntok * G * 4;
    for (int base = 0; base < nq; base += nthreads) {
        const int idx = base + tid;
        const bool on = idx < nq;
        const int q = on ? idx : 0;
        const int tk = q / (G * 4), rem = q - tk * G * 4, g = rem >> 2, tt = rem & 3;
        const uint16_t *src = xg + tk * ldx + 32 * g + 4 * tt;
        const uint2 lo = ldg_x64<kCoherent>(src);        // x[4t..4t+3]
        const uint2 hi = ldg_x64<kCoherent>(src + 16);   // x[4t+16..4t+19]
        a16_quad_store(lo, hi, on, tk, g, tt, L);
    }
}

// ---------------------------------------------------------------- per-stage compute
// DP4A (W4A8, 1 token): warp w owns row w of the 16-row tile; lane l the blocks l and
// l+32 of the chunk, in that order.  8 IDP.4A + deferred correction D = sumi - 8 sum_x
// + fp32 (d s) D per block.
__device__ __forceinline__ void chunk_dp4a(uint32_t st, int nblk, int blk0, uint32_t K2, const ActSmem &L, int warp,
                                           int lane, float &acc)
{
    const int r = warp;
    if (nblk == kChunkBlocks) {
        // full chunk: no predicates, both blocks' load/dp4a chains interleave
        const int g0 = blk0 + lane, g1 = g0 + 32;
        const uint4 w0 = lds128(st + nib_off(r, lane));
        const uint4 w1 = lds128(st + nib_off(r, lane + 32));
        const uint4 qa0 = lds128(L.act + 16u * g0), qb0 = lds128(L.act + K2 + 16u * g0);
        const uint4 qa1 = lds128(L.act + 16u * g1), qb1 = lds128(L.act + K2 + 16u * g1);
        const float d0 = h2f(lds16(st + scale_off(r, lane)));
        const float d1 = h2f(lds16(st + scale_off(r, lane + 32)));
        const uint2 p0 = lds64(L.ssq + 8u * g0), p1 = lds64(L.ssq + 8u * g1);
        const int D0 = block_D(w0, qa0, qb0, (int)p0.y);
        const int D1 = block_D(w1, qa1, qb1, (int)p1.y);
        acc = fmaf(d0 * __uint_as_float(p0.x), (float)D0, acc);
        acc = fmaf(d1 * __uint_as_float(p1.x), (float)D1, acc);
    } else {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int b = lane + 32 * h;
            if (b < nblk) {
                const int g = blk0 + b;
                const uint4 qa = lds128(L.act + 16u * g), qb = lds128(L.act + K2 + 16u * g);
                const uint4 w = lds128(st + nib_off(r, b));
                const uint2 p = lds64(L.ssq + 8u * g);
                const int D = block_D(w, qa, qb, (int)p.y);
                acc = fmaf(h2f(lds16(st + scale_off(r, b))) * __uint_as_float(p.x), (float)D, acc);
            }
        }
    }
}

// DUMP engine (test entry): chunk_dp4a's blocks and block_D, storing each block's D.
__device__ __forceinline__ void chunk_dump(uint32_t st, int nblk, int blk0, uint32_t K2, const ActSmem &L, int warp,
                                           int lane, int64_t row0, int64_t n, int G, int32_t *dump_d)
{
    const int r = warp;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int b = lane + 32 * h;
        if (b < nblk && row0 + r < n) {
            const int g = blk0 + b;
            const uint4 qa = lds128(L.act + 16u * g), qb = lds128(L.act + K2 + 16u * g);
            const uint4 w = lds128(st + nib_off(r, b));
            const uint2 p = lds64(L.ssq + 8u * g);
            dump_d[(row0 + r) * G + g] = block_D(w, qa, qb, (int)p.y);
        }
    }
}

// One lane's activation operands for two Q4_0 blocks (q words, {s, 8 sum q} pairs).
struct Dp4aAct {
    uint4 qa0, qb0, qa1, qb1;
    uint2 p0, p1;
};
// the two blocks (b0, b1) a lane of the step kernel's row-lane DP4A mapping meets in a
// chunk: q words and the {s, 8 sum q} pairs
__device__ __forceinline__ Dp4aAct dp4a_act_load_pair(const ActSmem &L, int b0, int b1, uint32_t K2)
{
    Dp4aAct r;
    r.qa0 = lds128(L.act + 16u * b0);
    r.qb0 = lds128(L.act + K2 + 16u * b0);
    r.qa1 = lds128(L.act + 16u * b1);
    r.qb1 = lds128(L.act + K2 + 16u * b1);
    r.p0 = lds64(L.ssq + 8u * b0);
    r.p1 = lds64(L.ssq + 8u * b1);
    return r;
}
// MMA engines: warp w owns blocks 4w..4w+3 of the chunk (contiguous, in that order)
// for all 16 rows; ldmatrix.x4 hands lane (gid, t) word t of rows gid / gid+8 of two
// blocks -- the m16n8k32.s8 / m16n8k16.bf16 A fragment of the split nibble layout.
//   IMMA  (W4A8, 2..8 tokens): one mma.sync per block -> exact int32 D, fp32 d s D.
//   HMMA  (W4A16, 2..8 tokens) / HMMA1 (1 token): A = 128 + c (exact bf16, one LOP3
//         per pair), two MMAs per block, D + corr restores sum (c - 8) x in fp32.
template <int E>
__device__ __forceinline__ void chunk_mma(uint32_t st, int nblk, int blk0, uint32_t K2, const ActSmem &L, int G,
                                          int ntok, int warp, int lane, uint32_t kNib2, uint32_t kMagic, float acc[4])
{
    const int gid = lane >> 2, t = lane & 3;
    const int mrow = (lane & 7) + ((lane >> 3) & 1) * 8;    // ldmatrix row of this lane
    const int mhalf = lane >> 4;                             // lanes 16-31 address the 2nd block
    const int bq = 4 * warp;
    if (bq >= nblk) return;
    uint32_t wv[8];   // [block j][row half]: wa(j) = wv[2j], wb(j) = wv[2j+1]
    ldmatrix_x4(st + nib_off(mrow, bq + mhalf), wv[0], wv[1], wv[2], wv[3]);
    ldmatrix_x4(st + nib_off(mrow, bq + 2 + mhalf), wv[4], wv[5], wv[6], wv[7]);
    // scales of rows gid / gid+8 for the 4 blocks: one 8-byte load each
    const uint2 sa = lds64(st + scale_off(gid, bq));
    const uint2 sbb = lds64(st + scale_off(gid + 8, bq));
    const float dA[4] = {h2f((uint16_t)(sa.x & 0xffff)), h2f((uint16_t)(sa.x >> 16)), h2f((uint16_t)(sa.y & 0xffff)),
                         h2f((uint16_t)(sa.y >> 16))};
    const float dB[4] = {h2f((uint16_t)(sbb.x & 0xffff)), h2f((uint16_t)(sbb.x >> 16)),
                         h2f((uint16_t)(sbb.y & 0xffff)), h2f((uint16_t)(sbb.y >> 16))};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t wa = wv[2 * j], wb = wv[2 * j + 1];
        const int g = blk0 + bq + j;
        if constexpr (E == IMMA) {
            uint32_t b0 = 0, b1 = 0;
            if (gid < ntok) {
                const uint32_t qt = L.act + (uint32_t)gid * L.tsz;
                b0 = lds32(qt + 16u * g + 4u * t);
                b1 = lds32(qt + K2 + 16u * g + 4u * t);
            }
            int c[4];
            imma(wa, wb, b0, b1, c);
            const int c0 = 2 * t, c1 = 2 * t + 1;
            const uint2 p0 = c0 < ntok ? lds64(L.ssq + 8u * (c0 * G + g)) : make_uint2(0u, 0u);
            const uint2 p1 = c1 < ntok ? lds64(L.ssq + 8u * (c1 * G + g)) : make_uint2(0u, 0u);
            const float s0 = __uint_as_float(p0.x), s1 = __uint_as_float(p1.x);
            acc[0] = fmaf(dA[j] * s0, (float)(c[0] - (int)p0.y), acc[0]);
            acc[1] = fmaf(dA[j] * s1, (float)(c[1] - (int)p1.y), acc[1]);
            acc[2] = fmaf(dB[j] * s0, (float)(c[2] - (int)p0.y), acc[2]);
            acc[3] = fmaf(dB[j] * s1, (float)(c[3] - (int)p1.y), acc[3]);
        } else {
            uint4 bx = make_uint4(0, 0, 0, 0);
            if (gid < ntok) bx = lds128(L.act + (uint32_t)gid * L.tsz + 64u * g + 16u * t);
            uint32_t pa[4], pb[4];
            magic_bf16(wa, kNib2, kMagic, pa);
            magic_bf16(wb, kNib2, kMagic, pb);
            float c[4];
            hmma_c(pa[0], pb[0], pa[2], pb[2], bx.x, bx.y, 0.f, 0.f, 0.f, 0.f, c);
            hmma(pa[1], pb[1], pa[3], pb[3], bx.z, bx.w, c);
            if constexpr (E == HMMA1) {
                // one token: only column 0 (lanes t == 0) is live
                const float crx = __uint_as_float(lds32(L.corr + 32u * g));
                acc[0] = fmaf(dA[j], c[0] + crx, acc[0]);
                acc[2] = fmaf(dB[j], c[2] + crx, acc[2]);
            } else {
                const uint2 cru = lds64(L.corr + 32u * g + 8u * t);
                const float crx = __uint_as_float(cru.x), cry = __uint_as_float(cru.y);
                acc[0] = fmaf(dA[j], c[0] + crx, acc[0]);
                acc[1] = fmaf(dA[j], c[1] + cry, acc[1]);
                acc[2] = fmaf(dB[j], c[2] + crx, acc[2]);
                acc[3] = fmaf(dB[j], c[3] + cry, acc[3]);
            }
        }
    }
}

// HMMA1 on a full chunk with the lane's loop-invariant shared-memory offsets computed once
// per kernel (the generic chunk_mma re-derives them every stage under the 60-register cap
// of two CTAs per SM).  Same loads, MMAs and fmaf order as chunk_mma<HMMA1>: bit-identical.
struct Hmma1Lane {
    uint32_t oa, ob;   // ldmatrix offsets in a stage: blocks bq + mhalf, bq + 2 + mhalf
    uint32_t sa, sb;   // scale offsets in a stage: rows gid / gid + 8, blocks bq .. bq + 3
    uint32_t xo;       // x of block bq, this lane's 16 B (token 0, lanes gid == 0)
    uint32_t co;       // corr of block bq
    bool xon;
};
__device__ __forceinline__ Hmma1Lane hmma1_lane(const ActSmem &L, int warp, int lane)
{
    const int gid = lane >> 2, t = lane & 3;
    const int mrow = (lane & 7) + ((lane >> 3) & 1) * 8, mhalf = lane >> 4;
    const int bq = 4 * warp;
    Hmma1Lane H;
    H.oa = nib_off(mrow, bq + mhalf);
    H.ob = nib_off(mrow, bq + 2 + mhalf);
    H.sa = scale_off(gid, bq);
    H.sb = scale_off(gid + 8, bq);
    H.xo = L.act + 64u * (uint32_t)bq + 16u * (uint32_t)t;
    H.co = L.corr + 32u * (uint32_t)bq;
    H.xon = gid == 0;
    return H;
}
// xo / co: the chunk's offsets (64 B of x and 32 B of corr per block of the chunk)
__device__ __forceinline__ void chunk_hmma1(uint32_t st, uint32_t xo, uint32_t co, const Hmma1Lane &H, uint32_t kNib2,
                                            uint32_t kMagic, float &acc0, float &acc2)
{
    uint32_t wv[8];
    ldmatrix_x4(st + H.oa, wv[0], wv[1], wv[2], wv[3]);
    ldmatrix_x4(st + H.ob, wv[4], wv[5], wv[6], wv[7]);
    const uint2 sa = lds64(st + H.sa);
    const uint2 sbb = lds64(st + H.sb);
    const float dA[4] = {h2f((uint16_t)(sa.x & 0xffff)), h2f((uint16_t)(sa.x >> 16)), h2f((uint16_t)(sa.y & 0xffff)),
                         h2f((uint16_t)(sa.y >> 16))};
    const float dB[4] = {h2f((uint16_t)(sbb.x & 0xffff)), h2f((uint16_t)(sbb.x >> 16)),
                         h2f((uint16_t)(sbb.y & 0xffff)), h2f((uint16_t)(sbb.y >> 16))};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        uint4 bx = make_uint4(0, 0, 0, 0);
        if (H.xon) bx = lds128(H.xo + xo + 64u * j);
        uint32_t pa[4], pb[4];
        magic_bf16(wv[2 * j], kNib2, kMagic, pa);
        magic_bf16(wv[2 * j + 1], kNib2, kMagic, pb);
        float c[4];
        hmma_c(pa[0], pb[0], pa[2], pb[2], bx.x, bx.y, 0.f, 0.f, 0.f, 0.f, c);
        hmma(pa[1], pb[1], pa[3], pb[3], bx.z, bx.w, c);
        const float crx = __uint_as_float(lds32(H.co + co + 32u * j));
        acc0 = fmaf(dA[j], c[0] + crx, acc0);
        acc2 = fmaf(dB[j], c[2] + crx, acc2);
    }
}

// ---------------------------------------------------------------- argmax keys (NEXT-2)
// A 64-bit key whose unsigned order is "larger fp32 value first, then smaller index":
// high word = the IEEE bits mapped to an unsigned total order (-0 folded onto +0, so
// equal values tie), low word = 0xffffffff - index.  max() over keys is exact and
// order-independent: any reduction tree gives the same argmax (first index on ties).
__device__ __forceinline__ unsigned long long argmax_key(float v, int64_t idx)
{
    uint32_t b = __float_as_uint(v);
    if (b == 0x80000000u) b = 0u;
    const uint32_t ord = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    return ((unsigned long long)ord << 32) | (unsigned long long)(0xffffffffu - (uint32_t)idx);
}
__device__ __forceinline__ float argmax_key_value(unsigned long long key)
{
    const uint32_t ord = (uint32_t)(key >> 32);
    return __uint_as_float((ord & 0x80000000u) ? (ord & 0x7fffffffu) : ~ord);
}

// ---------------------------------------------------------------- tile epilogues
// One output element: the local store, or (a8 fused epilogue) one store per LSA peer at
// its byte offset from the local address -- the local replica is one of them (delta 0).
__device__ __forceinline__ void store_out_peers(void *y, int ydt, int64_t idx, float v, const int64_t *delta,
                                                int npeers)
{
    if (npeers == 0) {
        dev::store_out(y, ydt, idx, v);
        return;
    }
    for (int p = 0; p < npeers; ++p) dev::store_out(reinterpret_cast<uint8_t *>(y) + delta[p], ydt, idx, v);
}

// DP4A: fixed xor butterfly; lane 0 of warp w stores row row0 + w.
__device__ __forceinline__ void epilogue_dp4a(float acc, int64_t row0, int64_t n, void *y, int ydt, int64_t off, int warp,
                                              int lane, const int64_t *delta = nullptr, int npeers = 0)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
        const int64_t row = row0 + warp;
        if (row < n) store_out_peers(y, ydt, off + row, acc, delta, npeers);
    }
}

// DP4A epilogue in greedy-decode mode: the same butterfly, the row's value folded into
// lane 0's running argmax key instead of stored
__device__ __forceinline__ void epilogue_dp4a_amax(float acc, int64_t row0, int64_t n, int64_t off, int warp, int lane,
                                                   unsigned long long &best)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    const int64_t row = row0 + warp;
    if (lane == 0 && row < n) {
        const unsigned long long key = argmax_key(acc, off + row);
        best = key > best ? key : best;
    }
}

// MMA: fixed-order cross-warp reduction through shared memory (red: 16 warps x 512 B).
// best != nullptr: greedy-decode mode (token 0's rows folded into a running argmax key).
__device__ __forceinline__ void epilogue_mma(const float acc[4], uint32_t red, int64_t row0, int64_t n, void *y,
                                             int ydt, int64_t ldy, int64_t tok0, int ntok, int warp, int lane,
                                             unsigned long long *best = nullptr, int64_t amax_off = 0,
                                             const int64_t *delta = nullptr, int npeers = 0)
{
    const int gid = lane >> 2, t = lane & 3;
    const uint32_t rw = red + 512u * warp;
    const int c0 = 2 * t, c1 = 2 * t + 1;
    sts32(rw + 4u * (gid * 8 + c0), __float_as_uint(acc[0]));
    sts32(rw + 4u * (gid * 8 + c1), __float_as_uint(acc[1]));
    sts32(rw + 4u * ((gid + 8) * 8 + c0), __float_as_uint(acc[2]));
    sts32(rw + 4u * ((gid + 8) * 8 + c1), __float_as_uint(acc[3]));
    bar_consumers();
    const int tid = warp * 32 + lane;
    if (tid < 128) {
        const int r = tid >> 3, tk = tid & 7;
        float sum = __uint_as_float(lds32(red + 4u * tid));
#pragma unroll
        for (int w = 1; w < kConsumerWarps; ++w) sum += __uint_as_float(lds32(red + 512u * w + 4u * tid));
        const int64_t row = row0 + r;
        if (best) {
            if (row < n && tk == 0) {
                const unsigned long long key = argmax_key(sum, amax_off + row);
                *best = key > *best ? key : *best;
            }
        } else if (row < n && tk < ntok) {
            store_out_peers(y, ydt, (tok0 + tk) * ldy + row, sum, delta, npeers);
        }
    }
    bar_consumers();
}
