// K3 round-function variants, one serial chain on one warp (the lookup's
// critical path): cycles per 64-round compression for each variant, and the
// final state (every variant must agree). Build + run on the box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_sha tools/microbench_sha.cu && /tmp/mb_sha
#include <cstdint>
#include <cstdio>

__constant__ uint32_t kK[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5, 0xd807aa98,
    0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174, 0xe49b69c1, 0xefbe4786,
    0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da, 0x983e5152, 0xa831c66d, 0xb00327c8,
    0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967, 0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13,
    0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85, 0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819,
    0xd6990624, 0xf40e3585, 0x106aa070, 0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a,
    0x5b9cca4f, 0x682e6ff3, 0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7,
    0xc67178f2};

__device__ __forceinline__ uint32_t rotr(uint32_t x, int n) { return __funnelshift_r(x, x, n); }
__device__ __forceinline__ uint32_t add_fixed(uint32_t x, uint32_t y) {
    uint32_t r;
    asm("add.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(y));
    return r;
}
__device__ __forceinline__ uint32_t add_fma(uint32_t x, uint32_t y) {  // IMAD pipe
    uint32_t r;
    asm("mad.lo.u32 %0, %1, 1, %2;" : "=r"(r) : "r"(x), "r"(y));
    return r;
}
__device__ __forceinline__ uint32_t rotr_fma(uint32_t x, int n) {  // x * 2^(32-n): hi | lo words
    const uint32_t m = 1u << (32 - n);
    uint32_t lo, hi;
    asm("mul.lo.u32 %0, %1, %2;" : "=r"(lo) : "r"(x), "r"(m));
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(hi) : "r"(x), "r"(m));
    return lo | hi;
}

// V0: round 1 (T1 = h + KW + S1 + Ch; e = d + T1)
__device__ __forceinline__ void c_v0(uint32_t h[8], const uint32_t* kw) {
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
#pragma unroll
    for (int t = 0; t < 64; ++t) {
        const uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
        const uint32_t ch = (e & f) ^ (~e & g);
        const uint32_t t1 = hh + kw[t] + S1 + ch;
        const uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
        const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + S0 + mj;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

// V1: Y/Yd prepared a round early (the product's compress_kw)
__device__ __forceinline__ void c_v1(uint32_t h[8], const uint32_t* kw) {
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    uint32_t y = hh + kw[0], yd = y + d;
#pragma unroll
    for (int t = 0; t < 64; ++t) {
        const uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
        const uint32_t ch = (e & f) ^ (~e & g);
        const uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
        const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        const uint32_t e_new = add_fixed(S1, add_fixed(ch, yd));
        const uint32_t t1 = add_fixed(S1, add_fixed(ch, y));
        const uint32_t a_new = add_fixed(t1, add_fixed(S0, mj));
        if (t + 1 < 64) { y = g + kw[t + 1]; yd = y + c; }
        hh = g; g = f; f = e; e = e_new; d = c; c = b; b = a; a = a_new;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

// V2: as V1, every add on the IMAD (FMA) pipe: the ALU pipe keeps only the
// 6 SHF + 4 LOP3 of a round
__device__ __forceinline__ void c_v2(uint32_t h[8], const uint32_t* kw) {
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    uint32_t y = add_fma(hh, kw[0]), yd = add_fma(y, d);
#pragma unroll
    for (int t = 0; t < 64; ++t) {
        const uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
        const uint32_t ch = (e & f) ^ (~e & g);
        const uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
        const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        const uint32_t e_new = add_fma(S1, add_fma(ch, yd));
        const uint32_t t1 = add_fma(S1, add_fma(ch, y));
        const uint32_t a_new = add_fma(t1, add_fma(S0, mj));
        if (t + 1 < 64) { y = add_fma(g, kw[t + 1]); yd = add_fma(y, c); }
        hh = g; g = f; f = e; e = e_new; d = c; c = b; b = a; a = a_new;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

// V3: V1 adds, and the off-path prepare (y, yd) on the FMA pipe only
__device__ __forceinline__ void c_v3(uint32_t h[8], const uint32_t* kw) {
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    uint32_t y = add_fma(hh, kw[0]), yd = add_fma(y, d);
#pragma unroll
    for (int t = 0; t < 64; ++t) {
        const uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
        const uint32_t ch = (e & f) ^ (~e & g);
        const uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
        const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        const uint32_t e_new = add_fixed(S1, add_fixed(ch, yd));
        const uint32_t t1 = add_fixed(S1, add_fixed(ch, y));
        const uint32_t a_new = add_fixed(t1, add_fixed(S0, mj));
        if (t + 1 < 64) { y = add_fma(g, kw[t + 1]); yd = add_fma(y, c); }
        hh = g; g = f; f = e; e = e_new; d = c; c = b; b = a; a = a_new;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

// V4: V2 with Maj and Ch written to stay single LOP3s, Sigma0's three
// rotates on the FMA pipe (IMAD.HI | IMAD.LO); Sigma1 stays on the ALU pipe
__device__ __forceinline__ void c_v4(uint32_t h[8], const uint32_t* kw) {
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    uint32_t y = add_fma(hh, kw[0]), yd = add_fma(y, d);
#pragma unroll
    for (int t = 0; t < 64; ++t) {
        const uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
        const uint32_t ch = (e & f) ^ (~e & g);
        const uint32_t S0 = rotr_fma(a, 2) ^ rotr_fma(a, 13) ^ rotr_fma(a, 22);
        const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        const uint32_t e_new = add_fma(S1, add_fma(ch, yd));
        const uint32_t t1 = add_fma(S1, add_fma(ch, y));
        const uint32_t a_new = add_fma(t1, add_fma(S0, mj));
        if (t + 1 < 64) { y = add_fma(g, kw[t + 1]); yd = add_fma(y, c); }
        hh = g; g = f; f = e; e = e_new; d = c; c = b; b = a; a = a_new;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

template <int N>
__device__ __forceinline__ uint32_t shr_(uint32_t x) {
    uint32_t r;
    asm("shr.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "n"(N));
    return r;
}
template <int N>
__device__ __forceinline__ uint32_t shl_(uint32_t x) {
    uint32_t r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "n"(N));
    return r;
}
template <int N>
__device__ __forceinline__ uint32_t shl_fma(uint32_t x) {  // x * 2^N on the FMA pipe
    uint32_t r;
    asm("mul.lo.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "n"(1u << N));
    return r;
}
__device__ __forceinline__ uint32_t xor3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
// Sigma from six disjoint shifted halves: the halves of each rotate share no
// bits, so the whole Sigma is the XOR of the six shifts.
template <int A, int B, int C, bool FMA>
__device__ __forceinline__ uint32_t sigma_shifts(uint32_t x) {
    const uint32_t l0 = FMA ? shl_fma<32 - A>(x) : shl_<32 - A>(x);
    const uint32_t l1 = FMA ? shl_fma<32 - B>(x) : shl_<32 - B>(x);
    const uint32_t l2 = FMA ? shl_fma<32 - C>(x) : shl_<32 - C>(x);
    return xor3(xor3(shr_<A>(x), shr_<B>(x), shr_<C>(x)), l0, l1 ^ l2);
}

template <bool FMA>
__device__ __forceinline__ void c_v56(uint32_t h[8], const uint32_t* kw) {
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    uint32_t y = add_fma(hh, kw[0]), yd = add_fma(y, d);
#pragma unroll
    for (int t = 0; t < 64; ++t) {
        const uint32_t S1 = sigma_shifts<6, 11, 25, FMA>(e);
        const uint32_t ch = (e & f) ^ (~e & g);
        const uint32_t S0 = sigma_shifts<2, 13, 22, FMA>(a);
        const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        const uint32_t e_new = add_fixed(S1, add_fixed(ch, yd));
        const uint32_t t1 = add_fixed(S1, add_fixed(ch, y));
        const uint32_t a_new = add_fixed(t1, add_fixed(S0, mj));
        if (t + 1 < 64) { y = add_fma(g, kw[t + 1]); yd = add_fma(y, c); }
        hh = g; g = f; f = e; e = e_new; d = c; c = b; b = a; a = a_new;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

// V7: V1 with Sigma1 on funnel shifts and Sigma0 from shifts (left halves on
// the FMA pipe): splits the rotate work across both pipes
__device__ __forceinline__ void c_v7(uint32_t h[8], const uint32_t* kw) {
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    uint32_t y = add_fma(hh, kw[0]), yd = add_fma(y, d);
#pragma unroll
    for (int t = 0; t < 64; ++t) {
        const uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
        const uint32_t ch = (e & f) ^ (~e & g);
        const uint32_t S0 = sigma_shifts<2, 13, 22, true>(a);
        const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        const uint32_t e_new = add_fixed(S1, add_fixed(ch, yd));
        const uint32_t t1 = add_fixed(S1, add_fixed(ch, y));
        const uint32_t a_new = add_fixed(t1, add_fixed(S0, mj));
        if (t + 1 < 64) { y = add_fma(g, kw[t + 1]); yd = add_fma(y, c); }
        hh = g; g = f; f = e; e = e_new; d = c; c = b; b = a; a = a_new;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

// V8: every add as IMAD with a multiplier the compiler cannot see is 1
// (ptxas folds `mad.lo x, 1, y` back into an ALU-pipe IADD3): the ALU pipe
// keeps only the 6 SHF + 4 LOP3, the adds go to the FMA pipe
__device__ __forceinline__ uint32_t add_rt(uint32_t x, uint32_t one, uint32_t y) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(one), "r"(y));
    return r;
}
__device__ __forceinline__ void c_v8(uint32_t h[8], const uint32_t* kw, uint32_t one) {
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    uint32_t y = add_rt(hh, one, kw[0]), yd = add_rt(y, one, d);
#pragma unroll
    for (int t = 0; t < 64; ++t) {
        const uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
        const uint32_t ch = (e & f) ^ (~e & g);
        const uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
        const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        const uint32_t e_new = add_rt(S1, one, add_rt(ch, one, yd));
        const uint32_t t1 = add_rt(S1, one, add_rt(ch, one, y));
        const uint32_t a_new = add_rt(t1, one, add_rt(S0, one, mj));
        if (t + 1 < 64) { y = add_rt(g, one, kw[t + 1]); yd = add_rt(y, one, c); }
        hh = g; g = f; f = e; e = e_new; d = c; c = b; b = a; a = a_new;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

// V9: V1, but only the e-chain adds on the ALU pipe (IADD3 e = S1 + ch + Yd)
// and everything else on the FMA pipe
__device__ __forceinline__ void c_v9(uint32_t h[8], const uint32_t* kw, uint32_t one) {
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    uint32_t y = add_rt(hh, one, kw[0]), yd = add_rt(y, one, d);
#pragma unroll
    for (int t = 0; t < 64; ++t) {
        const uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
        const uint32_t ch = (e & f) ^ (~e & g);
        const uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
        const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        const uint32_t e_new = add_fixed(S1, add_fixed(ch, yd));
        const uint32_t t1 = add_rt(S1, one, add_rt(ch, one, y));
        const uint32_t a_new = add_rt(t1, one, add_rt(S0, one, mj));
        if (t + 1 < 64) { y = add_rt(g, one, kw[t + 1]); yd = add_rt(y, one, c); }
        hh = g; g = f; f = e; e = e_new; d = c; c = b; b = a; a = a_new;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

// V10: the a chain rebuilt on e_{t+1}: T1 = e_{t+1} - d_t, so
//   e_{t+1} = Sigma1(e_t) + (Ch + Yd_t)          Yd_t = h_t + KW_t + d_t, off the chains
//   a_{t+1} = Sigma0(a_t) + (e_{t+1} + (Maj - d_t))
// each chain is SHF -> LOP3 -> one add per round and a trails e by one add;
// every add on the FMA pipe (runtime multiplier), the ALU pipe keeps the
// 6 SHF + 4 LOP3 (20-cycle issue bound)
__device__ __forceinline__ uint32_t wide_rot(uint32_t x, uint32_t m) {  // rotr via IMAD.WIDE + IMAD
    const uint64_t p = uint64_t(x) * m;
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(uint32_t(p)), "r"(1u), "r"(uint32_t(p >> 32)));
    return r;
}
template <int MODE>
__device__ __forceinline__ void c_v10(uint32_t h[8], const uint32_t* kw, uint32_t one) {
    const uint32_t mone = 0u - one;  // -1, opaque to ptxas
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    uint32_t yd = add_rt(add_rt(hh, one, kw[0]), one, d);
#pragma unroll
    for (int t = 0; t < 64; ++t) {
        uint32_t S1, S0;
        if (MODE == 3) S1 = rotr(e, 6) ^ rotr(e, 11) ^ wide_rot(e, one << 7);  // rotr25 = x * 2^7
        else S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
        if (MODE == 2 || MODE == 3) S0 = rotr(a, 2) ^ rotr(a, 13) ^ wide_rot(a, one << 10);  // rotr22
        else S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
        const uint32_t ch = (e & f) ^ (~e & g);
        const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        const uint32_t mjd = add_rt(d, mone, mj);
        uint32_t e_new;
        if (MODE == 1) e_new = S1 + ch + yd;  // one ALU IADD3
        else e_new = add_rt(S1, one, add_rt(ch, one, yd));
        const uint32_t a_new = add_rt(S0, one, add_rt(e_new, one, mjd));
        if (t + 1 < 64) yd = add_rt(add_rt(g, one, kw[t + 1]), one, c);
        hh = g; g = f; f = e; e = e_new; d = c; c = b; b = a; a = a_new;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

// V14: two lanes per chain. Lane E (even) runs the e chain, lane A (odd) the
// a chain one round behind; one instruction stream computes Sigma1(e_s) in E
// and Sigma0(a_{s-1}) in A (per-lane rotate counts), Ch in E and Maj in A,
// and one SHFL.BFLY per round trades e_{s+1} (A turns it into T1 = e - d)
// for a_s (E queues it as the d of round s+3).
__device__ __forceinline__ void c_v14(uint32_t hs[8], const uint32_t* kw_lane, uint32_t one) {
    const bool A = threadIdx.x & 1;
    const uint32_t r0 = A ? 2 : 6, r1 = A ? 13 : 11, r2 = A ? 22 : 25;
    const uint32_t msk = A ? ~0u : 0u;
    // E: x = (e, f, g, h); A before round 0: x = (b, c, d, -), a0 injected at round 0
    uint32_t x0 = A ? hs[1] : hs[4], x1 = A ? hs[2] : hs[5], x2 = A ? hs[3] : hs[6], x3 = A ? 0u : hs[7];
    const uint32_t a0 = hs[0];
    // d queue (E): after round s's push, q = (a_{s-3}, a_{s-2}, a_{s-1}, a_s);
    // before round 0: a_{-3}, a_{-2}, a_{-1} = d, c, b of the input state
    uint32_t q0 = 0, q1 = hs[3], q2 = hs[2], q3 = hs[1];
    // P for round 0: E: h + KW_0 + d_0; A: unused (its round 0 result is replaced by a0)
    uint32_t P = x3 + kw_lane[0] + hs[3];
    uint32_t fe0 = 0, fe1 = 0, fe2 = 0, fe3 = 0;
#pragma unroll
    for (int s = 0; s <= 64; ++s) {
        const uint32_t S = __funnelshift_r(x0, x0, r0) ^ __funnelshift_r(x0, x0, r1) ^ __funnelshift_r(x0, x0, r2);
        const uint32_t chv = (x0 & x1) ^ (~x0 & x2);
        const uint32_t mjv = (x0 & x1) ^ (x0 & x2) ^ (x1 & x2);
        const uint32_t cm = (chv & ~msk) | (mjv & msk);
        uint32_t nw = add_rt(S, one, add_rt(cm, one, P));
        if (s == 0) nw = A ? a0 : nw;
        if (s == 64) { fe0 = x0; fe1 = x1; fe2 = x2; fe3 = x3; }
        const uint32_t rv = __shfl_xor_sync(0xffffffffu, nw, 1);
        // shift the history
        x3 = x2; x2 = x1; x1 = x0; x0 = nw;
        // d queue (E): rv = a_s arrives; d_{s+1} = a_{s-2} = q1
        q0 = q1; q1 = q2; q2 = q3; q3 = rv;
        if (s + 1 <= 64) {
            // E: P = h_{s+1} + KW_{s+1} + d_{s+1};  A: P = e_{s+1} - d_s (T1_s), d_s = a_{s-3} = x3 (after shift)
            const uint32_t kwn = kw_lane[s + 1 < 64 ? s + 1 : 63];
            const uint32_t u = A ? rv : x3;
            const uint32_t w = A ? (0u - x3) : q1;
            P = u + kwn + w;
        }
    }
    // E: e f g h = fe0..fe3 (before round 64's shift); A: a b c d = x0..x3
    const uint32_t s0 = A ? x0 : fe0, s1 = A ? x1 : fe1, s2 = A ? x2 : fe2, s3 = A ? x3 : fe3;
    const uint32_t o0 = __shfl_xor_sync(0xffffffffu, s0, 1), o1 = __shfl_xor_sync(0xffffffffu, s1, 1);
    const uint32_t o2 = __shfl_xor_sync(0xffffffffu, s2, 1), o3 = __shfl_xor_sync(0xffffffffu, s3, 1);
    const uint32_t aa = A ? s0 : o0, bb = A ? s1 : o1, cc = A ? s2 : o2, dd = A ? s3 : o3;
    const uint32_t ee = A ? o0 : s0, ff = A ? o1 : s1, gg = A ? o2 : s2, hh = A ? o3 : s3;
    hs[0] += aa; hs[1] += bb; hs[2] += cc; hs[3] += dd; hs[4] += ee; hs[5] += ff; hs[6] += gg; hs[7] += hh;
}

// V15: V14 with lane A two rounds behind lane E: both transfers of the
// per-round SHFL.BFLY (e_{s+1} to A, a_{s-1} to E) get one round of slack,
// the lane-dependent sign of the d / T1 term is an IMAD with a per-lane +-1
// (no select), Ch / Maj picked with one LOP3 against a lane mask.
__device__ __forceinline__ void c_v15(uint32_t hs[8], const uint32_t* kw_lane, uint32_t one) {
    const bool A = threadIdx.x & 1;
    const uint32_t r0 = A ? 2 : 6, r1 = A ? 13 : 11, r2 = A ? 22 : 25;
    const uint32_t msk = A ? ~0u : 0u;
    const uint32_t sgn = A ? (0u - one) : one;  // x3 enters P with + (E) or - (A)
    // E: x = (e, f, g, h) = (e_0, e_-1, e_-2, e_-3).
    // A before round 0: x = (a_-2, a_-3, a_-4, a_-5); rounds 0 and 1 inject a_-1 (= b) and a_0 (= a).
    // a_-k for k = 1..3 are b, c, d; a_-4, a_-5 never enter a result (A's rounds 0, 1 are replaced).
    uint32_t x0 = A ? hs[2] : hs[4], x1 = A ? hs[3] : hs[5], x2 = A ? 0u : hs[6], x3 = A ? 0u : hs[7];
    // rv_prev: the value received one round earlier. E's P for round 0 / 1 needs
    // d_0 = a_-3 = d and d_1 = a_-2 = c, which no round delivers: seeded.
    uint32_t P = x3 + kw_lane[0] + hs[3];  // E: h_0 + KW_0 + d_0 (A: unused, round 0 replaced)
    uint32_t rv_prev = 0, rv = 0;
    uint32_t fe0 = 0, fe1 = 0, fe2 = 0, fe3 = 0;
#pragma unroll
    for (int s = 0; s <= 65; ++s) {
        const uint32_t S = __funnelshift_r(x0, x0, r0) ^ __funnelshift_r(x0, x0, r1) ^ __funnelshift_r(x0, x0, r2);
        const uint32_t chv = (x0 & x1) ^ (~x0 & x2);
        const uint32_t mjv = (x0 & x1) ^ (x0 & x2) ^ (x1 & x2);
        const uint32_t cm = (chv & ~msk) | (mjv & msk);
        uint32_t nw = S + cm + P;
        if (s == 0) nw = A ? hs[1] : nw;  // a_-1
        if (s == 1) nw = A ? hs[0] : nw;  // a_0
        if (s == 64) { fe0 = x0; fe1 = x1; fe2 = x2; fe3 = x3; }
        rv_prev = rv;
        rv = __shfl_xor_sync(0xffffffffu, nw, 1);  // E gets a_{s-1}, A gets e_{s+1}
        x3 = x2; x2 = x1; x1 = x0; x0 = nw;
        // P for round s + 1:
        //   E: h_{s+1} + KW_{s+1} + d_{s+1},  h = x3 (= e_{s-2}), d_{s+1} = a_{s-2} = rv_prev
        //   A: e_s - d_{s-1} (= T1_{s-1}, for a_s),  e_s = rv_prev, d_{s-1} = a_{s-4} = x3
        // with A's round s computing a_{s-1}: its history after the shift is
        // (a_{s-1}, a_{s-2}, a_{s-3}, a_{s-4}), so T1 for round s + 1 (a_s) is
        // e_s - a_{s-4}.
        uint32_t dE = rv_prev;
        if (s == 0 && !A) dE = hs[2];  // E: d_1 = a_-2 = c (no round delivered it)
        const uint32_t kwn = kw_lane[s + 1 < 64 ? s + 1 : 63];
        P = add_rt(x3, sgn, add_rt(dE, one, kwn));
    }
    // E: e f g h = fe0..fe3 (state before round 64's shift); A: a b c d after round 65
    const uint32_t s0 = A ? x0 : fe0, s1 = A ? x1 : fe1, s2 = A ? x2 : fe2, s3 = A ? x3 : fe3;
    const uint32_t o0 = __shfl_xor_sync(0xffffffffu, s0, 1), o1 = __shfl_xor_sync(0xffffffffu, s1, 1);
    const uint32_t o2 = __shfl_xor_sync(0xffffffffu, s2, 1), o3 = __shfl_xor_sync(0xffffffffu, s3, 1);
    hs[0] += A ? s0 : o0; hs[1] += A ? s1 : o1; hs[2] += A ? s2 : o2; hs[3] += A ? s3 : o3;
    hs[4] += A ? o0 : s0; hs[5] += A ? o1 : s1; hs[6] += A ? o2 : s2; hs[7] += A ? o3 : s3;
}

// op throughput / latency probes (one warp): 8 independent chains (rt) or
// one dependent chain (lat) of the same op
template <int OP, bool DEP>
__global__ void opbench(uint32_t seed, int iters, uint32_t* out, long long* cycles) {
    uint32_t x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = seed * (i + 3) + threadIdx.x;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int j = DEP ? 0 : i;
            if (OP == 0) x[j] = __funnelshift_r(x[j], x[j], 7);
            if (OP == 1) x[j] = shr_<7>(x[j]) ^ seed;
            if (OP == 2) x[j] = xor3(x[j], seed, 0x1234567u);
            if (OP == 3) x[j] = add_fixed(x[j], seed);
            if (OP == 4) x[j] = add_fma(x[j], seed);
            if (OP == 5) x[j] = shl_fma<7>(x[j]) ^ seed;
        }
    }
    const long long t1 = clock64();
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r ^= x[i];
    out[threadIdx.x] = r;
    if (threadIdx.x == 0) *cycles = t1 - t0;
}

template <int V>
__global__ void bench(const uint32_t* kw_g, int blocks, uint32_t* out, long long* cycles, uint32_t one) {
    __shared__ uint32_t kw[64], kwz[64];
    for (int i = threadIdx.x; i < 64; i += 32) { kw[i] = kw_g[i] + kK[i]; kwz[i] = 0; }
    __syncwarp();
    uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a, 0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    const long long t0 = clock64();
    for (int b = 0; b < blocks; ++b) {
        if (V == 0) c_v0(h, kw);
        if (V == 1) c_v1(h, kw);
        if (V == 2) c_v2(h, kw);
        if (V == 3) c_v3(h, kw);
        if (V == 4) c_v4(h, kw);
        if (V == 5) c_v56<false>(h, kw);
        if (V == 6) c_v56<true>(h, kw);
        if (V == 7) c_v7(h, kw);
        if (V == 8) c_v8(h, kw, one);
        if (V == 9) c_v9(h, kw, one);
        if (V >= 10 && V <= 13) c_v10<V - 10>(h, kw, one);
        if (V == 14) c_v14(h, (threadIdx.x & 1) ? kwz : kw, one);
        if (V == 15) c_v15(h, (threadIdx.x & 1) ? kwz : kw, one);
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) out[i] = h[i];
        *cycles = t1 - t0;
    }
}

int main() {
    uint32_t hw[64];
    for (int i = 0; i < 64; ++i) hw[i] = 0x9e3779b9u * (i + 1);
    uint32_t *kw, *out;
    long long* cyc;
    cudaMalloc(&kw, 256);
    cudaMalloc(&out, 32);
    cudaMalloc(&cyc, 8);
    cudaMemcpy(kw, hw, 256, cudaMemcpyHostToDevice);
    const int blocks = 2000;
    uint32_t ref[8] = {};
    for (int v = 0; v < 16; ++v) {
        for (int rep = 0; rep < 2; ++rep) {
            switch (v) {
                case 0: bench<0><<<1, 32>>>(kw, blocks, out, cyc, 1u); break;
                case 1: bench<1><<<1, 32>>>(kw, blocks, out, cyc, 1u); break;
                case 2: bench<2><<<1, 32>>>(kw, blocks, out, cyc, 1u); break;
                case 3: bench<3><<<1, 32>>>(kw, blocks, out, cyc, 1u); break;
                case 4: bench<4><<<1, 32>>>(kw, blocks, out, cyc, 1u); break;
                case 5: bench<5><<<1, 32>>>(kw, blocks, out, cyc, 1u); break;
                case 6: bench<6><<<1, 32>>>(kw, blocks, out, cyc, 1u); break;
                case 7: bench<7><<<1, 32>>>(kw, blocks, out, cyc, 1u); break;
                case 8: bench<8><<<1, 32>>>(kw, blocks, out, cyc, 1u); break;
                case 9: bench<9><<<1, 32>>>(kw, blocks, out, cyc, 1u); break;
                case 10: bench<10><<<1, 32>>>(kw, blocks, out, cyc, 1u); break;
                case 11: bench<11><<<1, 32>>>(kw, blocks, out, cyc, 1u); break;
                case 12: bench<12><<<1, 32>>>(kw, blocks, out, cyc, 1u); break;
                case 13: bench<13><<<1, 32>>>(kw, blocks, out, cyc, 1u); break;
                case 14: bench<14><<<1, 32>>>(kw, blocks, out, cyc, 1u); break;
                case 15: bench<15><<<1, 32>>>(kw, blocks, out, cyc, 1u); break;
            }
        }
        uint32_t h[8];
        long long c = 0;
        cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        if (v == 0)
            for (int i = 0; i < 8; ++i) ref[i] = h[i];
        bool same = true;
        for (int i = 0; i < 8; ++i) same &= h[i] == ref[i];
        printf("{\"variant\": %d, \"cycles_per_block\": %.1f, \"cycles_per_round\": %.2f, \"same_state\": %s}\n", v,
               double(c) / blocks, double(c) / blocks / 64, same ? "true" : "false");
    }
    const char* names[] = {"SHF.R.W funnel", "SHR+xor", "LOP3", "add (IADD)", "mad.lo (IMAD)", "mul.lo shl+xor"};
    uint32_t* o2;
    cudaMalloc(&o2, 128);
    const int iters = 4096;
    auto run = [&](auto kern, int op, bool dep) {
        kern<<<1, 32>>>(12345u, iters, o2, cyc);
        kern<<<1, 32>>>(12345u, iters, o2, cyc);
        long long c = 0;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("{\"op\": \"%s\", \"%s\": %.2f}\n", names[op], dep ? "cycles_dependent" : "cycles_per_instr_8way",
               double(c) / (iters * 8.0));
    };
    run(opbench<0, false>, 0, false); run(opbench<0, true>, 0, true);
    run(opbench<1, false>, 1, false); run(opbench<1, true>, 1, true);
    run(opbench<2, false>, 2, false); run(opbench<2, true>, 2, true);
    run(opbench<3, false>, 3, false); run(opbench<3, true>, 3, true);
    run(opbench<4, false>, 4, false); run(opbench<4, true>, 4, true);
    run(opbench<5, false>, 5, false); run(opbench<5, true>, 5, true);
    return 0;
}
