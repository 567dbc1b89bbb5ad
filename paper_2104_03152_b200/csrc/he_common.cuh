// he_common.cuh — device-side modular arithmetic, Philox and samplers for the
// B200 CKKS path.  Product code (independent of oracle/).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace he {

typedef uint64_t u64;
typedef uint32_t u32;
typedef int64_t i64;

// Per-prime constants read by every kernel (one 64-byte record per prime).
struct __align__(16) PrimeD {
  u64 q;       // the prime
  u64 two_q;   // 2q (lazy-reduction bound)
  u64 mu;      // Barrett: floor(2^{2k} / q)
  u64 ninv;    // N^{-1} mod q
  u64 ninvsh;  // floor(ninv 2^64 / q)
  u32 k;       // bit length of q
  u32 pad0;
  u64 mu64;    // floor(2^64 / q)
  u64 r64;     // 2^64 mod q
};

__device__ __forceinline__ PrimeD load_prime(const PrimeD* p, int i) {
  PrimeD r;
  const ulonglong2* s = reinterpret_cast<const ulonglong2*>(p + i);
  ulonglong2 a = __ldg(s), b = __ldg(s + 1), c = __ldg(s + 2);
  ulonglong2 d = __ldg(s + 3);
  r.q = a.x; r.two_q = a.y; r.mu = b.x; r.ninv = b.y; r.ninvsh = c.x; r.k = (u32)c.y;
  r.mu64 = d.x; r.r64 = d.y;
  return r;
}

// ---------------------------------------------------------------- modular ---
__device__ __forceinline__ u64 add_mod(u64 a, u64 b, u64 q) {
  u64 s = a + b;
  return s >= q ? s - q : s;
}
__device__ __forceinline__ u64 sub_mod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }
__device__ __forceinline__ u64 neg_mod(u64 a, u64 q) { return a ? q - a : 0; }

// Barrett reduction of a 128-bit x = (hi, lo) < 2^{2k} (HAC 14.42, base 2):
// q1 = x >> (k-1), q3 = (q1 mu) >> (k+1), r = x - q3 q in [0, 3q).
__device__ __forceinline__ u64 barrett128(u64 lo, u64 hi, u64 q, u64 mu, u32 k) {
  const u64 q1 = (lo >> (k - 1)) | (hi << (65 - k));
  const u64 l2 = q1 * mu, h2 = __umul64hi(q1, mu);
  const u64 q3 = (l2 >> (k + 1)) | (h2 << (63 - k));
  u64 r = lo - q3 * q;
  r = r >= q ? r - q : r;
  return r >= q ? r - q : r;
}
// Barrett for q < 2^31 (k <= 31) and x = a b < 2^{2k}: the same HAC 14.42
// steps with every intermediate in one 32x32->64 multiply.
__device__ __forceinline__ u64 barrett_small(u64 x, u64 q, u64 mu, u32 k) {
  const u32 q1 = (u32)(x >> (k - 1));
  const u32 q3 = (u32)(((u64)q1 * (u32)mu) >> (k + 1));
  u64 r = x - (u64)q3 * (u32)q;
  r = r >= q ? r - q : r;
  return r >= q ? r - q : r;
}
// a * b mod q for a, b < q.
__device__ __forceinline__ u64 mul_mod(u64 a, u64 b, const PrimeD& P) {
  if (P.k <= 31) return barrett_small((u64)(u32)a * (u32)b, P.q, P.mu, P.k);
  return barrett128(a * b, __umul64hi(a, b), P.q, P.mu, P.k);
}
// Reduce any 64-bit word mod q: qh = floor(x mu64 / 2^64) >= floor(x/q) - 2,
// so x - qh q is in [0, 3q).
__device__ __forceinline__ u64 reduce64(u64 x, const PrimeD& P) {
  u64 r = x - __umul64hi(x, P.mu64) * P.q;
  r = r >= P.q ? r - P.q : r;
  return r >= P.q ? r - P.q : r;
}
// x mod q for x < 2^32 and q < 2^31: q_hat = umulhi(x, floor(2^32 / q)) >= floor(x/q) - 1,
// so one conditional subtraction (as an unsigned min) finishes.
__device__ __forceinline__ u64 reduce32(u32 x, const PrimeD& P) {
  const u32 q = (u32)P.q, mu32 = (u32)(P.mu64 >> 32);
  const u32 r = x - __umulhi(x, mu32) * q;
  return min(r, r - q);
}
// Shoup: x * w mod q in [0, 2q) for any 64-bit x, w < q, wsh = floor(w 2^64 / q).
__device__ __forceinline__ u64 mul_shoup_lazy(u64 x, u64 w, u64 wsh, u64 q) {
  return x * w - __umul64hi(x, wsh) * q;
}
__device__ __forceinline__ u64 mul_shoup(u64 x, u64 w, u64 wsh, u64 q) {
  u64 r = mul_shoup_lazy(x, w, wsh, q);
  return r >= q ? r - q : r;
}
// Signed small integer -> residue.
__device__ __forceinline__ u64 from_signed(i64 v, const PrimeD& P) {
  if (v >= 0) return reduce64((u64)v, P);
  u64 r = reduce64((u64)(-v), P);
  return r ? P.q - r : 0;
}
// C16 centered lift of a residue of q_j, then reduction into prime t.
__device__ __forceinline__ u64 lift_centered(u64 r, u64 qj, const PrimeD& T) {
  if (r <= (qj - 1) / 2) return r >= T.q ? reduce64(r, T) : r;
  const u64 m = qj - r;  // |D| with D = r - qj < 0
  const u64 red = m >= T.q ? reduce64(m, T) : m;
  return red ? T.q - red : 0;
}

// C16 centered lift of r < q_j into q_t with 32-bit arithmetic (q_j, q_t < 2^31):
// [r]_t or q_t - [q_j - r]_t, each reduced by one umulhi Barrett (mut = floor(2^32 / q_t)).
__device__ __forceinline__ u32 lift32(u32 r, u32 qj, u32 qt, u32 mut) {
  const bool neg = r > (qj - 1) / 2;
  const u32 m = neg ? qj - r : r;
  const u32 v = min(m - __umulhi(m, mut) * qt, m - __umulhi(m, mut) * qt - qt);
  return neg ? (v ? qt - v : 0u) : v;
}

// C8/a8: NTT-domain automorphism index.  out[j] = in[pi_g(j)] with
// 2 brv(pi_g(j)) + 1 = g (2 brv(j) + 1) mod 2N.
__device__ __forceinline__ u32 brv_bits(u32 x, int logN) { return __brev(x) >> (32 - logN); }
__device__ __forceinline__ u32 galois_src(u32 j, u32 g, int logN) {
  const u32 mask2N = (2u << logN) - 1;
  const u32 e = 2u * brv_bits(j, logN) + 1u;
  const u32 e2 = (u32)(((u64)g * e) & mask2N);
  return brv_bits((e2 - 1u) >> 1, logN);
}

// ---------------------------------------------------------------- Philox ---
// Philox4x32-10 (Salmon et al. 2011) written from its round function; C9
// counter = (block_lo, block_hi, sid_lo, sid_hi), key = (seed_lo, seed_hi).
__device__ __forceinline__ uint4 philox10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const u32 lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const u32 lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}
__device__ __forceinline__ uint4 philox_block(u64 seed, u64 sid, u64 block) {
  return philox10(make_uint4((u32)block, (u32)(block >> 32), (u32)sid, (u32)(sid >> 32)),
                  make_uint2((u32)seed, (u32)(seed >> 32)));
}
__device__ __forceinline__ u32 uint4_at(const uint4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

// C9 stream id
enum Purpose : u64 {
  PUR_S = 1, PUR_PK_A = 2, PUR_PK_E = 3, PUR_RLK_A = 4, PUR_RLK_E = 5,
  PUR_GK_A = 6, PUR_GK_E = 7, PUR_ENC_V = 8, PUR_ENC_E0 = 9, PUR_ENC_E1 = 10,
  PUR_SYM_A = 11, PUR_SYM_E = 12   // symmetric encryption: a from a public seed, e from the context seed
};
__host__ __device__ __forceinline__ u64 stream_sid(u64 purpose, u64 object, u64 prime) {
  return (purpose << 56) | (object << 16) | prime;
}

// C10 ternary coefficient n: block n/4, word n%4, t = (w 3) >> 32, value t-1.
__device__ __forceinline__ i64 sample_ternary(u64 seed, u64 sid, u32 n) {
  const uint4 b = philox_block(seed, sid, n >> 2);
  const u32 w = uint4_at(b, n & 3);
  return (i64)(((u64)w * 3u) >> 32) - 1;
}
// C11 CDT coefficient n: block n/2, u = w[2h+1] << 32 | w[2h] (h = n%2);
// bit 63 = sign, magnitude = smallest k with (u mod 2^63) < T[k].
__device__ __forceinline__ i64 sample_cdt(u64 seed, u64 sid, u32 n, const u64* T) {
  const uint4 b = philox_block(seed, sid, n >> 1);
  const int h = n & 1;
  const u64 u = ((u64)uint4_at(b, 2 * h + 1) << 32) | uint4_at(b, 2 * h);
  const u64 mag = u & 0x7fffffffffffffffULL;
  int k = 0;
  while (k < 19 && mag >= T[k]) ++k;
  return ((u >> 63) && k) ? -(i64)k : (i64)k;
}
// C13 uniform residue n: block n, v = w3<<96 | w2<<64 | w1<<32 | w0, v mod q.
__device__ __forceinline__ u64 sample_uniform(u64 seed, u64 sid, u32 n, const PrimeD& P) {
  const uint4 b = philox_block(seed, sid, n);
  const u64 hi = ((u64)b.w << 32) | b.z, lo = ((u64)b.y << 32) | b.x;
  // (hi 2^64 + lo) mod q = ([hi]_q [2^64]_q + [lo]_q) mod q
  return add_mod(mul_mod(reduce64(hi, P), P.r64, P), reduce64(lo, P), P.q);
}

}  // namespace he
