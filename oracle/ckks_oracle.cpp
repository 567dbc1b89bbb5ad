// ============================================================================
// oracle/ckks_oracle.cpp — CPU ORACLE FOR THE CKKS HOT PATH.
//
// TEST INFRASTRUCTURE ONLY. This file is the slow, plain, obviously-correct
// reference that the CUDA path (paper_2104_03152_b200/csrc) is checked
// against. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load it. It shares no source, header, table or
// constant generator with the CUDA path, and never includes anything from it.
//
// What it computes: CKKS (Cheon et al. 2017, cited at PAPER.md:32 — "TenSEAL
// relies on the implementation of the CKKS scheme") over the RNS ring
// Z_Q[X]/(X^N+1), with the conventions C1–C20 of SURVEY.md §8(c), which are
// the readings recorded in DESIGN.md §3.  Every step follows SURVEY.md §8(c)
// "Oracle algorithm, step by step", in that order and notation.
//
// Deliberately plain:
//   * every modular product is (unsigned __int128)a*b % q — no Barrett,
//     Montgomery or Shoup;
//   * the NTT is "twist by psi^i, textbook cyclic radix-2 DFT with omega =
//     psi^2, bit-reverse the output" — written from definition C5, not from
//     the merged-twiddle Cooley–Tukey loop the GPU uses;
//   * CRT uses explicit multiword integers;
//   * encode/decode are the direct O(N*n) canonical-embedding sums in long
//     double (C6/C7);
//   * DivRound (rescale, ModDown) is done in the coefficient domain (C15).
// Parallelism: only over independent items (Galois keys) with std::thread.
// ============================================================================
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
#include <map>
#include <string>
#include <thread>
#include <stdexcept>
#include <algorithm>

namespace {

typedef uint64_t u64;
typedef uint32_t u32;
typedef int64_t i64;
typedef unsigned __int128 u128;

// ---------------------------------------------------------------- modular ---
u64 mulmod(u64 a, u64 b, u64 q) { return (u64)((u128)a * b % q); }
u64 addmod(u64 a, u64 b, u64 q) { return (u64)(((u128)a + b) % q); }
u64 submod(u64 a, u64 b, u64 q) { return (u64)(((u128)a + q - (b % q)) % q); }
u64 negmod(u64 a, u64 q) { return a % q == 0 ? 0 : q - a % q; }
u64 powmod(u64 a, u64 e, u64 q) {
  u64 r = 1 % q;
  a %= q;
  while (e) {
    if (e & 1) r = mulmod(r, a, q);
    a = mulmod(a, a, q);
    e >>= 1;
  }
  return r;
}
u64 invmod(u64 a, u64 q) { return powmod(a, q - 2, q); }  // q prime
u64 from_signed(i64 v, u64 q) {
  i64 r = v % (i64)q;
  return r < 0 ? (u64)(r + (i64)q) : (u64)r;
}

// Deterministic Miller–Rabin for 64-bit n (bases 2..37), SURVEY C2.
bool is_prime(u64 n) {
  static const u64 bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return false;
  for (u64 p : bases) {
    if (n % p == 0) return n == p;
  }
  u64 d = n - 1;
  int s = 0;
  while ((d & 1) == 0) { d >>= 1; ++s; }
  for (u64 a : bases) {
    u64 x = powmod(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int r = 1; r < s; ++r) {
      x = mulmod(x, x, n);
      if (x == n - 1) { comp = false; break; }
    }
    if (comp) return false;
  }
  return true;
}

unsigned bitrev(unsigned x, int bits) {
  unsigned r = 0;
  for (int i = 0; i < bits; ++i) { r = (r << 1) | (x & 1); x >>= 1; }
  return r;
}

// ------------------------------------------------------------- multiword ---
// Little-endian base-2^64 naturals; only what CRT / DivRound constants need.
typedef std::vector<u64> Big;
void big_trim(Big& a) { while (a.size() > 1 && a.back() == 0) a.pop_back(); }
Big big_from(u64 v) { return Big{v}; }
Big big_mul_small(const Big& a, u64 m) {
  Big r(a.size() + 1, 0);
  u128 carry = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    u128 t = (u128)a[i] * m + carry;
    r[i] = (u64)t;
    carry = t >> 64;
  }
  r[a.size()] = (u64)carry;
  big_trim(r);
  return r;
}
Big big_add(const Big& a, const Big& b) {
  size_t n = std::max(a.size(), b.size());
  Big r(n + 1, 0);
  u128 carry = 0;
  for (size_t i = 0; i < n; ++i) {
    u128 t = carry;
    if (i < a.size()) t += a[i];
    if (i < b.size()) t += b[i];
    r[i] = (u64)t;
    carry = t >> 64;
  }
  r[n] = (u64)carry;
  big_trim(r);
  return r;
}
int big_cmp(const Big& a0, const Big& b0) {
  Big a = a0, b = b0;
  big_trim(a); big_trim(b);
  if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
  for (size_t i = a.size(); i-- > 0;) {
    if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
  }
  return 0;
}
Big big_sub(const Big& a, const Big& b) {  // requires a >= b
  Big r(a.size(), 0);
  u64 borrow = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    u64 bi = i < b.size() ? b[i] : 0;
    u128 need = (u128)bi + borrow;
    r[i] = (u64)((u128)a[i] - need);  // wraps mod 2^64 when borrowing
    borrow = ((u128)a[i] < need) ? 1 : 0;
  }
  big_trim(r);
  return r;
}
u64 big_mod_small(const Big& a, u64 m) {  // Horner, most significant word first
  u128 r = 0;
  for (size_t i = a.size(); i-- > 0;) r = ((r << 64) | a[i]) % m;
  return (u64)r;
}
Big big_shr1(const Big& a) {
  Big r(a.size(), 0);
  for (size_t i = 0; i < a.size(); ++i) {
    r[i] = a[i] >> 1;
    if (i + 1 < a.size()) r[i] |= a[i + 1] << 63;
  }
  big_trim(r);
  return r;
}
long double big_to_ld(const Big& a) {
  long double r = 0;
  for (size_t i = a.size(); i-- > 0;) r = r * 18446744073709551616.0L + (long double)a[i];
  return r;
}

// ---------------------------------------------------------------- Philox ---
// Philox4x32-10 (Salmon et al., "Parallel random numbers: as easy as 1,2,3");
// restated from the published round function. Used as the counter-based
// generator of SURVEY C9; the GPU side implements the same generator itself.
void philox4x32_10(const u32 ctr[4], const u32 key[2], u32 out[4]) {
  const u32 M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  u32 c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  u32 k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += W0; k1 += W1; }
    u64 p0 = (u64)M0 * c0;
    u64 p1 = (u64)M1 * c2;
    u32 hi0 = (u32)(p0 >> 32), lo0 = (u32)p0;
    u32 hi1 = (u32)(p1 >> 32), lo1 = (u32)p1;
    u32 n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// C9: counter = (block_lo, block_hi, sid_lo, sid_hi), key = (seed_lo, seed_hi)
void philox_block(u64 seed, u64 sid, u64 block, u32 out[4]) {
  u32 ctr[4] = {(u32)block, (u32)(block >> 32), (u32)sid, (u32)(sid >> 32)};
  u32 key[2] = {(u32)seed, (u32)(seed >> 32)};
  philox4x32_10(ctr, key, out);
}

// C9 stream id: purpose<<56 | object<<16 | prime_index
enum Purpose : u64 {
  P_S = 1, P_PK_A = 2, P_PK_E = 3, P_RLK_A = 4, P_RLK_E = 5,
  P_GK_A = 6, P_GK_E = 7, P_ENC_V = 8, P_ENC_E0 = 9, P_ENC_E1 = 10,
  P_SYM_A = 11, P_SYM_E = 12   // symmetric encryption (DESIGN.md §3 reading "seeded symmetric")
};
u64 make_sid(u64 purpose, u64 object, u64 prime) {
  return (purpose << 56) | (object << 16) | prime;
}

// C10 ternary: coefficient n uses block n/4, word n%4; t=(w*3)>>32; value t-1
void sample_ternary(u64 seed, u64 sid, int N, i64* out) {
  for (int n = 0; n < N; n += 4) {
    u32 w[4];
    philox_block(seed, sid, (u64)(n / 4), w);
    for (int k = 0; k < 4 && n + k < N; ++k) {
      u64 t = ((u64)w[k] * 3u) >> 32;
      out[n + k] = (i64)t - 1;
    }
  }
}

// C11 CDT Gaussian: coefficient n uses block n/2; u = w[2(n%2)+1]<<32 | w[2(n%2)];
// bit 63 = sign; magnitude = smallest k with (u & (2^63-1)) < T[k].
void sample_cdt(u64 seed, u64 sid, int N, const u64* T, int T_len, i64* out) {
  for (int n = 0; n < N; n += 2) {
    u32 w[4];
    philox_block(seed, sid, (u64)(n / 2), w);
    for (int h = 0; h < 2 && n + h < N; ++h) {
      u64 u = ((u64)w[2 * h + 1] << 32) | (u64)w[2 * h];
      u64 sign = u >> 63;
      u64 mag = u & 0x7fffffffffffffffULL;
      int k = 0;
      while (k < T_len - 1 && !(mag < T[k])) ++k;
      out[n + h] = (sign && k > 0) ? -(i64)k : (i64)k;
    }
  }
}

// C13 uniform residue drawn directly as an NTT-domain word: coefficient n uses
// block n; u128 = w3<<96|w2<<64|w1<<32|w0; value = u128 mod q.
void sample_uniform(u64 seed, u64 sid, u64 q, int N, u64* out) {
  for (int n = 0; n < N; ++n) {
    u32 w[4];
    philox_block(seed, sid, (u64)n, w);
    u128 v = ((u128)w[3] << 96) | ((u128)w[2] << 64) | ((u128)w[1] << 32) | (u128)w[0];
    out[n] = (u64)(v % q);
  }
}

// ------------------------------------------------------------------- NTT ---
// C5: NTT(a)[j] = sum_i a_i psi^{(2 brv(j) + 1) i}.
// Written as: b_i = a_i psi^i (twist); A = cyclic DFT of b with omega = psi^2
// (A[k] = sum_i b_i omega^{ik}); NTT(a)[j] = A[brv(j)].
void cyclic_dft(std::vector<u64>& x, u64 w, u64 q, int logN) {
  const int N = 1 << logN;
  for (int i = 0; i < N; ++i) {
    int r = (int)bitrev((unsigned)i, logN);
    if (i < r) std::swap(x[i], x[r]);
  }
  for (int len = 2; len <= N; len <<= 1) {
    u64 wl = powmod(w, (u64)(N / len), q);
    for (int i = 0; i < N; i += len) {
      u64 ww = 1;
      for (int j = 0; j < len / 2; ++j) {
        u64 u = x[i + j];
        u64 v = mulmod(x[i + j + len / 2], ww, q);
        x[i + j] = addmod(u, v, q);
        x[i + j + len / 2] = submod(u, v, q);
        ww = mulmod(ww, wl, q);
      }
    }
  }
}

void ntt_forward(u64* a, int logN, u64 q, u64 psi) {
  const int N = 1 << logN;
  std::vector<u64> b(N);
  u64 pw = 1;
  for (int i = 0; i < N; ++i) { b[i] = mulmod(a[i] % q, pw, q); pw = mulmod(pw, psi, q); }
  cyclic_dft(b, mulmod(psi, psi, q), q, logN);
  for (int j = 0; j < N; ++j) a[j] = b[bitrev((unsigned)j, logN)];
}

void ntt_inverse(u64* a, int logN, u64 q, u64 psi) {
  const int N = 1 << logN;
  std::vector<u64> b(N);
  for (int k = 0; k < N; ++k) b[k] = a[bitrev((unsigned)k, logN)];
  u64 ipsi = invmod(psi, q);
  cyclic_dft(b, mulmod(ipsi, ipsi, q), q, logN);
  u64 ninv = invmod((u64)N, q);
  u64 pw = ninv;
  for (int i = 0; i < N; ++i) { a[i] = mulmod(b[i], pw, q); pw = mulmod(pw, ipsi, q); }
}

// C8 automorphism in the coefficient domain: a(X) -> a(X^g).
void automorph_coeff(const u64* a, u64* out, int N, u64 g, u64 q) {
  const u64 twoN = 2 * (u64)N;
  for (int i = 0; i < N; ++i) {
    u64 e = ((u64)i * g) % twoN;
    if (e < (u64)N) out[e] = a[i] % q;
    else out[e - N] = negmod(a[i], q);
  }
}

// --------------------------------------------------------------- context ---
struct Ctx {
  int logN = 0, N = 0, L = 0, K = 0;   // L data primes, K special primes
  std::vector<u64> q;                  // L + K primes (specials last)
  std::vector<u64> psi;
  u64 seed = 0;
  std::vector<u64> cdt;                // C11 table T[0..19]
  bool has_keys = false;
  std::vector<i64> s_coeff;            // N
  std::vector<u64> s_ntt;              // (L+K) x N
  std::vector<u64> pk;                 // [2][L][N]  (b, a)
  std::vector<u64> rlk;                // [L][2][L+K][N]
  std::map<u64, std::vector<u64>> gk;  // galois element -> [L][2][L+K][N]
  std::string err;
};

int LK(const Ctx& c) { return c.L + c.K; }

// C2: for each requested size b, in order: the largest unused prime
// 2^{b-1} < p < 2^b with p = 1 mod 2N.
std::vector<u64> select_primes(const std::vector<int>& bits, int N) {
  const u64 M = 2 * (u64)N;
  std::vector<u64> out;
  for (int b : bits) {
    if (b < 2 || b > 62) throw std::runtime_error("prime bit size out of range");
    u64 top = 1ULL << b, low = 1ULL << (b - 1);
    u64 p = ((top - 1) / M) * M + 1;
    if (p >= top) p -= M;
    while (true) {
      if (p <= low || p < M) throw std::runtime_error("not enough NTT primes");
      if (std::find(out.begin(), out.end(), p) == out.end() && is_prime(p)) break;
      p -= M;
    }
    out.push_back(p);
  }
  return out;
}

// C4: psi = min over odd e of r^e, r any primitive 2N-th root of unity mod q.
u64 min_psi(u64 q, int N) {
  const u64 M = 2 * (u64)N;
  u64 r = 0;
  for (u64 x = 2;; ++x) {
    u64 c = powmod(x, (q - 1) / M, q);
    if (powmod(c, (u64)N, q) == q - 1) { r = c; break; }
  }
  u64 r2 = mulmod(r, r, q), cur = r, best = r;
  for (u64 e = 3; e < M; e += 2) {
    cur = mulmod(cur, r2, q);
    if (cur < best) best = cur;
  }
  return best;
}

// C6: galois element for a left rotation by k (k<0 -> 5^{n_s+k}); k = n_s -> 1.
u64 galois_elt(const Ctx& c, int k) {
  const int ns = c.N / 2;
  int e = k > 0 ? k : ns + k;
  return powmod(5, (u64)e, 2 * (u64)c.N);
}

void ntt_limb(const Ctx& c, int t, u64* a) { ntt_forward(a, c.logN, c.q[t], c.psi[t]); }
void intt_limb(const Ctx& c, int t, u64* a) { ntt_inverse(a, c.logN, c.q[t], c.psi[t]); }

void signed_to_ntt(const Ctx& c, const i64* v, int t, u64* out) {
  for (int n = 0; n < c.N; ++n) out[n] = from_signed(v[n], c.q[t]);
  ntt_limb(c, t, out);
}

// C12: key-switching key for s' (NTT words over all L+K limbs).
// ksk_j = (b_j, a_j):  b_j = -a_j s + e_j + [P]_{q_j} s'  (last term on limb j only)
void make_ksk(const Ctx& c, const std::vector<u64>& sprime, u64 pa, u64 pe, u64 objbase,
              std::vector<u64>& out) {
  const int N = c.N, lk = LK(c);
  out.assign((size_t)c.L * 2 * lk * N, 0);
  std::vector<i64> e(N);
  std::vector<u64> a(N), et(N);
  for (int j = 0; j < c.L; ++j) {
    const u64 obj = objbase | (u64)j;
    sample_cdt(c.seed, make_sid(pe, obj, 0), N, c.cdt.data(), (int)c.cdt.size(), e.data());
    u64 P_qj = 1;
    for (int k = 0; k < c.K; ++k) P_qj = mulmod(P_qj, c.q[c.L + k] % c.q[j], c.q[j]);
    for (int t = 0; t < lk; ++t) {
      const u64 qt = c.q[t];
      sample_uniform(c.seed, make_sid(pa, obj, (u64)t), qt, N, a.data());
      signed_to_ntt(c, e.data(), t, et.data());
      u64* bo = &out[(((size_t)j * 2 + 0) * lk + t) * N];
      u64* ao = &out[(((size_t)j * 2 + 1) * lk + t) * N];
      for (int n = 0; n < N; ++n) {
        u64 b = addmod(negmod(mulmod(a[n], c.s_ntt[(size_t)t * N + n], qt), qt), et[n], qt);
        if (t == j) b = addmod(b, mulmod(P_qj, sprime[(size_t)t * N + n], qt), qt);
        bo[n] = b;
        ao[n] = a[n];
      }
    }
  }
}

void galois_key(const Ctx& c, u64 g, std::vector<u64>& out) {
  const int N = c.N, lk = LK(c);
  // s' = phi_g(s), built in the coefficient domain (C8) then NTT per limb
  std::vector<u64> sp((size_t)lk * N), tmp(N);
  for (int t = 0; t < lk; ++t) {
    for (int n = 0; n < N; ++n) tmp[n] = from_signed(c.s_coeff[n], c.q[t]);
    automorph_coeff(tmp.data(), &sp[(size_t)t * N], N, g, c.q[t]);
    ntt_limb(c, t, &sp[(size_t)t * N]);
  }
  make_ksk(c, sp, P_GK_A, P_GK_E, g << 8, out);
}

void keygen(Ctx& c, const std::vector<int>& steps, int nthreads) {
  const int N = c.N, lk = LK(c);
  // s: ternary, one signed polynomial, NTT into every limb
  c.s_coeff.assign(N, 0);
  sample_ternary(c.seed, make_sid(P_S, 0, 0), N, c.s_coeff.data());
  c.s_ntt.assign((size_t)lk * N, 0);
  for (int t = 0; t < lk; ++t) signed_to_ntt(c, c.s_coeff.data(), t, &c.s_ntt[(size_t)t * N]);
  // pk = (-a s + e, a) over the data limbs
  c.pk.assign((size_t)2 * c.L * N, 0);
  std::vector<i64> e(N);
  std::vector<u64> et(N);
  sample_cdt(c.seed, make_sid(P_PK_E, 0, 0), N, c.cdt.data(), (int)c.cdt.size(), e.data());
  for (int i = 0; i < c.L; ++i) {
    const u64 qi = c.q[i];
    u64* b = &c.pk[(size_t)i * N];
    u64* a = &c.pk[((size_t)c.L + i) * N];
    sample_uniform(c.seed, make_sid(P_PK_A, 0, (u64)i), qi, N, a);
    signed_to_ntt(c, e.data(), i, et.data());
    for (int n = 0; n < N; ++n)
      b[n] = addmod(negmod(mulmod(a[n], c.s_ntt[(size_t)i * N + n], qi), qi), et[n], qi);
  }
  // relinearisation key: s' = s^2
  std::vector<u64> s2((size_t)lk * N);
  for (int t = 0; t < lk; ++t)
    for (int n = 0; n < N; ++n)
      s2[(size_t)t * N + n] = mulmod(c.s_ntt[(size_t)t * N + n], c.s_ntt[(size_t)t * N + n], c.q[t]);
  make_ksk(c, s2, P_RLK_A, P_RLK_E, 0, c.rlk);
  // Galois keys, one per distinct element; threads over independent keys
  std::vector<u64> gs;
  for (int k : steps) {
    u64 g = galois_elt(c, k);
    if (std::find(gs.begin(), gs.end(), g) == gs.end()) gs.push_back(g);
  }
  std::vector<std::vector<u64>> keys(gs.size());
  if (nthreads < 1) nthreads = 1;
  std::vector<std::thread> th;
  for (int w = 0; w < nthreads; ++w) {
    th.emplace_back([&, w]() {
      for (size_t i = w; i < gs.size(); i += nthreads) galois_key(c, gs[i], keys[i]);
    });
  }
  for (auto& t : th) t.join();
  c.gk.clear();
  for (size_t i = 0; i < gs.size(); ++i) c.gk[gs[i]] = std::move(keys[i]);
  c.has_keys = true;
}

// C15 DivRound by basis B = {q[drop_k]} on coefficient-domain residues.
// h = floor(B/2); y_k = [x_{b_k} + [h]_{b_k}]_{b_k};
// conv_i = sum_k [y_k (B/b_k)^{-1}]_{b_k} [B/b_k]_{q_i};
// out_i = (x_i + [h]_{q_i} - conv_i) [B^{-1}]_{q_i}.
void divround(const Ctx& c, const std::vector<int>& keep, const std::vector<int>& drop,
              const std::vector<const u64*>& x_keep, const std::vector<const u64*>& x_drop,
              const std::vector<u64*>& out) {
  const int N = c.N;
  Big B = big_from(1);
  for (int d : drop) B = big_mul_small(B, c.q[d]);
  Big h = big_shr1(B);  // B odd: floor(B/2)
  const size_t nd = drop.size(), nk = keep.size();
  std::vector<u64> hk(nd), invk(nd);
  std::vector<std::vector<u64>> Bk_qi(nd, std::vector<u64>(nk));
  for (size_t k = 0; k < nd; ++k) {
    Big Bk = big_from(1);
    for (size_t l = 0; l < nd; ++l)
      if (l != k) Bk = big_mul_small(Bk, c.q[drop[l]]);
    const u64 bk = c.q[drop[k]];
    hk[k] = big_mod_small(h, bk);
    invk[k] = invmod(big_mod_small(Bk, bk), bk);
    for (size_t i = 0; i < nk; ++i) Bk_qi[k][i] = big_mod_small(Bk, c.q[keep[i]]);
  }
  std::vector<u64> hi(nk), Binv(nk);
  for (size_t i = 0; i < nk; ++i) {
    hi[i] = big_mod_small(h, c.q[keep[i]]);
    Binv[i] = invmod(big_mod_small(B, c.q[keep[i]]), c.q[keep[i]]);
  }
  std::vector<u64> t(nd);
  for (int n = 0; n < N; ++n) {
    for (size_t k = 0; k < nd; ++k) {
      const u64 bk = c.q[drop[k]];
      u64 y = addmod(x_drop[k][n], hk[k], bk);
      t[k] = mulmod(y, invk[k], bk);
    }
    for (size_t i = 0; i < nk; ++i) {
      const u64 qi = c.q[keep[i]];
      u64 conv = 0;
      for (size_t k = 0; k < nd; ++k) conv = addmod(conv, mulmod(t[k] % qi, Bk_qi[k][i], qi), qi);
      u64 v = submod(addmod(x_keep[i][n], hi[i], qi), conv, qi);
      out[i][n] = mulmod(v, Binv[i], qi);
    }
  }
}

// C16 centered lift of a residue of q_j.
i64 centered(u64 r, u64 q) { return r <= (q - 1) / 2 ? (i64)r : (i64)r - (i64)q; }

// Step 7: KS_{s'}(d) at level l. d: (l+1) x N NTT words. ksk: [L][2][L+K][N].
// Returns u: [2][l+1][N] NTT words.
void keyswitch(const Ctx& c, const u64* d, int level, const std::vector<u64>& ksk, u64* u) {
  const int N = c.N, lk = LK(c), Lc = level + 1;
  // INTT d into residues [d]_{q_j}; centered lift D_j
  std::vector<std::vector<i64>> D(Lc, std::vector<i64>(N));
  std::vector<u64> tmp(N);
  for (int j = 0; j < Lc; ++j) {
    std::memcpy(tmp.data(), d + (size_t)j * N, N * 8);
    intt_limb(c, j, tmp.data());
    for (int n = 0; n < N; ++n) D[j][n] = centered(tmp[n], c.q[j]);
  }
  // targets: data limbs 0..l then the specials
  std::vector<int> targets;
  for (int i = 0; i < Lc; ++i) targets.push_back(i);
  for (int k = 0; k < c.K; ++k) targets.push_back(c.L + k);
  const size_t nt = targets.size();
  std::vector<std::vector<u64>> acc0(nt, std::vector<u64>(N, 0)), acc1(nt, std::vector<u64>(N, 0));
  std::vector<u64> Dt(N);
  for (size_t ti = 0; ti < nt; ++ti) {
    const int t = targets[ti];
    const u64 qt = c.q[t];
    for (int j = 0; j < Lc; ++j) {
      signed_to_ntt(c, D[j].data(), t, Dt.data());
      const u64* b = &ksk[(((size_t)j * 2 + 0) * lk + t) * N];
      const u64* a = &ksk[(((size_t)j * 2 + 1) * lk + t) * N];
      for (int n = 0; n < N; ++n) {
        acc0[ti][n] = addmod(acc0[ti][n], mulmod(Dt[n], b[n], qt), qt);
        acc1[ti][n] = addmod(acc1[ti][n], mulmod(Dt[n], a[n], qt), qt);
      }
    }
  }
  // ModDown: INTT everything, DivRound by P in the coefficient domain, NTT back
  std::vector<int> keep(targets.begin(), targets.begin() + Lc);
  std::vector<int> drop(targets.begin() + Lc, targets.end());
  for (int part = 0; part < 2; ++part) {
    auto& acc = part == 0 ? acc0 : acc1;
    for (size_t ti = 0; ti < nt; ++ti) intt_limb(c, targets[ti], acc[ti].data());
    std::vector<const u64*> xk, xd;
    std::vector<u64*> out;
    for (int i = 0; i < Lc; ++i) {
      xk.push_back(acc[i].data());
      out.push_back(u + ((size_t)part * Lc + i) * N);
    }
    for (size_t k = 0; k < drop.size(); ++k) xd.push_back(acc[Lc + k].data());
    divround(c, keep, drop, xk, xd, out);
    for (int i = 0; i < Lc; ++i) ntt_limb(c, i, out[i]);
  }
}

// Step 9: rescale a size-`size` ciphertext at level l (NTT words) -> level l-1.
void rescale(const Ctx& c, const u64* ct, int size, int level, u64* out) {
  const int N = c.N, Lc = level + 1;
  std::vector<int> keep, drop{level};
  for (int i = 0; i < level; ++i) keep.push_back(i);
  std::vector<std::vector<u64>> x(Lc, std::vector<u64>(N));
  for (int p = 0; p < size; ++p) {
    for (int i = 0; i < Lc; ++i) {
      std::memcpy(x[i].data(), ct + ((size_t)p * Lc + i) * N, N * 8);
      intt_limb(c, i, x[i].data());
    }
    std::vector<const u64*> xk, xd{x[level].data()};
    std::vector<u64*> o;
    for (int i = 0; i < level; ++i) {
      xk.push_back(x[i].data());
      o.push_back(out + ((size_t)p * level + i) * N);
    }
    divround(c, keep, drop, xk, xd, o);
    for (int i = 0; i < level; ++i) ntt_limb(c, i, o[i]);
  }
}

// cos(pi k / N) table in long double for k in [0, 2N)
std::vector<long double> cos_table(int N) {
  const long double pi = acosl(-1.0L);
  std::vector<long double> t(2 * (size_t)N);
  for (int k = 0; k < 2 * N; ++k) t[k] = cosl(pi * (long double)k / (long double)N);
  return t;
}

}  // namespace

// =================================================================== C API ===
extern "C" {

void* orc_create(int logN, int n_primes, const int* bits, int n_special, uint64_t seed,
                 const uint64_t* cdt, int cdt_len) {
  try {
    Ctx* c = new Ctx();
    c->logN = logN;
    c->N = 1 << logN;
    c->K = n_special;
    c->L = n_primes - n_special;
    if (c->L < 1 || c->K < 0) throw std::runtime_error("bad prime split");
    c->q = select_primes(std::vector<int>(bits, bits + n_primes), c->N);
    for (u64 q : c->q) c->psi.push_back(min_psi(q, c->N));
    c->seed = seed;
    c->cdt.assign(cdt, cdt + cdt_len);
    return c;
  } catch (...) {
    return nullptr;
  }
}

void orc_destroy(void* h) { delete (Ctx*)h; }

int orc_dims(void* h, int* out) {
  Ctx* c = (Ctx*)h;
  out[0] = c->logN; out[1] = c->N; out[2] = c->L; out[3] = c->K;
  return 0;
}

void orc_primes(void* h, uint64_t* out) {
  Ctx* c = (Ctx*)h;
  for (size_t i = 0; i < c->q.size(); ++i) out[i] = c->q[i];
}

void orc_psis(void* h, uint64_t* out) {
  Ctx* c = (Ctx*)h;
  for (size_t i = 0; i < c->psi.size(); ++i) out[i] = c->psi[i];
}

// Standalone helpers used by the pins.
int orc_select_primes(int logN, int n, const int* bits, uint64_t* out) {
  try {
    auto v = select_primes(std::vector<int>(bits, bits + n), 1 << logN);
    for (int i = 0; i < n; ++i) out[i] = v[i];
    return 0;
  } catch (...) {
    return -1;
  }
}
uint64_t orc_min_psi(uint64_t q, int N) { return min_psi(q, N); }
int orc_is_prime(uint64_t n) { return is_prime(n) ? 1 : 0; }
void orc_ntt_raw(uint64_t* a, int logN, uint64_t q, uint64_t psi) { ntt_forward(a, logN, q, psi); }
void orc_intt_raw(uint64_t* a, int logN, uint64_t q, uint64_t psi) { ntt_inverse(a, logN, q, psi); }
void orc_philox(const uint32_t* ctr, const uint32_t* key, uint32_t* out) { philox4x32_10(ctr, key, out); }

void orc_ntt(void* h, int t, uint64_t* a) { ntt_limb(*(Ctx*)h, t, a); }
void orc_intt(void* h, int t, uint64_t* a) { intt_limb(*(Ctx*)h, t, a); }

void orc_sample_ternary(void* h, uint64_t sid, int64_t* out) {
  Ctx* c = (Ctx*)h;
  sample_ternary(c->seed, sid, c->N, out);
}
void orc_sample_cdt(void* h, uint64_t sid, int64_t* out) {
  Ctx* c = (Ctx*)h;
  sample_cdt(c->seed, sid, c->N, c->cdt.data(), (int)c->cdt.size(), out);
}
void orc_sample_uniform(void* h, uint64_t sid, int t, uint64_t* out) {
  Ctx* c = (Ctx*)h;
  sample_uniform(c->seed, sid, c->q[t], c->N, out);
}
uint64_t orc_sid(uint64_t purpose, uint64_t object, uint64_t prime) {
  return make_sid(purpose, object, prime);
}
uint64_t orc_galois_elt(void* h, int k) { return galois_elt(*(Ctx*)h, k); }

int orc_keygen(void* h, const int* steps, int n_steps, int nthreads) {
  Ctx* c = (Ctx*)h;
  try {
    keygen(*c, std::vector<int>(steps, steps + n_steps), nthreads);
    return 0;
  } catch (const std::exception& e) {
    c->err = e.what();
    return -1;
  }
}

void orc_sk(void* h, int64_t* coeffs, uint64_t* ntt_words) {
  Ctx* c = (Ctx*)h;
  if (coeffs) std::memcpy(coeffs, c->s_coeff.data(), c->N * 8);
  if (ntt_words) std::memcpy(ntt_words, c->s_ntt.data(), c->s_ntt.size() * 8);
}
void orc_pk(void* h, uint64_t* out) {
  Ctx* c = (Ctx*)h;
  std::memcpy(out, c->pk.data(), c->pk.size() * 8);
}
void orc_relin_key(void* h, uint64_t* out) {
  Ctx* c = (Ctx*)h;
  std::memcpy(out, c->rlk.data(), c->rlk.size() * 8);
}
int orc_galois_key(void* h, int step, uint64_t* out) {
  Ctx* c = (Ctx*)h;
  auto it = c->gk.find(galois_elt(*c, step));
  if (it == c->gk.end()) return -1;
  std::memcpy(out, it->second.data(), it->second.size() * 8);
  return 0;
}

// C6/C7 encode: m_i = round(scale * (2/N) * Re sum_{j<n} z_j zeta^{-i 5^j}),
// zeta = exp(i pi / N), round half away from zero. Writes the pre-rounding
// values (as double) and the integer coefficients.
int orc_encode(void* h, const double* z, int n, double scale, double* pre, int64_t* m) {
  Ctx* c = (Ctx*)h;
  const int N = c->N;
  const u64 twoN = 2 * (u64)N, mask = twoN - 1;
  if (n > N / 2) return -1;
  auto ct = cos_table(N);
  std::vector<u64> g(n);
  u64 p = 1;
  for (int j = 0; j < n; ++j) { g[j] = p; p = (p * 5) & mask; }
  const long double f = (long double)scale * 2.0L / (long double)N;
  const long double lim = 4611686018427387904.0L;  // 2^62
  int rc = 0;
  for (int i = 0; i < N; ++i) {
    long double acc = 0;
    for (int j = 0; j < n; ++j) {
      u64 e = (twoN - (((u64)i * g[j]) & mask)) & mask;
      acc += (long double)z[j] * ct[e];
    }
    long double v = f * acc;
    if (pre) pre[i] = (double)v;
    if (fabsl(v) >= lim) { rc = -2; v = 0; }
    m[i] = (int64_t)llroundl(v);
  }
  return rc;
}

// Signed integer coefficients -> NTT words [level+1][N].
void orc_coeffs_to_pt(void* h, const int64_t* m, int level, uint64_t* pt) {
  Ctx* c = (Ctx*)h;
  for (int i = 0; i <= level; ++i) signed_to_ntt(*c, m, i, pt + (size_t)i * c->N);
}

// C6 decode: INTT, CRT to X in [0, Q_l), centre, long double,
// z_j = Re sum_i X_i zeta^{i 5^j} / scale for j < n. Also returns the centred
// coefficients as doubles when coeffs != nullptr.
void orc_decode(void* h, const uint64_t* pt, int level, double scale, int n, double* z,
                double* coeffs) {
  Ctx* c = (Ctx*)h;
  const int N = c->N, Lc = level + 1;
  std::vector<std::vector<u64>> x(Lc, std::vector<u64>(N));
  for (int i = 0; i < Lc; ++i) {
    std::memcpy(x[i].data(), pt + (size_t)i * N, N * 8);
    intt_limb(*c, i, x[i].data());
  }
  Big Q = big_from(1);
  for (int i = 0; i < Lc; ++i) Q = big_mul_small(Q, c->q[i]);
  std::vector<Big> Qi(Lc);
  std::vector<u64> Qi_inv(Lc);
  for (int i = 0; i < Lc; ++i) {
    Big t = big_from(1);
    for (int l = 0; l < Lc; ++l)
      if (l != i) t = big_mul_small(t, c->q[l]);
    Qi[i] = t;
    Qi_inv[i] = invmod(big_mod_small(t, c->q[i]), c->q[i]);
  }
  std::vector<long double> X(N);
  for (int k = 0; k < N; ++k) {
    Big acc = big_from(0);
    for (int i = 0; i < Lc; ++i)
      acc = big_add(acc, big_mul_small(Qi[i], mulmod(x[i][k], Qi_inv[i], c->q[i])));
    while (big_cmp(acc, Q) >= 0) acc = big_sub(acc, Q);
    Big twice = big_add(acc, acc);
    if (big_cmp(twice, Q) > 0) X[k] = -big_to_ld(big_sub(Q, acc));
    else X[k] = big_to_ld(acc);
    if (coeffs) coeffs[k] = (double)X[k];
  }
  if (z && n > 0) {
    auto ct = cos_table(N);
    const u64 twoN = 2 * (u64)N, mask = twoN - 1;
    u64 g = 1;
    for (int j = 0; j < n; ++j) {
      long double acc = 0;
      for (int i = 0; i < N; ++i) acc += X[i] * ct[((u64)i * g) & mask];
      z[j] = (double)(acc / (long double)scale);
      g = (g * 5) & mask;
    }
  }
}

// Step 4 (C13): c0 = v b + e0 + m, c1 = v a + e1 (NTT domain, level l).
void orc_encrypt(void* h, const uint64_t* pt, int level, uint64_t stream_id, uint64_t* ct) {
  Ctx* c = (Ctx*)h;
  const int N = c->N, Lc = level + 1;
  std::vector<i64> v(N), e0(N), e1(N);
  sample_ternary(c->seed, make_sid(P_ENC_V, stream_id, 0), N, v.data());
  sample_cdt(c->seed, make_sid(P_ENC_E0, stream_id, 0), N, c->cdt.data(), (int)c->cdt.size(), e0.data());
  sample_cdt(c->seed, make_sid(P_ENC_E1, stream_id, 0), N, c->cdt.data(), (int)c->cdt.size(), e1.data());
  std::vector<u64> vt(N), e0t(N), e1t(N);
  for (int i = 0; i < Lc; ++i) {
    const u64 qi = c->q[i];
    signed_to_ntt(*c, v.data(), i, vt.data());
    signed_to_ntt(*c, e0.data(), i, e0t.data());
    signed_to_ntt(*c, e1.data(), i, e1t.data());
    const u64* b = &c->pk[(size_t)i * N];
    const u64* a = &c->pk[((size_t)c->L + i) * N];
    u64* c0 = ct + (size_t)i * N;
    u64* c1 = ct + ((size_t)Lc + i) * N;
    for (int n = 0; n < N; ++n) {
      c0[n] = addmod(addmod(mulmod(vt[n], b[n], qi), e0t[n], qi), pt[(size_t)i * N + n], qi);
      c1[n] = addmod(mulmod(vt[n], a[n], qi), e1t[n], qi);
    }
  }
}

// Symmetric encryption (DESIGN.md §3 "seeded symmetric encryption"):
// a_i = Uniform(a_seed, (P_SYM_A, stream_id, i)) -- the PUBLIC seed --, e = CDT(seed, (P_SYM_E,
// stream_id, 0)); c0 = -a s + e + m, c1 = a (NTT domain, level l).
void orc_encrypt_symmetric(void* h, const uint64_t* pt, int level, uint64_t stream_id, uint64_t a_seed,
                           uint64_t* ct) {
  Ctx* c = (Ctx*)h;
  const int N = c->N, Lc = level + 1;
  std::vector<i64> e(N);
  sample_cdt(c->seed, make_sid(P_SYM_E, stream_id, 0), N, c->cdt.data(), (int)c->cdt.size(), e.data());
  std::vector<u64> et(N);
  for (int i = 0; i < Lc; ++i) {
    const u64 qi = c->q[i];
    u64* c0 = ct + (size_t)i * N;
    u64* c1 = ct + ((size_t)Lc + i) * N;
    sample_uniform(a_seed, make_sid(P_SYM_A, stream_id, (u64)i), qi, N, c1);
    signed_to_ntt(*c, e.data(), i, et.data());
    for (int n = 0; n < N; ++n)
      c0[n] = addmod(addmod(negmod(mulmod(c1[n], c->s_ntt[(size_t)i * N + n], qi), qi), et[n], qi),
                     pt[(size_t)i * N + n], qi);
  }
}

// Step 10: m = c0 + c1 s (+ c2 s^2), NTT domain.
void orc_decrypt(void* h, const uint64_t* ct, int size, int level, uint64_t* pt) {
  Ctx* c = (Ctx*)h;
  const int N = c->N, Lc = level + 1;
  for (int i = 0; i < Lc; ++i) {
    const u64 qi = c->q[i];
    for (int n = 0; n < N; ++n) {
      u64 s = c->s_ntt[(size_t)i * N + n];
      u64 acc = 0, sp = 1;
      for (int p = 0; p < size; ++p) {
        acc = addmod(acc, mulmod(ct[((size_t)p * Lc + i) * N + n], sp, qi), qi);
        sp = mulmod(sp, s, qi);
      }
      pt[(size_t)i * N + n] = acc;
    }
  }
}

// Step 5/6: limb-wise ring ops on [parts][l+1][N] word arrays.
// op: 0 add, 1 sub, 2 negate(a), 3 mul (pointwise, b has the same parts count or 1)
void orc_pointwise(void* h, int op, const uint64_t* a, const uint64_t* b, int parts_a, int parts_b,
                   int level, uint64_t* out) {
  Ctx* c = (Ctx*)h;
  const int N = c->N, Lc = level + 1;
  for (int p = 0; p < parts_a; ++p) {
    const int pb = parts_b == 1 ? 0 : p;
    for (int i = 0; i < Lc; ++i) {
      const u64 qi = c->q[i];
      for (int n = 0; n < N; ++n) {
        const size_t ia = ((size_t)p * Lc + i) * N + n;
        const size_t ib = ((size_t)pb * Lc + i) * N + n;
        u64 r = 0;
        switch (op) {
          case 0: r = addmod(a[ia], b[ib], qi); break;
          case 1: r = submod(a[ia], b[ib], qi); break;
          case 2: r = negmod(a[ia], qi); break;
          case 3: r = mulmod(a[ia], b[ib], qi); break;
        }
        out[ia] = r;
      }
    }
  }
}

// Step 6: (c0 c0', c0 c1' + c1 c0', c1 c1').
void orc_tensor(void* h, const uint64_t* x, const uint64_t* y, int level, uint64_t* out) {
  Ctx* c = (Ctx*)h;
  const int N = c->N, Lc = level + 1;
  const size_t P = (size_t)Lc * N;
  for (int i = 0; i < Lc; ++i) {
    const u64 qi = c->q[i];
    for (int n = 0; n < N; ++n) {
      const size_t k = (size_t)i * N + n;
      out[k] = mulmod(x[k], y[k], qi);
      out[P + k] = addmod(mulmod(x[k], y[P + k], qi), mulmod(x[P + k], y[k], qi), qi);
      out[2 * P + k] = mulmod(x[P + k], y[P + k], qi);
    }
  }
}

// Step 7 exposed: key = 0 -> relinearisation key, else Galois key of `step`.
int orc_keyswitch(void* h, const uint64_t* d, int level, int use_galois, int step, uint64_t* u) {
  Ctx* c = (Ctx*)h;
  const std::vector<u64>* k = &c->rlk;
  if (use_galois) {
    auto it = c->gk.find(galois_elt(*c, step));
    if (it == c->gk.end()) return -1;
    k = &it->second;
  }
  keyswitch(*c, d, level, *k, u);
  return 0;
}

// Step 8: relinearise (d0 + u0, d1 + u1), u = KS_{s^2}(d2).
void orc_relinearize(void* h, const uint64_t* ct3, int level, uint64_t* out) {
  Ctx* c = (Ctx*)h;
  const int N = c->N, Lc = level + 1;
  const size_t P = (size_t)Lc * N;
  std::vector<u64> u(2 * P);
  keyswitch(*c, ct3 + 2 * P, level, c->rlk, u.data());
  for (int i = 0; i < Lc; ++i)
    for (int n = 0; n < N; ++n) {
      const size_t k = (size_t)i * N + n;
      out[k] = addmod(ct3[k], u[k], c->q[i]);
      out[P + k] = addmod(ct3[P + k], u[P + k], c->q[i]);
    }
}

// Step 8: rotate left by k: (phi_g(c0) + u0, u1), u = KS_{phi_g(s)}(phi_g(c1)).
// phi_g is applied in the coefficient domain (INTT, C8, NTT).
int orc_rotate(void* h, const uint64_t* ct, int level, int step, uint64_t* out) {
  Ctx* c = (Ctx*)h;
  const int N = c->N, Lc = level + 1;
  const size_t P = (size_t)Lc * N;
  const u64 g = galois_elt(*c, step);
  auto it = c->gk.find(g);
  if (it == c->gk.end()) return -1;
  std::vector<u64> phi(2 * P), tmp(N);
  for (int p = 0; p < 2; ++p)
    for (int i = 0; i < Lc; ++i) {
      std::memcpy(tmp.data(), ct + (size_t)p * P + (size_t)i * N, N * 8);
      intt_limb(*c, i, tmp.data());
      u64* o = &phi[(size_t)p * P + (size_t)i * N];
      automorph_coeff(tmp.data(), o, N, g, c->q[i]);
      ntt_limb(*c, i, o);
    }
  std::vector<u64> u(2 * P);
  keyswitch(*c, phi.data() + P, level, it->second, u.data());
  for (int i = 0; i < Lc; ++i)
    for (int n = 0; n < N; ++n) {
      const size_t k = (size_t)i * N + n;
      out[k] = addmod(phi[k], u[k], c->q[i]);
      out[P + k] = u[P + k];
    }
  return 0;
}

// C8 automorphism on NTT words of one limb, done through the coefficient domain.
void orc_automorph_ntt(void* h, const uint64_t* a, int t, uint64_t g, uint64_t* out) {
  Ctx* c = (Ctx*)h;
  const int N = c->N;
  std::vector<u64> tmp(a, a + N);
  intt_limb(*c, t, tmp.data());
  automorph_coeff(tmp.data(), out, N, g, c->q[t]);
  ntt_limb(*c, t, out);
}

void orc_rescale(void* h, const uint64_t* ct, int size, int level, uint64_t* out) {
  rescale(*(Ctx*)h, ct, size, level, out);
}

// DivRound exposed for the big-integer pin: coefficient-domain residues.
void orc_divround(void* h, const int* keep, int nkeep, const int* drop, int ndrop,
                  const uint64_t* x_keep, const uint64_t* x_drop, uint64_t* out) {
  Ctx* c = (Ctx*)h;
  const int N = c->N;
  std::vector<const u64*> xk, xd;
  std::vector<u64*> o;
  for (int i = 0; i < nkeep; ++i) { xk.push_back(x_keep + (size_t)i * N); o.push_back(out + (size_t)i * N); }
  for (int i = 0; i < ndrop; ++i) xd.push_back(x_drop + (size_t)i * N);
  divround(*c, std::vector<int>(keep, keep + nkeep), std::vector<int>(drop, drop + ndrop), xk, xd, o);
}

// vec_mat with ONE ModDown (DESIGN.md §3 "lazy ModDown"): the key-switch
// inner products of all rotations are weighted by their diagonals and summed
// in the extended basis Q_l P before a single DivRound by P:
//   acc_p[t] = sum_{k>=1} D_k[t] . sum_j NTT_t([D_j(phi_k(c1))]_t) . ksk_k[j][p][t]
//            + [t data limb] [P]_t (D_0[t] . c_p[t] + [p=0] sum_{k>=1} D_k[t] . phi_k(c0)[t])
//   out_p = ModDown(acc_p)   (INTT, C15 DivRound by P, NTT; exact: ModDown(P X + Y) = X + ModDown(Y)).
// diags: [n][l+1+K][N] NTT words, data limbs 0..l then the K special limbs.
// Written unhoisted (phi_k applied to the ciphertext in the coefficient domain,
// then the textbook key-switch digit lift), i.e. from the definitions.
int orc_vec_mat_lazy_step(void* h, const uint64_t* ct, int level, const uint64_t* diags, int n, int step,
                          uint64_t* out);
int orc_vec_mat_lazy(void* h, const uint64_t* ct, int level, const uint64_t* diags, int n, uint64_t* out) {
  return orc_vec_mat_lazy_step(h, ct, level, diags, n, 1, out);
}
// Same with diagonal k applied to rot(ct, k * step) (strided rotation sums).
int orc_vec_mat_lazy_step(void* h, const uint64_t* ct, int level, const uint64_t* diags, int n, int step,
                          uint64_t* out) {
  Ctx* c = (Ctx*)h;
  const int N = c->N, Lc = level + 1, lk = LK(*c), nt = Lc + c->K;
  const size_t P_ = (size_t)Lc * N;
  std::vector<int> targets;
  for (int i = 0; i < Lc; ++i) targets.push_back(i);
  for (int k = 0; k < c->K; ++k) targets.push_back(c->L + k);
  std::vector<u64> Pmod(nt);
  for (int ti = 0; ti < nt; ++ti) {
    u64 p = 1;
    for (int k = 0; k < c->K; ++k) p = mulmod(p, c->q[c->L + k] % c->q[targets[ti]], c->q[targets[ti]]);
    Pmod[ti] = p;
  }
  // acc[part][ti][n]
  std::vector<u64> acc((size_t)2 * nt * N, 0);
  auto A = [&](int p, int ti) { return &acc[((size_t)p * nt + ti) * N]; };
  auto D = [&](int k, int ti) { return diags + ((size_t)k * nt + ti) * N; };
  // k = 0: P D_0 c_p on the data limbs
  for (int p = 0; p < 2; ++p)
    for (int i = 0; i < Lc; ++i)
      for (int m = 0; m < N; ++m)
        A(p, i)[m] = addmod(A(p, i)[m], mulmod(Pmod[i], mulmod(D(0, i)[m], ct[p * P_ + (size_t)i * N + m], c->q[i]),
                                               c->q[i]), c->q[i]);
  std::vector<u64> phi(2 * P_), tmp(N), Dt(N);
  std::vector<std::vector<i64>> Dj(Lc, std::vector<i64>(N));
  for (int k = 1; k < n; ++k) {
    const u64 g = galois_elt(*c, k * step);
    auto it = c->gk.find(g);
    if (it == c->gk.end()) return -1;
    const std::vector<u64>& ksk = it->second;
    for (int p = 0; p < 2; ++p)
      for (int i = 0; i < Lc; ++i) {
        std::memcpy(tmp.data(), ct + (size_t)p * P_ + (size_t)i * N, N * 8);
        intt_limb(*c, i, tmp.data());
        u64* o = &phi[(size_t)p * P_ + (size_t)i * N];
        automorph_coeff(tmp.data(), o, N, g, c->q[i]);
        ntt_limb(*c, i, o);
      }
    // P D_k phi_k(c0) on the data limbs
    for (int i = 0; i < Lc; ++i)
      for (int m = 0; m < N; ++m)
        A(0, i)[m] = addmod(A(0, i)[m], mulmod(Pmod[i], mulmod(D(k, i)[m], phi[(size_t)i * N + m], c->q[i]), c->q[i]),
                            c->q[i]);
    // digits of phi_k(c1): INTT, centered lift (C16)
    for (int j = 0; j < Lc; ++j) {
      std::memcpy(tmp.data(), &phi[P_ + (size_t)j * N], N * 8);
      intt_limb(*c, j, tmp.data());
      for (int m = 0; m < N; ++m) Dj[j][m] = centered(tmp[m], c->q[j]);
    }
    for (int ti = 0; ti < nt; ++ti) {
      const int t = targets[ti];
      const u64 qt = c->q[t];
      for (int j = 0; j < Lc; ++j) {
        signed_to_ntt(*c, Dj[j].data(), t, Dt.data());
        const u64* kb = &ksk[(((size_t)j * 2 + 0) * lk + t) * N];
        const u64* ka = &ksk[(((size_t)j * 2 + 1) * lk + t) * N];
        for (int m = 0; m < N; ++m) {
          const u64 d = mulmod(D(k, ti)[m], Dt[m], qt);
          A(0, ti)[m] = addmod(A(0, ti)[m], mulmod(d, kb[m], qt), qt);
          A(1, ti)[m] = addmod(A(1, ti)[m], mulmod(d, ka[m], qt), qt);
        }
      }
    }
  }
  // one ModDown per part
  std::vector<int> keep(targets.begin(), targets.begin() + Lc), drop(targets.begin() + Lc, targets.end());
  for (int p = 0; p < 2; ++p) {
    for (int ti = 0; ti < nt; ++ti) intt_limb(*c, targets[ti], A(p, ti));
    std::vector<const u64*> xk, xd;
    std::vector<u64*> o;
    for (int i = 0; i < Lc; ++i) {
      xk.push_back(A(p, i));
      o.push_back(out + (size_t)p * P_ + (size_t)i * N);
    }
    for (int k = 0; k < c->K; ++k) xd.push_back(A(p, Lc + k));
    divround(*c, keep, drop, xk, xd, o);
    for (int i = 0; i < Lc; ++i) ntt_limb(*c, i, o[i]);
  }
  return 0;
}

// Signed coefficients -> NTT words on data limbs 0..l and the K special limbs.
void orc_coeffs_to_pt_qp(void* h, const int64_t* m, int level, uint64_t* pt) {
  Ctx* c = (Ctx*)h;
  for (int i = 0; i <= level; ++i) signed_to_ntt(*c, m, i, pt + (size_t)i * c->N);
  for (int k = 0; k < c->K; ++k) signed_to_ntt(*c, m, c->L + k, pt + (size_t)(level + 1 + k) * c->N);
}

}  // extern "C"
