// he_host.cpp — host precomputation for the B200 CKKS context
// ("Primes (C2), psi (C4), twiddles psi^brv and Shoup
// companions, inverse twiddles and N^{-1}, q_l^{-1} mod q_i, [P]_{q_j},
// P^{-1} mod q_i, (P/p_k)^{-1} mod p_k, [P/p_k]_{q_i}, Galois elements").
//
// Product code: written independently of oracle/ (which the product never
// includes or links).  Compiled with g++ (needs libquadmath for the CDT).
#include "he_host.h"

#include <quadmath.h>

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace he {

static u64 mul_mod(u64 a, u64 b, u64 q) { return (u64)((u128)a * b % q); }

u64 pow_mod(u64 a, u64 e, u64 q) {
  u64 r = 1 % q;
  a %= q;
  for (; e; e >>= 1) {
    if (e & 1) r = mul_mod(r, a, q);
    a = mul_mod(a, a, q);
  }
  return r;
}

static u64 inv_mod(u64 a, u64 q) { return pow_mod(a, q - 2, q); }  // q prime

// Miller-Rabin with the first 12 prime bases: deterministic below 3.3e24.
bool is_prime_u64(u64 n) {
  if (n < 2) return false;
  const u64 small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  for (u64 p : small)
    if (n % p == 0) return n == p;
  u64 d = n - 1;
  int r = 0;
  while (!(d & 1)) { d >>= 1; ++r; }
  for (u64 a : small) {
    u64 x = pow_mod(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool witness = true;
    for (int i = 1; i < r && witness; ++i) {
      x = mul_mod(x, x, n);
      if (x == n - 1) witness = false;
    }
    if (witness) return false;
  }
  return true;
}

static int bit_length(u64 x) { return 64 - __builtin_clzll(x); }

static unsigned brv(unsigned x, int bits) {
  unsigned r = 0;
  for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1u) << (bits - 1 - i);
  return r;
}

// C2: per requested size b (list order), the largest unused prime
// 2^{b-1} < p < 2^b with p = 1 (mod 2N).
static std::vector<u64> choose_primes(const std::vector<int>& bits, int N) {
  const u64 step = 2 * (u64)N;
  std::vector<u64> out;
  for (int b : bits) {
    if (b < 20 || b > 60) throw std::runtime_error("prime bit size must be in [20, 60]");
    const u64 hi = 1ULL << b, lo = 1ULL << (b - 1);
    u64 c = ((hi - 2) / step) * step + 1;  // largest candidate < 2^b with c = 1 mod 2N
    for (;; c -= step) {
      if (c <= lo) throw std::runtime_error("not enough NTT-friendly primes of the requested size");
      if (std::find(out.begin(), out.end(), c) == out.end() && is_prime_u64(c)) break;
    }
    out.push_back(c);
  }
  return out;
}

// C4: the smallest primitive 2N-th root of unity mod q.  The primitive roots
// are exactly x^{(q-1)/2N} raised to odd powers, for any x whose
// x^{(q-1)/2N} has order 2N (i.e. its N-th power is -1).
static u64 smallest_psi(u64 q, int N) {
  const u64 M = 2 * (u64)N;
  u64 g = 0;
  for (u64 x = 2; !g; ++x) {
    u64 c = pow_mod(x, (q - 1) / M, q);
    if (pow_mod(c, (u64)N, q) == q - 1) g = c;
  }
  const u64 g2 = mul_mod(g, g, q);
  u64 best = g, cur = g;
  for (u64 e = 3; e < M; e += 2) {
    cur = mul_mod(cur, g2, q);
    best = std::min(best, cur);
  }
  return best;
}

u64 galois_element(int N, int step) {
  const int ns = N / 2;
  const int e = step > 0 ? step : ns + step;
  return pow_mod(5, (u64)e, 2 * (u64)N);
}

ConvGeom conv_geometry(int H, int W, int kh, int kw, int stride) {
  ConvGeom g;
  g.oh = (H - kh) / stride + 1;
  g.ow = (W - kw) / stride + 1;
  g.windows = g.oh * g.ow;
  g.chunk = 1;
  while (g.chunk < g.windows) g.chunk <<= 1;
  return g;
}

// ------------------------------------------------------------ multiword ---
// Little-endian base-2^64 integers, just enough for the CRT constants.
typedef std::vector<u64> Words;
static Words w_mul(const Words& a, u64 m) {
  Words r(a.size() + 1, 0);
  u128 c = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    u128 t = (u128)a[i] * m + c;
    r[i] = (u64)t;
    c = t >> 64;
  }
  r[a.size()] = (u64)c;
  return r;
}
static u64 w_mod(const Words& a, u64 q) {
  u128 r = 0;
  for (size_t i = a.size(); i-- > 0;) r = ((r << 64) | a[i]) % q;
  return (u64)r;
}
static Words w_half(const Words& a) {
  Words r(a.size(), 0);
  for (size_t i = 0; i < a.size(); ++i) r[i] = (a[i] >> 1) | (i + 1 < a.size() ? a[i + 1] << 63 : 0);
  return r;
}
static Words w_resize(Words a, size_t n) {
  for (size_t i = n; i < a.size(); ++i)
    if (a[i]) throw std::runtime_error("multiword overflow");
  a.resize(n, 0);
  return a;
}

// C11: T[k] = floor(2^63 Pr(|X| <= k)) for the discrete Gaussian with
// rho(x) = exp(-x^2 / (2 sigma^2)), sigma = 3.2, support |x| <= 19, in
// binary128 arithmetic (113-bit significand); T[19] = 2^63 exactly.
static std::vector<u64> cdt_table() {
  const int bound = 19;
  const __float128 sigma = strtoflt128("3.2", nullptr);
  __float128 rho[bound + 1], total = 0;
  for (int x = 0; x <= bound; ++x) {
    rho[x] = expq(-(__float128)(x * x) / (2 * sigma * sigma));
    total += x == 0 ? rho[x] : 2 * rho[x];
  }
  std::vector<u64> T(bound + 1);
  __float128 run = 0;
  const __float128 two63 = ldexpq((__float128)1, 63);
  for (int k = 0; k <= bound; ++k) {
    run += k == 0 ? rho[0] : 2 * rho[k];
    T[k] = (u64)floorq(two63 * run / total);
  }
  T[bound] = 1ULL << 63;
  return T;
}

HostParams make_params(int logN, const std::vector<int>& bits, int n_special) {
  if (logN < 10 || logN > 15) throw std::runtime_error("log2N must be in [10, 15]");
  if (bits.empty() || bits.size() > 64) throw std::runtime_error("n_primes must be in [1, 64]");
  if (n_special < 0 || n_special > 2) throw std::runtime_error("n_special must be 0, 1 or 2");
  if ((int)bits.size() - n_special < 1) throw std::runtime_error("need at least one data prime");
  HostParams h;
  h.logN = logN;
  h.N = 1 << logN;
  h.K = n_special;
  h.L = (int)bits.size() - n_special;
  const int N = h.N, NP = h.L + h.K;
  h.q = choose_primes(bits, N);
  for (u64 q : h.q) {
    h.psi.push_back(smallest_psi(q, N));
    const int k = bit_length(q);
    h.kbits.push_back(k);
    h.mu.push_back((u64)(((u128)1 << (2 * k)) / q));
  }
  // twiddles: psi^{brv(i)} (forward, merged-psi Cooley-Tukey) and
  // psi^{-brv(i)} (inverse, Gentleman-Sande), with Shoup companions.
  h.tw.resize((size_t)NP * N);
  h.twsh.resize((size_t)NP * N);
  h.itw.resize((size_t)NP * N);
  h.itwsh.resize((size_t)NP * N);
  for (int t = 0; t < NP; ++t) {
    const u64 q = h.q[t], psi = h.psi[t], ipsi = inv_mod(psi, q);
    std::vector<u64> pw(N), ipw(N);
    pw[0] = ipw[0] = 1;
    for (int i = 1; i < N; ++i) {
      pw[i] = mul_mod(pw[i - 1], psi, q);
      ipw[i] = mul_mod(ipw[i - 1], ipsi, q);
    }
    for (int i = 0; i < N; ++i) {
      const unsigned r = brv((unsigned)i, logN);
      const size_t o = (size_t)t * N + i;
      h.tw[o] = pw[r];
      h.itw[o] = ipw[r];
      h.twsh[o] = (u64)(((u128)pw[r] << 64) / q);
      h.itwsh[o] = (u64)(((u128)ipw[r] << 64) / q);
    }
    const u64 ni = inv_mod((u64)N % q, q);
    h.ninv.push_back(ni);
    h.ninvsh.push_back((u64)(((u128)ni << 64) / q));
  }
  // ModDown constants (C15 with B = P).
  Words P{1};
  for (int k = 0; k < h.K; ++k) P = w_mul(P, h.q[h.L + k]);
  const Words Ph = w_half(P);
  h.P_mod.resize(NP);
  h.Pinv_mod.assign(NP, 0);
  h.Ph_mod.resize(NP);
  for (int t = 0; t < NP; ++t) {
    h.P_mod[t] = w_mod(P, h.q[t]);
    h.Ph_mod[t] = w_mod(Ph, h.q[t]);
    if (t < h.L && h.K > 0) h.Pinv_mod[t] = inv_mod(h.P_mod[t], h.q[t]);
  }
  h.Phat_inv.resize(h.K);
  h.Phat_mod.resize((size_t)h.K * NP);
  for (int k = 0; k < h.K; ++k) {
    Words Pk{1};
    for (int l = 0; l < h.K; ++l)
      if (l != k) Pk = w_mul(Pk, h.q[h.L + l]);
    h.Phat_inv[k] = inv_mod(w_mod(Pk, h.q[h.L + k]), h.q[h.L + k]);
    for (int t = 0; t < NP; ++t) h.Phat_mod[(size_t)k * NP + t] = w_mod(Pk, h.q[t]);
  }
  // rescale constants (C15 with B = q_l)
  h.rs_qinv.assign((size_t)h.L * h.L, 0);
  h.rs_h.assign((size_t)h.L * h.L, 0);
  for (int l = 1; l < h.L; ++l)
    for (int i = 0; i < l; ++i) {
      h.rs_qinv[(size_t)l * h.L + i] = inv_mod(h.q[l] % h.q[i], h.q[i]);
      h.rs_h[(size_t)l * h.L + i] = ((h.q[l] - 1) / 2) % h.q[i];
    }
  // CRT decode constants per level: Qhat_inv[Lc] | Qhat[Lc][Lc] | Q[Lc] | Qhalf[Lc]
  for (int l = 0; l < h.L; ++l) {
    const int Lc = l + 1;
    h.crt_off.push_back(h.crt_words.size());
    Words Q{1};
    for (int i = 0; i < Lc; ++i) Q = w_mul(Q, h.q[i]);
    std::vector<Words> Qhat(Lc);
    for (int i = 0; i < Lc; ++i) {
      Words t{1};
      for (int j = 0; j < Lc; ++j)
        if (j != i) t = w_mul(t, h.q[j]);
      Qhat[i] = w_resize(t, Lc);
      h.crt_words.push_back(inv_mod(w_mod(t, h.q[i]), h.q[i]));
    }
    for (int i = 0; i < Lc; ++i)
      for (int w = 0; w < Lc; ++w) h.crt_words.push_back(Qhat[i][w]);
    const Words Qr = w_resize(Q, Lc), Qh = w_resize(w_half(Q), Lc);
    for (int w = 0; w < Lc; ++w) h.crt_words.push_back(Qr[w]);
    for (int w = 0; w < Lc; ++w) h.crt_words.push_back(Qh[w]);
  }
  h.cdt = cdt_table();
  // canonical embedding (C6): slot j <-> zeta^{5^j}, 5^j = 4 r_j + 1 (mod 2N)
  const int M = N / 2;
  h.slot_index.resize(M);
  u64 g = 1;
  for (int j = 0; j < M; ++j) {
    h.slot_index[j] = (int)((g - 1) / 4);
    g = (g * 5) % (2 * (u64)N);
  }
  h.fft_w.resize(2 * (size_t)M);
  h.zeta_pow.resize(2 * (size_t)M);
  const long double pi = acosl(-1.0L);
  for (int k = 0; k < M; ++k) {
    const long double a = 2.0L * pi * (long double)k / (long double)M;
    h.fft_w[2 * k] = (double)cosl(a);
    h.fft_w[2 * k + 1] = (double)sinl(a);
    const long double b = pi * (long double)k / (long double)N;
    h.zeta_pow[2 * k] = (double)cosl(b);
    h.zeta_pow[2 * k + 1] = (double)sinl(b);
  }
  return h;
}

}  // namespace he
