// he_host.h — host-side parameter precomputation for the CKKS context
// (SURVEY.md §8(a) a1).  Product code; independent of oracle/.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace he {

typedef uint64_t u64;
typedef unsigned __int128 u128;

// Everything a1 lists: primes (C2), psi (C4), twiddles + Shoup companions,
// N^{-1}, Barrett constants, RNS constants for rescale / ModDown / keygen /
// CRT decode, the CDT table (C11) and the float64 FFT tables of the
// canonical embedding (C6).
struct HostParams {
  int logN = 0, N = 0, L = 0, K = 0;
  std::vector<u64> q, psi;          // L+K primes (specials last) and their psi
  std::vector<int> kbits;           // bit length of q
  std::vector<u64> mu;              // floor(2^{2k} / q)  (Barrett, k = bit length)
  std::vector<u64> tw, twsh;        // [NP][N] psi^{brv(i)} and floor(w 2^64 / q)
  std::vector<u64> itw, itwsh;      // [NP][N] psi^{-brv(i)} and Shoup companions
  std::vector<u64> ninv, ninvsh;    // N^{-1} mod q and its Shoup companion
  // ModDown by P = prod p_k (C15 with B = P), indexed by absolute prime index
  std::vector<u64> P_mod;           // [NP] P mod q_t (keygen: [P]_{q_j})
  std::vector<u64> Pinv_mod;        // [NP] P^{-1} mod q_i (data primes only; 0 for specials)
  std::vector<u64> Ph_mod;          // [NP] floor(P/2) mod q_t
  std::vector<u64> Phat_inv;        // [K] (P/p_k)^{-1} mod p_k
  std::vector<u64> Phat_mod;        // [K][NP] (P/p_k) mod q_t
  // rescale at level l (drop q_l): [l][i] for i < l
  std::vector<u64> rs_qinv;         // [L][L] q_l^{-1} mod q_i
  std::vector<u64> rs_h;            // [L][L] ((q_l-1)/2) mod q_i
  // CRT decode at level l (Lc = l+1): offsets into crt_* arrays
  std::vector<size_t> crt_off;      // [L]  start of level l's block
  std::vector<u64> crt_words;       // per level: Qhat_inv[Lc], Qhat[Lc][Lc words], Q[Lc], Qhalf[Lc]
  std::vector<u64> cdt;             // 20 words, T[k] = floor(2^63 Pr(|X| <= k))
  std::vector<int> slot_index;      // [N/2]  r_j = (5^j mod 2N - 1) / 4
  std::vector<double> fft_w;        // [N/2][2] exp(2 pi i k / (N/2))
  std::vector<double> zeta_pow;     // [N/2][2] exp(pi i k / N)
};

// Throws std::runtime_error with a message on invalid parameters.
HostParams make_params(int logN, const std::vector<int>& bits, int n_special);

// Utilities also used by the C-ABI layer.
bool is_prime_u64(u64 n);
u64 pow_mod(u64 a, u64 e, u64 q);
u64 galois_element(int N, int step);   // C6: 5^k (k>0) or 5^{n_s+k} (k<0) mod 2N

// C17-C19 slot layouts (host, float64) used by the composite ops.
struct ConvGeom { int oh, ow, windows, chunk; };
ConvGeom conv_geometry(int H, int W, int kh, int kw, int stride);

}  // namespace he
