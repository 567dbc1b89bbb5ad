// he_jobs.cuh — load/store functors that fuse each CKKS step into the NTT
// kernels of he_ntt.cuh (SURVEY.md §8(a) kernels K1-K7).  Product code.
#pragma once
#include <type_traits>
#include <utility>

#include "he_common.cuh"

namespace he {

// ---- per-block binding for the 32-bit engine (k_ntt32) ----------------------
// A job may provide bind32(blk, P) returning an object with load(n) / store(n, v): the block's
// decomposition, row pointers and 32-bit constants are computed once per CTA instead of per
// element.  k_ntt32 runs only on contexts whose primes are all < 2^31, so bound jobs use u32
// arithmetic.  Jobs without bind32 go through JobAt (their per-element load/store).
__device__ __forceinline__ u32 add32(u32 a, u32 b, u32 q) { return min(a + b, a + b - q); }
__device__ __forceinline__ u32 sub32(u32 a, u32 b, u32 q) { return min(a - b, a - b + q); }
__device__ __forceinline__ u32 red32(u32 x, u32 q, u32 mu32) {   // x mod q, mu32 = floor(2^32 / q)
  const u32 r = x - __umulhi(x, mu32) * q;
  return min(r, r - q);
}
__device__ __forceinline__ u32 mulsh32(u32 x, u32 w, u32 wsh, u32 q) {   // Shoup, x < 2^32, w < q
  const u32 r = x * w - __umulhi(x, wsh) * q;
  return min(r, r - q);
}
__device__ __forceinline__ u32 shoup_companion32(u32 w, u32 q) { return (u32)(((u64)w << 32) / q); }
__device__ __forceinline__ u32 mu32_of(const PrimeD& P) { return (u32)(P.mu64 >> 32); }

template <class B, class = void>
struct has_store4 : std::false_type {};
template <class B>
struct has_store4<B, std::void_t<decltype(std::declval<const B&>().store4(0u, 0u, (const u32*)nullptr))>>
    : std::true_type {};

// Epilogue operand rows a pipelined block will read after its passes: one thread asks the TMA engine
// to pull them into L2 when the block starts (cp.async.bulk.prefetch.L2), so the epilogue's loads hit
// L2 instead of waiting on DRAM.  Rows are 16-byte aligned and N * 4 or N * 8 bytes.
__device__ __forceinline__ void prefetch_l2(const void* p, u32 bytes) {
  if (p) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}
template <class B, class = void>
struct has_prefetch : std::false_type {};
template <class B>
struct has_prefetch<B, std::void_t<decltype(std::declval<const B&>().prefetch(0u))>> : std::true_type {};
// Pipelined jobs whose input is the staged u32 row combined with a second row read from global memory
// in the first pass (load_raw_at(staged word, index)): the rescale-fused ModDown (JobKsDataRs).
template <class B, class = void>
struct has_load_raw_at : std::false_type {};
template <class B>
struct has_load_raw_at<B, std::void_t<decltype(std::declval<const B&>().load_raw_at(0u, 0u))>> : std::true_type {};

template <class J, class = void>
struct has_gather_src : std::false_type {};
template <class J>
struct has_gather_src<J, std::void_t<decltype(std::declval<const J&>().gather_src(0u))>> : std::true_type {};

template <class B, class = void>
struct has_load4 : std::false_type {};
template <class B>
struct has_load4<B, std::void_t<decltype(std::declval<const B&>().load4(0u))>> : std::true_type {};

// Words a thread of the NTT kernels keeps in flight in its HBM-facing loops (chunks that are not
// interleaved, so registers stay bounded).  Jobs whose per-word load / store is itself a long
// computation (the key-switch inner products) set kIoWords lower.
template <class J, class = void>
struct io_words_of { static constexpr int value = 8; };
template <class J>
struct io_words_of<J, std::void_t<decltype(J::kIoWords)>> { static constexpr int value = J::kIoWords; };

template <class Job>
struct JobAt {
  const Job& j;
  int blk;
  const PrimeD& P;
  __device__ __forceinline__ u64 load(u32 i) const { return j.load(blk, i, P); }
  __device__ __forceinline__ void store(u32 i, u64 v) const { j.store(blk, i, v, P); }
};
template <class Job>
__device__ __forceinline__ auto bind_job(const Job& j, int blk, const PrimeD& P, int) -> decltype(j.bind32(blk, P)) {
  return j.bind32(blk, P);
}
template <class Job>
__device__ __forceinline__ JobAt<Job> bind_job(const Job& j, int blk, const PrimeD& P, long) {
  return JobAt<Job>{j, blk, P};
}

// Plain transform of limbs: blk -> (item = blk / nl, limb = blk % nl), limb l
// modulo prime l; items at strides src_bs / dst_bs words.
struct JobLimbs {
  static constexpr const char* kName = "ntt_limbs";
  const u64* src;
  u64* dst;
  int N, nl;
  size_t src_bs, dst_bs;
  __device__ int prime(int blk) const { return blk % nl; }
  __device__ u64 load(int blk, u32 i, const PrimeD&) const {
    return src[(size_t)(blk / nl) * src_bs + (size_t)(blk % nl) * N + i];
  }
  __device__ void store(int blk, u32 i, u64 v, const PrimeD&) const {
    dst[(size_t)(blk / nl) * dst_bs + (size_t)(blk % nl) * N + i] = v;
  }
  struct B32 {
    const u64* s;
    u64* d;
    __device__ __forceinline__ u64 load(u32 i) const { return s[i]; }
    __device__ __forceinline__ void store(u32 i, u64 v) const { d[i] = v; }
  };
  __device__ B32 bind32(int blk, const PrimeD&) const {
    const size_t it = (size_t)(blk / nl), l = (size_t)(blk % nl);
    return B32{src + it * src_bs + l * N, dst + it * dst_bs + l * N};
  }
};

// Plain transform writing u32 words (small-prime contexts: every residue < 2^31).
struct JobLimbsTo32 {
  static constexpr const char* kName = "ntt_limbs";
  const u64* src;
  u32* dst;
  int N, nl;
  size_t src_bs, dst_bs;
  int sq = 0;   // 1: transform src^2 (the square's d2 = x1^2, formed here instead of by a tensor)
  __device__ int prime(int blk) const { return blk % nl; }
  __device__ u64 load(int blk, u32 i, const PrimeD& P) const {
    const u64 v = src[(size_t)(blk / nl) * src_bs + (size_t)(blk % nl) * N + i];
    return sq ? mul_mod(v, v, P) : v;
  }
  __device__ void store(int blk, u32 i, u64 v, const PrimeD&) const {
    dst[(size_t)(blk / nl) * dst_bs + (size_t)(blk % nl) * N + i] = (u32)v;
  }
  struct B32 {
    const u64* s;
    u32* d;
    const PrimeD* P;
    int sq;
    __device__ __forceinline__ u64 load(u32 i) const { return sq ? mul_mod(s[i], s[i], *P) : s[i]; }
    __device__ __forceinline__ void store(u32 i, u64 v) const { d[i] = (u32)v; }
  };
  __device__ B32 bind32(int blk, const PrimeD& P) const {
    const size_t it = (size_t)(blk / nl), l = (size_t)(blk % nl);
    return B32{src + it * src_bs + l * N, dst + it * dst_bs + l * N, &P, sq};
  }
};
inline double alg_bytes(const JobLimbsTo32& j, int nblk) { return 12.0 * j.N * nblk; }

// Fused ring product out = INTT(NTT(a) (.) b) (config 2 "fwd -> modmul -> inv").
struct JobRingMul {
  static constexpr const char* kName = "ntt_mul_intt";
  const u64* a;
  const u64* b;
  u64* out;
  int N, nl;
  __device__ int prime(int blk) const { return blk % nl; }
  __device__ u64 load(int blk, u32 i, const PrimeD&) const { return a[(size_t)blk * N + i]; }
  __device__ u64 factor(int blk, u32 i, const PrimeD&) const { return b[(size_t)blk * N + i]; }
  __device__ void store(int blk, u32 i, u64 v, const PrimeD&) const { out[(size_t)blk * N + i] = v; }
};

// Signed small polynomials -> NTT words (encode injection, encryption noise,
// key generation): blk -> (item = blk / nl, limb = blk % nl); reads
// poly[item * src_bs + i] (int64), writes dst[item * dst_bs + limb * N + i].
struct JobSignedToNtt {
  static constexpr const char* kName = "ntt_small";
  const i64* poly;
  u64* dst;
  int N, nl;
  size_t src_bs, dst_bs;
  int lc, L;   // limbs >= lc are special limbs (prime L + limb - lc); lc = nl: data limbs only
  __device__ int prime(int blk) const {
    const int l = blk % nl;
    return l < lc ? l : L + (l - lc);
  }
  __device__ u64 load(int blk, u32 i, const PrimeD& P) const {
    return from_signed(poly[(size_t)(blk / nl) * src_bs + i], P);
  }
  __device__ void store(int blk, u32 i, u64 v, const PrimeD&) const {
    dst[(size_t)(blk / nl) * dst_bs + (size_t)(blk % nl) * N + i] = v;
  }
};

// Fused encryption (C13, kernel K8): the small polynomial of one draw (v
// ternary C10, e0 / e1 CDT C11) is sampled inside the transform's load from
// Philox stream (purpose, stream_id + b), and the transform's store
// accumulates it into the ciphertext:
//   which 0 (v):  c0 = v b + m,  c1 = v a;   which 1 (e0): c0 += e0;   which 2 (e1): c1 += e1.
struct JobEncrypt {
  static constexpr const char* kName = "encrypt_ntt";
  u64* ct;                 // [B][2][Lc][N]
  const u64* pk;           // [2][L][N]
  const u64* pt;           // [Bp][Lc][N]
  size_t pt_bs;
  const u64* cdt;          // 20-entry table
  u64 seed, stream0;
  int N, Lc, L, which;
  // fused encode + encrypt (he_encode_encrypt): the message's signed coefficients [B][N] instead of
  // plaintext words; the e0 pass transforms e0 + m (NTT is linear, so c0 has the same words)
  const i64* mco = nullptr;
  __device__ int prime(int blk) const { return blk % Lc; }
  __device__ u64 load(int blk, u32 n, const PrimeD& P) const {
    const u64 obj = stream0 + (u64)(blk / Lc);
    if (which == 0) return from_signed(sample_ternary(seed, stream_sid(PUR_ENC_V, obj, 0), n), P);
    i64 e = sample_cdt(seed, stream_sid(which == 1 ? PUR_ENC_E0 : PUR_ENC_E1, obj, 0), n, cdt);
    if (which == 1 && mco) e += mco[(size_t)(blk / Lc) * N + n];
    return from_signed(e, P);
  }
  __device__ void store(int blk, u32 n, u64 v, const PrimeD& P) const {
    const int b = blk / Lc, i = blk % Lc;
    const size_t LN = (size_t)Lc * N;
    u64* c0 = ct + (size_t)b * 2 * LN + (size_t)i * N + n;
    u64* c1 = c0 + LN;
    if (which == 0) {
      const u64 m = pt ? pt[(size_t)b * pt_bs + (size_t)i * N + n] : 0;
      *c0 = add_mod(mul_mod(v, pk[(size_t)i * N + n], P), m, P.q);
      *c1 = mul_mod(v, pk[((size_t)L + i) * N + n], P);
    } else if (which == 1) {
      *c0 = add_mod(*c0, v, P.q);
    } else {
      *c1 = add_mod(*c1, v, P.q);
    }
  }
  // 32-bit engine: load4(j) draws coefficients 4j..4j+3 from one Philox block (ternary) or two
  // (CDT) instead of one block per coefficient; the store is u32 arithmetic on bound rows
  struct B32 {
    const PrimeD* P;
    const u64* cdt;
    u64 seed, sid;
    u64* c0;
    u64* c1;
    const u64* pkb;
    const u64* pka;
    const u64* m;
    u32 q;
    int which;
    const i64* mc;   // fused encode + encrypt: this item's message coefficients (e0 pass), else null
    __device__ __forceinline__ u32 res(i64 v) const { return v < 0 ? q - (u32)(-v) : (u32)v; }
    // e0 + m (m up to 2^62 in magnitude): a full signed reduction
    __device__ __forceinline__ u32 resm(i64 e, u32 n) const { return (u32)from_signed(e + mc[n], *P); }
    __device__ __forceinline__ uint4 load4(u32 j) const {
      if (which == 0) {
        const uint4 b = philox_block(seed, sid, j);
        auto t = [&](u32 w) { return res((i64)(((u64)w * 3u) >> 32) - 1); };
        return make_uint4(t(b.x), t(b.y), t(b.z), t(b.w));
      }
      if (mc)
        return make_uint4(resm(sample_cdt(seed, sid, 4 * j, cdt), 4 * j),
                          resm(sample_cdt(seed, sid, 4 * j + 1, cdt), 4 * j + 1),
                          resm(sample_cdt(seed, sid, 4 * j + 2, cdt), 4 * j + 2),
                          resm(sample_cdt(seed, sid, 4 * j + 3, cdt), 4 * j + 3));
      return make_uint4(res(sample_cdt(seed, sid, 4 * j, cdt)), res(sample_cdt(seed, sid, 4 * j + 1, cdt)),
                        res(sample_cdt(seed, sid, 4 * j + 2, cdt)), res(sample_cdt(seed, sid, 4 * j + 3, cdt)));
    }
    __device__ __forceinline__ u64 load(u32 n) const {
      if (which == 0) return res(sample_ternary(seed, sid, n));
      return mc ? resm(sample_cdt(seed, sid, n, cdt), n) : res(sample_cdt(seed, sid, n, cdt));
    }
    __device__ __forceinline__ void store(u32 n, u64 v) const {
      if (which == 0) {
        c0[n] = m ? add32((u32)mul_mod(v, pkb[n], *P), (u32)m[n], q) : (u32)mul_mod(v, pkb[n], *P);
        c1[n] = (u32)mul_mod(v, pka[n], *P);
      } else if (which == 1) {
        c0[n] = add32((u32)c0[n], (u32)v, q);
      } else {
        c1[n] = add32((u32)c1[n], (u32)v, q);
      }
    }
  };
  __device__ B32 bind32(int blk, const PrimeD& P) const {
    const int b = blk / Lc, i = blk % Lc;
    const size_t LN = (size_t)Lc * N;
    const u64 obj = stream0 + (u64)b;
    const u64 pur = which == 0 ? PUR_ENC_V : which == 1 ? PUR_ENC_E0 : PUR_ENC_E1;
    u64* c0 = ct + (size_t)b * 2 * LN + (size_t)i * N;
    return B32{&P, cdt, seed, stream_sid(pur, obj, 0), c0, c0 + LN, pk + (size_t)i * N, pk + ((size_t)L + i) * N,
               pt ? pt + (size_t)b * pt_bs + (size_t)i * N : nullptr, (u32)P.q, which,
               mco && which == 1 ? mco + (size_t)b * N : nullptr};
  }
};
inline double alg_bytes(const JobEncrypt& j, int nblk) {
  return j.which == 0 ? 8.0 * j.N * nblk * 4 : 8.0 * j.N * nblk * 2;
}

// ModUp (a9, first half): digit j's coefficient residues [d]_{q_j} (already
// INTT'd), centered lift (C16) into target t != j, NTT_t.
//   coef: [B][Lc][N]; ext: [B][Lc][Lc+K][N] (t < Lc data, t >= Lc special).
struct JobModUp {
  static constexpr const char* kName = "ks_modup";
  const u64* coef;
  u64* ext;
  const u64* qtab;   // device table of all primes
  int N, Lc, K, L;
  // gal != 1: the extended digits are stored already permuted by the rotation, ext[n] = X[pi_g(n)]
  // (gathered from shared memory in the transform's epilogue), so the inner product reads them
  // coalesced (k_ks_ip64).  pi_g keeps the top index bit for g = 5^k (the halves of a 2-CTA limb).
  u32 gal = 1;
  int logN = 0;
  __device__ __forceinline__ u32 gather_src(u32 n) const { return gal == 1 ? n : galois_src(n, gal, logN); }
  __device__ void dec(int blk, int& b, int& j, int& t) const {
    const int nt = Lc + K - 1;
    b = blk / (Lc * nt);
    const int r = blk % (Lc * nt);
    j = r / nt;
    const int tt = r % nt;
    t = tt < j ? tt : tt + 1;
  }
  __device__ int prime(int blk) const {
    int b, j, t;
    dec(blk, b, j, t);
    return t < Lc ? t : L + (t - Lc);
  }
  __device__ u64 load(int blk, u32 i, const PrimeD& P) const {
    int b, j, t;
    dec(blk, b, j, t);
    return lift_centered(coef[((size_t)b * Lc + j) * N + i], __ldg(qtab + j), P);
  }
  __device__ void store(int blk, u32 i, u64 v, const PrimeD&) const {
    int b, j, t;
    dec(blk, b, j, t);
    ext[(((size_t)b * Lc + j) * (Lc + K) + t) * N + i] = v;
  }
};

// ModUp for small primes: u32 INTT'd digits in, u32 extended digits out
// (half the traffic of JobModUp); the 32-bit centered lift (C16).
struct JobModUp32 {
  static constexpr const char* kName = "ks_modup";
  const u32* coef;
  u32* ext;
  const u64* qtab;
  int N, Lc, K, L;
  __device__ void dec(int blk, int& b, int& j, int& t) const {
    const int nt = Lc + K - 1;
    b = blk / (Lc * nt);
    const int r = blk % (Lc * nt);
    j = r / nt;
    const int tt = r % nt;
    t = tt < j ? tt : tt + 1;
  }
  __device__ int prime(int blk) const {
    int b, j, t;
    dec(blk, b, j, t);
    return t < Lc ? t : L + (t - Lc);
  }
  __device__ u64 load(int blk, u32 i, const PrimeD& P) const {
    int b, j, t;
    dec(blk, b, j, t);
    return lift32(coef[((size_t)b * Lc + j) * N + i], (u32)__ldg(qtab + j), (u32)P.q, (u32)(P.mu64 >> 32));
  }
  __device__ void store(int blk, u32 i, u64 v, const PrimeD&) const {
    int b, j, t;
    dec(blk, b, j, t);
    ext[(((size_t)b * Lc + j) * (Lc + K) + t) * N + i] = (u32)v;
  }
  struct B32 {
    const u32* c;
    u32* e;
    u32 qj, q, mut;
    __device__ __forceinline__ u64 load(u32 i) const { return lift32(c[i], qj, q, mut); }
    __device__ __forceinline__ u64 load_raw(u32 x) const { return lift32(x, qj, q, mut); }
    __device__ __forceinline__ void store(u32 i, u64 v) const { e[i] = (u32)v; }
  };
  // pipelined transform (k_ntt32_pipe): the block's input is one u32 row
  __host__ __device__ bool pipe_ok() const { return true; }
  __host__ __device__ const u32* raw32(int blk) const {
    const int nt = Lc + K - 1;
    return coef + ((size_t)(blk / (Lc * nt)) * Lc + (blk % (Lc * nt)) / nt) * N;
  }
  __device__ B32 bind32(int blk, const PrimeD& P) const {
    int b, j, t;
    dec(blk, b, j, t);
    return B32{coef + ((size_t)b * Lc + j) * N, ext + (((size_t)b * Lc + j) * (Lc + K) + t) * N,
               (u32)__ldg(qtab + j), (u32)P.q, mu32_of(P)};
  }
};
inline double alg_bytes(const JobModUp32& j, int nblk) {
  const int nt = j.Lc + j.K - 1;
  return 4.0 * j.N * (nblk + (double)nblk / nt);
}

constexpr int KS_KB_MAX = 32;

// Everything the key-switch inner product + ModDown jobs need (a9/a10, C15).
struct KsArgs {
  int N, logN, Lc, L, K, NP, B, KB;
  const u64* ext;          // [B][Lc][Lc+K][N]
  const u64* dsrc;         // digit source (NTT words): item b at dsrc + b*dsrc_bs, limb j at +j*N
  size_t dsrc_bs;
  const u64* keys[KS_KB_MAX];  // per rotation of this launch: [L][2][NP][N]
  u32 gal[KS_KB_MAX];          // Galois element per rotation (1 = identity)
  u64* tb;                 // [KB][B][2][K][N] ModDown intermediates (coefficient domain)
  const u64* Ph_mod;       // floor(P/2) mod q_t  [NP]
  const u64* Pinv_mod;     // P^{-1} mod q_i     [NP]
  const u64* Phat_inv;     // (P/p_k)^{-1} mod p_k [K]
  const u64* Phat_mod;     // (P/p_k) mod q_t   [K][NP]
  const u64* P_mod;        // P mod q_t         [NP] (ModDown fused with the rescale)
  // epilogue (KsData only): out_p = acc_in_p[n] + D (.) (u_p + [p < add_parts] addsrc_p[pi?(n)])
  u64* out;                // item b at out + kk*out_ks + b*out_bs + p*Lc*N + i*N
  size_t out_bs, out_ks;
  const u64* acc_in;       // nullable, same strides as out (may alias out)
  const u64* addsrc;       // nullable, item stride add_bs
  size_t add_bs;
  int add_parts;           // 0, 1 or 2
  int add_gather;          // apply pi_g to the addsrc index
  const u64* D;            // nullable plaintext factor: D + kk*D_ks + i*N
  size_t D_ks;
  // lazy ModDown: when set, the inner products are replaced by the extended-basis
  // accumulator accx[b][part][Lc+K][N] (data limbs then specials), KB = 1;
  // accx32: the accumulator words are u32 (small-prime fused key switch)
  const u64* accx;
  int accx32;
  // square (he_square): poly 0 gets + x0^2 and poly 1 + 2 x0 x1 from x = sq_src (item stride
  // sq_bs, 2 polys), i.e. the tensor's d0 / d1 formed in the epilogue instead of read
  const u64* sq_src = nullptr;
  size_t sq_bs = 0;
};

__device__ __forceinline__ u64 accx_word(const KsArgs& a, size_t i) {
  return a.accx32 ? (u64)reinterpret_cast<const u32*>(a.accx)[i] : a.accx[i];
}

// Inner product over digits at target limb t for source position sn.  The products (each < q^2)
// are summed in 128 bits and reduced once per 8 terms (q < 2^60, so 8 q^2 < 2^123 and the high
// word stays below q): hi 2^64 + lo = [hi (2^64 mod q)]_q + [lo]_q, one Barrett product and one
// 64-bit reduction instead of a Barrett reduction per term.
__device__ __forceinline__ u64 ks_inner(const KsArgs& a, int kk, int b, int part, int t, int tprime,
                                        u32 sn, u32 n, const PrimeD& P) {
  const u64* key = a.keys[kk];
  u64 acc = 0;
  for (int j0 = 0; j0 < a.Lc; j0 += 8) {
    u64 lo = 0, hi = 0;
    const int j1 = min(a.Lc, j0 + 8);
    for (int j = j0; j < j1; ++j) {
      const u64 x = (t == j) ? a.dsrc[(size_t)b * a.dsrc_bs + (size_t)j * a.N + sn]
                             : a.ext[(((size_t)b * a.Lc + j) * (a.Lc + a.K) + t) * a.N + sn];
      const u64 k = key[(((size_t)j * 2 + part) * a.NP + tprime) * a.N + n];
      const u64 pl = x * k, ph = __umul64hi(x, k);
      lo += pl;
      hi += ph + (lo < pl);
    }
    acc = add_mod(acc, add_mod(mul_mod(hi, P.r64, P), reduce64(lo, P), P.q), P.q);
  }
  return acc;
}

// a9 special limbs: inner product at p_k, INTT, then
// tb = [ (x + [P/2]_{p_k}) (P/p_k)^{-1} ]_{p_k}    (C15 y_k and its CRT weight)
struct JobKsSpecial {
  static constexpr const char* kName = "ks_special";
  static constexpr int kIoWords = 2;   // load = an Lc-term 64-bit inner product
  KsArgs a;
  __device__ void dec(int blk, int& kk, int& b, int& part, int& k) const {
    k = blk % a.K;
    int r = blk / a.K;
    part = r & 1;
    r >>= 1;
    b = r % a.B;
    kk = r / a.B;
  }
  __device__ int prime(int blk) const { return a.L + blk % a.K; }
  __device__ u64 load(int blk, u32 n, const PrimeD& P) const {
    int kk, b, part, k;
    dec(blk, kk, b, part, k);
    if (a.accx) return accx_word(a, (((size_t)b * 2 + part) * (a.Lc + a.K) + a.Lc + k) * a.N + n);
    const u32 g = a.gal[kk];
    const u32 sn = g == 1 ? n : galois_src(n, g, a.logN);
    return ks_inner(a, kk, b, part, a.Lc + k, a.L + k, sn, n, P);
  }
  __device__ void store(int blk, u32 n, u64 v, const PrimeD& P) const {
    int kk, b, part, k;
    dec(blk, kk, b, part, k);
    const u64 y = add_mod(v, __ldg(a.Ph_mod + a.L + k), P.q);
    // one special prime: (P/p_0)^{-1} = 1
    a.tb[((((size_t)kk * a.B + b) * 2 + part) * a.K + k) * a.N + n] =
        a.K == 1 ? y : mul_mod(y, __ldg(a.Phat_inv + k), P);
  }
  // lazy ModDown with u32 accumulators and one special prime (the small-prime fused path)
  struct B32 {
    const JobKsSpecial* j;
    int blk;
    const PrimeD* P;
    bool fast;
    const u32* ax;
    u32* tb;
    u32 q, ph;
    __device__ __forceinline__ u64 load(u32 n) const { return fast ? (u64)ax[n] : j->load(blk, n, *P); }
    __device__ __forceinline__ u64 load_raw(u32 x) const { return x; }
    __device__ __forceinline__ void store(u32 n, u64 v) const {
      if (fast) tb[n] = add32((u32)v, ph, q);   // fast path: tb holds u32 words (read by JobKsData)
      else j->store(blk, n, v, *P);
    }
  };
  __device__ B32 bind32(int blk, const PrimeD& P) const {
    int kk, b, part, k;
    dec(blk, kk, b, part, k);
    const bool fast = pipe_ok();
    B32 r{this, blk, &P, fast, nullptr, nullptr, (u32)P.q, 0};
    if (fast) {
      r.ax = raw32(blk);
      r.tb = reinterpret_cast<u32*>(a.tb) + (((size_t)kk * a.B + b) * 2 + part) * a.N;
      r.ph = (u32)__ldg(a.Ph_mod + a.L + k);
    }
    return r;
  }
  // pipelined kernel (pipe_ok): the fast form only, without the generic fallback's registers
  struct P32 {
    u32* tb;
    u32 q, ph;
    __device__ __forceinline__ u64 load_raw(u32 x) const { return x; }
    __device__ __forceinline__ void store(u32 n, u64 v) const { tb[n] = add32((u32)v, ph, q); }
  };
  __device__ P32 bind_pipe(int blk, const PrimeD& P) const {
    int kk, b, part, k;
    dec(blk, kk, b, part, k);
    return P32{reinterpret_cast<u32*>(a.tb) + (((size_t)kk * a.B + b) * 2 + part) * a.N, (u32)P.q,
               (u32)__ldg(a.Ph_mod + a.L + k)};
  }
  // lazy ModDown with u32 accumulators and one special prime: input = one u32 accumulator row
  __host__ __device__ bool pipe_ok() const { return a.accx && a.accx32 && a.K == 1; }
  __host__ __device__ const u32* raw32(int blk) const {
    const int b = (blk >> 1) % a.B, part = blk & 1;   // K == 1: blk = (kk B + b) 2 + part
    return reinterpret_cast<const u32*>(a.accx) + (((size_t)b * 2 + part) * (a.Lc + a.K) + a.Lc) * a.N;
  }
};

// a9 data limbs: c_i = sum_k tb_k [P/p_k]_{q_i} - [P/2]_{q_i} (coefficient
// domain), NTT, then u = (IP_i - NTT(c_i)) P^{-1} and the epilogue.
struct JobKsData {
  static constexpr const char* kName = "ks_data";
  static constexpr int kIoWords = 2;   // store = an Lc-term 64-bit inner product + epilogue
  KsArgs a;
  __device__ void dec(int blk, int& kk, int& b, int& part, int& i) const {
    i = blk % a.Lc;
    int r = blk / a.Lc;
    part = r & 1;
    r >>= 1;
    b = r % a.B;
    kk = r / a.B;
  }
  __device__ int prime(int blk) const { return blk % a.Lc; }
  __device__ u64 load(int blk, u32 n, const PrimeD& P) const {
    int kk, b, part, i;
    dec(blk, kk, b, part, i);
    u64 conv = 0;
    if (a.K == 1 && P.k <= 31) {   // one special prime: weight P/p_0 = 1, residues < 2^31
      conv = reduce32((u32)a.tb[(((size_t)kk * a.B + b) * 2 + part) * a.N + n], P);
    } else {
      for (int k = 0; k < a.K; ++k) {
        const u64 t = a.tb[((((size_t)kk * a.B + b) * 2 + part) * a.K + k) * a.N + n];
        conv = add_mod(conv, mul_mod(reduce64(t, P), __ldg(a.Phat_mod + (size_t)k * a.NP + i), P), P.q);
      }
    }
    // the +[P/2]_{q_i} of C15 is added to every COEFFICIENT, so it is folded
    // here (coefficient domain) rather than after the transform
    return sub_mod(conv, __ldg(a.Ph_mod + i), P.q);
  }
  __device__ void store(int blk, u32 n, u64 v, const PrimeD& P) const {
    int kk, b, part, i;
    dec(blk, kk, b, part, i);
    const u32 g = a.gal[kk];
    const u32 sn = g == 1 ? n : galois_src(n, g, a.logN);
    const u64 ip = a.accx ? accx_word(a, (((size_t)b * 2 + part) * (a.Lc + a.K) + i) * a.N + n)
                          : ks_inner(a, kk, b, part, i, i, sn, n, P);
    u64 u = mul_mod(sub_mod(ip, v, P.q), __ldg(a.Pinv_mod + i), P);
    const size_t LN = (size_t)a.Lc * a.N;
    if (part < a.add_parts)
      u = add_mod(u, a.addsrc[(size_t)b * a.add_bs + part * LN + (size_t)i * a.N + (a.add_gather ? sn : n)], P.q);
    if (a.sq_src) {
      const u64 x0 = a.sq_src[(size_t)b * a.sq_bs + (size_t)i * a.N + n];
      const u64 x1 = a.sq_src[(size_t)b * a.sq_bs + LN + (size_t)i * a.N + n];
      const u64 t = part == 0 ? mul_mod(x0, x0, P) : mul_mod(x0, x1, P);
      u = add_mod(u, part == 0 ? t : add_mod(t, t, P.q), P.q);
    }
    if (a.D) u = mul_mod(u, a.D[(size_t)kk * a.D_ks + (size_t)i * a.N + n], P);
    const size_t o = (size_t)kk * a.out_ks + (size_t)b * a.out_bs + part * LN + (size_t)i * a.N + n;
    if (a.acc_in) u = add_mod(u, a.acc_in[o], P.q);
    a.out[o] = u;
  }
  // lazy ModDown with u32 accumulators and one special prime (the small-prime fused path): the
  // same arithmetic in u32 with the block's rows and constants bound once
  struct B32 {
    const JobKsData* j;
    int blk;
    const PrimeD* P;
    bool fast, gather;
    // 4 outputs (n0 + u st): every operand load of the 4 is issued before the arithmetic, so the
    // epilogue's global loads overlap instead of serialising behind the stores
    __device__ __forceinline__ void store4(u32 n0, u32 st, const u32* v) const {
      if (!fast || D || acc) {   // (the plaintext-factor / accumulating forms: one output at a time)
#pragma unroll
        for (int u = 0; u < 4; ++u) store(n0 + u * st, v[u]);
        return;
      }
      u32 axv[4], adv[4] = {0, 0, 0, 0}, s0[4] = {0, 0, 0, 0}, s1[4] = {0, 0, 0, 0};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const u32 n = n0 + u * st;
        axv[u] = ax[n];
        if (add) adv[u] = (u32)add[gather ? galois_src(n, g, logN) : n];
        if (sq0) {
          s0[u] = (u32)sq0[n];
          s1[u] = sq1 ? (u32)sq1[n] : s0[u];
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        u32 r = mulsh32(sub32(axv[u], v[u], q), pinv, pinvsh, q);
        if (add) r = add32(r, adv[u], q);
        if (sq0) {
          const u32 t = (u32)mul_mod(s0[u], s1[u], *P);
          r = add32(r, sq1 ? add32(t, t, q) : t, q);
        }
        out[n0 + u * st] = r;
      }
    }
    const u32* tb;
    const u32* ax;
    const u64* add;
    const u64* D;
    const u64* acc;
    u64* out;
    const u64* sq0;   // square: x0 row of this limb (poly 0: + x0^2; poly 1 with sq1 = x1: + 2 x0 x1)
    const u64* sq1;
    u32 q, mu32, ph, pinv, pinvsh, g;
    int logN;
    __device__ __forceinline__ u64 load(u32 n) const {
      if (!fast) return j->load(blk, n, *P);
      return sub32(red32(tb[n], q, mu32), ph, q);
    }
    __device__ __forceinline__ u64 load_raw(u32 x) const { return sub32(red32(x, q, mu32), ph, q); }
    __device__ __forceinline__ void store(u32 n, u64 v) const {
      if (!fast) {
        j->store(blk, n, v, *P);
        return;
      }
      u32 u = mulsh32(sub32(ax[n], (u32)v, q), pinv, pinvsh, q);
      if (add) u = add32(u, (u32)add[gather ? galois_src(n, g, logN) : n], q);
      if (sq0) {
        const u32 t = (u32)mul_mod(sq0[n], sq1 ? sq1[n] : sq0[n], *P);
        u = add32(u, sq1 ? add32(t, t, q) : t, q);
      }
      if (D) u = (u32)mul_mod(u, D[n], *P);
      if (acc) u = add32(u, (u32)acc[n], q);
      out[n] = u;
    }
  };
  __device__ B32 bind32(int blk, const PrimeD& P) const {
    int kk, b, part, i;
    dec(blk, kk, b, part, i);
    const bool fast = pipe_ok();
    B32 r{this, blk, &P, fast, false, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
          (u32)P.q, mu32_of(P), 0, 0, 0, 1, a.logN};
    if (fast) {
      const size_t LN = (size_t)a.Lc * a.N;
      r.tb = raw32(blk);
      r.ax = reinterpret_cast<const u32*>(a.accx) + (((size_t)b * 2 + part) * (a.Lc + a.K) + i) * a.N;
      r.ph = (u32)__ldg(a.Ph_mod + i);
      r.pinv = (u32)__ldg(a.Pinv_mod + i);
      r.pinvsh = shoup_companion32(r.pinv, r.q);
      r.g = a.gal[kk];
      r.gather = a.add_gather && r.g != 1;
      if (part < a.add_parts) r.add = a.addsrc + (size_t)b * a.add_bs + part * LN + (size_t)i * a.N;
      if (a.D) r.D = a.D + (size_t)kk * a.D_ks + (size_t)i * a.N;
      const size_t o = (size_t)kk * a.out_ks + (size_t)b * a.out_bs + part * LN + (size_t)i * a.N;
      if (a.acc_in) r.acc = a.acc_in + o;
      r.out = a.out + o;
      if (a.sq_src) {
        r.sq0 = a.sq_src + (size_t)b * a.sq_bs + (size_t)i * a.N;
        if (part == 1) r.sq1 = r.sq0 + LN;
      }
    }
    return r;
  }
  // pipelined kernel (pipe_ok, accx mode: no plaintext factor D): the fast form only
  struct P32 {
    const u32* ax;
    const u64* add;
    const u64* acc;
    u64* out;
    const u64* sq0;
    const u64* sq1;
    const PrimeD* P;
    u32 q, mu32, ph, pinv, pinvsh, g;
    int logN;
    bool gather;
    __device__ __forceinline__ u64 load_raw(u32 x) const { return sub32(red32(x, q, mu32), ph, q); }
    __device__ __forceinline__ u32 fin(u32 n, u32 v, u32 axv, u32 adv, u32 s0, u32 s1, u32 acv) const {
      u32 r = mulsh32(sub32(axv, v, q), pinv, pinvsh, q);
      if (add) r = add32(r, adv, q);
      if (sq0) {
        const u32 t = (u32)mul_mod(s0, s1, *P);
        r = add32(r, sq1 ? add32(t, t, q) : t, q);
      }
      if (acc) r = add32(r, acv, q);
      return r;
    }
    __device__ __forceinline__ void store(u32 n, u64 v) const {
      const u32 s0 = sq0 ? (u32)sq0[n] : 0u;
      out[n] = fin(n, (u32)v, ax[n], add ? (u32)add[gather ? galois_src(n, g, logN) : n] : 0u, s0,
                   sq1 ? (u32)sq1[n] : s0, acc ? (u32)acc[n] : 0u);
    }
    __device__ __forceinline__ void prefetch(u32 N) const {
      prefetch_l2(ax, N * 4);
      prefetch_l2(add, N * 8);
      prefetch_l2(acc, N * 8);
      prefetch_l2(sq0, N * 8);
      prefetch_l2(sq1, N * 8);
    }
    // 4 outputs n0 + u st: the operand loads of all 4 are issued before the arithmetic
    __device__ __forceinline__ void store4(u32 n0, u32 st, const u32* v) const {
      u32 axv[4], adv[4] = {0, 0, 0, 0}, s0[4] = {0, 0, 0, 0}, s1[4] = {0, 0, 0, 0}, acv[4] = {0, 0, 0, 0};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const u32 n = n0 + u * st;
        axv[u] = ax[n];
        if (add) adv[u] = (u32)add[gather ? galois_src(n, g, logN) : n];
        if (sq0) {
          s0[u] = (u32)sq0[n];
          s1[u] = sq1 ? (u32)sq1[n] : s0[u];
        }
        if (acc) acv[u] = (u32)acc[n];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) out[n0 + u * st] = fin(n0 + u * st, v[u], axv[u], adv[u], s0[u], s1[u], acv[u]);
    }
  };
  __device__ P32 bind_pipe(int blk, const PrimeD& P) const {
    int kk, b, part, i;
    dec(blk, kk, b, part, i);
    const size_t LN = (size_t)a.Lc * a.N;
    P32 r{reinterpret_cast<const u32*>(a.accx) + (((size_t)b * 2 + part) * (a.Lc + a.K) + i) * a.N, nullptr,
          nullptr, nullptr, nullptr, nullptr, &P, (u32)P.q, mu32_of(P), (u32)__ldg(a.Ph_mod + i),
          (u32)__ldg(a.Pinv_mod + i), 0, a.gal[kk], a.logN, false};
    r.pinvsh = shoup_companion32(r.pinv, r.q);
    r.gather = a.add_gather && r.g != 1;
    if (part < a.add_parts) r.add = a.addsrc + (size_t)b * a.add_bs + part * LN + (size_t)i * a.N;
    const size_t o = (size_t)kk * a.out_ks + (size_t)b * a.out_bs + part * LN + (size_t)i * a.N;
    if (a.acc_in) r.acc = a.acc_in + o;
    r.out = a.out + o;
    if (a.sq_src) {
      r.sq0 = a.sq_src + (size_t)b * a.sq_bs + (size_t)i * a.N;
      if (part == 1) r.sq1 = r.sq0 + LN;
    }
    return r;
  }
  // fast path input = one u32 row of tb (written by JobKsSpecial's fast store); accx mode has no D
  __host__ __device__ bool pipe_ok() const { return a.accx && a.accx32 && a.K == 1; }
  __host__ __device__ const u32* raw32(int blk) const {
    const int r = blk / a.Lc;   // (kk B + b) 2 + part
    return reinterpret_cast<const u32*>(a.tb) + (size_t)r * a.N;
  }
};

// ---- ModDown fused with the rescale that follows it (small primes, one special prime, accx) --------
// Sequentially (JobKsData then JobRescaleLast / JobRescaleData), limb i of the result is
//   u_i = (ax_i - NTT(conv_i)) P^{-1} + E_i,   y = INTT(u_l) + (q_l - 1)/2,
//   out_i = (u_i - NTT([y]_{q_i} - [h]_{q_i})) q_l^{-1}  (+ bias),
// with E_i the ModDown epilogue's NTT-domain terms (gathered c0, square terms, accumulated input).
// Both transforms are linear mod q_i, so with y'_i = [y]_{q_i} - [h]_{q_i}:
//   INTT(u_l) = (INTT(ax_l + P E_l) - conv_l) P^{-1}                       (JobKsDrop: one INTT)
//   out_i     = (ax_i + P E_i - NTT(conv_i + P y'_i)) (P q_l)^{-1}          (JobKsDataRs: one NTT)
// -- the same residues as the two-step form, with Lc + 1 transforms per part instead of 2 Lc + 1.
struct KsEpi32 {   // the epilogue terms E(n) of a bound block (as JobKsData::P32::fin adds them)
  const u64* add;
  const u64* acc;
  const u64* sq0;
  const u64* sq1;
  u32 g;
  int logN;
  bool gather;
  __device__ __forceinline__ u32 at(u32 n, u32 q, const PrimeD& P) const {
    u32 e = add ? (u32)add[gather ? galois_src(n, g, logN) : n] : 0u;
    if (sq0) {
      const u32 t = (u32)mul_mod(sq0[n], sq1 ? sq1[n] : sq0[n], P);
      e = add32(e, sq1 ? add32(t, t, q) : t, q);
    }
    if (acc) e = add32(e, (u32)acc[n], q);
    return e;
  }
};
__device__ __forceinline__ KsEpi32 bind_epi32(const KsArgs& a, int b, int part, int i) {
  const size_t LN = (size_t)a.Lc * a.N;
  KsEpi32 e{nullptr, nullptr, nullptr, nullptr, a.gal[0], a.logN, false};
  e.gather = a.add_gather && e.g != 1;
  if (part < a.add_parts) e.add = a.addsrc + (size_t)b * a.add_bs + part * LN + (size_t)i * a.N;
  if (a.acc_in) e.acc = a.acc_in + (size_t)b * a.out_bs + part * LN + (size_t)i * a.N;
  if (a.sq_src) {
    e.sq0 = a.sq_src + (size_t)b * a.sq_bs + (size_t)i * a.N;
    if (part == 1) e.sq1 = e.sq0 + LN;
  }
  return e;
}

// The dropped limb l = Lc - 1: y[b][part] = INTT(ax_l + P E_l) - conv_l) P^{-1} + (q_l - 1)/2 (u32 rows).
struct JobKsDrop {
  static constexpr const char* kName = "ks_rescale_drop";
  KsArgs a;
  u32* y;   // [B][2][N]
  int N;
  __device__ int prime(int) const { return a.Lc - 1; }
  struct B32 {
    KsEpi32 e;
    const PrimeD* P;
    const u32* ax;
    const u32* tb;
    u32* y;
    u32 q, mu32, ph, pinv, pinvsh, pm, pmsh, h;
    __device__ __forceinline__ u64 load(u32 n) const {
      return add32(ax[n], mulsh32(e.at(n, q, *P), pm, pmsh, q), q);
    }
    __device__ __forceinline__ void store(u32 n, u64 v) const {
      const u32 conv = sub32(red32(tb[n], q, mu32), ph, q);
      y[n] = add32(mulsh32(sub32((u32)v, conv, q), pinv, pinvsh, q), h, q);
    }
  };
  __device__ B32 bind32(int blk, const PrimeD& P) const {
    const int b = blk >> 1, part = blk & 1, l = a.Lc - 1;
    const u32 q = (u32)P.q, pinv = (u32)__ldg(a.Pinv_mod + l), pm = (u32)__ldg(a.P_mod + l);
    return B32{bind_epi32(a, b, part, l), &P,
               reinterpret_cast<const u32*>(a.accx) + (((size_t)b * 2 + part) * (a.Lc + a.K) + l) * a.N,
               reinterpret_cast<const u32*>(a.tb) + ((size_t)b * 2 + part) * a.N, y + ((size_t)b * 2 + part) * a.N,
               q, mu32_of(P), (u32)__ldg(a.Ph_mod + l), pinv, shoup_companion32(pinv, q), pm,
               shoup_companion32(pm, q), (u32)((P.q - 1) >> 1)};
  }
  // generic form (only small-prime contexts take this path; the 64-bit engine instantiates it)
  __device__ u64 load(int blk, u32 n, const PrimeD& P) const { return bind32(blk, P).load(n); }
  __device__ void store(int blk, u32 n, u64 v, const PrimeD& P) const { bind32(blk, P).store(n, v); }
};

// Data limbs i < l of the rescaled result: out_i = (ax_i + P E_i - NTT(conv_i + P y'_i)) (P q_l)^{-1} + bias.
struct JobKsDataRs {
  static constexpr const char* kName = "ks_rescale";
  KsArgs a;
  const u32* y;       // JobKsDrop's rows
  u64* out;           // [B][2][Lc-1][N] (item stride out_bs)
  size_t out_bs;
  const u64* rs_h;    // row l of rs_h: (q_l - 1)/2 mod q_i
  const u64* rs_qinv; // row l of rs_qinv: q_l^{-1} mod q_i
  const u64* bias;    // nullable: poly 0 gets + bias[b * bias_bs + i * N + n]
  size_t bias_bs;
  int N;
  __device__ int prime(int blk) const { return blk % (a.Lc - 1); }
  struct B32 {
    KsEpi32 e;
    const PrimeD* P;
    const u32* ax;
    const u32* tb;
    const u32* y;
    u64* out;
    const u64* bias;
    u32 q, mu32, ph, hr, pm, pmsh, cinv, cinvsh;
    __device__ __forceinline__ u64 load(u32 n) const {
      const u32 conv = sub32(red32(tb[n], q, mu32), ph, q);
      const u32 yy = sub32(red32(y[n], q, mu32), hr, q);
      return add32(conv, mulsh32(yy, pm, pmsh, q), q);
    }
    // pipelined kernel: x is the staged word tb[n]; the y row (shared by the Lc-1 blocks of one
    // (item, part): L2-resident) is read here, in the transform's first pass
    __device__ __forceinline__ u64 load_raw_at(u32 x, u32 n) const {
      const u32 conv = sub32(red32(x, q, mu32), ph, q);
      const u32 yy = sub32(red32(__ldg(y + n), q, mu32), hr, q);
      return add32(conv, mulsh32(yy, pm, pmsh, q), q);
    }
    __device__ __forceinline__ u64 load_raw(u32 x) const { return x; }   // (interface; load_raw_at is used)
    __device__ __forceinline__ void prefetch(u32 N) const {
      prefetch_l2(ax, N * 4);
      prefetch_l2(e.add, N * 8);
      prefetch_l2(e.acc, N * 8);
      prefetch_l2(e.sq0, N * 8);
      prefetch_l2(e.sq1, N * 8);
    }
    __device__ __forceinline__ u32 fin(u32 n, u32 v, u32 axv, u32 ev, u32 bv) const {
      const u32 w = add32(axv, mulsh32(ev, pm, pmsh, q), q);
      u32 o = mulsh32(sub32(w, v, q), cinv, cinvsh, q);
      return bias ? add32(o, bv, q) : o;
    }
    __device__ __forceinline__ void store(u32 n, u64 v) const {
      out[n] = fin(n, (u32)v, ax[n], e.at(n, q, *P), bias ? (u32)bias[n] : 0u);
    }
    // 4 outputs n0 + u st: every operand load of the 4 is issued before the arithmetic
    __device__ __forceinline__ void store4(u32 n0, u32 st, const u32* v) const {
      u32 axv[4], ev[4], bv[4] = {0, 0, 0, 0};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const u32 n = n0 + u * st;
        axv[u] = ax[n];
        ev[u] = e.at(n, q, *P);
        if (bias) bv[u] = (u32)bias[n];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) out[n0 + u * st] = fin(n0 + u * st, v[u], axv[u], ev[u], bv[u]);
    }
  };
  __device__ B32 bind32(int blk, const PrimeD& P) const {
    const int i = blk % (a.Lc - 1), r = blk / (a.Lc - 1), b = r >> 1, part = r & 1;
    const u32 q = (u32)P.q, pm = (u32)__ldg(a.P_mod + i);
    const u32 cinv = (u32)mul_mod(__ldg(a.Pinv_mod + i), __ldg(rs_qinv + i), P);
    return B32{bind_epi32(a, b, part, i), &P,
               reinterpret_cast<const u32*>(a.accx) + (((size_t)b * 2 + part) * (a.Lc + a.K) + i) * a.N,
               reinterpret_cast<const u32*>(a.tb) + (size_t)r * a.N, y + (size_t)r * a.N,
               out + (size_t)b * out_bs + ((size_t)part * (a.Lc - 1) + i) * a.N,
               bias && part == 0 ? bias + (size_t)b * bias_bs + (size_t)i * a.N : nullptr, q, mu32_of(P),
               (u32)__ldg(a.Ph_mod + i), (u32)__ldg(rs_h + i), pm, shoup_companion32(pm, q), cinv,
               shoup_companion32(cinv, q)};
  }
  __device__ u64 load(int blk, u32 n, const PrimeD& P) const { return bind32(blk, P).load(n); }
  __device__ void store(int blk, u32 n, u64 v, const PrimeD& P) const { bind32(blk, P).store(n, v); }
  // pipelined transform (k_ntt32_pipe): the staged row is the block's tb row, y joins in load_raw_at.
  // OFF: measured slower than the one-shot kernel on B200 (A/B, the CNN step at batch 512: ks_rescale
  // 1.11 -> 1.58 ms per step) - the y loads sit on the critical path of every block's first pass and the
  // wider binding spills in the 40-register persistent kernel; kept for the experiment's record.
#ifndef HE_KSRS_PIPE
#define HE_KSRS_PIPE 0
#endif
  __host__ __device__ bool pipe_ok() const { return HE_KSRS_PIPE != 0; }
  __host__ __device__ const u32* raw32(int blk) const {
    return reinterpret_cast<const u32*>(a.tb) + (size_t)(blk / (a.Lc - 1)) * a.N;
  }
};

// Rescale source: row r of x, or (conv, C18) the product ct_b (.) K_c formed on
// the fly for row r = (b C + c) 2 + p, so the products never reach HBM.
struct RescaleSrc {
  const u64* x;     // [R][Lc][N], or ciphertexts (see mask_sum / K)
  const u64* K;     // nullable: [C][Lc][N] plaintexts
  int C, N, Lc;
  int mask_sum = 0; // 1: row r = b 2 + p is sum_c x[b C + c][p] (.) K_c (conv masks, C19)
  __device__ __forceinline__ u64 at(int r, int i, u32 n, const PrimeD& P) const {
    if (!K) return x[((size_t)r * Lc + i) * N + n];
    if (mask_sum) {
      const int b = r >> 1, p = r & 1;
      u64 acc = 0;
      for (int c = 0; c < C; ++c)
        acc = add_mod(acc, mul_mod(x[((((size_t)b * C + c) * 2 + p) * Lc + i) * N + n], K[((size_t)c * Lc + i) * N + n], P),
                      P.q);
      return acc;
    }
    const int b = r / (2 * C), rem = r % (2 * C), c = rem >> 1, p = rem & 1;
    return mul_mod(x[(((size_t)b * 2 + p) * Lc + i) * N + n], K[((size_t)c * Lc + i) * N + n], P);
  }
};

// a11 rescale, step 1: INTT of the last limb l, y = [x_l + (q_l-1)/2]_{q_l}.
struct JobRescaleLast {
  static constexpr const char* kName = "rescale_last";
  RescaleSrc src;
  u64* y;           // [R][N]
  int N, Lc;
  __device__ int prime(int) const { return Lc - 1; }
  __device__ u64 load(int blk, u32 n, const PrimeD& P) const { return src.at(blk, Lc - 1, n, P); }
  __device__ void store(int blk, u32 n, u64 v, const PrimeD& P) const {
    y[(size_t)blk * N + n] = add_mod(v, (P.q - 1) >> 1, P.q);
  }
  // 32-bit engine: y holds u32 words (read by JobRescaleData's bound / pipelined load)
  struct B32 {
    const RescaleSrc* src;
    const PrimeD* P;
    u32* y;
    int blk, l;
    u32 q, h;
    __device__ __forceinline__ u64 load(u32 n) const { return src->at(blk, l, n, *P); }
    __device__ __forceinline__ void store(u32 n, u64 v) const { y[n] = add32((u32)v, h, q); }
  };
  __device__ B32 bind32(int blk, const PrimeD& P) const {
    return B32{&src, &P, reinterpret_cast<u32*>(y) + (size_t)blk * N, blk, Lc - 1, (u32)P.q, (u32)((P.q - 1) >> 1)};
  }
};
// a11 rescale, step 2: out_i = (x_i - NTT_i([y]_{q_i} - [h]_{q_i})) [q_l^{-1}]_{q_i}.
struct JobRescaleData {
  static constexpr const char* kName = "rescale_data";
  RescaleSrc src;
  const u64* y;
  u64* out;         // [R][Lc-1][N]
  const u64* h;     // [Lc-1] (q_l-1)/2 mod q_i   (row l of rs_h)
  const u64* qinv;  // [Lc-1] q_l^{-1} mod q_i
  int N, Lc;
  // optional fused bias (vec_mat): poly 0 of item r / size gets + bias[item * bias_bs + i * N + n]
  const u64* bias = nullptr;
  size_t bias_bs = 0;
  int size = 2;
  __device__ int prime(int blk) const { return blk % (Lc - 1); }
  __device__ u64 load(int blk, u32 n, const PrimeD& P) const {
    // [y]_{q_i} - [h]_{q_i}: h is added to every coefficient (C15), so it is
    // folded in before the forward transform
    const u64 yv = y[(size_t)(blk / (Lc - 1)) * N + n];
    return sub_mod(P.k <= 31 && yv < (1ULL << 32) ? reduce32((u32)yv, P) : reduce64(yv, P), __ldg(h + blk % (Lc - 1)),
                   P.q);
  }
  __device__ void store(int blk, u32 n, u64 v, const PrimeD& P) const {
    const int r = blk / (Lc - 1), i = blk % (Lc - 1);
    const u64 t = sub_mod(src.at(r, i, n, P), v, P.q);
    u64 o = mul_mod(t, __ldg(qinv + i), P);
    if (bias && r % size == 0) o = add_mod(o, bias[(size_t)(r / size) * bias_bs + (size_t)i * N + n], P.q);
    out[((size_t)r * (Lc - 1) + i) * N + n] = o;
  }
  struct B32 {
    const RescaleSrc* src;
    const PrimeD* P;
    const u32* y;
    u64* out;
    const u64* bias;   // bias row (poly 0 only) or null
    int r, i;
    u32 q, mu32, h, qi, qish;
    __device__ __forceinline__ void store4(u32 n0, u32 st, const u32* v) const {
      u32 xv[4], bv[4] = {0, 0, 0, 0};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        xv[u] = (u32)src->at(r, i, n0 + u * st, *P);
        if (bias) bv[u] = (u32)bias[n0 + u * st];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        u32 o = mulsh32(sub32(xv[u], v[u], q), qi, qish, q);
        if (bias) o = add32(o, bv[u], q);
        out[n0 + u * st] = o;
      }
    }
    __device__ __forceinline__ void prefetch(u32 N) const {
      if (!src->K) prefetch_l2(src->x + ((size_t)r * src->Lc + i) * N, N * 8);
      prefetch_l2(bias, N * 8);
    }
    __device__ __forceinline__ u64 load(u32 n) const { return sub32(red32(y[n], q, mu32), h, q); }
    __device__ __forceinline__ u64 load_raw(u32 x) const { return sub32(red32(x, q, mu32), h, q); }
    __device__ __forceinline__ void store(u32 n, u64 v) const {
      u32 o = mulsh32(sub32((u32)src->at(r, i, n, *P), (u32)v, q), qi, qish, q);
      if (bias) o = add32(o, (u32)bias[n], q);
      out[n] = o;
    }
  };
  __device__ B32 bind32(int blk, const PrimeD& P) const {
    const int r = blk / (Lc - 1), i = blk % (Lc - 1);
    const u32 q = (u32)P.q, qi = (u32)__ldg(qinv + i);
    const u64* brow = bias && r % size == 0 ? bias + (size_t)(r / size) * bias_bs + (size_t)i * N : nullptr;
    return B32{&src, &P, raw32(blk), out + ((size_t)r * (Lc - 1) + i) * N, brow, r, i, q, mu32_of(P),
               (u32)__ldg(h + i), qi, shoup_companion32(qi, q)};
  }
  __host__ __device__ bool pipe_ok() const { return true; }
  __host__ __device__ const u32* raw32(int blk) const {
    return reinterpret_cast<const u32*>(y) + (size_t)(blk / (Lc - 1)) * N;
  }
};

// Algorithmic bytes of one launch of nblk blocks: every distinct input word
// read once and every output word written once.
inline double alg_bytes(const JobLimbs& j, int nblk) { return 16.0 * j.N * nblk; }
inline double alg_bytes(const JobRingMul& j, int nblk) { return 24.0 * j.N * nblk; }
inline double alg_bytes(const JobSignedToNtt& j, int nblk) { return 8.0 * j.N * (nblk + nblk / j.nl); }
inline double alg_bytes(const JobModUp& j, int nblk) {
  const int nt = j.Lc + j.K - 1;
  return 8.0 * j.N * (nblk + (double)nblk / nt);
}
inline double alg_bytes(const JobKsSpecial& j, int nblk) {
  const KsArgs& a = j.a;
  const double N8 = 8.0 * a.N;
  if (a.accx) return N8 * 2.0 * nblk;
  return N8 * ((double)a.B * a.Lc * a.K + (double)a.KB * 2 * a.Lc * a.K + (double)a.KB * a.B * 2 * a.K);
}
inline double alg_bytes(const JobKsData& j, int nblk) {
  const KsArgs& a = j.a;
  const double N8 = 8.0 * a.N;
  if (a.accx) return N8 * ((double)nblk * 2 + (double)a.B * 2 * a.K);
  double w = (double)a.KB * a.B * 2 * a.K                  // tb
             + (double)a.B * a.Lc * a.Lc                   // ext data limbs (+ digit source diagonal)
             + (double)a.KB * 2 * a.Lc * a.Lc              // key rows of the data limbs
             + (double)a.KB * a.B * 2 * a.Lc;              // output
  if (a.add_parts) w += (double)a.B * a.add_parts * a.Lc;
  if (a.D) w += (double)a.KB * a.Lc;
  if (a.acc_in) w += (double)a.KB * a.B * 2 * a.Lc;
  return N8 * w;
}
inline double alg_bytes(const JobRescaleLast& j, int nblk) { return 16.0 * j.N * nblk; }
inline double alg_bytes(const JobKsDrop& j, int nblk) { return 4.0 * j.N * nblk * 3 + 8.0 * j.N * nblk; }
inline double alg_bytes(const JobKsDataRs& j, int nblk) { return 4.0 * j.N * nblk * 3 + 16.0 * j.N * nblk; }
inline double alg_bytes(const JobRescaleData& j, int nblk) {
  return 8.0 * j.N * (2.0 * nblk + (double)nblk / (j.Lc - 1));
}

// Algorithmic modular operations of one launch (DESIGN.md §5 ALU roofline):
// (N/2) log2 N butterflies per limb transform, plus one per modular
// multiply-accumulate of the fused inner products / epilogues.
inline double ntt_ops(int N, int logN) { return 0.5 * N * logN; }
template <class Job>
inline double alg_ops(const Job& j, int nblk, int logN) { return nblk * ntt_ops(j.N, logN); }
inline double alg_ops(const JobKsSpecial& j, int nblk, int logN) {
  const KsArgs& a = j.a;
  return nblk * (ntt_ops(a.N, logN) + (a.accx ? 0.0 : (double)a.Lc * a.N) + a.N);
}
inline double alg_ops(const JobKsData& j, int nblk, int logN) {
  const KsArgs& a = j.a;
  return nblk * (ntt_ops(a.N, logN) + (a.accx ? 0.0 : (double)a.Lc * a.N) + (double)a.K * a.N + 2.0 * a.N);
}

}  // namespace he
