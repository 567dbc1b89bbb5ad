// he_ntt.cuh — batched negacyclic NTT / INTT for sm_100a (SURVEY.md §8(a) a6,
// kernels K1/K2), templated on load / store functors so that every producer
// and consumer of a transform (digit lift, key inner product, ModDown,
// rescale, encode, decrypt, ...) is fused into the transform's single pass
// over HBM.
//
// Transform (C5): NTT(a)[j] = sum_i a_i psi^{(2 brv(j)+1) i} mod q, computed
// by the merged-psi Cooley-Tukey network (twiddle of stage s, butterfly group
// i: psi^{brv(2^s + i)}), output in bit-reversed order; the inverse is the
// Gentleman-Sande network with psi^{-brv(.)} followed by N^{-1}.
//
// Layout: one CTA (or a 2-CTA cluster for N = 32768) owns one limb of N
// words in shared memory (padded one word per 16 against bank conflicts).
// Each thread owns 2^R words per pass and runs R radix-2 stages in registers
// (Harvey lazy butterflies, Shoup twiddle products, values kept in [0, 4q)),
// so a 2^13 transform makes 4 passes over shared memory and exactly one
// coalesced read and one coalesced write of the limb in HBM.
#pragma once
#include <cooperative_groups.h>

#include "he_common.cuh"
#include "he_jobs.cuh"

namespace he {

template <int LOGN, int CL>
struct NttGeom {
  static constexpr int N = 1 << LOGN;
  static constexpr int LOGNL = LOGN - (CL == 2 ? 1 : 0);  // bits owned by one CTA
  static constexpr int NL = 1 << LOGNL;
#ifndef HE_NTT64_R14
#define HE_NTT64_R14 4
#endif
  // log2 words per thread (a 2^14 limb per CTA: HE_NTT64_R14, 4 = 1024 threads x 16 words)
  static constexpr int R = LOGNL == 14 ? HE_NTT64_R14 : (LOGNL - 10 > 4 ? LOGNL - 10 : 4);
  static constexpr int T = NL >> R;                            // threads per CTA
  // CTAs per SM the register budget is sized for (shared memory allows 3 at N=2^13)
#ifndef HE_NTT64_MINB
#define HE_NTT64_MINB 2
#endif
  static constexpr int MINB = NL <= 8192 ? HE_NTT64_MINB : 1;
  static constexpr int NPASS = (LOGNL + R - 1) / R;
  static constexpr int SMEM = (NL + NL / 16) * 8;
};

__device__ __forceinline__ u32 spad(u32 i) { return i + (i >> 4); }

// Cooley-Tukey butterfly, inputs/outputs in [0, 4q).  (An approximate-quotient Shoup product --
// three 32-bit high products instead of the 64x64 high product, result in [0, 4q) -- was measured
// slower in round 2: the extra 64-bit conditional subtraction and register pressure cost more than
// the fmaheavy cycles it saves; cfg2 forward 955 vs 999 GB/s.)
__device__ __forceinline__ void ct_bfly(u64& x, u64& y, u64 w, u64 wsh, u64 q, u64 two_q) {
  u64 X = x >= two_q ? x - two_q : x;
  u64 T = mul_shoup_lazy(y, w, wsh, q);
  x = X + T;
  y = X - T + two_q;
}
// Gentleman-Sande butterfly, inputs/outputs in [0, 2q).
__device__ __forceinline__ void gs_bfly(u64& x, u64& y, u64 w, u64 wsh, u64 q, u64 two_q) {
  u64 U = x + y;
  U = U >= two_q ? U - two_q : U;
  u64 V = x - y + two_q;
  x = U;
  y = mul_shoup_lazy(V, w, wsh, q);
}

// One pass over local bits [LO, LO+NB): each thread reads 2^NB words per group through ld(i)
// (2^(R-NB) groups), runs NB stages in registers and hands them to st(i, v).  ld / st are shared
// memory for the inner passes; the first forward pass reads the job's input straight from HBM and
// the last inverse pass scales by N^{-1} and writes the job's output (the top bit group: both
// coalesced, consecutive threads own consecutive indices), which saves two shared-memory round trips
// and two barriers per transform.
// WORDS bounds the words a thread has in flight (its groups run in chunks of max(1, WORDS / 2^NB)
// groups, chunks not interleaved): HBM-facing passes take 8 so that all of a chunk's loads are issued
// together without spilling; shared-memory passes are fully unrolled.
template <int LOGN, int CL, bool INV, int LO, int NB, int WORDS = 0, class LD, class ST>
__device__ __forceinline__ void ntt_pass_io(u32 tid, u32 gbase, const ulonglong2* __restrict__ tw, u64 q,
                                            u64 two_q, LD ld, ST st) {
  typedef NttGeom<LOGN, CL> G;
  constexpr int NG = 1 << (G::R - NB);
  constexpr int E = 1 << NB;
  constexpr int CH0 = WORDS > E ? WORDS / E : 1;
  constexpr int CH = (WORDS == 0 || CH0 > NG) ? NG : CH0;
#pragma unroll 1
  for (int c = 0; c < NG / CH; ++c)
#pragma unroll
  for (int gg = 0; gg < CH; ++gg) {
    const int gi = c * CH + gg;
    const u32 g = tid + gi * G::T;
    const u32 base = ((g >> LO) << (LO + NB)) | (g & ((1u << LO) - 1u));
    u64 x[E];
#pragma unroll
    for (int k = 0; k < E; ++k) x[k] = ld(base + (k << LO));
    // twiddle of the butterfly on bit b at index j = gbase | hi << (LO+NB) | k << LO | lo:
    // tw[2^s + (j >> (b+1))], s = LOGN-1-b, and j >> (b+1) = (gbase >> (b+1)) + (hi << (LO+NB-1-b)) +
    // (k >> (b+1-LO)): one base pointer per stage and compile-time offsets, so the butterflies of a
    // group that share a twiddle share one load
    const u32 hi = g >> LO;
#pragma unroll
    for (int ss = 0; ss < NB; ++ss) {
      const int b = INV ? LO + ss : LO + NB - 1 - ss;   // local == global bit being paired
      const int s = LOGN - 1 - b;                        // stage index
      const int half = INV ? 1 << ss : 1 << (NB - 1 - ss);
      const ulonglong2* tws = tw + (1u << s) + (gbase >> (b + 1)) + (hi << (LO + NB - 1 - b));
#pragma unroll
      for (int k = 0; k < E; ++k) {
        if (k & half) continue;
        const ulonglong2 w = __ldg(tws + (k >> (b + 1 - LO)));
        if (!INV) ct_bfly(x[k], x[k + half], w.x, w.y, q, two_q);
        else gs_bfly(x[k], x[k + half], w.x, w.y, q, two_q);
      }
    }
#pragma unroll
    for (int k = 0; k < E; ++k) st(base + (k << LO), x[k]);
  }
}

template <int LOGN, int CL, bool INV, int LO, int NB>
__device__ __forceinline__ void ntt_pass(u64* sm, u32 tid, u32 gbase, const ulonglong2* __restrict__ tw,
                                         u64 q, u64 two_q) {
  ntt_pass_io<LOGN, CL, INV, LO, NB>(
      tid, gbase, tw, q, two_q, [&](u32 i) { return sm[spad(i)]; }, [&](u32 i, u64 v) { sm[spad(i)] = v; });
}

// Passes P .. PEND-1 over the local problem: pass P covers bit group GP = INV ? P : NPASS-1-P,
// local bits [GP R, min(GP R + R, LOGNL)); each ends with a barrier.
// Two consecutive full passes (NB = R, one group per thread) over bits below 5 + R exchange data inside
// one warp only (its 32 2^R words; see Pass32 below): __syncwarp() orders them instead of the barrier.
#ifndef HE_NTT64_WARPSYNC
#define HE_NTT64_WARPSYNC 1
#endif
template <int LOGN, int CL, bool INV, int P>
struct Pass64 {
  typedef NttGeom<LOGN, CL> G;
  static constexpr int GP = INV ? P : G::NPASS - 1 - P;  // forward runs top-down
  static constexpr int LO = GP * G::R;
  static constexpr int NB = (LO + G::R <= G::LOGNL) ? G::R : G::LOGNL - LO;
  static constexpr bool WL = HE_NTT64_WARPSYNC && P >= 0 && P < G::NPASS && NB == G::R && LO <= 5 && G::T % 32 == 0;
};
template <int LOGN, int CL, bool INV, int P, int PEND = NttGeom<LOGN, CL>::NPASS>
__device__ __forceinline__ void ntt_passes(u64* sm, u32 tid, u32 gbase, const ulonglong2* tw, u64 q,
                                           u64 two_q) {
  if constexpr (P < PEND) {
    typedef Pass64<LOGN, CL, INV, P> PS;
    ntt_pass<LOGN, CL, INV, PS::LO, PS::NB>(sm, tid, gbase, tw, q, two_q);
    constexpr bool next_wl = (P + 1 < PEND) && Pass64<LOGN, CL, INV, (P + 1 < PEND ? P + 1 : P)>::WL;
    if constexpr (PS::WL && next_wl) __syncwarp();
    else __syncthreads();
    ntt_passes<LOGN, CL, INV, P + 1, PEND>(sm, tid, gbase, tw, q, two_q);
  }
}

// Cluster barrier halves (release / acquire): a CTA must not exit while its peer still reads its
// shared memory, and remote stores must be visible before the peer's next pass.
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::); }
__device__ __forceinline__ void cluster_sync_all() {
  cluster_arrive();
  cluster_wait();
}

// Forward cross-CTA stage (bit LOGN-1) of the 2-CTA cluster transform fused with the job's loads:
// CTA r owns the pairs (i, i + NL), i in [r NL/2, (r+1) NL/2); every load of a thread is issued
// before the first butterfly, the two outputs go to local index i of CTA 0 and CTA 1 (DSMEM).
template <int LOGN, class Job>
__device__ __forceinline__ void ntt_cross_load(const Job& job, int blk, const PrimeD& P, u64* sm, u32 tid,
                                               u32 rank, const ulonglong2* tw) {
  namespace cg = cooperative_groups;
  typedef NttGeom<LOGN, 2> G;
  constexpr int PAIRS = G::NL / 2 / G::T;
  cg::cluster_group cl = cg::this_cluster();
  u64* s0 = cl.map_shared_rank(sm, 0);
  u64* s1 = cl.map_shared_rank(sm, 1);
  constexpr int W2 = io_words_of<Job>::value / 2 > 0 ? io_words_of<Job>::value / 2 : 1;
  constexpr int CH = PAIRS < W2 ? PAIRS : W2;   // io_words_of<Job> words in flight per chunk
  const ulonglong2 tw1 = __ldg(tw + 1);
#pragma unroll 1
  for (int c = 0; c < PAIRS / CH; ++c) {
    u64 x[CH], y[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const u32 i = rank * (G::NL / 2) + tid + (c * CH + k) * G::T;
      x[k] = job.load(blk, i, P);
      y[k] = job.load(blk, i + G::NL, P);
    }
    if (c == 0) cluster_wait();   // the peer CTA is running (its shared memory exists): arrived at entry
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const u32 i = rank * (G::NL / 2) + tid + (c * CH + k) * G::T;
      ct_bfly(x[k], y[k], tw1.x, tw1.y, P.q, P.two_q);
      s0[spad(i)] = x[k];
      s1[spad(i)] = y[k];
    }
  }
}

// Inverse cross-CTA stage fused with the N^{-1} scaling and the job's stores (global indices i and
// i + NL).  Arrives on the cluster barrier once the peer's shared memory has been read.
template <int LOGN, class Job>
__device__ __forceinline__ void ntt_cross_store(const Job& job, int blk, const PrimeD& P, u64* sm, u32 tid,
                                                u32 rank, const ulonglong2* tw) {
  namespace cg = cooperative_groups;
  typedef NttGeom<LOGN, 2> G;
  constexpr int PAIRS = G::NL / 2 / G::T;
  cg::cluster_group cl = cg::this_cluster();
  const u64* s0 = cl.map_shared_rank(sm, 0);
  const u64* s1 = cl.map_shared_rank(sm, 1);
  const ulonglong2 tw1 = __ldg(tw + 1);
  u64 x[PAIRS], y[PAIRS];
#pragma unroll
  for (int k = 0; k < PAIRS; ++k) {
    const u32 i = rank * (G::NL / 2) + tid + k * G::T;
    x[k] = s0[spad(i)];
    y[k] = s1[spad(i)];
  }
  cluster_arrive();
#pragma unroll
  for (int k = 0; k < PAIRS; ++k) {
    const u32 i = rank * (G::NL / 2) + tid + k * G::T;
    gs_bfly(x[k], y[k], tw1.x, tw1.y, P.q, P.two_q);
    job.store(blk, i, mul_shoup(x[k], P.ninv, P.ninvsh, P.q), P);
    job.store(blk, i + G::NL, mul_shoup(y[k], P.ninv, P.ninvsh, P.q), P);
  }
}

// Generic batched transform.  Job provides:
//   int  prime(int blk)                           absolute prime index of limb blk
//   u64  load(int blk, u32 i, const PrimeD&)      canonical input word i (natural index)
//   void store(int blk, u32 i, u64 v, const PrimeD&)  canonical output word i
// blk = blockIdx.x / CL.  The launch uses exactly G::T threads, so every per-thread loop has a
// compile-time trip count and is unrolled: all of a thread's HBM loads are in flight together
// (round 2: the rolled loops serialised one DRAM latency per word).
//   forward:  [CL=2: loads + cross stage -> DSMEM]  or  [CL=1: loads + top pass]  -> shared passes
//             -> reduce + store (shared memory read back in coalesced order)
//   inverse:  coalesced loads -> shared passes -> [CL=1: top pass + N^{-1} + store]
//             or [CL=2: cross stage + N^{-1} + store]
template <int LOGN, int CL, bool INV, class Job>
__global__ void __launch_bounds__(NttGeom<LOGN, CL>::T, NttGeom<LOGN, CL>::MINB)
k_ntt(Job job, const PrimeD* __restrict__ primes, const ulonglong2* __restrict__ tw_all) {
  typedef NttGeom<LOGN, CL> G;
  constexpr int PER = G::NL / G::T;
  constexpr int LO_TOP = (G::NPASS - 1) * G::R, NB_TOP = G::LOGNL - LO_TOP;
  extern __shared__ u64 sm[];
  const u32 tid = threadIdx.x;
  const int blk = blockIdx.x / CL;
  const u32 rank = CL == 2 ? (blockIdx.x & 1) : 0;
  const u32 gbase = rank * G::NL;
  const int pi = job.prime(blk);
  const PrimeD P = load_prime(primes, pi);
  const ulonglong2* tw = tw_all + (size_t)pi * G::N;
  auto sld = [&](u32 i) { return sm[spad(i)]; };
  auto sst = [&](u32 i, u64 v) { sm[spad(i)] = v; };
  if constexpr (!INV) {
    if constexpr (CL == 2) {
      cluster_arrive();
      ntt_cross_load<LOGN>(job, blk, P, sm, tid, rank, tw);
      cluster_sync_all();
      ntt_passes<LOGN, CL, false, 0>(sm, tid, gbase, tw, P.q, P.two_q);
    } else {
      ntt_pass_io<LOGN, CL, false, LO_TOP, NB_TOP, io_words_of<Job>::value>(
          tid, gbase, tw, P.q, P.two_q, [&](u32 i) { return job.load(blk, i, P); }, sst);
      __syncthreads();
      ntt_passes<LOGN, CL, false, 1>(sm, tid, gbase, tw, P.q, P.two_q);
    }
    constexpr int CS = PER < io_words_of<Job>::value ? PER : io_words_of<Job>::value;
#pragma unroll 1
    for (int c = 0; c < PER / CS; ++c)
#pragma unroll
    for (int kk = 0; kk < CS; ++kk) {
      const u32 i = tid + (c * CS + kk) * G::T;
      u32 si = i;   // jobs storing a permuted transform read word gather_src(n) of their own half
      if constexpr (has_gather_src<Job>::value) si = job.gather_src(gbase + i) - gbase;
      u64 v = sm[spad(si)];
      v = v >= P.two_q ? v - P.two_q : v;
      v = v >= P.q ? v - P.q : v;
      job.store(blk, gbase + i, v, P);
    }
  } else {
    constexpr int CH = PER < io_words_of<Job>::value ? PER : io_words_of<Job>::value;
#pragma unroll 1
    for (int c = 0; c < PER / CH; ++c) {
      u64 v[CH];
#pragma unroll
      for (int k = 0; k < CH; ++k) v[k] = job.load(blk, gbase + tid + (c * CH + k) * G::T, P);
#pragma unroll
      for (int k = 0; k < CH; ++k) sm[spad(tid + (c * CH + k) * G::T)] = v[k];
    }
    __syncthreads();
    if constexpr (CL == 2) {
      ntt_passes<LOGN, CL, true, 0>(sm, tid, gbase, tw, P.q, P.two_q);
      cluster_sync_all();
      ntt_cross_store<LOGN>(job, blk, P, sm, tid, rank, tw);
      cluster_wait();   // the peer has read this CTA's shared memory
    } else {
      ntt_passes<LOGN, CL, true, 0, G::NPASS - 1>(sm, tid, gbase, tw, P.q, P.two_q);
      ntt_pass_io<LOGN, CL, true, LO_TOP, NB_TOP, io_words_of<Job>::value>(
          tid, gbase, tw, P.q, P.two_q, sld,
          [&](u32 i, u64 v) { job.store(blk, i, mul_shoup(v, P.ninv, P.ninvsh, P.q), P); });
    }
  }
}

// Fused ring product: out = INTT(NTT(a) (.) b), one CTA per limb (CL = 1).
// Job provides prime(blk), load(blk,i,P) (coefficient-domain a),
// factor(blk,i,P) (NTT-domain b at bit-reversed position i) and store.
template <int LOGN, class Job>
__global__ void __launch_bounds__(NttGeom<LOGN, 1>::T, NttGeom<LOGN, 1>::MINB)
k_ntt_mul_intt(Job job, const PrimeD* __restrict__ primes, const ulonglong2* __restrict__ tw_all,
               const ulonglong2* __restrict__ itw_all) {
  typedef NttGeom<LOGN, 1> G;
  extern __shared__ u64 sm[];
  const u32 tid = threadIdx.x;
  const int blk = blockIdx.x;
  const int pi = job.prime(blk);
  const PrimeD P = load_prime(primes, pi);
  constexpr int PER = G::NL / G::T;
  constexpr int LO_TOP = (G::NPASS - 1) * G::R, NB_TOP = G::LOGNL - LO_TOP;
  const ulonglong2* tw = tw_all + (size_t)pi * G::N;
  const ulonglong2* itw = itw_all + (size_t)pi * G::N;
  ntt_pass_io<LOGN, 1, false, LO_TOP, NB_TOP, 8>(
      tid, 0, tw, P.q, P.two_q, [&](u32 i) { return job.load(blk, i, P); },
      [&](u32 i, u64 v) { sm[spad(i)] = v; });
  __syncthreads();
  ntt_passes<LOGN, 1, false, 1>(sm, tid, 0, tw, P.q, P.two_q);
#pragma unroll 4
  for (int k = 0; k < PER; ++k) {
    const u32 i = tid + k * G::T;
    u64 v = sm[spad(i)];
    v = v >= P.two_q ? v - P.two_q : v;
    v = v >= P.q ? v - P.q : v;
    sm[spad(i)] = mul_mod(v, job.factor(blk, i, P), P);
  }
  __syncthreads();
  ntt_passes<LOGN, 1, true, 0, G::NPASS - 1>(sm, tid, 0, itw, P.q, P.two_q);
  ntt_pass_io<LOGN, 1, true, LO_TOP, NB_TOP, 8>(
      tid, 0, itw, P.q, P.two_q, [&](u32 i) { return sm[spad(i)]; },
      [&](u32 i, u64 v) { job.store(blk, i, mul_shoup(v, P.ninv, P.ninvsh, P.q), P); });
}

// ===================================================== 32-bit arithmetic ===
// Contexts whose primes are all < 2^31 (BASELINE config 4) run the same
// network on u32 registers and shared memory (half the smem, 32x32-bit Shoup
// products); ciphertext words in HBM stay u64 (scratch rows, digits and keys are u32).  Strict butterflies: values stay in [0, q)
// (2q < 2^32, but 4q may not be).  Twiddle table entries are (w, floor(w 2^32 / q));
// entry 0 of the inverse table holds (N^{-1}, its companion).
__device__ __forceinline__ u32 spad32(u32 i) { return i + (i >> 5); }
// words a thread keeps in flight in the HBM-facing loops of the 32-bit engine (chunks, as ntt_pass_io)
#ifndef NTT32_IO_WORDS
#define NTT32_IO_WORDS 8
#endif

// Geometry of the 32-bit engine: 2^R words per thread, T = N / 2^R threads, NPASS passes of R bits.
// Measured at N = 2^13 (profiles/r01_ncu_summary.md): R = 4 with 3 CTAs/SM is the best of R 4/5 x
// 2..5 CTAs/SM; the transforms are latency-bound (load -> passes -> store per CTA, ~35% issue
// utilisation; twiddle loads cost ~10%), the next step is a persistent double-buffered kernel.
#ifndef HE_NTT32_R
#define HE_NTT32_R 0   // 0: the 64-bit engine's choice (R = 4 for N <= 2^14)
#endif
template <int LOGN>
struct NttGeomS {
  static constexpr int N = 1 << LOGN;
  static constexpr int LOGNL = LOGN;
  static constexpr int NL = N;
  static constexpr int R = HE_NTT32_R ? HE_NTT32_R : NttGeom<LOGN, 1>::R;
  static constexpr int T = NL >> R;
  static constexpr int NPASS = (LOGNL + R - 1) / R;
};

// Conditional subtraction as an unsigned min: x - q wraps above 2^31 when
// x < q (all values < 2q < 2^32), so min(x, x - q) is the reduced value; one
// VIADDMNMX instead of ISETP + SEL.
__device__ __forceinline__ u32 csub32(u32 x, u32 q) { return min(x, x - q); }
__device__ __forceinline__ u32 shoup32(u32 x, u32 w, u32 wsh, u32 q) {
  return csub32(x * w - __umulhi(x, wsh) * q, q);   // [0, 2q) -> [0, q)
}
__device__ __forceinline__ void ct_bfly32(u32& x, u32& y, u32 w, u32 wsh, u32 q) {
  const u32 T = shoup32(y, w, wsh, q);
  const u32 u = csub32(x + T, q);
  y = csub32(x - T + q, q);
  x = u;
}
__device__ __forceinline__ void gs_bfly32(u32& x, u32& y, u32 w, u32 wsh, u32 q) {
  const u32 u = csub32(x + y, q);
  const u32 v = x - y + q;   // (0, 2q)
  x = u;
  y = shoup32(v, w, wsh, q);
}

// Harvey-lazy 32-bit butterflies for q < 2^30 (4q < 2^32): CT keeps values in
// [0, 4q), GS in [0, 2q); one conditional subtraction per butterfly.
__device__ __forceinline__ void ct_bfly32_lazy(u32& x, u32& y, u32 w, u32 wsh, u32 q) {
  const u32 X = min(x, x - 2 * q);
  const u32 T = y * w - __umulhi(y, wsh) * q;   // [0, 2q)
  x = X + T;
  y = X - T + 2 * q;
}
__device__ __forceinline__ void gs_bfly32_lazy(u32& x, u32& y, u32 w, u32 wsh, u32 q) {
  const u32 u = min(x + y, x + y - 2 * q);
  const u32 v = x - y + 2 * q;                   // (0, 4q)
  x = u;
  y = v * w - __umulhi(v, wsh) * q;              // [0, 2q)
}

// One pass over bits [LO, LO+NB) reading its inputs through ld(i) and writing its
// outputs through st(i, v): shared memory for the inner passes; the job's
// load (first forward pass) or the final scaling + store (last inverse pass)
// when fused, which saves a shared-memory round trip and a barrier.
template <int LOGN, bool INV, int LO, int NB, bool LAZY, int WORDS = 0, class LD, class ST>
__device__ __forceinline__ void ntt_pass32_io(u32 tid, const uint2* __restrict__ tw, u32 q, LD ld, ST st) {
  typedef NttGeomS<LOGN> G;
  constexpr int NG = 1 << (G::R - NB);
  constexpr int E = 1 << NB;
  constexpr int CH0 = WORDS > E ? WORDS / E : 1;   // groups per chunk (as ntt_pass_io)
  constexpr int CH = (WORDS == 0 || CH0 > NG) ? NG : CH0;
#pragma unroll 1
  for (int c = 0; c < NG / CH; ++c)
#pragma unroll
  for (int gg = 0; gg < CH; ++gg) {
    const int gi = c * CH + gg;
    const u32 g = tid + gi * G::T;
    const u32 base = ((g >> LO) << (LO + NB)) | (g & ((1u << LO) - 1u));
    u32 x[E];
#pragma unroll
    for (int k = 0; k < E; ++k) x[k] = ld(base + (k << LO));
    // twiddle of the butterfly on bit b at index j: tw[2^s + (j >> (b + 1))], s = LOGN-1-b.  With
    // j = hi << (LO+NB) | k << LO | lo, j >> (b+1) = (hi << (LO+NB-1-b)) | (k >> (b+1-LO)): one
    // base pointer per stage and compile-time offsets (identical offsets share one load).
    const u32 hi = g >> LO;
#pragma unroll
    for (int ss = 0; ss < NB; ++ss) {
      const int b = INV ? LO + ss : LO + NB - 1 - ss;
      const int s = LOGN - 1 - b;
      const int half = INV ? 1 << ss : 1 << (NB - 1 - ss);
      const uint2* tws = tw + (1u << s) + (hi << (LO + NB - 1 - b));
#pragma unroll
      for (int k = 0; k < E; ++k) {
        if (k & half) continue;
        const uint2 w = __ldg(tws + (k >> (b + 1 - LO)));
        if (LAZY) {
          if (!INV) ct_bfly32_lazy(x[k], x[k + half], w.x, w.y, q);
          else gs_bfly32_lazy(x[k], x[k + half], w.x, w.y, q);
        } else {
          if (!INV) ct_bfly32(x[k], x[k + half], w.x, w.y, q);
          else gs_bfly32(x[k], x[k + half], w.x, w.y, q);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < E; ++k) st(base + (k << LO), x[k]);
  }
}

// Shared-memory pass.  base has zero bits in [LO, LO+NB), so base + (k << LO) is base | (k << LO)
// and spad32(base + (k << LO)) = spad32(base) + (k << LO) + ((k << LO) >> 5): one padded base
// pointer per group and compile-time offsets (LDS/STS with immediate offsets).
template <int LOGN, bool INV, int LO, int NB, bool LAZY = false>
__device__ __forceinline__ void ntt_pass32(u32* sm, u32 tid, const uint2* __restrict__ tw, u32 q) {
  typedef NttGeomS<LOGN> G;
  constexpr int NG = 1 << (G::R - NB);
  constexpr int E = 1 << NB;
#pragma unroll
  for (int gi = 0; gi < NG; ++gi) {
    const u32 g = tid + gi * G::T;
    const u32 base = ((g >> LO) << (LO + NB)) | (g & ((1u << LO) - 1u));
    u32* p = sm + spad32(base);
    u32 x[E];
#pragma unroll
    for (int k = 0; k < E; ++k) x[k] = p[(k << LO) + ((k << LO) >> 5)];
    const u32 hi = g >> LO;
#pragma unroll
    for (int ss = 0; ss < NB; ++ss) {
      const int b = INV ? LO + ss : LO + NB - 1 - ss;
      const int s = LOGN - 1 - b;
      const int half = INV ? 1 << ss : 1 << (NB - 1 - ss);
      const uint2* tws = tw + (1u << s) + (hi << (LO + NB - 1 - b));
#pragma unroll
      for (int k = 0; k < E; ++k) {
        if (k & half) continue;
        const uint2 w = __ldg(tws + (k >> (b + 1 - LO)));
        if (LAZY) {
          if (!INV) ct_bfly32_lazy(x[k], x[k + half], w.x, w.y, q);
          else gs_bfly32_lazy(x[k], x[k + half], w.x, w.y, q);
        } else {
          if (!INV) ct_bfly32(x[k], x[k + half], w.x, w.y, q);
          else gs_bfly32(x[k], x[k + half], w.x, w.y, q);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < E; ++k) p[(k << LO) + ((k << LO) >> 5)] = x[k];
  }
}

// Warp-local passes.  A full pass (NB = R: one group per thread, g = tid) over bits [LO, LO+R) with
// LO + R <= 5 + R touches, for warp w, exactly the words [w 2^(5+R), (w+1) 2^(5+R)): word =
// (tid >> 5) << (5+R) | ... for every LO <= 5.  Two consecutive such passes (and a warp-ordered
// epilogue) exchange data inside one warp only, so __syncwarp() orders them and the warps of a CTA
// drift apart instead of meeting at a block barrier (at N = 2^13: the passes over bits [7:4], [3:0]).
#ifndef HE_NTT32_WARPSYNC
#define HE_NTT32_WARPSYNC 1
#endif
template <int LOGN, bool INV, int P>
struct Pass32 {
  typedef NttGeomS<LOGN> G;
  static constexpr int GP = INV ? P : G::NPASS - 1 - P;
  static constexpr int LO = GP * G::R;
  static constexpr int NB = (LO + G::R <= G::LOGNL) ? G::R : G::LOGNL - LO;
  static constexpr bool WL = HE_NTT32_WARPSYNC && P >= 0 && P < G::NPASS && NB == G::R && LO <= 5 && G::T % 32 == 0;
};

// Passes P0 .. PEND-1 (pass P covers bit group GP = INV ? P : NPASS-1-P).  TAIL_WL: what follows the
// last pass reads only the words of the thread's own warp region (ntt32_epilogue<.., WL = true>).
template <int LOGN, bool INV, int P, bool LAZY = false, int PEND = NttGeomS<LOGN>::NPASS, bool TAIL_WL = false>
__device__ __forceinline__ void ntt_passes32(u32* sm, u32 tid, const uint2* tw, u32 q) {
  if constexpr (P < PEND) {
    typedef Pass32<LOGN, INV, P> PS;
    ntt_pass32<LOGN, INV, PS::LO, PS::NB, LAZY>(sm, tid, tw, q);
    constexpr bool next_wl = (P + 1 < PEND) ? Pass32<LOGN, INV, (P + 1 < PEND ? P + 1 : P)>::WL : TAIL_WL;
    if constexpr (PS::WL && next_wl) __syncwarp();
    else __syncthreads();
    ntt_passes32<LOGN, INV, P + 1, LAZY, PEND, TAIL_WL>(sm, tid, tw, q);
  }
}

// Forward transform whose first pass reads the input through ld(i) (no staging
// of the input in shared memory); result left in sm (lazy range when q < 2^30).
template <int LOGN, int WORDS = NTT32_IO_WORDS, class LD>
__device__ __forceinline__ void ntt_fwd32_from(u32* sm, u32 tid, const uint2* tw, u32 q, LD ld) {
  typedef NttGeomS<LOGN> G;
  constexpr int LO = (G::NPASS - 1) * G::R, NB = G::LOGNL - LO;
  auto st = [&](u32 i, u32 v) { sm[spad32(i)] = v; };
  if (q < (1u << 30)) {
    ntt_pass32_io<LOGN, false, LO, NB, true, WORDS>(tid, tw, q, ld, st);
    __syncthreads();
    ntt_passes32<LOGN, false, 1, true>(sm, tid, tw, q);
  } else {
    ntt_pass32_io<LOGN, false, LO, NB, false, WORDS>(tid, tw, q, ld, st);
    __syncthreads();
    ntt_passes32<LOGN, false, 1, false>(sm, tid, tw, q);
  }
}

// Inverse transform of the values in sm whose last pass hands each output,
// scaled by N^{-1} (canonical), to st(i, v) instead of shared memory.
template <int LOGN, class ST>
__device__ __forceinline__ void ntt_inv32_to(u32* sm, u32 tid, const uint2* tw, u32 q, ST st) {
  typedef NttGeomS<LOGN> G;
  constexpr int LO = (G::NPASS - 1) * G::R, NB = G::LOGNL - LO;
  const uint2 ni = __ldg(tw);
  auto ld = [&](u32 i) { return sm[spad32(i)]; };
  auto fin = [&](u32 i, u32 v) { st(i, shoup32(v, ni.x, ni.y, q)); };
  if (q < (1u << 30)) {
    ntt_passes32<LOGN, true, 0, true, G::NPASS - 1>(sm, tid, tw, q);
    ntt_pass32_io<LOGN, true, LO, NB, true>(tid, tw, q, ld, fin);
  } else {
    ntt_passes32<LOGN, true, 0, false, G::NPASS - 1>(sm, tid, tw, q);
    ntt_pass32_io<LOGN, true, LO, NB, false>(tid, tw, q, ld, fin);
  }
}

// Runs the lazy network when q < 2^30; outputs are then in [0, 4q) (forward) or
// [0, 2q) (inverse) and must be reduced by the caller (ntt_reduce32).
template <int LOGN, bool INV>
__device__ __forceinline__ void ntt_run32(u32* sm, u32 tid, const uint2* tw, u32 q) {
  if (q < (1u << 30)) ntt_passes32<LOGN, INV, 0, true>(sm, tid, tw, q);
  else ntt_passes32<LOGN, INV, 0, false>(sm, tid, tw, q);
}
__device__ __forceinline__ u32 ntt_reduce32(u32 v, u32 q) {
  v = min(v, v - 2 * q);   // no-op unless q < 2^30 (then v < 4q)
  return min(v, v - q);
}

// Final scaling (inverse) or reduction (forward) of the transform in sm and the job's store; jobs
// with store4 get 4 outputs per call (their operand loads batched ahead of the arithmetic).
// WL: warp w stores the words of its own region [w 32 PER, (w+1) 32 PER) (lane + 32 k: still one
// coalesced 32-word run per instruction), so a warp-local last pass needs only __syncwarp() before it.
template <int LOGN, bool INV, class JB, bool WL = false>
__device__ __forceinline__ void ntt32_epilogue(const JB& jb, const u32* sm, u32 tid, uint2 ni, u32 q) {
  typedef NttGeomS<LOGN> G;
  constexpr int PER = G::NL / G::T;   // the launch has exactly T threads: unrolled, loads batched
  constexpr u32 ST = WL ? 32u : (u32)G::T;
  const u32 i00 = WL ? (tid >> 5) * (32u * PER) + (tid & 31u) : tid;
  if constexpr (has_store4<JB>::value && PER % 4 == 0) {
#pragma unroll 2
    for (int c = 0; c < PER / 4; ++c) {
      const u32 i0 = i00 + 4 * c * ST;
      u32 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const u32 x = sm[spad32(i0 + u * ST)];
        v[u] = INV ? shoup32(x, ni.x, ni.y, q) : ntt_reduce32(x, q);
      }
      jb.store4(i0, ST, v);
    }
  } else {
#pragma unroll 4
    for (int k = 0; k < PER; ++k) {
      const u32 i = i00 + k * ST;
      u32 v = sm[spad32(i)];
      v = INV ? shoup32(v, ni.x, ni.y, q) : ntt_reduce32(v, q);
      jb.store(i, (u64)v);
    }
  }
}

template <int LOGN>
struct NttGeom32 {
  static constexpr int SMEM = ((1 << LOGN) + (1 << LOGN) / 32) * 4;
#ifndef HE_NTT32_MINB
#define HE_NTT32_MINB 3
#endif
  static constexpr int MINB = (1 << LOGN) <= 8192 ? HE_NTT32_MINB : 2;   // 3 CTAs/SM at N = 2^13 (2: -17%)
};

// ---- pipelined persistent variant (jobs with a single u32 input row: raw32 / load_raw) ----------
// Each CTA loops over job blocks blk = blockIdx.x, blockIdx.x + gridDim.x, ...; while block k's
// passes and epilogue run, cp.async streams block k+1's raw input row into a staging buffer, so
// the load latency that a one-shot CTA exposes (load -> passes -> store) is overlapped.
template <int LOGN>
__device__ __forceinline__ void stage_row32(u32* stage, const u32* __restrict__ src, u32 tid) {
  typedef NttGeomS<LOGN> G;
  const u32 base = (u32)__cvta_generic_to_shared(stage);
#pragma unroll
  for (u32 c = tid; c < G::NL / 4; c += G::T)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(base + c * 16), "l"(src + c * 4));
  asm volatile("cp.async.commit_group;\n" ::);
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

// Jobs may give the pipelined kernel a lighter binding (bind_pipe: the fast form only).
template <class Job>
__device__ __forceinline__ auto bind_pipe_job(const Job& j, int blk, const PrimeD& P, int)
    -> decltype(j.bind_pipe(blk, P)) {
  return j.bind_pipe(blk, P);
}
template <class Job>
__device__ __forceinline__ auto bind_pipe_job(const Job& j, int blk, const PrimeD& P, long)
    -> decltype(j.bind32(blk, P)) {
  return j.bind32(blk, P);
}

// The first pass of a block reads its input straight from the staged row (no copy into sm32 and
// no extra barrier): forward = the top bit group (the 1-bit pass at N = 2^13), inverse = bits
// [0, R).  Ends with the barrier after which the staging buffer may be refilled.
template <int LOGN, bool INV, bool LAZY, class JB>
__device__ __forceinline__ void ntt32_pipe_block(const JB& jb, u32* sm, const u32* stage, u32 tid,
                                                 const uint2* tw, u32 q) {
  typedef NttGeomS<LOGN> G;
  constexpr int LO = INV ? 0 : (G::NPASS - 1) * G::R;
  constexpr int NB = (LO + G::R <= G::LOGNL) ? G::R : G::LOGNL - LO;
  auto ld = [&](u32 i) {
    if constexpr (has_load_raw_at<JB>::value) return (u32)jb.load_raw_at(stage[i], i);
    else return (u32)jb.load_raw(stage[i]);
  };
  auto st = [&](u32 i, u32 v) { sm[spad32(i)] = v; };
  ntt_pass32_io<LOGN, INV, LO, NB, LAZY>(tid, tw, q, ld, st);
  __syncthreads();
}

// Inverse: the last pass (the top bit group) fused with the N^{-1} scaling and the job's store.
// Thread tid's outputs are n = tid + m T (m < 2^R) exactly as in ntt32_epilogue: group gi of the
// pass holds m = gi + k NG (k < 2^NB), so four consecutive groups give store4 runs of 4.
template <int LOGN, bool LAZY, class JB>
__device__ __forceinline__ void ntt32_inv_last_store(const JB& jb, const u32* sm, u32 tid, const uint2* tw, u32 q) {
  typedef NttGeomS<LOGN> G;
  constexpr int LO = (G::NPASS - 1) * G::R, NB = G::LOGNL - LO, E = 1 << NB, NG = 1 << (G::R - NB);
  const uint2 ni = __ldg(tw);
#pragma unroll
  for (int c = 0; c < NG / 4; ++c) {
    u32 out[E][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const u32 g = tid + (4 * c + j) * G::T;   // < 2^LO, so the group's base is g
      u32 x[E];
#pragma unroll
      for (int k = 0; k < E; ++k) x[k] = sm[spad32(g + (k << LO))];
#pragma unroll
      for (int ss = 0; ss < NB; ++ss) {
        const int b = LO + ss, s = LOGN - 1 - b, half = 1 << ss;
        const uint2* tws = tw + (1u << s);
#pragma unroll
        for (int k = 0; k < E; ++k) {
          if (k & half) continue;
          const uint2 w = __ldg(tws + (k >> (b + 1 - LO)));
          if (LAZY) gs_bfly32_lazy(x[k], x[k + half], w.x, w.y, q);
          else gs_bfly32(x[k], x[k + half], w.x, w.y, q);
        }
      }
#pragma unroll
      for (int k = 0; k < E; ++k) out[k][j] = shoup32(x[k], ni.x, ni.y, q);
    }
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const u32 n0 = tid + (4 * c + k * NG) * G::T;
      if constexpr (has_store4<JB>::value) {
        jb.store4(n0, G::T, out[k]);
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) jb.store(n0 + u * G::T, (u64)out[k][u]);
      }
    }
  }
}

// The remaining passes of a pipelined block and its epilogue.
template <int LOGN, bool INV, class JB>
__device__ __forceinline__ void ntt32_pipe_rest(const JB& jb, u32* sm, u32 tid, const uint2* tw, u32 q) {
  typedef NttGeomS<LOGN> G;
  constexpr int LO_LAST = (G::NPASS - 1) * G::R, NB_LAST = G::LOGNL - LO_LAST;
  constexpr bool FUSE_LAST = INV && G::NPASS >= 3 && (1 << (G::R - NB_LAST)) % 4 == 0;
  if (!INV) {
    constexpr bool TWL = Pass32<LOGN, false, G::NPASS - 1>::WL;   // the last pass is warp-local: so is the epilogue
    if (q < (1u << 30)) ntt_passes32<LOGN, false, 1, true, G::NPASS, TWL>(sm, tid, tw, q);
    else ntt_passes32<LOGN, false, 1, false, G::NPASS, TWL>(sm, tid, tw, q);
    ntt32_epilogue<LOGN, false, JB, TWL>(jb, sm, tid, __ldg(tw), q);
  } else if constexpr (FUSE_LAST) {
    if (q < (1u << 30)) {
      ntt_passes32<LOGN, true, 1, true, G::NPASS - 1>(sm, tid, tw, q);
      ntt32_inv_last_store<LOGN, true>(jb, sm, tid, tw, q);
    } else {
      ntt_passes32<LOGN, true, 1, false, G::NPASS - 1>(sm, tid, tw, q);
      ntt32_inv_last_store<LOGN, false>(jb, sm, tid, tw, q);
    }
  } else {
    if (q < (1u << 30)) ntt_passes32<LOGN, true, 1, true>(sm, tid, tw, q);
    else ntt_passes32<LOGN, true, 1, false>(sm, tid, tw, q);
    ntt32_epilogue<LOGN, true>(jb, sm, tid, __ldg(tw), q);
  }
}

template <int LOGN, bool INV, class Job>
__global__ void __launch_bounds__(NttGeomS<LOGN>::T, NttGeom32<LOGN>::MINB)
k_ntt32(Job job, const PrimeD* __restrict__ primes, const uint2* __restrict__ tw_all) {
  typedef NttGeomS<LOGN> G;
  extern __shared__ u32 sm32[];
  const u32 tid = threadIdx.x;
  const int blk = blockIdx.x;
  const int pi = job.prime(blk);
  const PrimeD P = load_prime(primes, pi);
  const uint2* tw = tw_all + (size_t)pi * G::N;
  const u32 q = (u32)P.q;
  const auto jb = bind_job(job, blk, P, 0);   // block decomposition + constants, once per CTA
  constexpr int PER = G::NL / G::T;            // the launch has exactly T threads: unrolled loops
  if constexpr (has_load4<decltype(jb)>::value) {   // 4 consecutive words per call (shared draws)
#pragma unroll 2
    for (int k = 0; k < PER / 4; ++k) {
      const u32 j = tid + k * G::T;
      const uint4 v = jb.load4(j);
      sm32[spad32(4 * j)] = v.x;
      sm32[spad32(4 * j + 1)] = v.y;
      sm32[spad32(4 * j + 2)] = v.z;
      sm32[spad32(4 * j + 3)] = v.w;
    }
    __syncthreads();
    ntt_run32<LOGN, INV>(sm32, tid, tw, q);
  } else if constexpr (!INV) {
    // first pass (the top bit group: coalesced) straight from the job's loads
    ntt_fwd32_from<LOGN, io_words_of<Job>::value>(sm32, tid, tw, q, [&](u32 i) { return (u32)jb.load(i); });
  } else {
    constexpr int CH = PER < io_words_of<Job>::value ? PER : io_words_of<Job>::value;
#pragma unroll 1
    for (int c = 0; c < PER / CH; ++c) {
      u32 v[CH];
#pragma unroll
      for (int k = 0; k < CH; ++k) v[k] = (u32)jb.load(tid + (c * CH + k) * G::T);
#pragma unroll
      for (int k = 0; k < CH; ++k) sm32[spad32(tid + (c * CH + k) * G::T)] = v[k];
    }
    __syncthreads();
    constexpr int NB_LAST = G::LOGNL - (G::NPASS - 1) * G::R;
    if constexpr (G::NPASS >= 3 && (1 << (G::R - NB_LAST)) % 4 == 0) {
      // last pass (the top bit group: coalesced) fused with N^{-1} and the job's store
      if (q < (1u << 30)) {
        ntt_passes32<LOGN, true, 0, true, G::NPASS - 1>(sm32, tid, tw, q);
        ntt32_inv_last_store<LOGN, true>(jb, sm32, tid, tw, q);
      } else {
        ntt_passes32<LOGN, true, 0, false, G::NPASS - 1>(sm32, tid, tw, q);
        ntt32_inv_last_store<LOGN, false>(jb, sm32, tid, tw, q);
      }
      return;
    }
    ntt_run32<LOGN, INV>(sm32, tid, tw, q);
  }
  const uint2 ni = __ldg(tw);
  ntt32_epilogue<LOGN, INV>(jb, sm32, tid, ni, q);
}

template <int LOGN>
struct NttGeom32Pipe {
  static constexpr int SMEM = NttGeom32<LOGN>::SMEM + (1 << LOGN) * 4 + 16;   // + staging row + mbarrier
};

// One-thread bulk copies (TMA engine, cp.async.bulk) of a block's input row into the staging buffer,
// completing on an mbarrier (round 2; HE_NTT32_TMA=0 keeps the per-thread cp.async form).
#ifndef HE_NTT32_TMA
#define HE_NTT32_TMA 1
#endif
__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bulk_row_to_smem(u32* dst, const u32* src, u32 bytes, u64* bar) {
  // generic-proxy reads of dst (the previous block's first pass) are ordered before the async writes
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, u32 phase) {
  u32 ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!ok);
}

template <int LOGN, bool INV, class Job>
__global__ void __launch_bounds__(NttGeomS<LOGN>::T, NttGeom32<LOGN>::MINB)
k_ntt32_pipe(Job job, const PrimeD* __restrict__ primes, const uint2* __restrict__ tw_all, int nblk) {
  typedef NttGeomS<LOGN> G;
  extern __shared__ u32 sm32[];
  u32* stage = sm32 + G::NL + G::NL / 32;
  const u32 tid = threadIdx.x;
  int blk = blockIdx.x;
  if (blk >= nblk) return;
#if HE_NTT32_TMA
  u64* bar = reinterpret_cast<u64*>(stage + G::NL);   // 8-byte aligned: (2 NL + NL / 32) words
  u32 phase = 0;
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) bulk_row_to_smem(stage, job.raw32(blk), G::NL * 4, bar);
#else
  stage_row32<LOGN>(stage, job.raw32(blk), tid);
#endif
  for (; blk < nblk; blk += gridDim.x) {
    const int pi = job.prime(blk);
    const PrimeD P = load_prime(primes, pi);
    const uint2* tw = tw_all + (size_t)pi * G::N;
    const u32 q = (u32)P.q;
    const auto jb = bind_pipe_job(job, blk, P, 0);
#ifndef HE_NTT32_PREFETCH
#define HE_NTT32_PREFETCH 1
#endif
    if constexpr (HE_NTT32_PREFETCH && has_prefetch<decltype(jb)>::value) {
      if (tid == 0) jb.prefetch(G::NL);   // the epilogue's operand rows -> L2 while the passes run
    }
#if HE_NTT32_TMA
    mbar_wait(bar, phase);   // the staged row has landed
    phase ^= 1;
#else
    cp_async_wait_all();
#endif
    __syncthreads();   // staged row visible; the previous block's epilogue is done with sm32
    if (q < (1u << 30)) ntt32_pipe_block<LOGN, INV, true>(jb, sm32, stage, tid, tw, q);
    else ntt32_pipe_block<LOGN, INV, false>(jb, sm32, stage, tid, tw, q);
    // ntt32_pipe_block synchronised once the staged row was consumed (its first pass): prefetch
#if HE_NTT32_TMA
    if (tid == 0 && blk + (int)gridDim.x < nblk) bulk_row_to_smem(stage, job.raw32(blk + gridDim.x), G::NL * 4, bar);
#else
    if (blk + (int)gridDim.x < nblk) stage_row32<LOGN>(stage, job.raw32(blk + gridDim.x), tid);
#endif
    ntt32_pipe_rest<LOGN, INV>(jb, sm32, tid, tw, q);
  }
}

// ---- fused digit INTT + ModUp (small primes, the vec_mat paths' ModUp32) ------------------------
// One persistent CTA per (item b, digit j): INTT of limb j of the digit source straight into the
// staging row (u32 coefficients, scaled by N^{-1}), then for every target limb t != j the lift into
// q_t (C16) and the forward transform from that row, stored as u32 extended digits.  The digit's
// coefficient row never reaches HBM and the separate INTT launch (one-shot CTAs reading u64 rows)
// disappears; the words are those of JobLimbsTo32 followed by JobModUp32.
struct StageRowStore {
  u32* row;
  __device__ __forceinline__ void store(u32 n, u64 v) const { row[n] = (u32)v; }
  __device__ __forceinline__ void store4(u32 n0, u32 st, const u32* v) const {
#pragma unroll
    for (int u = 0; u < 4; ++u) row[n0 + u * st] = v[u];
  }
};

template <int LOGN>
__global__ void __launch_bounds__(NttGeomS<LOGN>::T, NttGeom32<LOGN>::MINB)
k_modup32_fused(const u64* __restrict__ dsrc, size_t bs, u32* __restrict__ ext, const u64* __restrict__ qtab,
                int Lc, int K, int L, int nitems, const PrimeD* __restrict__ primes,
                const uint2* __restrict__ tw_all, const uint2* __restrict__ itw_all) {
  typedef NttGeomS<LOGN> G;
  extern __shared__ u32 sm32[];
  u32* stage = sm32 + G::NL + G::NL / 32;
  const u32 tid = threadIdx.x;
  const int nt = Lc + K;
  constexpr int PER = G::NL / G::T, CH = PER < 8 ? PER : 8;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const int b = it / Lc, j = it % Lc;
    {   // INTT of limb j -> stage
      const PrimeD P = load_prime(primes, j);
      const u32 q = (u32)P.q;
      const uint2* itw = itw_all + (size_t)j * G::N;
      const u64* src = dsrc + (size_t)b * bs + (size_t)j * G::N;
#pragma unroll 1
      for (int c = 0; c < PER / CH; ++c) {
        u32 v[CH];
#pragma unroll
        for (int k = 0; k < CH; ++k) v[k] = (u32)src[tid + (c * CH + k) * G::T];
#pragma unroll
        for (int k = 0; k < CH; ++k) sm32[spad32(tid + (c * CH + k) * G::T)] = v[k];
      }
      __syncthreads();
      const StageRowStore st{stage};
      constexpr int NB_LAST = G::LOGNL - (G::NPASS - 1) * G::R;
      if constexpr (G::NPASS >= 3 && (1 << (G::R - NB_LAST)) % 4 == 0) {
        if (q < (1u << 30)) {
          ntt_passes32<LOGN, true, 0, true, G::NPASS - 1>(sm32, tid, itw, q);
          ntt32_inv_last_store<LOGN, true>(st, sm32, tid, itw, q);
        } else {
          ntt_passes32<LOGN, true, 0, false, G::NPASS - 1>(sm32, tid, itw, q);
          ntt32_inv_last_store<LOGN, false>(st, sm32, tid, itw, q);
        }
      } else {
        ntt_run32<LOGN, true>(sm32, tid, itw, q);
        ntt32_epilogue<LOGN, true>(st, sm32, tid, __ldg(itw), q);
      }
      __syncthreads();   // the coefficient row is complete; sm32 is free
    }
    // the next item's digit row -> L2 while this item's nt - 1 forward transforms run
    if (tid == 0 && it + (int)gridDim.x < nitems) {
      const int nx = it + (int)gridDim.x;
      prefetch_l2(dsrc + (size_t)(nx / Lc) * bs + (size_t)(nx % Lc) * G::N, G::N * 8);
    }
    const u32 qj = (u32)__ldg(qtab + j);
    for (int tt = 0; tt < nt - 1; ++tt) {
      const int t = tt < j ? tt : tt + 1;
      const int tp = t < Lc ? t : L + (t - Lc);
      const PrimeD P = load_prime(primes, tp);
      const u32 q = (u32)P.q;
      const uint2* tw = tw_all + (size_t)tp * G::N;
      const JobModUp32::B32 jb{stage, ext + (((size_t)b * Lc + j) * nt + t) * G::N, qj, q, mu32_of(P)};
      if (q < (1u << 30)) ntt32_pipe_block<LOGN, false, true>(jb, sm32, stage, tid, tw, q);
      else ntt32_pipe_block<LOGN, false, false>(jb, sm32, stage, tid, tw, q);
      ntt32_pipe_rest<LOGN, false>(jb, sm32, tid, tw, q);
      __syncthreads();   // the (warp-ordered) epilogue is done with sm32 before the next first pass
    }
  }
}

}  // namespace he
