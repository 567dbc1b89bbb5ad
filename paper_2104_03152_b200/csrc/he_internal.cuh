// he_internal.cuh — context / handle structs and launch helpers shared by the
// kernel translation units of the B200 CKKS library.  Product code.
#pragma once
#include <cuda_runtime.h>

#include <cstdio>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>
#include <type_traits>
#include <utility>
#include <algorithm>

#include "../../include/he_ckks.h"
#include "he_common.cuh"
#include "he_host.h"
#include "he_jobs.cuh"
#include "he_ntt.cuh"

namespace he {

struct HeError : std::runtime_error {
  he_status code;
  HeError(he_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define HE_CK(call)                                                                       \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw ::he::HeError(e_ == cudaErrorMemoryAllocation ? HE_OUT_OF_MEMORY : HE_CUDA_ERROR, \
                          std::string(#call) + ": " + cudaGetErrorString(e_));            \
  } while (0)

}  // namespace he

struct he_context {
  he::HostParams hp;
  int logN = 0, N = 0, L = 0, K = 0, NP = 0;
  uint64_t seed = 0;
  int device = 0;
  cudaStream_t stream = nullptr;
  uint64_t launches = 0;
  bool small_primes = false;  // every prime < 2^31: 64-bit lazy sums of 62-bit products
  // test knob (env HE_PIPE_GRID_CAP at context creation): caps the persistent NTT grid so that the
  // multi-block prefetch loop of k_ntt32_pipe runs at small batch sizes too (tests only; 0 = off)
  int pipe_grid_cap = 0;
  // device tables
  he::PrimeD* d_primes = nullptr;
  ulonglong2 *d_tw2 = nullptr, *d_itw2 = nullptr;  // [NP][N] (w, floor(w 2^64 / q))
  uint2 *d_tw32 = nullptr, *d_itw32 = nullptr;      // [NP][N] (w, floor(w 2^32 / q)); small primes only
  he::u64* d_cdt = nullptr;
  int* d_err = nullptr;   // sticky device-side error flag (asynchronous he_encode_device overflow)
  he::u64 *d_P_mod = nullptr, *d_Pinv_mod = nullptr, *d_Ph_mod = nullptr;
  he::u64 *d_Phat_inv = nullptr, *d_Phat_mod = nullptr;
  he::u64 *d_rs_qinv = nullptr, *d_rs_h = nullptr, *d_crt = nullptr;
  he::u64* d_q = nullptr;
  int* d_slot_index = nullptr;
  double *d_fft_w = nullptr, *d_zeta = nullptr;
  // keys (NTT words)
  bool has_sk = false, has_pk = false, has_rlk = false;
  he::u64* d_sk = nullptr;   // [NP][N]
  he::u64* d_pk = nullptr;   // [2][L][N]
  he::u64* d_rlk = nullptr;  // [L][2][NP][N]
  uint32_t* d_rlk32 = nullptr;  // small primes: Montgomery-form u32 copy
  std::map<he::u64, he::u64*> gk;  // Galois element -> [L][2][NP][N]
  std::map<he::u64, uint32_t*> gk32;
  // device tables indexed by rotation step k in [0, n_s]: Galois element and key
  // pointers (null where no key), built at keygen so the vec_mat paths issue no
  // host-to-device copies (a pageable copy may synchronise the stream)
  uint32_t* d_step_gal = nullptr;
  const he::u64** d_step_key = nullptr;
  const uint32_t** d_step_key32 = nullptr;  // small primes: the same keys as u32 in Montgomery form (k 2^32 mod q)
  std::vector<void*> owned;        // device allocations freed with the context
  // Stream-ordered caching allocator (he_ops.cu dalloc/dfree): freed blocks are kept in
  // exact-size bins and reused by later work on c->stream (the steady-state pipeline asks for
  // the same sizes every step; cudaMallocAsync growing its pool stalled the host 30-530 ms).
  std::map<size_t, std::vector<void*>> free_bins;
  std::map<void*, size_t> live_bytes;
  size_t cached_bytes = 0;
  // caller-installed allocator (he_set_allocator): ciphertext, plaintext and scratch blocks come
  // from alloc(bytes, stream, user) and go back through free(ptr, bytes, stream, user) in stream
  // order (torch's caching allocator in the Python binding); user_owned marks those blocks
  he_alloc_fn user_alloc = nullptr;
  he_free_fn user_free = nullptr;
  void* user_ctx = nullptr;
  std::map<void*, bool> user_owned;
  // opt-in profiler: CUDA events around every NTT-family launch
  struct ProfRec { const char* tag; cudaEvent_t a, b; double bytes; int blocks; double ops; };
  bool prof_on = false;
  std::vector<ProfRec> prof;
  std::vector<cudaEvent_t> ev_pool;
  // CUDA-graph recording (he_graph_begin / he_graph_end): while rec is set, c->stream is the capture
  // stream, dalloc takes graph-owned blocks (cudaMalloc, relaxed capture) and dfree defers
  struct GraphRec {
    cudaStream_t cap = nullptr, orig = nullptr;
    uint64_t launches0 = 0;
    std::vector<void*> owned;     // allocated while recording: freed with the graph
    std::vector<void*> deferred;  // pre-existing blocks freed while recording: released with the graph
  };
  GraphRec* rec = nullptr;
  std::map<void*, bool> graph_owned;   // blocks owned by a live graph (dfree is a no-op for them)
  // Host-input upload path (he_encode / he_encode_encrypt with a host z): two context-owned device
  // buffers filled on a copy stream of the context's own, so the H2D of call i+1 overlaps the kernels
  // of call i on c->stream.  up_done[k]: copy k finished (c->stream waits for it); up_free[k]: the
  // kernels that read buffer k were enqueued (the copy stream waits for it before refilling).
  struct Upload {
    cudaStream_t stream = nullptr;
    double* buf[2] = {nullptr, nullptr};
    size_t cap[2] = {0, 0};
    cudaEvent_t done[2] = {nullptr, nullptr}, free_[2] = {nullptr, nullptr};
    int next = 0;
  } up;
};

struct he_graph {
  he_context* ctx;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  uint64_t kernels = 0;
  std::vector<void*> owned, deferred;
};

struct he_ciphertext {
  he_context* ctx;
  int B, size, level;
  double scale;
  he::u64* d;  // [B][size][level+1][N]
  // fresh symmetric ciphertext: c1 of item b is Uniform(a_seed, (PUR_SYM_A, stream0 + b, i)), so the
  // seeded wire form can omit it (set by he_encrypt_symmetric / seeded deserialization only)
  int seeded = 0;
  he::u64 a_seed = 0, stream0 = 0;
};

struct he_plaintext {
  he_context* ctx;
  int B, level;
  double scale;
  he::u64* d;  // [B][level+1 (+K if qp)][N]
  int qp = 0;  // 1: also carries the K special limbs (data limbs first), for lazy-ModDown products
  uint32_t* dm = nullptr;  // small primes: cached Montgomery-form u32 copy (lazy vec_mat)
  int bsgs_g = 0;          // > 0: vec_mat diagonals in baby-step/giant-step order E[k2][k1], baby step g
  int fold_n = 0, fold_step = 0;  // > 1: folded replicated-output vec_mat, sum_{t<fold_n} rot(., fold_step t)
};

namespace he {

// ---- memory (stream-ordered pool on the context stream) -----------------
void* dalloc(he_context* c, size_t bytes);
void dfree(he_context* c, void* p);
template <class T>
T* dalloc_t(he_context* c, size_t n) { return (T*)dalloc(c, n * sizeof(T)); }

// RAII scratch buffer
struct Scratch {
  he_context* c;
  void* p;
  Scratch(he_context* c_, size_t bytes) : c(c_), p(dalloc(c_, bytes)) {}
  ~Scratch() { dfree(c, p); }
  template <class T> T* as() const { return (T*)p; }
};

inline void check_launch(he_context* c) {
  c->launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw HeError(HE_CUDA_ERROR, std::string("kernel launch: ") + cudaGetErrorString(e));
}

inline cudaEvent_t prof_event(he_context* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  HE_CK(cudaEventCreate(&e));
  return e;
}

// RAII profiling scope around one launch (no-op unless c->prof_on).
struct ProfScope {
  he_context* c;
  he_context::ProfRec rec;
  ProfScope(he_context* c_, const char* tag, double bytes, int blocks, double ops = 0.0) : c(c_) {
    rec = he_context::ProfRec{tag, nullptr, nullptr, bytes, blocks, ops};
    if (c->prof_on) {
      rec.a = prof_event(c);
      rec.b = prof_event(c);
      HE_CK(cudaEventRecord(rec.a, c->stream));
    }
  }
  ~ProfScope() {
    if (c->prof_on && rec.b) {
      cudaEventRecord(rec.b, c->stream);
      c->prof.push_back(rec);
    }
  }
};

// ---- NTT launch with per-instantiation smem opt-in -----------------------
template <int LOGN, int CL, bool INV, class Job>
void launch_ntt_t(he_context* c, const Job& job, int nblk) {
  typedef NttGeom<LOGN, CL> G;
  static bool configured = false;
  auto kern = k_ntt<LOGN, CL, INV, Job>;
  if (!configured) {
    HE_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM));
    HE_CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    if (CL == 2) HE_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    configured = true;
  }
  if (nblk <= 0) return;
  const ulonglong2* tw = INV ? c->d_itw2 : c->d_tw2;
  ProfScope ps(c, Job::kName, c->prof_on ? alg_bytes(job, nblk) : 0.0, nblk,
               c->prof_on ? alg_ops(job, nblk, LOGN) : 0.0);
  if (CL == 1) {
    kern<<<nblk, G::T, G::SMEM, c->stream>>>(job, c->d_primes, tw);
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nblk * CL);
    cfg.blockDim = dim3(G::T);
    cfg.dynamicSmemBytes = G::SMEM;
    cfg.stream = c->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    HE_CK(cudaLaunchKernelEx(&cfg, kern, job, (const PrimeD*)c->d_primes, tw));
  }
  check_launch(c);
}

// Jobs with a single u32 input row (pipe_ok() on the host) run the persistent pipelined kernel.
template <class J, class = void>
struct has_raw32 : std::false_type {};
template <class J>
struct has_raw32<J, std::void_t<decltype(std::declval<const J&>().raw32(0))>> : std::true_type {};

#ifndef HE_NTT32_PIPE
#define HE_NTT32_PIPE 1
#endif

// Kernel attributes and the occupancy-sized grid are configured once per process: the library
// runs one process per GPU, so the first device's values hold for all calls.
template <int LOGN, bool INV, class Job>
void launch_ntt32_pipe(he_context* c, const Job& job, int nblk) {
  typedef NttGeomS<LOGN> G;
  static int grid = 0;
  auto kern = k_ntt32_pipe<LOGN, INV, Job>;
  if (!grid) {
    HE_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, NttGeom32Pipe<LOGN>::SMEM));
    HE_CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    int per_sm = 0, sms = 0;
    HE_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G::T, NttGeom32Pipe<LOGN>::SMEM));
    HE_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
    grid = std::max(1, per_sm) * sms;
  }
  ProfScope ps(c, Job::kName, c->prof_on ? alg_bytes(job, nblk) : 0.0, nblk,
               c->prof_on ? alg_ops(job, nblk, LOGN) : 0.0);
  int gr = std::min(nblk, grid);
  if (c->pipe_grid_cap > 0) gr = std::min(gr, c->pipe_grid_cap);
  kern<<<gr, G::T, NttGeom32Pipe<LOGN>::SMEM, c->stream>>>(
      job, c->d_primes, INV ? c->d_itw32 : c->d_tw32, nblk);
  check_launch(c);
}

template <int LOGN, bool INV, class Job>
void launch_ntt32_t(he_context* c, const Job& job, int nblk) {
  typedef NttGeomS<LOGN> G;
  if constexpr (has_raw32<Job>::value) {
    if (nblk > 0 && HE_NTT32_PIPE && job.pipe_ok()) {
      launch_ntt32_pipe<LOGN, INV>(c, job, nblk);
      return;
    }
  }
  static bool configured = false;
  auto kern = k_ntt32<LOGN, INV, Job>;
  if (!configured) {
    HE_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, NttGeom32<LOGN>::SMEM));
    HE_CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    configured = true;
  }
  if (nblk <= 0) return;
  ProfScope ps(c, Job::kName, c->prof_on ? alg_bytes(job, nblk) : 0.0, nblk,
               c->prof_on ? alg_ops(job, nblk, LOGN) : 0.0);
  kern<<<nblk, G::T, NttGeom32<LOGN>::SMEM, c->stream>>>(job, c->d_primes, INV ? c->d_itw32 : c->d_tw32);
  check_launch(c);
}

#ifndef HE_NTT64_CL14
#define HE_NTT64_CL14 2   // CTAs per 2^14-word limb on the 64-bit engine: a 2-CTA DSMEM cluster (2 per SM; +8% at cfg2)
#endif
template <bool INV, class Job>
void launch_ntt(he_context* c, const Job& job, int nblk) {
  if (c->small_primes && c->d_tw32 && c->logN <= 14) {
    switch (c->logN) {
      case 10: launch_ntt32_t<10, INV>(c, job, nblk); return;
      case 11: launch_ntt32_t<11, INV>(c, job, nblk); return;
      case 12: launch_ntt32_t<12, INV>(c, job, nblk); return;
      case 13: launch_ntt32_t<13, INV>(c, job, nblk); return;
      case 14: launch_ntt32_t<14, INV>(c, job, nblk); return;
    }
  }
  switch (c->logN) {
    case 10: launch_ntt_t<10, 1, INV>(c, job, nblk); break;
    case 11: launch_ntt_t<11, 1, INV>(c, job, nblk); break;
    case 12: launch_ntt_t<12, 1, INV>(c, job, nblk); break;
    case 13: launch_ntt_t<13, 1, INV>(c, job, nblk); break;
    case 14: launch_ntt_t<14, HE_NTT64_CL14, INV>(c, job, nblk); break;
    case 15: launch_ntt_t<15, 2, INV>(c, job, nblk); break;
    default: throw HeError(HE_INVALID_PARAMS, "unsupported log2N");
  }
}

// Grid for row-wise pointwise kernels: x covers N, y covers rows.
inline dim3 rows_grid(he_context* c, size_t rows, int threads = 256) {
  unsigned gx = (unsigned)((c->N + threads - 1) / threads);
  unsigned gy = (unsigned)std::min<size_t>(rows, 65535);
  return dim3(gx, gy ? gy : 1);
}

}  // namespace he
