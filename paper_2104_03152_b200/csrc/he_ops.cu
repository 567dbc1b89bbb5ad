#include <mutex>
#include <unordered_map>
// he_ops.cu — kernels and internal operations of the B200 CKKS hot path
// (SURVEY.md §8(a) a1-a16).  Product code: shares nothing with oracle/.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "he_internal.cuh"
#include "he_jobs.cuh"
#include "he_ops.h"

namespace he {

// ======================================================== memory / setup ===
// Blocks are binned by exact size (rounded to 512 B).  All kernels of a context run on
// c->stream, so a block freed after enqueuing its last use can be handed to work enqueued
// later on the same stream; he_set_stream synchronizes the old stream before switching.
static size_t bin_size(size_t bytes) { return (std::max<size_t>(bytes, 8) + 511) & ~(size_t)511; }

void trim_cache(he_context* c) {
  if (c->free_bins.empty()) return;
  cudaStreamSynchronize(c->stream);
  for (auto& kv : c->free_bins)
    for (void* p : kv.second) cudaFree(p);
  c->free_bins.clear();
  c->cached_bytes = 0;
}

void* dalloc(he_context* c, size_t bytes) {
  const size_t sz = bin_size(bytes);
  if (c->rec) {   // recording a graph: a block only the graph uses (cudaMalloc is legal in relaxed capture)
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, sz);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw HeError(e == cudaErrorMemoryAllocation ? HE_OUT_OF_MEMORY : HE_CUDA_ERROR,
                    std::string("cudaMalloc (graph): ") + cudaGetErrorString(e));
    }
    c->rec->owned.push_back(p);
    c->graph_owned[p] = true;
    c->live_bytes[p] = sz;
    return p;
  }
  if (c->user_alloc) {
    void* p = c->user_alloc(sz, (void*)c->stream, c->user_ctx);
    if (!p) throw HeError(HE_OUT_OF_MEMORY, "the installed allocator returned NULL");
    c->live_bytes[p] = sz;
    c->user_owned[p] = true;
    return p;
  }
  auto it = c->free_bins.find(sz);
  if (it != c->free_bins.end() && !it->second.empty()) {
    void* p = it->second.back();
    it->second.pop_back();
    c->cached_bytes -= sz;
    c->live_bytes[p] = sz;
    return p;
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, sz);
  if (e == cudaErrorMemoryAllocation && c->cached_bytes) {
    cudaGetLastError();
    trim_cache(c);
    e = cudaMalloc(&p, sz);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw HeError(e == cudaErrorMemoryAllocation ? HE_OUT_OF_MEMORY : HE_CUDA_ERROR,
                  std::string("cudaMalloc: ") + cudaGetErrorString(e));
  }
  c->live_bytes[p] = sz;
  return p;
}
void dfree(he_context* c, void* p) {
  if (!p) return;
  auto it = c->live_bytes.find(p);
  if (it == c->live_bytes.end()) return;
  if (c->graph_owned.count(p)) return;   // released by he_graph_free
  if (c->rec) {                            // recorded kernels may still read it: release with the graph
    c->rec->deferred.push_back(p);
    c->graph_owned[p] = true;
    return;
  }
  auto uo = c->user_owned.find(p);
  if (uo != c->user_owned.end()) {   // back to the caller's allocator, in stream order
    c->user_owned.erase(uo);
    c->user_free(p, it->second, (void*)c->stream, c->user_ctx);
    c->live_bytes.erase(it);
    return;
  }
  c->free_bins[it->second].push_back(p);
  c->cached_bytes += it->second;
  c->live_bytes.erase(it);
}

// cudaFuncSetAttribute waits for the device when the kernel is in flight, so a per-call attribute
// set inside a launch path drains the stream; each kernel's dynamic smem limit is raised once.
static void smem_limit_once(const void* f, int bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> done;
  std::lock_guard<std::mutex> lk(mu);
  int& have = done[f];
  if (have >= bytes) return;
  HE_CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  have = bytes;
}

template <class T>
static T* upload(he_context* c, const std::vector<T>& v) {
  T* d = nullptr;
  HE_CK(cudaMalloc(&d, std::max<size_t>(1, v.size()) * sizeof(T)));
  if (!v.empty()) HE_CK(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  c->owned.push_back(d);
  return d;
}

void context_init(he_context* c, const HostParams& hp, u64 seed) {
  c->hp = hp;
  c->logN = hp.logN;
  c->N = hp.N;
  c->L = hp.L;
  c->K = hp.K;
  c->NP = hp.L + hp.K;
  c->seed = seed;
  if (const char* cap = getenv("HE_PIPE_GRID_CAP")) c->pipe_grid_cap = atoi(cap);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    throw HeError(HE_CUDA_ERROR, "no CUDA device available (the library has no CPU fallback)");
  }
  HE_CK(cudaGetDevice(&c->device));
  {
    // Kernel attributes (dynamic smem opt-in) and occupancy-sized persistent grids are configured
    // once per process (he_internal.cuh launch helpers), which holds for one device per process
    // (one process per GPU).  A second device would miss those attributes, so it is
    // refused here instead of failing later at a launch.
    static std::mutex mu;
    static int first_device = -1;
    std::lock_guard<std::mutex> lk(mu);
    if (first_device < 0) first_device = c->device;
    if (first_device != c->device)
      throw HeError(HE_INVALID_PARAMS, "contexts on more than one CUDA device in one process are not supported "
                                       "(one process per GPU)");
  }
  std::vector<PrimeD> pd(c->NP);
  for (int t = 0; t < c->NP; ++t) {
    PrimeD& p = pd[t];
    memset(&p, 0, sizeof(p));
    p.q = hp.q[t];
    p.two_q = 2 * hp.q[t];
    p.mu = hp.mu[t];
    p.ninv = hp.ninv[t];
    p.ninvsh = hp.ninvsh[t];
    p.k = (u32)hp.kbits[t];
    p.mu64 = (u64)((~(u128)0 >> 64) / hp.q[t]);  // floor((2^64 - 1) / q) == floor(2^64 / q) for odd q
    p.r64 = (u64)((((u128)1) << 64) % hp.q[t]);
  }
  c->d_primes = upload(c, pd);
  c->small_primes = true;
  for (u64 q : hp.q) c->small_primes = c->small_primes && q < (1ULL << 31);
  if (c->small_primes) {
    std::vector<uint2> t32(hp.tw.size()), i32(hp.tw.size());
    for (size_t k = 0; k < hp.tw.size(); ++k) {
      const u64 q = hp.q[k / hp.N];
      t32[k] = make_uint2((u32)hp.tw[k], (u32)(((u64)hp.tw[k] << 32) / q));
      i32[k] = make_uint2((u32)hp.itw[k], (u32)(((u64)hp.itw[k] << 32) / q));
    }
    for (int t = 0; t < c->NP; ++t) {   // entry 0 of the inverse table: N^{-1} and its companion
      const u64 q = hp.q[t], ni = hp.ninv[t];
      i32[(size_t)t * hp.N] = make_uint2((u32)ni, (u32)((ni << 32) / q));
    }
    c->d_tw32 = upload(c, t32);
    c->d_itw32 = upload(c, i32);
  }
  {
    std::vector<ulonglong2> t2(hp.tw.size()), i2(hp.tw.size());
    for (size_t k = 0; k < hp.tw.size(); ++k) {
      t2[k] = make_ulonglong2(hp.tw[k], hp.twsh[k]);
      i2[k] = make_ulonglong2(hp.itw[k], hp.itwsh[k]);
    }
    c->d_tw2 = upload(c, t2);
    c->d_itw2 = upload(c, i2);
  }
  c->d_cdt = upload(c, hp.cdt);
  c->d_err = upload(c, std::vector<int>(1, 0));
  c->d_P_mod = upload(c, hp.P_mod);
  c->d_Pinv_mod = upload(c, hp.Pinv_mod);
  c->d_Ph_mod = upload(c, hp.Ph_mod);
  c->d_Phat_inv = upload(c, hp.Phat_inv);
  c->d_Phat_mod = upload(c, hp.Phat_mod);
  c->d_rs_qinv = upload(c, hp.rs_qinv);
  c->d_rs_h = upload(c, hp.rs_h);
  c->d_crt = upload(c, hp.crt_words);
  c->d_slot_index = upload(c, hp.slot_index);
  c->d_fft_w = upload(c, hp.fft_w);
  c->d_zeta = upload(c, hp.zeta_pow);
  c->d_q = upload(c, hp.q);
}

void context_destroy(he_context* c) {
  cudaStreamSynchronize(c->stream);
  if (c->up.stream) {
    cudaStreamSynchronize(c->up.stream);
    for (int k = 0; k < 2; ++k) {
      if (c->up.buf[k]) cudaFree(c->up.buf[k]);
      if (c->up.done[k]) cudaEventDestroy(c->up.done[k]);
      if (c->up.free_[k]) cudaEventDestroy(c->up.free_[k]);
    }
    cudaStreamDestroy(c->up.stream);
    c->up = he_context::Upload();
  }
  for (void* p : c->owned) cudaFree(p);
  for (auto& kv : c->gk) cudaFree(kv.second);
  for (auto& kv : c->gk32) cudaFree(kv.second);
  if (c->d_sk) cudaFree(c->d_sk);
  if (c->d_pk) cudaFree(c->d_pk);
  if (c->d_rlk) cudaFree(c->d_rlk);
  if (c->d_rlk32) cudaFree(c->d_rlk32);
  trim_cache(c);
  for (auto& kv : c->live_bytes) {
    if (c->user_owned.count(kv.first)) c->user_free(kv.first, kv.second, (void*)c->stream, c->user_ctx);
    else cudaFree(kv.first);
  }
  c->live_bytes.clear();
  c->user_owned.clear();
}

void set_allocator(he_context* c, he_alloc_fn alloc, he_free_fn free_fn, void* user) {
  trim_cache(c);   // cached blocks of the internal pool go back to the driver (stream synchronized)
  c->user_alloc = alloc;
  c->user_free = free_fn;
  c->user_ctx = user;
}

// ============================================================== handles ===
he_ciphertext* ct_new(he_context* c, int B, int size, int level, double scale) {
  he_ciphertext* ct = new he_ciphertext{c, B, size, level, scale, nullptr};
  try {
    ct->d = dalloc_t<u64>(c, ct_words(ct));
  } catch (...) {
    delete ct;
    throw;
  }
  return ct;
}
he_plaintext* pt_new(he_context* c, int B, int level, double scale, int qp) {
  he_plaintext* pt = new he_plaintext{c, B, level, scale, nullptr, qp};
  try {
    pt->d = dalloc_t<u64>(c, pt_words(pt));
  } catch (...) {
    delete pt;
    throw;
  }
  return pt;
}
void ct_free(he_ciphertext* ct) {
  if (!ct) return;
  dfree(ct->ctx, ct->d);
  delete ct;
}
void pt_free(he_plaintext* pt) {
  if (!pt) return;
  dfree(pt->ctx, pt->dm);
  dfree(pt->ctx, pt->d);
  delete pt;
}

// ===================================================== pointwise kernels ===
// Rows of N words; row r of a [B][size][Lc][N] array is limb r % Lc.
enum BinOp { OP_ADD = 0, OP_SUB = 1, OP_MUL = 2 };

template <int OP>
__global__ void k_binop(const u64* __restrict__ a, const u64* __restrict__ b, u64* __restrict__ out,
                        const PrimeD* __restrict__ primes, int N, int Lc, size_t rows, size_t a_bs,
                        size_t b_bs, size_t item_rows, size_t b_limb_bs, size_t o_bs) {
  // a_bs / b_bs: item strides in words (0 = broadcast); item_rows = size*Lc.
  // b_limb_bs: stride between b's polys inside an item (0 = same poly for every part).
  for (size_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const size_t item = r / item_rows, ir = r % item_rows;
    const int limb = (int)(ir % Lc);
    const size_t part = ir / Lc;
    const PrimeD P = load_prime(primes, limb);
    const u64* pa = a + item * a_bs + ir * N;
    const u64* pb = b + item * b_bs + part * b_limb_bs + (size_t)limb * N;
    u64* po = out + item * o_bs + ir * N;
    for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
      const u64 x = pa[n], y = pb[n];
      po[n] = OP == OP_ADD ? add_mod(x, y, P.q) : OP == OP_SUB ? sub_mod(x, y, P.q) : mul_mod(x, y, P);
    }
  }
}

__global__ void k_negate(const u64* __restrict__ a, u64* __restrict__ out, const PrimeD* __restrict__ primes,
                         int N, int Lc, size_t rows) {
  for (size_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const u64 q = load_prime(primes, (int)(r % Lc)).q;
    for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x)
      out[r * N + n] = neg_mod(a[r * N + n], q);
  }
}

// (c0 c0', c0 c1' + c1 c0', c1 c1')  (SURVEY a7 tensor)
__global__ void k_tensor(const u64* __restrict__ x, const u64* __restrict__ y, u64* __restrict__ out,
                         const PrimeD* __restrict__ primes, int N, int Lc, size_t rows, size_t x_bs,
                         size_t y_bs) {
  // rows = B * Lc
  const size_t LN = (size_t)Lc * N;
  for (size_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const size_t b = r / Lc;
    const int i = (int)(r % Lc);
    const PrimeD P = load_prime(primes, i);
    const u64* x0 = x + b * x_bs + (size_t)i * N;
    const u64* y0 = y + b * y_bs + (size_t)i * N;
    u64* o = out + b * 3 * LN + (size_t)i * N;
    for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
      const u64 a0 = x0[n], a1 = x0[LN + n], b0 = y0[n], b1 = y0[LN + n];
      o[n] = mul_mod(a0, b0, P);
      o[LN + n] = add_mod(mul_mod(a0, b1, P), mul_mod(a1, b0, P), P.q);
      o[2 * LN + n] = mul_mod(a1, b1, P);
    }
  }
}

// m = c0 + c1 s (+ c2 s^2)
__global__ void k_decrypt(const u64* __restrict__ ct, const u64* __restrict__ sk, u64* __restrict__ out,
                          const PrimeD* __restrict__ primes, int N, int Lc, int size, size_t rows) {
  const size_t LN = (size_t)Lc * N;
  for (size_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const size_t b = r / Lc;
    const int i = (int)(r % Lc);
    const PrimeD P = load_prime(primes, i);
    const u64* c = ct + b * size * LN + (size_t)i * N;
    for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
      const u64 s = sk[(size_t)i * N + n];
      u64 acc = c[n], sp = s;
      for (int p = 1; p < size; ++p) {
        acc = add_mod(acc, mul_mod(c[p * LN + n], sp, P), P.q);
        sp = mul_mod(sp, s, P);
      }
      out[r * N + n] = acc;
    }
  }
}

// c0 = v b + e0 + m, c1 = v a + e1 (C13). noise: [B][3][Lc][N] NTT words (v, e0, e1).
__global__ void k_encrypt_combine(const u64* __restrict__ noise, const u64* __restrict__ pk,
                                  const u64* __restrict__ pt, size_t pt_bs, u64* __restrict__ out,
                                  const PrimeD* __restrict__ primes, int N, int Lc, int L, size_t rows) {
  const size_t LN = (size_t)Lc * N;
  for (size_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const size_t b = r / Lc;
    const int i = (int)(r % Lc);
    const PrimeD P = load_prime(primes, i);
    const u64* v = noise + b * 3 * LN + (size_t)i * N;
    const u64* pb = pk + (size_t)i * N;
    const u64* pa = pk + ((size_t)L + i) * N;
    const u64* m = pt + b * pt_bs + (size_t)i * N;
    u64* o = out + b * 2 * LN + (size_t)i * N;
    for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
      const u64 vv = v[n];
      o[n] = add_mod(add_mod(mul_mod(vv, pb[n], P), v[LN + n], P.q), m[n], P.q);
      o[LN + n] = add_mod(mul_mod(vv, pa[n], P), v[2 * LN + n], P.q);
    }
  }
}

// Small-coefficient sampling (C10 ternary / C11 CDT): row r uses stream
// (pur << 56) | ((obj0 + r) << 16).
__global__ void k_sample_small(i64* __restrict__ out, int N, int rows, u64 seed, u64 pur, u64 obj0, int kind,
                               const u64* __restrict__ cdt) {
  __shared__ u64 T[20];
  if (threadIdx.x < 20) T[threadIdx.x] = cdt[threadIdx.x];
  __syncthreads();
  for (int r = blockIdx.y; r < rows; r += gridDim.y) {
    const u64 sid = stream_sid(pur, obj0 + (u64)r, 0);
    for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x)
      out[(size_t)r * N + n] = kind == 0 ? sample_ternary(seed, sid, n) : sample_cdt(seed, sid, n, T);
  }
}

// Uniform residues drawn as NTT words (C13): row (j, t) for j < nj, t < nt
// writes out + j*j_stride + t*N with stream (pur<<56)|((obj0+j)<<16)|t.
__global__ void k_sample_uniform(u64* __restrict__ out, size_t j_stride, int nj, int nt, int N, u64 seed,
                                 u64 pur, u64 obj0, const PrimeD* __restrict__ primes) {
  for (int r = blockIdx.y; r < nj * nt; r += gridDim.y) {
    const int j = r / nt, t = r % nt;
    const PrimeD P = load_prime(primes, t);
    const u64 sid = stream_sid(pur, obj0 + (u64)j, (u64)t);
    for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x)
      out[(size_t)j * j_stride + (size_t)t * N + n] = sample_uniform(seed, sid, n, P);
  }
}

// pk: b_i = -a_i s_i + e_i over data limbs (a already in pk[1]).
__global__ void k_pk_combine(u64* __restrict__ pk, const u64* __restrict__ e_ntt, const u64* __restrict__ sk,
                             const PrimeD* __restrict__ primes, int N, int L) {
  for (int i = blockIdx.y; i < L; i += gridDim.y) {
    const PrimeD P = load_prime(primes, i);
    for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
      const size_t o = (size_t)i * N + n;
      const u64 a = pk[(size_t)L * N + o];
      pk[o] = add_mod(neg_mod(mul_mod(a, sk[o], P), P.q), e_ntt[o], P.q);
    }
  }
}

// ksk_j = (b_j, a_j): b_j[t] = -a_j[t] s_t + e_j[t] + [t == j] [P]_{q_j} s'_t  (C12).
// key: [L][2][NP][N] with a_j already in part 1; e_ntt: [L][NP][N].
// s' = s^2 (gal == 0) or phi_g(s) in the NTT domain (gal = g).
__global__ void k_ksk_combine(u64* __restrict__ key, const u64* __restrict__ e_ntt, const u64* __restrict__ sk,
                              const u64* __restrict__ P_mod, const PrimeD* __restrict__ primes, int N, int logN,
                              int L, int NP, u32 gal) {
  for (int r = blockIdx.y; r < L * NP; r += gridDim.y) {
    const int j = r / NP, t = r % NP;
    const PrimeD P = load_prime(primes, t);
    const u64 Pq = P_mod[t];
    for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
      const size_t sn = (size_t)t * N + n;
      const u64 a = key[(((size_t)j * 2 + 1) * NP + t) * N + n];
      u64 b = add_mod(neg_mod(mul_mod(a, sk[sn], P), P.q), e_ntt[((size_t)j * NP + t) * N + n], P.q);
      if (t == j) {
        u64 sp;
        if (gal == 0) sp = mul_mod(sk[sn], sk[sn], P);
        else sp = sk[(size_t)t * N + galois_src(n, gal, logN)];
        b = add_mod(b, mul_mod(Pq, sp, P), P.q);
      }
      key[(((size_t)j * 2 + 0) * NP + t) * N + n] = b;
    }
  }
}

__global__ void k_narrow(const u64* __restrict__ src, u32* __restrict__ dst, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = (u32)src[i];
}

// Sum over kk of tmp[kk][item] into acc (vec_mat rotation chunks).
__global__ void k_accumulate(u64* __restrict__ acc, const u64* __restrict__ tmp, int KB, size_t chunk_words,
                             const PrimeD* __restrict__ primes, int N, int Lc, size_t rows) {
  for (size_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const u64 q = load_prime(primes, (int)(r % Lc)).q;
    for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
      u64 s = acc[r * N + n];
      for (int kk = 0; kk < KB; ++kk) s = add_mod(s, tmp[kk * chunk_words + r * N + n], q);
      acc[r * N + n] = s;
    }
  }
}



__global__ void k_check_words(const u64* __restrict__ w, const PrimeD* __restrict__ primes, int N, int Lc,
                              size_t rows, int* bad) {
  for (size_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const u64 q = load_prime(primes, (int)(r % Lc)).q;
    for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x)
      if (w[r * N + n] >= q) atomicOr(bad, 1);
  }
}

// vec_mat with one lazy ModDown: extended-basis accumulator
//   acc_p[t] = sum_{k>=1} D_k[t] sum_j x_j^{(k)}[t] ksk_k[j][p][t]
//            + [t < Lc] [P]_t (D_0 c_p + [p = 0] sum_{k>=1} D_k phi_k(c0))
// with x_j^{(k)}[t][n] = ext[j][t][pi_k(n)] (t != j) or c1[j][pi_k(n)] (t == j): the
// hoisted digits of c1, permuted by the automorphism as they are gathered.
struct LazyArgs {
  int N, logN, Lc, K, L, NP, n;
  const u64* ext;               // [B][Lc][Lc+K][N]
  const u64* ct;                // [B][2][Lc][N]
  const u64* diags;             // [n][Lc+K][N]
  const u64* const* keys;       // [n] device pointers (entry 0 unused)
  const u32* gal;               // [n]
  const u64* P_mod;             // [NP]
  u64* accx;                    // [B][2][Lc+K][N]
  int step = 1;                 // diagonal k multiplies rot(x, k * step) (tables indexed by step)
  const u32* ext32 = nullptr;   // small primes: the extended digits as u32 (replaces ext)
};
constexpr int LAZY_EPT = 2;
constexpr size_t kMaxSmem = 232448;   // opt-in dynamic shared memory per block on sm_100 (227 KB)
// SMALL: every prime < 2^31, so a product of two residues is < 2^62 and up to
// four products (plus a reduced value) sum without overflow in 64 bits: one
// IMAD.WIDE.U32 per term and one reduction per four terms.
template <bool SMALL>
__device__ __forceinline__ u64 mac_reduce(u64 acc, u64 a, u64 b, const PrimeD& P) {
  if (SMALL) return reduce64(acc + (u64)(u32)a * (u32)b, P);
  return add_mod(acc, mul_mod(a, b, P), P.q);
}

template <bool SMALL>
__global__ void __launch_bounds__(256) k_vecmat_lazy(LazyArgs a, const PrimeD* __restrict__ primes) {
  const int t = blockIdx.y, b = blockIdx.z, nt = a.Lc + a.K;
  const int tp = t < a.Lc ? t : a.L + (t - a.Lc);
  const PrimeD P = load_prime(primes, tp);
  const size_t N = a.N, LN = (size_t)a.Lc * N;
  const u64* c0 = a.ct + (size_t)b * 2 * LN;
  const u64* c1 = c0 + LN;
  const u64* ext = a.ext + (size_t)b * a.Lc * nt * N;
  const bool data = t < a.Lc;
  u32 nn[LAZY_EPT];
  u64 acc0[LAZY_EPT], acc1[LAZY_EPT], cc0[LAZY_EPT], cc1[LAZY_EPT];
#pragma unroll
  for (int e = 0; e < LAZY_EPT; ++e) {
    nn[e] = (blockIdx.x * LAZY_EPT + e) * blockDim.x + threadIdx.x;
    acc0[e] = acc1[e] = cc0[e] = cc1[e] = 0;
    if (data) {
      const u64 d0 = a.diags[(size_t)t * N + nn[e]];
      cc0[e] = mac_reduce<SMALL>(0, d0, c0[(size_t)t * N + nn[e]], P);
      cc1[e] = mac_reduce<SMALL>(0, d0, c1[(size_t)t * N + nn[e]], P);
    }
  }
  for (int k = 1; k < a.n; ++k) {
    const u32 g = __ldg(a.gal + k * a.step);
    const u64* key = a.keys[k * a.step];
    const u64* Dk = a.diags + ((size_t)k * nt + t) * N;
#pragma unroll
    for (int e = 0; e < LAZY_EPT; ++e) {
      const u32 n = nn[e], sn = galois_src(n, g, a.logN);
      u64 ip0 = 0, ip1 = 0;
      for (int j = 0; j < a.Lc; ++j) {
        const u64 x = (t == j) ? c1[(size_t)j * N + sn] : ext[((size_t)j * nt + t) * N + sn];
        const u64 kb = __ldg(key + (((size_t)j * 2 + 0) * a.NP + tp) * N + n);
        const u64 ka = __ldg(key + (((size_t)j * 2 + 1) * a.NP + tp) * N + n);
        if (SMALL) {
          ip0 += (u64)(u32)x * (u32)kb;
          ip1 += (u64)(u32)x * (u32)ka;
          if ((j & 3) == 3) {
            ip0 = reduce64(ip0, P);
            ip1 = reduce64(ip1, P);
          }
        } else {
          ip0 = add_mod(ip0, mul_mod(x, kb, P), P.q);
          ip1 = add_mod(ip1, mul_mod(x, ka, P), P.q);
        }
      }
      if (SMALL) {
        ip0 = reduce64(ip0, P);
        ip1 = reduce64(ip1, P);
      }
      const u64 d = __ldg(Dk + n);
      acc0[e] = mac_reduce<SMALL>(acc0[e], d, ip0, P);
      acc1[e] = mac_reduce<SMALL>(acc1[e], d, ip1, P);
      if (data) cc0[e] = mac_reduce<SMALL>(cc0[e], d, c0[(size_t)t * N + sn], P);
    }
  }
  const u64 Pt = __ldg(a.P_mod + tp);
#pragma unroll
  for (int e = 0; e < LAZY_EPT; ++e) {
    if (data) {
      acc0[e] = mac_reduce<SMALL>(acc0[e], Pt, cc0[e], P);
      acc1[e] = mac_reduce<SMALL>(acc1[e], Pt, cc1[e], P);
    }
    a.accx[(((size_t)b * 2 + 0) * nt + t) * N + nn[e]] = acc0[e];
    a.accx[(((size_t)b * 2 + 1) * nt + t) * N + nn[e]] = acc1[e];
  }
}

// Small-prime lazy accumulator (all primes < 2^31): the item's digits for
// target t are staged in shared memory as u32 (the automorphism gathers hit
// smem), keys and diagonals are read as u32 copies in Montgomery form
// (k' = k 2^32 mod q), and every product is reduced with one 32-bit
// Montgomery REDC per PAIR of products (x0 k0' + x1 k1' < q 2^32).  Results
// are the exact residues, bit-identical to the generic path.  One CTA per
// (target limb t, item b).
constexpr int LAZY_SM_T = 1024, LAZY_SM_EPT = 2;
#ifndef HE_BSGS_UNIT_UNROLL
#define HE_BSGS_UNIT_UNROLL 2
#endif
#ifndef HE_BSGS_FIXED
#define HE_BSGS_FIXED 1   // 0: always the runtime-geometry BSGS kernels (A/B experiments)
#endif

__device__ __forceinline__ u32 redc32(u64 T, u32 q, u32 qneg_inv) {
  const u32 m = (u32)T * qneg_inv;
  const u32 t = (u32)((T + (u64)m * q) >> 32);   // < 2q
  return csub32(t, q);
}
__device__ __forceinline__ u32 mont_neg_inv(u32 q) {  // -q^{-1} mod 2^32 (q odd)
  u32 inv = q;
  for (int i = 0; i < 5; ++i) inv *= 2u - q * inv;
  return 0u - inv;
}
__device__ __forceinline__ u32 addq(u32 a, u32 b, u32 q) { return csub32(a + b, q); }

template <int LC>
__global__ void __launch_bounds__(LAZY_SM_T, 1)
k_vecmat_lazy_mont(LazyArgs a, const u32* const* __restrict__ keys32, const u32* __restrict__ dm,
                   const PrimeD* __restrict__ primes) {
  // each thread owns 4 consecutive coefficients: key rows, diagonals and the
  // outputs move as 16-byte vectors; the automorphism gathers come from smem
  constexpr int V = 4;
  extern __shared__ u32 xs[];
  const int t = blockIdx.x, b = blockIdx.y, nt = LC + a.K;
  const int tp = t < LC ? t : a.L + (t - LC);
  const PrimeD P = load_prime(primes, tp);
  const u32 q = (u32)P.q, qi = mont_neg_inv(q);
  const u32 N = a.N, NP = a.NP;
  const u64* c0 = a.ct + (size_t)b * 2 * LC * N;
  const u64* c1 = c0 + (size_t)LC * N;
  const bool data = t < LC;
#pragma unroll
  for (int j = 0; j < LC; ++j) {
    if (t == j || !a.ext32) {
      const u64* src = (t == j) ? c1 + (size_t)j * N : a.ext + (((size_t)b * LC + j) * nt + t) * N;
      for (u32 i = threadIdx.x; i < N; i += LAZY_SM_T) xs[j * N + i] = (u32)src[i];
    } else {
      const u32* src = a.ext32 + (((size_t)b * LC + j) * nt + t) * N;
      for (u32 i = threadIdx.x * 4; i < N; i += LAZY_SM_T * 4)
        *reinterpret_cast<uint4*>(xs + j * N + i) = __ldg(reinterpret_cast<const uint4*>(src + i));
    }
  }
  u32* c0s = xs + LC * N;
  if (data)
    for (u32 i = threadIdx.x; i < N; i += LAZY_SM_T) c0s[i] = (u32)c0[(size_t)t * N + i];
  __syncthreads();
  const u32 Pm = (u32)((((u64)__ldg(a.P_mod + tp)) << 32) % q);
  const u32 keyrow = tp * N, kpart = NP * N, kdig = 2 * NP * N;
  for (u32 tile = 0; tile < N; tile += LAZY_SM_T * V) {
    const u32 n0 = tile + threadIdx.x * V;
    u32 acc0[V], acc1[V], cc0[V], cc1[V];
    {
      uint4 d0 = make_uint4(0, 0, 0, 0);
      if (data) d0 = __ldg(reinterpret_cast<const uint4*>(dm + t * N + n0));
      const u32 dd[V] = {d0.x, d0.y, d0.z, d0.w};
#pragma unroll
      for (int e = 0; e < V; ++e) {
        acc0[e] = acc1[e] = cc0[e] = cc1[e] = 0;
        if (data) {
          cc0[e] = redc32((u64)dd[e] * c0s[n0 + e], q, qi);
          cc1[e] = redc32((u64)dd[e] * xs[t * N + n0 + e], q, qi);   // the t == j digit is c1[t]
        }
      }
    }
    for (int k = 1; k < a.n; ++k) {
      const u32 g = __ldg(a.gal + k * a.step);
      const u32* key = keys32[k * a.step] + keyrow + n0;
      const uint4 dv = __ldg(reinterpret_cast<const uint4*>(dm + ((u32)k * nt + t) * N + n0));
      const u32 dd[V] = {dv.x, dv.y, dv.z, dv.w};
      u32 sn[V];
#pragma unroll
      for (int e = 0; e < V; ++e) sn[e] = galois_src(n0 + e, g, a.logN);
      u32 ip0[V], ip1[V];
#pragma unroll
      for (int e = 0; e < V; ++e) ip0[e] = ip1[e] = 0;
#pragma unroll
      for (int j = 0; j < LC; j += 2) {
        const uint4 kb0 = __ldg(reinterpret_cast<const uint4*>(key + j * kdig));
        const uint4 ka0 = __ldg(reinterpret_cast<const uint4*>(key + j * kdig + kpart));
        uint4 kb1 = make_uint4(0, 0, 0, 0), ka1 = make_uint4(0, 0, 0, 0);
        if (j + 1 < LC) {
          kb1 = __ldg(reinterpret_cast<const uint4*>(key + (j + 1) * kdig));
          ka1 = __ldg(reinterpret_cast<const uint4*>(key + (j + 1) * kdig + kpart));
        }
        const u32 b0[V] = {kb0.x, kb0.y, kb0.z, kb0.w}, a0[V] = {ka0.x, ka0.y, ka0.z, ka0.w};
        const u32 b1[V] = {kb1.x, kb1.y, kb1.z, kb1.w}, a1[V] = {ka1.x, ka1.y, ka1.z, ka1.w};
#pragma unroll
        for (int e = 0; e < V; ++e) {
          const u32 x0 = xs[j * N + sn[e]];
          u64 s0 = (u64)x0 * b0[e], s1 = (u64)x0 * a0[e];
          if (j + 1 < LC) {
            const u32 x1 = xs[(j + 1) * N + sn[e]];
            s0 += (u64)x1 * b1[e];
            s1 += (u64)x1 * a1[e];
          }
          ip0[e] = addq(ip0[e], redc32(s0, q, qi), q);
          ip1[e] = addq(ip1[e], redc32(s1, q, qi), q);
        }
      }
#pragma unroll
      for (int e = 0; e < V; ++e) {
        acc0[e] = addq(acc0[e], redc32((u64)dd[e] * ip0[e], q, qi), q);
        acc1[e] = addq(acc1[e], redc32((u64)dd[e] * ip1[e], q, qi), q);
        if (data) cc0[e] = addq(cc0[e], redc32((u64)dd[e] * c0s[sn[e]], q, qi), q);
      }
    }
    u64* o0 = a.accx + (((size_t)b * 2 + 0) * nt + t) * N + n0;
    u64* o1 = a.accx + (((size_t)b * 2 + 1) * nt + t) * N + n0;
#pragma unroll
    for (int e = 0; e < V; ++e) {
      if (data) {
        acc0[e] = addq(acc0[e], redc32((u64)Pm * cc0[e], q, qi), q);
        acc1[e] = addq(acc1[e], redc32((u64)Pm * cc1[e], q, qi), q);
      }
    }
    reinterpret_cast<ulonglong2*>(o0)[0] = make_ulonglong2(acc0[0], acc0[1]);
    reinterpret_cast<ulonglong2*>(o0)[1] = make_ulonglong2(acc0[2], acc0[3]);
    reinterpret_cast<ulonglong2*>(o1)[0] = make_ulonglong2(acc1[0], acc1[1]);
    reinterpret_cast<ulonglong2*>(o1)[1] = make_ulonglong2(acc1[2], acc1[3]);
  }
}

// Baby-step/giant-step lazy accumulator (small primes): for baby steps k1 < g
// the inner product of rot(x, k1) is computed ONCE and accumulated into all G
// giant-step groups with their own (pre-rotated, Montgomery u32) diagonals
// E[k2][k1]; P (.) c0 is staged so the c0 term joins before the diagonal:
//   acc_p[k2] += E[k2][k1] (ip_p + [p = 0] P c0[pi_k1(n)]).
// accx: [G][B][2][Lc+K][N] u32.
//
// Image-pair / half-ring tiling.  Every rotation element g = 5^k is 1 mod 4, so the NTT-domain
// automorphism pi_g (a8) keeps the top index bit: 2 brv(pi(n)) + 1 = g (2 brv(n) + 1) mod 2N agrees
// with 2 brv(n) + 1 mod 4, i.e. bit 0 of brv, the top bit of n.  A CTA therefore owns one half of
// the ring (top bit h) and needs only that half of the digits - and with the smem of one full-ring
// image it holds the halves of IB = 2 images, so every key row and diagonal it loads serves both
// images (half the key traffic and half the key / diagonal / galois_src instructions per image).
// CTA (t, h, pair): target limb t, coefficients [h N/2, (h+1) N/2), images IB pair + {0, 1}.
//
// Two reduction schedules, chosen per CTA from its target prime q (uniform branch):
// * LAZY (LC q < 2^32 and g q < 2^32, e.g. every 26-bit prime of BASELINE config 4): the LC
//   digit products of one inner product are summed in 64 bits (each < q^2) and reduced by ONE
//   Montgomery REDC (T < LC q^2 < q 2^32, so the result is < 2q); the G diagonal products are
//   accumulated in 64 bits over all g baby steps (sum < g q^2 < 2^64) and reduced once at the
//   end (acc < g q^2 < q 2^32).  Keys and diagonals are stored as k 2^32 mod q, so each REDC
//   removes exactly the one factor 2^32 its products carry: the results are the same residues.
// * PAIRED (q up to 2^31): one REDC per pair of products and per diagonal product (x0 k0' +
//   x1 k1' < 2 q^2 < q 2^32), the sums kept reduced.
// * UNIT (rotation sums: every diagonal is the plaintext polynomial 1, G = 1): no diagonal loads or
//   products.  acc_p = [data] P c_p + sum_k (ip_p,k + [p = 0] P c0[pi_k(n)]); in the lazy schedule the
//   Montgomery-form inner products of ALL baby steps are summed in 64 bits (< g LC q^2 < q 2^32) and
//   reduced by one REDC at the end, the P c terms summed as plain residues: the same residues as the
//   general schedule with the diagonal 2^32 mod q (Montgomery 1), one REDC and one product fewer per
//   baby step, part and coefficient.
template <int LC, int G, int IB, bool LAZY, bool UNIT = false>
__device__ __forceinline__ void bsgs_hp_run(const LazyArgs& a, int g, int B, const u32* const* __restrict__ keys32,
                                            const u32* __restrict__ dm, const u32* xs, const u32* c0p, int t,
                                            int b0, int nimg, int nt, bool data, u32 q, u32 qi, u32 Pm, u32 keyrow,
                                            u32 kpart, u32 kdig, size_t gstride, u32 h0, u32 NH, u32 N, int logN) {
  typedef typename std::conditional<LAZY, u64, u32>::type acc_t;
  if constexpr (UNIT) {
    static_assert(G == 1, "rotation sums have one group");
    for (u32 l = threadIdx.x; l < NH; l += LAZY_SM_T) {
      const u32 n = h0 + l;
      acc_t T0[IB], T1[IB];   // LAZY: 64-bit sums of Montgomery-form products; else reduced residues
      u32 s0[IB], s1[IB];     // plain residues: P c0 terms of every step, P c1 of step 0
#pragma unroll
      for (int i = 0; i < IB; ++i) {
        T0[i] = T1[i] = 0;
        s0[i] = data ? c0p[i * NH + l] : 0u;
        s1[i] = data ? redc32((u64)xs[(i * LC + t) * NH + l] * Pm, q, qi) : 0u;
      }
      constexpr int kStepsInFlight = HE_BSGS_UNIT_UNROLL;   // the key loads of that many baby steps are issued together
#pragma unroll kStepsInFlight
      for (int k = 1; k < g; ++k) {
        const u32 gal = __ldg(a.gal + k * a.step);
        const u32* key = keys32[k * a.step] + keyrow + n;
        const u32 sl = galois_src(n, gal, logN) - h0;
        if (LAZY) {
#pragma unroll
          for (int j = 0; j < LC; ++j) {
            const u32 kb = __ldg(key + j * kdig), ka = __ldg(key + j * kdig + kpart);
#pragma unroll
            for (int i = 0; i < IB; ++i) {
              const u32 x = xs[(i * LC + j) * NH + sl];
              T0[i] += (u64)x * kb;
              T1[i] += (u64)x * ka;
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < LC; j += 2) {
            const u32 kb0 = __ldg(key + j * kdig), ka0 = __ldg(key + j * kdig + kpart);
            const u32 kb1 = j + 1 < LC ? __ldg(key + (j + 1) * kdig) : 0u;
            const u32 ka1 = j + 1 < LC ? __ldg(key + (j + 1) * kdig + kpart) : 0u;
#pragma unroll
            for (int i = 0; i < IB; ++i) {
              const u32 x0 = xs[(i * LC + j) * NH + sl];
              u64 p0 = (u64)x0 * kb0, p1 = (u64)x0 * ka0;
              if (j + 1 < LC) {
                const u32 x1 = xs[(i * LC + j + 1) * NH + sl];
                p0 += (u64)x1 * kb1;
                p1 += (u64)x1 * ka1;
              }
              T0[i] = addq((u32)T0[i], redc32(p0, q, qi), q);
              T1[i] = addq((u32)T1[i], redc32(p1, q, qi), q);
            }
          }
        }
        if (data) {
#pragma unroll
          for (int i = 0; i < IB; ++i) s0[i] = addq(s0[i], c0p[i * NH + sl], q);
        }
      }
      u32* out = reinterpret_cast<u32*>(a.accx);
#pragma unroll
      for (int i = 0; i < IB; ++i) {
        if (i < nimg) {
          const size_t base = ((((size_t)b0 + i) * 2) * nt + t) * N + n;
          out[base] = addq(LAZY ? redc32(T0[i], q, qi) : (u32)T0[i], s0[i], q);
          out[base + (size_t)nt * N] = addq(LAZY ? redc32(T1[i], q, qi) : (u32)T1[i], s1[i], q);
        }
      }
    }
  } else {
  for (u32 l = threadIdx.x; l < NH; l += LAZY_SM_T) {
    const u32 n = h0 + l;
    acc_t acc0[IB][G], acc1[IB][G];
#pragma unroll
    for (int k2 = 0; k2 < G; ++k2) {
      const u32 d = __ldg(dm + k2 * gstride + (size_t)t * N + n);
#pragma unroll
      for (int i = 0; i < IB; ++i) {
        if (data) {   // k1 = 0: P E[k2][0] (.) c
          const u32 pc1 = redc32((u64)xs[(i * LC + t) * NH + l] * Pm, q, qi);
          const u32 pc0 = c0p[i * NH + l];
          if (LAZY) {
            acc0[i][k2] = (u64)d * pc0;
            acc1[i][k2] = (u64)d * pc1;
          } else {
            acc0[i][k2] = redc32((u64)d * pc0, q, qi);
            acc1[i][k2] = redc32((u64)d * pc1, q, qi);
          }
        } else {
          acc0[i][k2] = acc1[i][k2] = 0;
        }
      }
    }
    for (int k = 1; k < g; ++k) {
      const u32 gal = __ldg(a.gal + k * a.step);
      const u32* key = keys32[k * a.step] + keyrow + n;
      const u32 sl = galois_src(n, gal, logN) - h0;   // same half (see above)
      u32 y0[IB], y1[IB];
      if (LAZY) {
        u64 T0[IB], T1[IB];
#pragma unroll
        for (int i = 0; i < IB; ++i) T0[i] = T1[i] = 0;
#pragma unroll
        for (int j = 0; j < LC; ++j) {
          const u32 kb = __ldg(key + j * kdig), ka = __ldg(key + j * kdig + kpart);
#pragma unroll
          for (int i = 0; i < IB; ++i) {
            const u32 x = xs[(i * LC + j) * NH + sl];
            T0[i] += (u64)x * kb;
            T1[i] += (u64)x * ka;
          }
        }
#pragma unroll
        for (int i = 0; i < IB; ++i) {
          y0[i] = redc32(T0[i], q, qi);
          if (data) y0[i] = addq(y0[i], c0p[i * NH + sl], q);
          y1[i] = redc32(T1[i], q, qi);
        }
      } else {
#pragma unroll
        for (int i = 0; i < IB; ++i) {
          y0[i] = data ? c0p[i * NH + sl] : 0u;
          y1[i] = 0;
        }
#pragma unroll
        for (int j = 0; j < LC; j += 2) {
          const u32 kb0 = __ldg(key + j * kdig), ka0 = __ldg(key + j * kdig + kpart);
          const u32 kb1 = j + 1 < LC ? __ldg(key + (j + 1) * kdig) : 0u;
          const u32 ka1 = j + 1 < LC ? __ldg(key + (j + 1) * kdig + kpart) : 0u;
#pragma unroll
          for (int i = 0; i < IB; ++i) {
            const u32 x0 = xs[(i * LC + j) * NH + sl];
            u64 s0 = (u64)x0 * kb0, s1 = (u64)x0 * ka0;
            if (j + 1 < LC) {
              const u32 x1 = xs[(i * LC + j + 1) * NH + sl];
              s0 += (u64)x1 * kb1;
              s1 += (u64)x1 * ka1;
            }
            y0[i] = addq(y0[i], redc32(s0, q, qi), q);
            y1[i] = addq(y1[i], redc32(s1, q, qi), q);
          }
        }
      }
#pragma unroll
      for (int k2 = 0; k2 < G; ++k2) {
        const u32 d = __ldg(dm + k2 * gstride + ((size_t)k * nt + t) * N + n);
#pragma unroll
        for (int i = 0; i < IB; ++i) {
          if (LAZY) {
            acc0[i][k2] += (u64)d * y0[i];
            acc1[i][k2] += (u64)d * y1[i];
          } else {
            acc0[i][k2] = addq(acc0[i][k2], redc32((u64)d * y0[i], q, qi), q);
            acc1[i][k2] = addq(acc1[i][k2], redc32((u64)d * y1[i], q, qi), q);
          }
        }
      }
    }
    u32* out = reinterpret_cast<u32*>(a.accx);
#pragma unroll
    for (int i = 0; i < IB; ++i) {
      if (i < nimg) {
#pragma unroll
        for (int k2 = 0; k2 < G; ++k2) {
          const size_t base = ((((size_t)k2 * B + b0 + i) * 2) * nt + t) * N + n;
          out[base] = LAZY ? redc32(acc0[i][k2], q, qi) : (u32)acc0[i][k2];
          out[base + (size_t)nt * N] = LAZY ? redc32(acc1[i][k2], q, qi) : (u32)acc1[i][k2];
        }
      }
    }
  }
  }   // !UNIT
}

// NFIX / NPFIX != 0: the ring degree and the key's limb count are compile-time constants (the launch
// checks a.N == NFIX, a.NP == NPFIX).  Every key row of a baby step (digit j, part p) is then the one
// 64-bit key pointer plus an immediate, and every staged digit one shared address plus an immediate:
// the general form spends ~40% of its fmaheavy-pipe cycles on 64-bit address products and adds
// (IMAD.WIDE x 4 for the row offsets) and spills loop invariants (profiles/r02, SASS of the per-k loop).
template <int LC, int G, int IB, bool UNIT = false, int NFIX = 0, int NPFIX = 0>
__global__ void __launch_bounds__(LAZY_SM_T, 1)
k_vecmat_bsgs_hp(LazyArgs a, int g, int B, const u32* const* __restrict__ keys32, const u32* __restrict__ dm,
                 const PrimeD* __restrict__ primes) {
  extern __shared__ u32 xs[];   // [IB][LC][N/2] digits of this half, then c0p [IB][N/2]
  // grid (image pairs, halves, targets): the image pairs vary fastest, so the CTAs resident together
  // share one (target, half) and its key rows / diagonals stay in L2 (round 2; targets fastest
  // re-read them from DRAM, ~2.8x the unique bytes)
  const u32 N = NFIX ? (u32)NFIX : (u32)a.N, NP = NPFIX ? (u32)NPFIX : (u32)a.NP;
  constexpr int LOGNFIX = NFIX == 8192 ? 13 : NFIX == 4096 ? 12 : NFIX == 16384 ? 14 : 0;
  static_assert(NFIX == 0 || LOGNFIX != 0, "fixed ring degree: 2^12, 2^13 or 2^14");
  const int logN = NFIX ? LOGNFIX : a.logN;
  const int t = blockIdx.z, nt = LC + a.K;
  const u32 NH = N / 2, h0 = blockIdx.y * NH;
  const int b0 = blockIdx.x * IB, nimg = min(IB, B - b0);
  const int tp = t < LC ? t : a.L + (t - LC);
  const PrimeD P = load_prime(primes, tp);
  const u32 q = (u32)P.q, qi = mont_neg_inv(q);
  const bool data = t < LC;
  const u32 Pm = (u32)((((u64)__ldg(a.P_mod + tp)) << 32) % q);
  u32* c0p = xs + IB * LC * NH;
  for (int i = 0; i < IB; ++i) {
    const int b = b0 + (i < nimg ? i : 0);   // a missing second image repeats the first (never stored)
    const u64* c0 = a.ct + (size_t)b * 2 * LC * N;
    const u64* c1 = c0 + (size_t)LC * N;
#pragma unroll
    for (int j = 0; j < LC; ++j) {
      u32* dst = xs + (i * LC + j) * NH;
      // (loops unrolled by 4: a thread's row loads are issued together, not one DRAM latency each)
      if (t == j || !a.ext32) {
        const u64* src = ((t == j) ? c1 + (size_t)j * N : a.ext + (((size_t)b * LC + j) * nt + t) * N) + h0;
#pragma unroll 4
        for (u32 l = threadIdx.x; l < NH; l += LAZY_SM_T) dst[l] = (u32)src[l];
      } else {
        const u32* src = a.ext32 + (((size_t)b * LC + j) * nt + t) * N + h0;
#pragma unroll 4
        for (u32 l = threadIdx.x * 4; l < NH; l += LAZY_SM_T * 4)
          *reinterpret_cast<uint4*>(dst + l) = __ldg(reinterpret_cast<const uint4*>(src + l));
      }
    }
    if (data)
#pragma unroll 4
      for (u32 l = threadIdx.x; l < NH; l += LAZY_SM_T)
        c0p[i * NH + l] = redc32((u64)(u32)c0[(size_t)t * N + h0 + l] * Pm, q, qi);
  }
  __syncthreads();
  const u32 keyrow = tp * N, kpart = NP * N, kdig = 2 * NP * N;
  const size_t gstride = (size_t)g * nt * N;   // between giant-step groups in dm
  if constexpr (UNIT) {
    if ((u64)LC * g * q < (1ULL << 32))
      bsgs_hp_run<LC, G, IB, true, true>(a, g, B, keys32, dm, xs, c0p, t, b0, nimg, nt, data, q, qi, Pm, keyrow,
                                         kpart, kdig, gstride, h0, NH, N, logN);
    else
      bsgs_hp_run<LC, G, IB, false, true>(a, g, B, keys32, dm, xs, c0p, t, b0, nimg, nt, data, q, qi, Pm, keyrow,
                                          kpart, kdig, gstride, h0, NH, N, logN);
  } else if ((u64)LC * q < (1ULL << 32) && (u64)g * q < (1ULL << 32))
    bsgs_hp_run<LC, G, IB, true>(a, g, B, keys32, dm, xs, c0p, t, b0, nimg, nt, data, q, qi, Pm, keyrow, kpart,
                                 kdig, gstride, h0, NH, N, logN);
  else
    bsgs_hp_run<LC, G, IB, false>(a, g, B, keys32, dm, xs, c0p, t, b0, nimg, nt, data, q, qi, Pm, keyrow, kpart,
                                  kdig, gstride, h0, NH, N, logN);
}

// Fused ModUp + key inner product for small primes (a9 without materialising
// the extended digits): CTA (target limb t, item b) loops over the digits j:
// lift [d]_{q_j} (coefficients) into q_t (C16), 32-bit NTT in smem, then
// accx_p[t][n] += X_j[pi_g(n)] ksk[j][p][t][n] with the Montgomery-form key.
// For j == t the digit is the NTT word itself (dsrc).  Output feeds the
// accx-mode ModDown jobs.
struct FusedArgs {
  int N, logN, Lc, K, L, NP;
  u32 gal;
  const u32* coef;     // [B][Lc][N] INTT'd digits (u32)
  const u64* dsrc;     // digit source NTT words, item stride dsrc_bs
  size_t dsrc_bs;
  const u32* key32;    // [L][2][NP][N] Montgomery form
  const u64* qtab;
  u64* accx;           // [B][2][Lc+K][N]
  int sq = 0;          // 1: the digits are dsrc^2 (square: d2 = x1^2 formed on load)
};
template <int LOGN>
__global__ void __launch_bounds__(NttGeomS<LOGN>::T, (1 << LOGN) <= 8192 ? 2 : 1)
k_modup_ip32(FusedArgs a, const PrimeD* __restrict__ primes, const uint2* __restrict__ tw_all) {
  typedef NttGeomS<LOGN> G;
  extern __shared__ u32 sm32[];
  u32* buf = sm32;                                  // NTT workspace (padded)
  u32* acc = sm32 + G::N + G::N / 32;               // [2][N]
  const int t = blockIdx.x, b = blockIdx.y, nt = a.Lc + a.K;
  const int tp = t < a.Lc ? t : a.L + (t - a.Lc);
  const PrimeD P = load_prime(primes, tp);
  const u32 q = (u32)P.q, qi = mont_neg_inv(q);
  const uint2* tw = tw_all + (size_t)tp * G::N;
  const u32 tid = threadIdx.x;
  for (u32 i = tid; i < 2 * G::N; i += G::T) acc[i] = 0;
  const u32* key = a.key32 + (size_t)tp * G::N;
  const u32 kpart = (u32)a.NP * G::N, kdig = 2 * kpart;
  const u32 mut = (u32)((1ULL << 32) / q);
  for (int j = 0; j < a.Lc; ++j) {
    if (j == t) {
      // compile-time trip counts (the launch has exactly T threads): 8 loads in flight per chunk
      const u64* src = a.dsrc + (size_t)b * a.dsrc_bs + (size_t)j * G::N;
      constexpr int PER = G::N / G::T, CH = PER < 8 ? PER : 8;
#pragma unroll 1
      for (int c = 0; c < PER / CH; ++c) {
        u64 v[CH];
#pragma unroll
        for (int k = 0; k < CH; ++k) v[k] = src[tid + (c * CH + k) * G::T];
#pragma unroll
        for (int k = 0; k < CH; ++k)
          buf[spad32(tid + (c * CH + k) * G::T)] = a.sq ? (u32)mul_mod(v[k], v[k], P) : (u32)v[k];
      }
    } else {
      const u32* src = a.coef + ((size_t)b * a.Lc + j) * G::N;
      const u32 qj = (u32)__ldg(a.qtab + j);
      // the lift feeds the first butterfly pass directly; values end in [0, 4q)
      // when q < 2^30: x k' < 4q^2 < q 2^32 still REDCs
      ntt_fwd32_from<LOGN>(buf, tid, tw, q, [&](u32 i) { return lift32(src[i], qj, q, mut); });
    }
    __syncthreads();
    // 4 consecutive coefficients per step: 16-byte key loads and accumulator updates (compile-time
    // trip count: every step's key loads are issued together)
#pragma unroll
    for (int s4 = 0; s4 < G::N / (4 * G::T); ++s4) {
      const u32 n0 = tid * 4 + s4 * 4 * G::T;
      const uint4 kb = __ldg(reinterpret_cast<const uint4*>(key + j * kdig + n0));
      const uint4 ka = __ldg(reinterpret_cast<const uint4*>(key + j * kdig + kpart + n0));
      uint4 a0 = *reinterpret_cast<uint4*>(acc + n0), a1 = *reinterpret_cast<uint4*>(acc + G::N + n0);
      const u32 kbv[4] = {kb.x, kb.y, kb.z, kb.w}, kav[4] = {ka.x, ka.y, ka.z, ka.w};
      u32 r0[4] = {a0.x, a0.y, a0.z, a0.w}, r1[4] = {a1.x, a1.y, a1.z, a1.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const u32 n = n0 + e;
        const u32 sn = a.gal == 1 ? n : galois_src(n, a.gal, LOGN);
        const u32 x = buf[spad32(sn)];
        r0[e] = addq(r0[e], redc32((u64)x * kbv[e], q, qi), q);
        r1[e] = addq(r1[e], redc32((u64)x * kav[e], q, qi), q);
      }
      *reinterpret_cast<uint4*>(acc + n0) = make_uint4(r0[0], r0[1], r0[2], r0[3]);
      *reinterpret_cast<uint4*>(acc + G::N + n0) = make_uint4(r1[0], r1[1], r1[2], r1[3]);
    }
    __syncthreads();
  }
  // accumulators leave as u32 (every residue < 2^31); the accx-mode ModDown reads u32
  u32* out = reinterpret_cast<u32*>(a.accx);
  for (u32 n0 = tid * 4; n0 < G::N; n0 += G::T * 4) {
    *reinterpret_cast<uint4*>(out + (((size_t)b * 2 + 0) * nt + t) * G::N + n0) =
        *reinterpret_cast<const uint4*>(acc + n0);
    *reinterpret_cast<uint4*>(out + (((size_t)b * 2 + 1) * nt + t) * G::N + n0) =
        *reinterpret_cast<const uint4*>(acc + G::N + n0);
  }
}

// Montgomery-form u32 copy of residues: out[i] = in[i] 2^32 mod q_{prime(i)}.
// rows of N words; row r is limb r % nl with limbs >= lc special (prime L + l - lc).
__global__ void k_to_mont32(const u64* __restrict__ in, u32* __restrict__ out, const PrimeD* __restrict__ primes,
                            int N, int nl, int lc, int L, size_t rows) {
  for (size_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const int l = (int)(r % nl);
    const u64 q = load_prime(primes, l < lc ? l : L + (l - lc)).q;
    for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x)
      out[r * N + n] = (u32)((in[r * N + n] << 32) % q);
  }
}

// The canonical u64 residues of a Montgomery-form u32 row: out[i] = in[i] 2^-32 mod q (one REDC).
// Small-prime contexts keep their switching keys as u32 only; the 64-bit forms
// (key export, the unfused fallback paths) are materialised from them on demand.
__global__ void k_from_mont32(const u32* __restrict__ in, u64* __restrict__ out, const PrimeD* __restrict__ primes,
                              int N, int nl, int lc, int L, size_t rows) {
  for (size_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const int l = (int)(r % nl);
    const u32 q = (u32)load_prime(primes, l < lc ? l : L + (l - lc)).q;
    u32 inv = q;   // Newton: q^-1 mod 2^32 (q odd; 3 correct bits double each step)
    for (int it = 0; it < 5; ++it) inv *= 2u - q * inv;
    const u32 qneg = 0u - inv;
    for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
      const u64 T = in[r * N + n];
      const u32 m = (u32)T * qneg;
      u32 v = (u32)((T + (u64)m * q) >> 32);   // < 2q
      out[r * N + n] = v >= q ? v - q : v;
    }
  }
}

// ============================================================ wire format ===
// (DESIGN.md §3): limb segment (b, p, i) holds N words of w_i = bitlen(q_i) bits,
// LSB first, in 64-bit words; N w_i is a multiple of 64, so segments are aligned.
// Pack: one thread per output word, gathering the <= 64/w + 2 residues it covers.
__global__ void k_wire_pack(const u64* __restrict__ src, u64* __restrict__ out, const u32* __restrict__ width,
                            const u64* __restrict__ seg_word, int N, int Lc, size_t nseg) {
  for (size_t sg = blockIdx.y; sg < nseg; sg += gridDim.y) {
    const int i = (int)(sg % Lc);
    const u32 w = width[i];
    const u64* x = src + sg * N;
    u64* o = out + seg_word[sg];
    const u32 nw = (u32)((u64)N * w / 64);
    for (u32 k = blockIdx.x * blockDim.x + threadIdx.x; k < nw; k += gridDim.x * blockDim.x) {
      const u64 bit0 = (u64)k * 64;
      u32 c = (u32)(bit0 / w);
      long pos = (long)((u64)c * w) - (long)bit0;   // <= 0
      u64 acc = 0;
      for (; pos < 64 && c < (u32)N; ++c, pos += w) acc |= pos < 0 ? x[c] >> (-pos) : x[c] << pos;
      o[k] = acc;
    }
  }
}
// Unpack: one thread per residue; flags any residue >= q (corrupt input).
__global__ void k_wire_unpack(const u64* __restrict__ in, u64* __restrict__ dst, const u32* __restrict__ width,
                              const u64* __restrict__ seg_word, const PrimeD* __restrict__ primes, int N, int Lc,
                              size_t nseg, int* bad) {
  for (size_t sg = blockIdx.y; sg < nseg; sg += gridDim.y) {
    const int i = (int)(sg % Lc);
    const u32 w = width[i];
    const u64 q = load_prime(primes, i).q;
    const u64* s = in + seg_word[sg];
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gridDim.x * blockDim.x) {
      const u64 bit = (u64)c * w;
      const u32 k = (u32)(bit >> 6), off = (u32)(bit & 63);
      u64 v = s[k] >> off;
      if (off + w > 64) v |= s[k + 1] << (64 - off);
      v &= (w == 64) ? ~0ULL : ((1ULL << w) - 1);
      if (v >= q) atomicOr(bad, 1);
      dst[sg * N + c] = v;
    }
  }
}

static void wire_tables(he_context* c, int level, size_t B, int size, std::vector<u32>& width,
                        std::vector<u64>& seg_word, u64& total_words) {
  const int Lc = level + 1;
  width.resize(Lc);
  for (int i = 0; i < Lc; ++i) width[i] = (u32)c->hp.kbits[i];
  seg_word.resize(B * size * Lc);
  u64 off = 0;
  for (size_t sg = 0; sg < seg_word.size(); ++sg) {
    seg_word[sg] = off;
    off += (u64)c->N * width[sg % Lc] / 64;
  }
  total_words = off;
}

size_t wire_payload_bytes(he_context* c, const he_ciphertext* ct) {
  std::vector<u32> w;
  std::vector<u64> sw;
  u64 tot;
  wire_tables(c, ct->level, ct->B, ct->size, w, sw, tot);
  return tot * 8;
}

void wire_pack(he_context* c, const he_ciphertext* ct, u64* out_dev) {
  std::vector<u32> w;
  std::vector<u64> sw;
  u64 tot;
  wire_tables(c, ct->level, ct->B, ct->size, w, sw, tot);
  Scratch dw(c, w.size() * 4), ds(c, sw.size() * 8);
  HE_CK(cudaMemcpyAsync(dw.p, w.data(), w.size() * 4, cudaMemcpyHostToDevice, c->stream));
  HE_CK(cudaMemcpyAsync(ds.p, sw.data(), sw.size() * 8, cudaMemcpyHostToDevice, c->stream));
  const size_t nseg = sw.size();
  {
    ProfScope ps_(c, "wire_pack", 8.0 * c->N * nseg + 8.0 * tot, 0);
    k_wire_pack<<<dim3((c->N * 62 / 64 + 255) / 256, (unsigned)std::min<size_t>(nseg, 65535)), 256, 0, c->stream>>>(
        ct->d, out_dev, dw.as<u32>(), ds.as<u64>(), c->N, ct->level + 1, nseg);
  }
  check_launch(c);
  HE_CK(cudaStreamSynchronize(c->stream));   // the scratch tables are freed on return
}

he_ciphertext* wire_unpack(he_context* c, const u64* in_dev, size_t B, int size, int level, double scale) {
  std::vector<u32> w;
  std::vector<u64> sw;
  u64 tot;
  wire_tables(c, level, B, size, w, sw, tot);
  Scratch dw(c, w.size() * 4), ds(c, sw.size() * 8), flag(c, 4);
  HE_CK(cudaMemcpyAsync(dw.p, w.data(), w.size() * 4, cudaMemcpyHostToDevice, c->stream));
  HE_CK(cudaMemcpyAsync(ds.p, sw.data(), sw.size() * 8, cudaMemcpyHostToDevice, c->stream));
  HE_CK(cudaMemsetAsync(flag.p, 0, 4, c->stream));
  he_ciphertext* ct = ct_new(c, (int)B, size, level, scale);
  const size_t nseg = sw.size();
  {
    ProfScope ps_(c, "wire_unpack", 8.0 * c->N * nseg + 8.0 * tot, 0);
    k_wire_unpack<<<dim3((c->N + 255) / 256, (unsigned)std::min<size_t>(nseg, 65535)), 256, 0, c->stream>>>(
        in_dev, ct->d, dw.as<u32>(), ds.as<u64>(), c->d_primes, c->N, level + 1, nseg, flag.as<int>());
  }
  check_launch(c);
  int h = 0;
  HE_CK(cudaMemcpyAsync(&h, flag.p, 4, cudaMemcpyDeviceToHost, c->stream));
  HE_CK(cudaStreamSynchronize(c->stream));
  if (h) {
    ct_free(ct);
    throw HeError(HE_INVALID_ARGUMENT, "wire: residue not reduced mod its prime (corrupt payload)");
  }
  return ct;
}

// ======================================================== encode / decode ===
// Canonical embedding (C6) with a length-M = N/2 complex FFT:
//   encode  w_i = zeta^{-i} sum_r Z[r] omega^{-i r},  Z[r_j] = z_j,
//           m_i = round(c Re w_i), m_{i+M} = round(c Im w_i), c = 2 scale / N;
//   decode  y_i = (X_i + i X_{i+M}) zeta^i,  z_j = Re(sum_i y_i omega^{i r_j}) / scale,
// with omega = exp(2 pi i / M), 5^j = 4 r_j + 1 (mod 2N).
__device__ void fft_inplace(double2* buf, int M, const double* __restrict__ w, double sign) {
  for (int len = 2; len <= M; len <<= 1) {
    const int half = len >> 1, step = M / len;
    for (int t = threadIdx.x; t < M / 2; t += blockDim.x) {
      const int pos = t % half;
      const int i0 = (t / half) * len + pos, i1 = i0 + half;
      const double c = w[2 * pos * step], s = sign * w[2 * pos * step + 1];
      const double2 u = buf[i0], v = buf[i1];
      const double2 vw = make_double2(v.x * c - v.y * s, v.x * s + v.y * c);
      buf[i0] = make_double2(u.x + vw.x, u.y + vw.y);
      buf[i1] = make_double2(u.x - vw.x, u.y - vw.y);
    }
    __syncthreads();
  }
}

__global__ void k_encode_fft(const double* __restrict__ z, size_t n, double scale, i64* __restrict__ m_out,
                             int* overflow, const int* __restrict__ slot_index, const double* __restrict__ w,
                             const double* __restrict__ zeta, int N, int logM, double2* gscratch,
                             double* __restrict__ pre_out = nullptr) {
  extern __shared__ double2 fbuf[];
  const int M = N / 2;
  const int b = blockIdx.x;
  double2* buf = gscratch ? gscratch + (size_t)b * M : fbuf;
  for (int i = threadIdx.x; i < M; i += blockDim.x) buf[i] = make_double2(0.0, 0.0);
  __syncthreads();
  for (size_t j = threadIdx.x; j < n; j += blockDim.x)
    buf[__brev((unsigned)slot_index[j]) >> (32 - logM)] = make_double2(z[(size_t)b * n + j], 0.0);
  __syncthreads();
  fft_inplace(buf, M, w, -1.0);
  const double c = 2.0 * scale / (double)N;
  const double lim = 4611686018427387904.0;  // 2^62
  for (int i = threadIdx.x; i < M; i += blockDim.x) {
    const double zr = zeta[2 * i], zi = -zeta[2 * i + 1];  // zeta^{-i}
    const double2 v = buf[i];
    const double re = c * (v.x * zr - v.y * zi), im = c * (v.x * zi + v.y * zr);
    if (pre_out) {   // he_encode_unrounded: the values this kernel rounds
      pre_out[(size_t)b * N + i] = re;
      pre_out[(size_t)b * N + i + M] = im;
    }
    if (!(fabs(re) < lim) || !(fabs(im) < lim)) {
      atomicOr(overflow, 1);
      m_out[(size_t)b * N + i] = 0;
      m_out[(size_t)b * N + i + M] = 0;
    } else {
      m_out[(size_t)b * N + i] = llround(re);
      m_out[(size_t)b * N + i + M] = llround(im);
    }
  }
}

__global__ void k_decode_fft(const double* __restrict__ X, size_t n, double scale, double* __restrict__ z,
                             const int* __restrict__ slot_index, const double* __restrict__ w,
                             const double* __restrict__ zeta, int N, int logM, double2* gscratch) {
  extern __shared__ double2 fbuf[];
  const int M = N / 2;
  const int b = blockIdx.x;
  double2* buf = gscratch ? gscratch + (size_t)b * M : fbuf;
  const double* x = X + (size_t)b * N;
  for (int i = threadIdx.x; i < M; i += blockDim.x) {
    const double a = x[i], c = x[i + M], zr = zeta[2 * i], zi = zeta[2 * i + 1];
    buf[__brev((unsigned)i) >> (32 - logM)] = make_double2(a * zr - c * zi, a * zi + c * zr);
  }
  __syncthreads();
  fft_inplace(buf, M, w, 1.0);
  for (size_t j = threadIdx.x; j < n; j += blockDim.x) z[(size_t)b * n + j] = buf[slot_index[j]].x / scale;
}

// CRT compose (a13): X = sum_i [x_i Qhat_i^{-1}]_{q_i} Qhat_i mod Q, centred, to double.
constexpr int CRT_MAXW = 40;
__global__ void k_crt_compose(const u64* __restrict__ coef, double* __restrict__ X, const u64* __restrict__ crt,
                              const PrimeD* __restrict__ primes, int N, int Lc, size_t total,
                              i64* __restrict__ Xi = nullptr, int* ovf = nullptr) {
  const u64* Qhat_inv = crt;
  const u64* Qhat = crt + Lc;
  const u64* Q = Qhat + (size_t)Lc * Lc;
  const u64* Qh = Q + Lc;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const size_t b = idx / N;
    const int n = (int)(idx % N);
    u64 acc[CRT_MAXW + 1];
    for (int w = 0; w <= Lc; ++w) acc[w] = 0;
    for (int i = 0; i < Lc; ++i) {
      const PrimeD P = load_prime(primes, i);
      const u64 a = mul_mod(coef[(b * Lc + i) * N + n], Qhat_inv[i], P);
      u64 carry = 0;
      for (int w = 0; w < Lc; ++w) {
        const u64 m = Qhat[(size_t)i * Lc + w];
        const u64 lo = a * m, hi = __umul64hi(a, m);
        u64 s = acc[w] + lo;
        u64 c1 = s < lo;
        s += carry;
        c1 += s < carry;
        acc[w] = s;
        carry = hi + c1;
      }
      for (int w = Lc; w <= Lc && carry; ++w) {
        acc[w] += carry;
        carry = 0;
      }
    }
    // reduce mod Q: acc < Lc Q
    for (int it = 0; it < Lc + 1; ++it) {
      bool ge = acc[Lc] != 0;
      if (!ge) {
        ge = true;
        for (int w = Lc - 1; w >= 0; --w) {
          if (acc[w] != Q[w]) { ge = acc[w] > Q[w]; break; }
        }
      }
      if (!ge) break;
      u64 borrow = 0;
      for (int w = 0; w < Lc; ++w) {
        const u64 d = acc[w] - Q[w] - borrow;
        borrow = (acc[w] < Q[w] + borrow) || (Q[w] + borrow < Q[w]) ? 1 : 0;
        acc[w] = d;
      }
      acc[Lc] -= borrow;
    }
    // centre: X > floor(Q/2) -> X - Q
    bool gt = false;
    for (int w = Lc - 1; w >= 0; --w) {
      if (acc[w] != Qh[w]) { gt = acc[w] > Qh[w]; break; }
    }
    double v = 0.0;
    if (gt) {
      u64 borrow = 0;
      for (int w = 0; w < Lc; ++w) {  // mag = Q - acc
        const u64 d = Q[w] - acc[w] - borrow;
        borrow = (Q[w] < acc[w] + borrow) || (acc[w] + borrow < acc[w]) ? 1 : 0;
        acc[w] = d;
      }
    }
    if (Xi) {   // exact centred integer (|X| < 2^63), else flagged
      bool fits = acc[0] < (1ULL << 63);
      for (int w = 1; w < Lc; ++w) fits = fits && acc[w] == 0;
      if (!fits) atomicOr(ovf, 1);
      Xi[idx] = fits ? (gt ? -(i64)acc[0] : (i64)acc[0]) : 0;
      continue;
    }
    for (int w = Lc - 1; w >= 0; --w) v = v * 18446744073709551616.0 + (double)acc[w];
    X[idx] = gt ? -v : v;
  }
}

// ======================================================== internal ops ===
static dim3 rows_grid2(he_context* c, size_t rows) { return rows_grid(c, rows, 256); }

void ntt_rows(he_context* c, const u64* src, u64* dst, size_t items, int nl, size_t src_bs, size_t dst_bs,
              bool inverse) {
  JobLimbs j{src, dst, c->N, nl, src_bs, dst_bs};
  if (inverse) launch_ntt<true>(c, j, (int)(items * nl));
  else launch_ntt<false>(c, j, (int)(items * nl));
}

void ring_mul(he_context* c, const u64* a, const u64* b, u64* out, size_t items, int nl) {
  JobRingMul j{a, b, out, c->N, nl};
  const int nblk = (int)(items * nl);
  auto run = [&](auto kern, int T, int smem) {
    static_cast<void>(T);
    smem_limit_once((const void*)kern, smem);
    {
      ProfScope ps_(c, "ntt_mul_intt", alg_bytes(j, nblk), nblk, nblk * (2 * ntt_ops(c->N, c->logN) + c->N));
      kern<<<nblk, T, smem, c->stream>>>(j, c->d_primes, c->d_tw2, c->d_itw2);
    }
    check_launch(c);
  };
  switch (c->logN) {
    case 10: run(k_ntt_mul_intt<10, JobRingMul>, NttGeom<10, 1>::T, NttGeom<10, 1>::SMEM); break;
    case 11: run(k_ntt_mul_intt<11, JobRingMul>, NttGeom<11, 1>::T, NttGeom<11, 1>::SMEM); break;
    case 12: run(k_ntt_mul_intt<12, JobRingMul>, NttGeom<12, 1>::T, NttGeom<12, 1>::SMEM); break;
    case 13: run(k_ntt_mul_intt<13, JobRingMul>, NttGeom<13, 1>::T, NttGeom<13, 1>::SMEM); break;
    case 14: run(k_ntt_mul_intt<14, JobRingMul>, NttGeom<14, 1>::T, NttGeom<14, 1>::SMEM); break;
    default: {
      // N = 32768: three passes (the fused single-CTA form needs 256 KB of smem)
      Scratch t(c, items * nl * (size_t)c->N * 8);
      const size_t bs = (size_t)nl * c->N;
      ntt_rows(c, a, t.as<u64>(), items, nl, bs, bs, false);
      modmul_rows(c, t.as<u64>(), b, t.as<u64>(), items, nl);
      ntt_rows(c, t.as<u64>(), out, items, nl, bs, bs, true);
    }
  }
}

void modmul_rows(he_context* c, const u64* a, const u64* b, u64* out, size_t items, int nl) {
  const size_t rows = items * nl;
  {
    ProfScope ps_(c, "pw_mul", 0.0, 0);
    k_binop<OP_MUL><<<rows_grid2(c, rows), 256, 0, c->stream>>>(a, b, out, c->d_primes, c->N, nl, rows,
                                                                (size_t)nl * c->N, (size_t)nl * c->N, nl, 0,
                                                                (size_t)nl * c->N);
  }
  check_launch(c);
}

void signed_to_ntt(he_context* c, const i64* poly, u64* dst, size_t items, int nl, int lc) {
  JobSignedToNtt j{poly, dst, c->N, nl, (size_t)c->N, (size_t)nl * c->N, lc < 0 ? nl : lc, c->L};
  launch_ntt<false>(c, j, (int)(items * nl));
}

// ---- arithmetic -----------------------------------------------------------
he_ciphertext* ct_binop(he_context* c, int op, const he_ciphertext* a, const he_ciphertext* b, he_ciphertext* into) {
  const int B = std::max(a->B, b->B), Lc = a->level + 1;
  he_ciphertext* o = into ? into : ct_new(c, B, a->size, a->level, a->scale);
  const size_t rows = (size_t)B * a->size * Lc, LN = (size_t)Lc * c->N;
  const size_t a_bs = a->B == 1 ? 0 : a->size * LN, b_bs = b->B == 1 ? 0 : b->size * LN;
  // b indexed like a: pass b_limb_bs = LN with b pointer per part
  dim3 g = rows_grid2(c, rows);
  if (op == OP_ADD)
    {
      ProfScope ps_(c, "pw_add", 0.0, 0);
      k_binop<OP_ADD><<<g, 256, 0, c->stream>>>(a->d, b->d, o->d, c->d_primes, c->N, Lc, rows, a_bs, b_bs,
                                                (size_t)a->size * Lc, LN, a->size * LN);
    }
  else
    {
      ProfScope ps_(c, "pw_sub", 0.0, 0);
      k_binop<OP_SUB><<<g, 256, 0, c->stream>>>(a->d, b->d, o->d, c->d_primes, c->N, Lc, rows, a_bs, b_bs,
                                                (size_t)a->size * Lc, LN, a->size * LN);
    }
  check_launch(c);
  return o;
}

he_ciphertext* ct_negate(he_context* c, const he_ciphertext* a) {
  const int Lc = a->level + 1;
  he_ciphertext* o = ct_new(c, a->B, a->size, a->level, a->scale);
  const size_t rows = (size_t)a->B * a->size * Lc;
  {
    ProfScope ps_(c, "pw_negate", 0.0, 0);
    k_negate<<<rows_grid2(c, rows), 256, 0, c->stream>>>(a->d, o->d, c->d_primes, c->N, Lc, rows);
  }
  check_launch(c);
  return o;
}

he_ciphertext* ct_mul_plain(he_context* c, const he_ciphertext* a, const he_plaintext* p, he_ciphertext* into) {
  const int Lc = a->level + 1;
  const int B = std::max(a->B, p->B);
  const double scale = a->scale * p->scale;
  he_ciphertext* o = into ? into : ct_new(c, B, a->size, a->level, scale);
  o->scale = scale;
  const size_t LN = (size_t)Lc * c->N, rows = (size_t)B * a->size * Lc;
  {
    ProfScope ps_(c, "pw_mul", 0.0, 0);
    k_binop<OP_MUL><<<rows_grid2(c, rows), 256, 0, c->stream>>>(a->d, p->d, o->d, c->d_primes, c->N, Lc, rows,
                                                                a->B == 1 ? 0 : a->size * LN, p->B == 1 ? 0 : LN,
                                                                (size_t)a->size * Lc, 0, a->size * LN);
  }
  check_launch(c);
  return o;
}

he_ciphertext* ct_add_plain(he_context* c, const he_ciphertext* a, const he_plaintext* p, he_ciphertext* into) {
  const int Lc = a->level + 1;
  const int B = std::max(a->B, p->B);
  he_ciphertext* o = into ? into : ct_new(c, B, a->size, a->level, a->scale);
  const size_t LN = (size_t)Lc * c->N;
  // poly 0 of every item: a + p (items as size-1 rows at stride size*LN) ...
  const size_t rows = (size_t)B * Lc;
  {
    ProfScope ps_(c, "pw_add", 0.0, 0);
    k_binop<OP_ADD><<<rows_grid2(c, rows), 256, 0, c->stream>>>(a->d, p->d, o->d, c->d_primes, c->N, Lc, rows,
                                                                a->B == 1 ? 0 : a->size * LN, p->B == 1 ? 0 : LN,
                                                                Lc, 0, a->size * LN);
  }
  check_launch(c);
  // ... and polys 1..size-1 copied: one strided copy (a per-item loop only to broadcast a single item)
  if (a->size > 1 && o != a) {
    const size_t w = (size_t)(a->size - 1) * LN * 8, pitch = (size_t)a->size * LN * 8;
    if (a->B == B) {
      HE_CK(cudaMemcpy2DAsync(o->d + LN, pitch, a->d + LN, pitch, w, B, cudaMemcpyDeviceToDevice, c->stream));
    } else {
      for (int b = 0; b < B; ++b)
        HE_CK(cudaMemcpyAsync(o->d + (size_t)b * a->size * LN + LN, a->d + LN, w, cudaMemcpyDeviceToDevice,
                              c->stream));
    }
  }
  return o;
}

he_ciphertext* ct_tensor(he_context* c, const he_ciphertext* x, const he_ciphertext* y) {
  const int Lc = x->level + 1;
  const int B = std::max(x->B, y->B);
  he_ciphertext* o = ct_new(c, B, 3, x->level, x->scale * y->scale);
  const size_t LN = (size_t)Lc * c->N, rows = (size_t)B * Lc;
  {
    ProfScope ps_(c, "pw_tensor", 0.0, 0);
    k_tensor<<<rows_grid2(c, rows), 256, 0, c->stream>>>(x->d, y->d, o->d, c->d_primes, c->N, Lc, rows,
                                                         x->B == 1 ? 0 : 2 * LN, y->B == 1 ? 0 : 2 * LN);
  }
  check_launch(c);
  return o;
}

// ---- rescale (a11, C15) ----------------------------------------------------
// rows R of polynomials at level l (src: rows of x, or ct (.) K products) -> out [R][l][N]
static void rescale_rows(he_context* c, const RescaleSrc& src, size_t R, int l, u64* out,
                         const he_plaintext* bias = nullptr, int size = 2) {
  const int Lc = l + 1;
  Scratch y(c, R * c->N * 8);
  JobRescaleLast j1{src, y.as<u64>(), c->N, Lc};
  launch_ntt<true>(c, j1, (int)R);
  JobRescaleData j2{src, y.as<u64>(), out, c->d_rs_h + (size_t)l * c->L, c->d_rs_qinv + (size_t)l * c->L, c->N, Lc};
  if (bias) {   // + bias on poly 0 (the same words as a following add_plain: modular addition is exact)
    j2.bias = bias->d;
    j2.bias_bs = bias->B == 1 ? 0 : (size_t)(Lc - 1) * c->N;
    j2.size = size;
  }
  launch_ntt<false>(c, j2, (int)(R * (Lc - 1)));
}

he_ciphertext* ct_rescale(he_context* c, const he_ciphertext* a, const he_plaintext* bias) {
  const int l = a->level;
  he_ciphertext* o = ct_new(c, a->B, a->size, l - 1, a->scale / (double)c->hp.q[l]);
  RescaleSrc src{a->d, nullptr, 0, c->N, l + 1};
  rescale_rows(c, src, (size_t)a->B * a->size, l, o->d, bias, a->size);
  return o;
}

// ---- key switching (a9/a10, C12/C15/C16) -------------------------------------
// ModUp of the digit source (NTT words, item stride bs): returns ext [B][Lc][Lc+K][N].
static u64* modup(he_context* c, const u64* dsrc, size_t bs, int B, int Lc, u32 gal = 1) {
  const size_t N = c->N;
  Scratch coef(c, (size_t)B * Lc * N * 8);
  ntt_rows(c, dsrc, coef.as<u64>(), B, Lc, bs, (size_t)Lc * N, true);
  u64* ext = dalloc_t<u64>(c, (size_t)B * Lc * (Lc + c->K) * N);
  JobModUp j{coef.as<u64>(), ext, c->d_q, c->N, Lc, c->K, c->L, gal, c->logN};
  launch_ntt<false>(c, j, B * Lc * (Lc + c->K - 1));
  return ext;
}

// Key inner products of a (non-hoisted) key switch as one coalesced pass (64-bit contexts): for every
// item b, target limb t < Lc + K and position n,
//   accx[b][p][t][n] = sum_j X_j[t][n] ksk[j][p][t][n],  p = 0, 1,
// with X_j[t] the extended digit already permuted by pi_g (modup with gal) and, for t == j, the digit's
// own NTT word at pi_g(n).  Both parts share every digit load; the ModDown then runs in accx mode.
// Products (< q^2 < 2^120) are summed in 128 bits and reduced once per 8 terms (as ks_inner).
__global__ void k_ks_ip64(const u64* __restrict__ ext, const u64* __restrict__ dsrc, size_t dsrc_bs,
                          const u64* __restrict__ key, u64* __restrict__ accx, const PrimeD* __restrict__ primes,
                          int N, int logN, int Lc, int K, int L, int NP, u32 gal, int ext_permuted) {
  const int nt = Lc + K, t = blockIdx.y, b = blockIdx.z;
  const int tp = t < Lc ? t : L + (t - Lc);
  const PrimeD P = load_prime(primes, tp);
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
    const u32 sn = gal == 1 ? (u32)n : galois_src((u32)n, gal, logN);
    u64 acc0 = 0, acc1 = 0;
    for (int j0 = 0; j0 < Lc; j0 += 8) {
      u64 lo0 = 0, hi0 = 0, lo1 = 0, hi1 = 0;
      const int j1 = min(Lc, j0 + 8);
      for (int j = j0; j < j1; ++j) {
        const u64 x = (t == j) ? __ldg(dsrc + (size_t)b * dsrc_bs + (size_t)j * N + sn)
                               : __ldg(ext + (((size_t)b * Lc + j) * nt + t) * N + (ext_permuted ? (u32)n : sn));
        const u64 k0 = __ldg(key + (((size_t)j * 2 + 0) * NP + tp) * N + n);
        const u64 k1 = __ldg(key + (((size_t)j * 2 + 1) * NP + tp) * N + n);
        u64 pl = x * k0, ph = __umul64hi(x, k0);
        lo0 += pl;
        hi0 += ph + (lo0 < pl);
        pl = x * k1;
        ph = __umul64hi(x, k1);
        lo1 += pl;
        hi1 += ph + (lo1 < pl);
      }
      acc0 = add_mod(acc0, add_mod(mul_mod(hi0, P.r64, P), reduce64(lo0, P), P.q), P.q);
      acc1 = add_mod(acc1, add_mod(mul_mod(hi1, P.r64, P), reduce64(lo1, P), P.q), P.q);
    }
    accx[(((size_t)b * 2 + 0) * nt + t) * N + n] = acc0;
    accx[(((size_t)b * 2 + 1) * nt + t) * N + n] = acc1;
  }
}

static void ks_launch(he_context* c, KsArgs& a);
// ModUp (permuted by gal) + k_ks_ip64 + the accx-mode ModDown with the caller's epilogue (64-bit path).
static void ks_materialized(he_context* c, const u64* dsrc, size_t bs, int B, int Lc, const u64* key, u32 g,
                            KsArgs& epi) {
  const size_t N = c->N;
  const int nt = Lc + c->K;
  // the 2-CTA transforms (N >= 2^14) can permute inside a half only: pi_g keeps the top index bit iff
  // g = 1 mod 4 (every rotation element 5^k); otherwise the inner product gathers
  const bool permute = g == 1 || g % 4 == 1 || c->logN < 14;
  u64* ext = modup(c, dsrc, bs, B, Lc, permute ? g : 1);
  try {
    Scratch accx(c, (size_t)B * 2 * nt * N * 8);
    {
      const double bytes = 8.0 * N * ((double)B * Lc * nt + 2.0 * Lc * nt + 2.0 * B * nt);
      ProfScope ps_(c, "ks_ip", bytes, B * nt, (double)B * nt * Lc * 2 * N);
      k_ks_ip64<<<dim3((unsigned)((N + 255) / 256), (unsigned)nt, (unsigned)B), 256, 0, c->stream>>>(
          ext, dsrc, bs, key, accx.as<u64>(), c->d_primes, (int)N, c->logN, Lc, c->K, c->L, c->NP, g,
          permute ? 1 : 0);
    }
    check_launch(c);
    epi.ext = nullptr;
    epi.accx = accx.as<u64>();
    epi.accx32 = 0;
    epi.gal[0] = g;
    ks_launch(c, epi);
  } catch (...) {
    dfree(c, ext);
    throw;
  }
  dfree(c, ext);
}

// Small-prime ModUp: u32 digits and u32 extended digits ([B][Lc][Lc+K][N] u32).
#ifndef HE_MODUP_FUSED
#define HE_MODUP_FUSED 1   // 0: digit INTT (JobLimbsTo32) and ModUp32 as two launches
#endif
template <int LOGN>
static void launch_modup32_fused(he_context* c, const u64* dsrc, size_t bs, u32* ext, int B, int Lc) {
  typedef NttGeomS<LOGN> G;
  static int grid = 0;   // once per process (one device per process, as launch_ntt32_pipe)
  auto kern = k_modup32_fused<LOGN>;
  if (!grid) {
    HE_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, NttGeom32Pipe<LOGN>::SMEM));
    HE_CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    int per_sm = 0, sms = 0;
    HE_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G::T, NttGeom32Pipe<LOGN>::SMEM));
    HE_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
    grid = std::max(1, per_sm) * sms;
  }
  const int nitems = B * Lc, nt = Lc + c->K;
  // algorithmic bytes: the u64 digit rows read once, the u32 extended digits written once; one
  // butterfly network per transform (1 inverse + nt - 1 forward per digit)
  ProfScope ps(c, "ks_modup", c->prof_on ? (double)G::N * nitems * (8.0 + 4.0 * (nt - 1)) : 0.0, nitems * nt,
               c->prof_on ? 0.5 * G::N * LOGN * (double)nitems * nt : 0.0);
  int gr = std::min(nitems, grid);
  if (c->pipe_grid_cap > 0) gr = std::min(gr, c->pipe_grid_cap);
  kern<<<gr, G::T, NttGeom32Pipe<LOGN>::SMEM, c->stream>>>(dsrc, bs, ext, c->d_q, Lc, c->K, c->L, nitems,
                                                           c->d_primes, c->d_tw32, c->d_itw32);
  check_launch(c);
}

static u32* modup32(he_context* c, const u64* dsrc, size_t bs, int B, int Lc) {
  const size_t N = c->N;
  if (HE_MODUP_FUSED && c->logN >= 11 && c->logN <= 13) {
    u32* ext = dalloc_t<u32>(c, (size_t)B * Lc * (Lc + c->K) * N);
    try {
      switch (c->logN) {
        case 11: launch_modup32_fused<11>(c, dsrc, bs, ext, B, Lc); break;
        case 12: launch_modup32_fused<12>(c, dsrc, bs, ext, B, Lc); break;
        default: launch_modup32_fused<13>(c, dsrc, bs, ext, B, Lc); break;
      }
    } catch (...) {
      dfree(c, ext);
      throw;
    }
    return ext;
  }
  Scratch coef(c, (size_t)B * Lc * N * 4);
  {
    JobLimbsTo32 j{dsrc, coef.as<u32>(), c->N, Lc, bs, (size_t)Lc * N};
    launch_ntt<true>(c, j, B * Lc);
  }
  u32* ext = dalloc_t<u32>(c, (size_t)B * Lc * (Lc + c->K) * N);
  JobModUp32 j{coef.as<u32>(), ext, c->d_q, c->N, Lc, c->K, c->L};
  launch_ntt<false>(c, j, B * Lc * (Lc + c->K - 1));
  return ext;
}

static KsArgs ks_base(he_context* c, int B, int Lc, const u64* ext, const u64* dsrc, size_t dsrc_bs) {
  KsArgs a;
  memset(&a, 0, sizeof(a));
  a.N = c->N;
  a.logN = c->logN;
  a.Lc = Lc;
  a.L = c->L;
  a.K = c->K;
  a.NP = c->NP;
  a.B = B;
  a.KB = 1;
  a.ext = ext;
  a.dsrc = dsrc;
  a.dsrc_bs = dsrc_bs;
  a.Ph_mod = c->d_Ph_mod;
  a.Pinv_mod = c->d_Pinv_mod;
  a.Phat_inv = c->d_Phat_inv;
  a.Phat_mod = c->d_Phat_mod;
  a.P_mod = c->d_P_mod;
  return a;
}

static void ks_launch(he_context* c, KsArgs& a) {
  // the accx-mode ModDown (pipelined, JobKsData::P32) has no plaintext-factor epilogue
  if (a.accx && a.D) throw HeError(HE_INVALID_ARGUMENT, "internal: plaintext factor with an accx ModDown");
  Scratch tb(c, (size_t)a.KB * a.B * 2 * a.K * a.N * 8);
  a.tb = tb.as<u64>();
  JobKsSpecial js{a};
  launch_ntt<true>(c, js, a.KB * a.B * 2 * a.K);
  JobKsData jd{a};
  launch_ntt<false>(c, jd, a.KB * a.B * 2 * a.Lc);
}

// ModDown fused with the rescale that follows it (JobKsDrop / JobKsDataRs, he_jobs.cuh): out holds
// [B][2][Lc-1][N] words at item stride out_bs, + bias on poly 0.  The same words as ks_launch then
// ct_rescale (exact: both transforms are linear), Lc + 1 transforms per part instead of 2 Lc + 1.
static bool ks_rescale_ok(const KsArgs& a) {
  return a.accx && a.accx32 && a.K == 1 && !a.D && a.KB == 1 && a.Lc >= 2;
}
static void ks_launch_rescale(he_context* c, KsArgs& a, u64* out, size_t out_bs, const he_plaintext* bias) {
  Scratch tb(c, (size_t)a.B * 2 * a.K * a.N * 8), y(c, (size_t)a.B * 2 * a.N * 4);
  a.tb = tb.as<u64>();
  JobKsSpecial js{a};
  launch_ntt<true>(c, js, a.B * 2 * a.K);
  JobKsDrop jd{a, y.as<u32>(), a.N};
  launch_ntt<true>(c, jd, a.B * 2);
  const int l = a.Lc - 1;
  JobKsDataRs jr{a, y.as<u32>(), out, out_bs, c->d_rs_h + (size_t)l * c->L, c->d_rs_qinv + (size_t)l * c->L,
                 bias ? bias->d : nullptr, bias && bias->B != 1 ? (size_t)(a.Lc - 1) * a.N : 0, a.N};
  launch_ntt<false>(c, jr, a.B * 2 * (a.Lc - 1));
}

// Fused small-prime key switch: INTT of the digit source, k_modup_ip32 (ModUp
// and inner product without the extended digits in HBM), then the accx-mode
// ModDown with the caller's epilogue (epi.out, addsrc, acc_in ...).
static bool fused_ks_ok(he_context* c) { return c->small_primes && c->d_tw32 && c->logN <= 14; }

static void ks_fused(he_context* c, const u64* dsrc, size_t bs, int B, int Lc, const u32* key32, u32 g,
                     KsArgs& epi, int sq = 0, u64* rs_out = nullptr, size_t rs_bs = 0,
                     const he_plaintext* rs_bias = nullptr) {
  const size_t N = c->N;
  const int nt = Lc + c->K;
  Scratch coef(c, (size_t)B * Lc * N * 4), accx(c, (size_t)B * 2 * nt * N * 4);
  {
    JobLimbsTo32 j{dsrc, coef.as<u32>(), c->N, Lc, bs, (size_t)Lc * N, sq};
    launch_ntt<true>(c, j, B * Lc);
  }
  FusedArgs fa{c->N, c->logN, Lc, c->K, c->L, c->NP, g, coef.as<u32>(), dsrc, bs, key32, c->d_q, accx.as<u64>(),
               sq};
  auto launch = [&](auto kern, int T) {
    const int smem = (int)((N + N / 32 + 2 * N) * 4);
    smem_limit_once((const void*)kern, smem);
    // algorithmic bytes: digits read once per item, key rows once per launch, accumulators written once
    const double bytes = 4.0 * N * B * Lc + 4.0 * N * B * 2 * nt + 4.0 * N * 2 * Lc * nt;
    const double ops = (double)B * (Lc * (nt - 1)) * ntt_ops((int)N, c->logN) + (double)B * nt * Lc * 2 * N;
    ProfScope ps_(c, "ks_modup_ip", bytes, B * nt, ops);
    kern<<<dim3(nt, B), T, smem, c->stream>>>(fa, c->d_primes, c->d_tw32);
  };
  switch (c->logN) {
    case 10: launch(k_modup_ip32<10>, NttGeomS<10>::T); break;
    case 11: launch(k_modup_ip32<11>, NttGeomS<11>::T); break;
    case 12: launch(k_modup_ip32<12>, NttGeomS<12>::T); break;
    case 13: launch(k_modup_ip32<13>, NttGeomS<13>::T); break;
    default: launch(k_modup_ip32<14>, NttGeomS<14>::T); break;
  }
  check_launch(c);
  epi.accx = accx.as<u64>();
  epi.accx32 = 1;
  epi.gal[0] = g;
  if (rs_out) ks_launch_rescale(c, epi, rs_out, rs_bs, rs_bias);
  else ks_launch(c, epi);
}

// Is there a Galois key for this rotation step (in either stored form)?
bool has_galois_key(he_context* c, int step, u32* gal_out) {
  const u64 g = galois_element(c->N, step);
  *gal_out = (u32)g;
  return c->gk.count(g) || c->gk32.count(g);
}

// u64 words of a u32-at-rest key: allocated and converted once, on the first caller that needs them
// (key export, the unfused fallback paths); the hot path of small-prime contexts never does.
// The conversion and the per-step table update run on a stream of their own and are waited for on
// the host, so they are never recorded into a CUDA graph when c->stream is capturing (the keys were
// synchronised at keygen; the consumers on c->stream are enqueued after this returns).
static cudaStream_t key_aux_stream() {
  static cudaStream_t s = nullptr;   // one device per process (context_init)
  if (!s) HE_CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  return s;
}
static u64* key64_from32(he_context* c, const u32* k32) {
  const size_t N = c->N, L = c->L, NP = c->NP, rows = L * 2 * NP;
  u64* key = nullptr;
  HE_CK(cudaMalloc(&key, rows * N * 8));
  cudaStream_t aux = key_aux_stream();
  k_from_mont32<<<dim3((unsigned)((N + 255) / 256), (unsigned)std::min<size_t>(rows, 65535)), 256, 0, aux>>>(
      k32, key, c->d_primes, (int)N, (int)NP, (int)NP, (int)L, rows);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFree(key);
    throw HeError(HE_CUDA_ERROR, std::string("k_from_mont32: ") + cudaGetErrorString(e));
  }
  HE_CK(cudaStreamSynchronize(aux));
  return key;
}

// The u64 form of a Galois key (null if there is no key for the step).
const u64* galois_key(he_context* c, int step, u32* gal_out) {
  const u64 g = galois_element(c->N, step);
  *gal_out = (u32)g;
  auto it = c->gk.find(g);
  if (it != c->gk.end()) return it->second;
  auto it32 = c->gk32.find(g);
  if (it32 == c->gk32.end()) return nullptr;
  u64* key = key64_from32(c, it32->second);
  c->gk[g] = key;
  if (c->d_step_key) {   // every step of the per-step table that maps to this Galois element
    const int ns = c->N / 2;
    cudaStream_t aux = key_aux_stream();
    for (int k = 0; k <= ns; ++k)
      if (galois_element(c->N, k == 0 ? ns : k) == g)
        HE_CK(cudaMemcpyAsync(c->d_step_key + k, &key, sizeof(u64*), cudaMemcpyHostToDevice, aux));
    HE_CK(cudaStreamSynchronize(aux));   // &key is a stack address
  }
  return key;
}

size_t key_bytes(he_context* c) {
  const size_t N = c->N, L = c->L, NP = c->NP, kw = L * 2 * NP * N;
  size_t b = c->d_pk ? 2 * L * N * 8 : 0;
  if (c->d_rlk) b += kw * 8;
  if (c->d_rlk32) b += kw * 4;
  return b + c->gk.size() * kw * 8 + c->gk32.size() * kw * 4;
}

// The u64 form of the relinearisation key (null if there is none).
const u64* relin_key(he_context* c) {
  if (!c->d_rlk && c->d_rlk32) c->d_rlk = key64_from32(c, c->d_rlk32);
  return c->d_rlk;
}

// Square + relinearize without the tensor: with the fused key switch, d2 = x1^2 is formed where
// the digits are loaded (INTT and own-digit load) and d0 = x0^2, d1 = 2 x0 x1 in the ModDown
// epilogue; the words equal ct_relinearize(ct_tensor(x, x)).  Other contexts take that path.
he_ciphertext* ct_square_relin(he_context* c, const he_ciphertext* x) {
  if (!(fused_ks_ok(c) && c->d_rlk32)) {
    he_ciphertext* t = ct_tensor(c, x, x);
    he_ciphertext* r = nullptr;
    try {
      r = ct_relinearize(c, t);
    } catch (...) {
      ct_free(t);
      throw;
    }
    ct_free(t);
    return r;
  }
  const int Lc = x->level + 1;
  const size_t LN = (size_t)Lc * c->N;
  he_ciphertext* o = ct_new(c, x->B, 2, x->level, x->scale * x->scale);
  KsArgs k = ks_base(c, x->B, Lc, nullptr, nullptr, 0);
  k.out = o->d;
  k.out_bs = 2 * LN;
  k.sq_src = x->d;
  k.sq_bs = 2 * LN;
  try {
    ks_fused(c, x->d + LN, 2 * LN, x->B, Lc, c->d_rlk32, 1, k, 1);
  } catch (...) {
    ct_free(o);
    throw;
  }
  return o;
}

// he_square on the fused path: square, relinearize and rescale with the rescale merged into the
// ModDown (ks_launch_rescale); other contexts: ct_square_relin then ct_rescale.
he_ciphertext* ct_square_rescale(he_context* c, const he_ciphertext* x) {
  if (!(fused_ks_ok(c) && c->d_rlk32 && c->K == 1 && x->level >= 1)) {
    he_ciphertext* r = ct_square_relin(c, x);
    he_ciphertext* o = nullptr;
    try {
      o = ct_rescale(c, r);
    } catch (...) {
      ct_free(r);
      throw;
    }
    ct_free(r);
    return o;
  }
  const int Lc = x->level + 1;
  const size_t LN = (size_t)Lc * c->N;
  he_ciphertext* o = ct_new(c, x->B, 2, x->level - 1, x->scale * x->scale / (double)c->hp.q[x->level]);
  KsArgs k = ks_base(c, x->B, Lc, nullptr, nullptr, 0);
  k.out_bs = 2 * LN;   // (level-l strides of the epilogue terms)
  k.sq_src = x->d;
  k.sq_bs = 2 * LN;
  try {
    ks_fused(c, x->d + LN, 2 * LN, x->B, Lc, c->d_rlk32, 1, k, 1, o->d, 2 * (LN - c->N));
  } catch (...) {
    ct_free(o);
    throw;
  }
  return o;
}

he_ciphertext* ct_relinearize(he_context* c, const he_ciphertext* a) {
  const int Lc = a->level + 1;
  const size_t LN = (size_t)Lc * c->N;
  he_ciphertext* o = ct_new(c, a->B, 2, a->level, a->scale);
  if (fused_ks_ok(c) && c->d_rlk32) {
    KsArgs k = ks_base(c, a->B, Lc, nullptr, nullptr, 0);
    k.out = o->d;
    k.out_bs = 2 * LN;
    k.addsrc = a->d;
    k.add_bs = 3 * LN;
    k.add_parts = 2;
    try {
      ks_fused(c, a->d + 2 * LN, 3 * LN, a->B, Lc, c->d_rlk32, 1, k);
    } catch (...) {
      ct_free(o);
      throw;
    }
    return o;
  }
  KsArgs k = ks_base(c, a->B, Lc, nullptr, a->d + 2 * LN, 3 * LN);
  k.out = o->d;
  k.out_bs = 2 * LN;
  k.addsrc = a->d;
  k.add_bs = 3 * LN;
  k.add_parts = 2;
  try {
    ks_materialized(c, a->d + 2 * LN, 3 * LN, a->B, Lc, relin_key(c), 1, k);
  } catch (...) {
    ct_free(o);
    throw;
  }
  return o;
}

// rotate (add_input = false) or x + rotate(x) (add_input = true)
he_ciphertext* ct_rotate(he_context* c, const he_ciphertext* a, int step, bool add_input) {
  const int Lc = a->level + 1;
  const size_t LN = (size_t)Lc * c->N;
  u32 g = 0;
  if (!has_galois_key(c, step, &g))
    throw HeError(HE_MISSING_GALOIS_KEY, "no Galois key for rotation step " + std::to_string(step));
  auto it32 = c->gk32.find(g);
  const u64* key = fused_ks_ok(c) && it32 != c->gk32.end() ? nullptr : galois_key(c, step, &g);
  he_ciphertext* o = ct_new(c, a->B, 2, a->level, a->scale);
  if (fused_ks_ok(c) && it32 != c->gk32.end()) {
    KsArgs k = ks_base(c, a->B, Lc, nullptr, nullptr, 0);
    k.out = o->d;
    k.out_bs = 2 * LN;
    k.addsrc = a->d;
    k.add_bs = 2 * LN;
    k.add_parts = 1;
    k.add_gather = 1;
    if (add_input) k.acc_in = a->d;
    try {
      ks_fused(c, a->d + LN, 2 * LN, a->B, Lc, it32->second, g, k);
    } catch (...) {
      ct_free(o);
      throw;
    }
    return o;
  }
  KsArgs k = ks_base(c, a->B, Lc, nullptr, a->d + LN, 2 * LN);
  k.out = o->d;
  k.out_bs = 2 * LN;
  k.addsrc = a->d;
  k.add_bs = 2 * LN;
  k.add_parts = 1;
  k.add_gather = 1;
  if (add_input) k.acc_in = a->d;
  try {
    ks_materialized(c, a->d + LN, 2 * LN, a->B, Lc, key, g, k);
  } catch (...) {
    ct_free(o);
    throw;
  }
  return o;
}

// acc + rot(a, step) with the addition in the rotation's ModDown epilogue (fused small-prime key
// switch: acc_in); other contexts: rotate, then add.
static he_ciphertext* ct_rotate_acc(he_context* c, const he_ciphertext* a, int step, const he_ciphertext* acc) {
  const int Lc = a->level + 1;
  const size_t LN = (size_t)Lc * c->N;
  u32 g = 0;
  if (!has_galois_key(c, step, &g))
    throw HeError(HE_MISSING_GALOIS_KEY, "no Galois key for rotation step " + std::to_string(step));
  auto it32 = c->gk32.find(g);
  if (!(fused_ks_ok(c) && it32 != c->gk32.end() && acc->level == a->level && acc->B == a->B && acc->size == 2)) {
    he_ciphertext* r = ct_rotate(c, a, step, false);
    he_ciphertext* s2 = nullptr;
    try {
      s2 = ct_binop(c, 0, acc, r);
    } catch (...) {
      ct_free(r);
      throw;
    }
    ct_free(r);
    return s2;
  }
  he_ciphertext* o = ct_new(c, a->B, 2, a->level, a->scale);
  KsArgs k = ks_base(c, a->B, Lc, nullptr, nullptr, 0);
  k.out = o->d;
  k.out_bs = 2 * LN;
  k.addsrc = a->d;
  k.add_bs = 2 * LN;
  k.add_parts = 1;
  k.add_gather = 1;
  k.acc_in = acc->d;
  try {
    ks_fused(c, a->d + LN, 2 * LN, a->B, Lc, it32->second, g, k);
  } catch (...) {
    ct_free(o);
    throw;
  }
  return o;
}

// vec_mat with pre-encoded diagonals (a14, C17): acc = sum_k rot(x, k) (.) D_k
// with all rotations hoisted (one ModUp of c1 shared by every k), then one
// rescale and the bias.
static he_ciphertext* ct_vec_mat_lazy(he_context* c, const he_ciphertext* x, const he_plaintext* diags,
                                      const std::vector<u32>& gals, int step = 1) {
  const int Lc = x->level + 1, n = diags->B, B = x->B, nt = Lc + c->K;
  const size_t LN = (size_t)Lc * c->N, N = c->N;
  // steps 1..n-1: the per-step device tables built at keygen (no host copies here)
  std::vector<const u32*> keys32;
  if (c->small_primes) {
    keys32.push_back(nullptr);
    for (int k = 1; k < n; ++k) {
      auto it = c->gk32.find(gals[k]);
      if (it == c->gk32.end()) break;
      keys32.push_back(it->second);
    }
  }
  const u64* const* kt = c->d_step_key;
  const u32* const* k32t = c->d_step_key32;
  const u32* gt = c->d_step_gal;
  const bool smem_path = c->small_primes && ((size_t)Lc + 1) * N * 4 <= kMaxSmem && Lc <= 8 &&
                         keys32.size() == (size_t)n && N % (LAZY_SM_T * 4) == 0 && step == 1;
  if (!smem_path)   // the generic kernel reads the u64 keys through d_step_key: materialise u32-at-rest keys
    for (int k = 1; k < n; ++k) {
      u32 gg;
      galois_key(c, k * step, &gg);
    }
  u64* ext = (n > 1 && !smem_path) ? modup(c, x->d + LN, 2 * LN, B, Lc) : nullptr;
  u32* ext32 = (n > 1 && smem_path) ? modup32(c, x->d + LN, 2 * LN, B, Lc) : nullptr;
  he_ciphertext* acc = nullptr;
  try {
    Scratch accx(c, (size_t)B * 2 * nt * N * 8);
    LazyArgs la{c->N, c->logN, Lc, c->K, c->L, c->NP, n, ext, x->d, diags->d, kt, gt,
                c->d_P_mod, accx.as<u64>(), step, ext32};
    {
      // algorithmic bytes: ext + ct + accumulators once per item, keys and diagonals once per launch
      const double bytes = 8.0 * N * ((double)B * Lc * nt + (double)B * 2 * Lc + (double)B * 2 * nt +
                                      (double)(n - 1) * 2 * Lc * nt + (double)n * nt);
      // one multiply-accumulate per key row, per diagonal product and per phi_k(c0) product
      const double ops = (double)B * (n - 1) * N * (nt * (2.0 * Lc + 2.0) + Lc);
      static const char* const tags[9] = {"vecmat_lazy", "vecmat_lazy_L1", "vecmat_lazy_L2", "vecmat_lazy_L3",
                                          "vecmat_lazy_L4", "vecmat_lazy_L5", "vecmat_lazy_L6", "vecmat_lazy_L7",
                                          "vecmat_lazy_L8"};
      ProfScope ps_(c, tags[Lc <= 8 ? Lc : 0], bytes, B * nt, ops);
      const size_t smem = ((size_t)Lc + 1) * N * 4;
      if (smem_path) {
        if (!diags->dm) {   // Montgomery u32 copy of the diagonals, cached on the plaintext
          const size_t rows = (size_t)n * nt;
          u32* dmp = dalloc_t<u32>(c, rows * N);
          k_to_mont32<<<dim3((unsigned)((N + 255) / 256), (unsigned)std::min<size_t>(rows, 65535)), 256, 0,
                        c->stream>>>(diags->d, dmp, c->d_primes, (int)N, nt, Lc, c->L, rows);
          check_launch(c);
          const_cast<he_plaintext*>(diags)->dm = dmp;
        }
        auto launch = [&](auto kern) {
          smem_limit_once((const void*)kern, (int)kMaxSmem);
          kern<<<dim3(nt, B), LAZY_SM_T, smem, c->stream>>>(la, k32t, diags->dm, c->d_primes);
        };
        switch (Lc) {
          case 1: launch(k_vecmat_lazy_mont<1>); break;
          case 2: launch(k_vecmat_lazy_mont<2>); break;
          case 3: launch(k_vecmat_lazy_mont<3>); break;
          case 4: launch(k_vecmat_lazy_mont<4>); break;
          case 5: launch(k_vecmat_lazy_mont<5>); break;
          case 6: launch(k_vecmat_lazy_mont<6>); break;
          case 7: launch(k_vecmat_lazy_mont<7>); break;
          default: launch(k_vecmat_lazy_mont<8>); break;
        }
      } else {
        const dim3 grid((unsigned)(N / (256 * LAZY_EPT)), nt, B);
        if (c->small_primes) k_vecmat_lazy<true><<<grid, 256, 0, c->stream>>>(la, c->d_primes);
        else k_vecmat_lazy<false><<<grid, 256, 0, c->stream>>>(la, c->d_primes);
      }
    }
    check_launch(c);
    acc = ct_new(c, B, 2, x->level, x->scale * diags->scale);
    KsArgs a = ks_base(c, B, Lc, nullptr, nullptr, 0);
    a.gal[0] = 1;
    a.accx = accx.as<u64>();
    a.out = acc->d;
    a.out_bs = 2 * LN;
    ks_launch(c, a);
  } catch (...) {
    dfree(c, ext);
    dfree(c, ext32);
    ct_free(acc);
    throw;
  }
  dfree(c, ext);
  dfree(c, ext32);
  return acc;
}

he_ciphertext* ct_vec_mat(he_context* c, const he_ciphertext* x, const he_plaintext* diags,
                          const he_plaintext* bias) {
  if (diags->bsgs_g > 0) return ct_vec_mat_bsgs(c, x, diags, diags->bsgs_g, bias);
  const int Lc = x->level + 1, n = diags->B, B = x->B;
  const size_t LN = (size_t)Lc * c->N;
  std::vector<const u64*> keys(n);
  std::vector<u32> gals(n);
  for (int k = 1; k < n; ++k)
    if (!has_galois_key(c, k, &gals[k]))
      throw HeError(HE_MISSING_GALOIS_KEY, "no Galois key for rotation step " + std::to_string(k));
  if (!diags->qp)   // the per-rotation form switches with the u64 keys
    for (int k = 1; k < n; ++k) keys[k] = galois_key(c, k, &gals[k]);
  if (diags->qp) {
    he_ciphertext* acc = ct_vec_mat_lazy(c, x, diags, gals);
    he_ciphertext* res = nullptr;
    try {
      res = ct_rescale(c, acc, bias);   // bias fused into the rescale's store
    } catch (...) {
      ct_free(acc);
      throw;
    }
    ct_free(acc);
    return res;
  }
  // k = 0 term
  he_plaintext d0{c, 1, diags->level, diags->scale, diags->d};
  he_ciphertext* acc = ct_mul_plain(c, x, &d0);
  he_ciphertext* res = nullptr;
  u64* ext = nullptr;
  try {
    if (n > 1) {
      ext = modup(c, x->d + LN, 2 * LN, B, Lc);
      const int per_rot = B * 2 * Lc;
      int KB = (4 * 148 + per_rot - 1) / per_rot;
      KB = std::max(1, std::min(KB, KS_KB_MAX));
      Scratch tmp(c, KB > 1 ? (size_t)KB * B * 2 * LN * 8 : 8);
      for (int k0 = 1; k0 < n; k0 += KB) {
        const int kb = std::min(KB, n - k0);
        KsArgs a = ks_base(c, B, Lc, ext, x->d + LN, 2 * LN);
        a.KB = kb;
        for (int kk = 0; kk < kb; ++kk) {
          a.keys[kk] = keys[k0 + kk];
          a.gal[kk] = gals[k0 + kk];
        }
        a.addsrc = x->d;
        a.add_bs = 2 * LN;
        a.add_parts = 1;
        a.add_gather = 1;
        a.D = diags->d + (size_t)k0 * LN;
        a.D_ks = LN;
        a.out_bs = 2 * LN;
        if (KB == 1) {
          a.out = acc->d;
          a.acc_in = acc->d;
          a.out_ks = 0;
          ks_launch(c, a);
        } else {
          a.out = tmp.as<u64>();
          a.out_ks = (size_t)B * 2 * LN;
          ks_launch(c, a);
          const size_t rows = (size_t)B * 2 * Lc;
          {
            ProfScope ps_(c, "vecmat_accumulate", 0.0, 0);
            k_accumulate<<<rows_grid2(c, rows), 256, 0, c->stream>>>(acc->d, tmp.as<u64>(), kb, (size_t)B * 2 * LN,
                                                                     c->d_primes, c->N, Lc, rows);
          }
          check_launch(c);
        }
      }
    }
    res = ct_rescale(c, acc);
  } catch (...) {
    dfree(c, ext);
    ct_free(acc);
    throw;
  }
  dfree(c, ext);
  ct_free(acc);
  if (bias) {
    he_ciphertext* r2 = ct_add_plain(c, res, bias);
    ct_free(res);
    res = r2;
  }
  return res;
}

__global__ void k_fill_u64(u64* __restrict__ p, size_t n, u64 v) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}

// BSGS vec_mat: diags = G groups of g QP diagonals E[k2][k1].
// Baby-step part: inner[k2] = ModDown(sum_{k1 < g} E[k2][k1] (.) rot(x, k1 step)) for the G
// groups of diags (unrescaled, scale x.scale * diags.scale).
// rescale (G == 1 only): inner[0] is returned rescaled (+ bias on poly 0), the rescale merged into
// the ModDown on the fused path (ks_launch_rescale).
static std::vector<he_ciphertext*> bsgs_inner(he_context* c, const he_ciphertext* x, const he_plaintext* diags,
                                              int g, int step, bool rescale = false,
                                              const he_plaintext* bias = nullptr,
                                              const he_plaintext* add_pt = nullptr) {
  // diags == nullptr: unit diagonals (a rotation sum of g terms, ct_rot_sum): the fused kernel's UNIT form
  // needs no plaintext; the other paths get the plaintext polynomial 1 (NTT words all 1) g times.
  const bool unit = diags == nullptr;
  const int Lc = x->level + 1, B = x->B, nt = Lc + c->K, G = unit ? 1 : diags->B / g;
  const double dscale = unit ? 1.0 : diags->scale;
  he_plaintext* ones = nullptr;
  const size_t N = c->N, LN = (size_t)Lc * N;
  std::vector<u32> gals(g, 1);
  for (int k = 1; k < g; ++k)
    if (!has_galois_key(c, k * step, &gals[k]))
      throw HeError(HE_MISSING_GALOIS_KEY, "no Galois key for baby step " + std::to_string(k * step));
  std::vector<const u32*> keys32;
  if (c->small_primes) {
    keys32.push_back(nullptr);
    for (int k = 1; k < g; ++k) {
      auto it = c->gk32.find(gals[k]);
      if (it == c->gk32.end()) break;
      keys32.push_back(it->second);
    }
  }
  const size_t smem = ((size_t)Lc + 1) * N * 4;
  // the fused kernel indexes the keygen tables d_step_key32 / d_step_gal (n_s + 1 entries) at k step
  const bool fused = c->small_primes && keys32.size() == (size_t)g && smem <= kMaxSmem && Lc <= 8 && G <= 4 &&
                     N % (LAZY_SM_T * 2) == 0 && B <= 65535 && (size_t)(g - 1) * step <= N / 2;
  std::vector<he_ciphertext*> inner(G, nullptr);
  auto cleanup = [&] {
    for (auto* p : inner) ct_free(p);
    pt_free(ones);
  };
  try {
    if (unit && !fused) {
      ones = pt_new(c, g, x->level, 1.0, 1);
      k_fill_u64<<<148 * 4, 256, 0, c->stream>>>(ones->d, pt_words(ones), 1);
      check_launch(c);
      diags = ones;
    }
    if (fused) {
      if (!unit && !diags->dm) {
        const size_t rows = (size_t)diags->B * nt;
        u32* dmp = dalloc_t<u32>(c, rows * N);
        k_to_mont32<<<dim3((unsigned)((N + 255) / 256), (unsigned)std::min<size_t>(rows, 65535)), 256, 0,
                      c->stream>>>(diags->d, dmp, c->d_primes, (int)N, nt, Lc, c->L, rows);
        check_launch(c);
        const_cast<he_plaintext*>(diags)->dm = dmp;
      }
      const u32* const* kt = c->d_step_key32;   // baby steps 1..g-1 (keygen tables)
      const u32* gt = c->d_step_gal;
      u32* ext = modup32(c, x->d + LN, 2 * LN, B, Lc);
      Scratch accx(c, (size_t)G * B * 2 * nt * N * 4);
      try {
        LazyArgs la{c->N, c->logN, Lc, c->K, c->L, c->NP, g, nullptr, x->d, nullptr, nullptr, gt, c->d_P_mod,
                    accx.as<u64>(), step, ext};
        {
          // unique bytes: u32 extended digits (t != j), the u64 own digit (c1) and c0 row, u32 accumulators
          // written, u32 key rows of the g-1 baby steps, u32 diagonals
          // (a rotation sum - unit diagonals - reads no diagonals and forms no diagonal products)
          const double bytes = 4.0 * N * B * Lc * (nt - 1) + 8.0 * N * 2.0 * B * Lc + 4.0 * N * G * B * 2 * nt +
                               4.0 * N * ((double)(g - 1) * 2 * Lc * nt + (unit ? 0.0 : (double)G * g * nt));
          const double ops = (double)B * (g - 1) * N * (nt * (2.0 * Lc + (unit ? 0.0 : 2.0 * G)) + Lc);
          static const char* const tags[9] = {"vecmat_bsgs", "vecmat_bsgs_L1", "vecmat_bsgs_L2", "vecmat_bsgs_L3",
                                              "vecmat_bsgs_L4", "vecmat_bsgs_L5", "vecmat_bsgs_L6", "vecmat_bsgs_L7",
                                              "vecmat_bsgs_L8"};
          ProfScope ps_(c, tags[Lc], bytes, B * nt, ops);
          // half-ring CTAs with image pairs (k_vecmat_bsgs_hp): same smem as one full-ring image
          const int IBv = B >= 2 ? 2 : 1;
          const size_t smem_hp = (size_t)IBv * (Lc + 1) * (N / 2) * 4;
          const dim3 grid((unsigned)((B + IBv - 1) / IBv), 2, nt);
          auto launch = [&](auto kern) {
            smem_limit_once((const void*)kern, (int)kMaxSmem);
            kern<<<grid, LAZY_SM_T, smem_hp, c->stream>>>(la, g, B, kt, unit ? nullptr : diags->dm, c->d_primes);
          };
          // BASELINE config 4's geometry (N = 2^13, L + K = 8) with image pairs: compile-time strides
          const bool fixg = N == 8192 && c->NP == 8 && IBv == 2 && HE_BSGS_FIXED;
#define HE_BSGS_G(LCV, IBV, NF, NPF)                                             \
    if (unit) launch(k_vecmat_bsgs_hp<LCV, 1, IBV, true, NF, NPF>);              \
    else if (G == 1) launch(k_vecmat_bsgs_hp<LCV, 1, IBV, false, NF, NPF>);      \
    else if (G == 2) launch(k_vecmat_bsgs_hp<LCV, 2, IBV, false, NF, NPF>);      \
    else if (G == 3) launch(k_vecmat_bsgs_hp<LCV, 3, IBV, false, NF, NPF>);      \
    else launch(k_vecmat_bsgs_hp<LCV, 4, IBV, false, NF, NPF>);
#define HE_BSGS_CASE(LCV)                                                        \
  case LCV:                                                                      \
    if (fixg) { HE_BSGS_G(LCV, 2, 8192, 8) }                                     \
    else if (IBv == 2) { HE_BSGS_G(LCV, 2, 0, 0) } else { HE_BSGS_G(LCV, 1, 0, 0) } \
    break;
          switch (Lc) {
            HE_BSGS_CASE(1) HE_BSGS_CASE(2) HE_BSGS_CASE(3) HE_BSGS_CASE(4)
            HE_BSGS_CASE(5) HE_BSGS_CASE(6) HE_BSGS_CASE(7) default: HE_BSGS_CASE(8)
          }
#undef HE_BSGS_G
#undef HE_BSGS_CASE
        }
        check_launch(c);
        for (int k2 = 0; k2 < G; ++k2) {
          KsArgs a = ks_base(c, B, Lc, nullptr, nullptr, 0);
          a.gal[0] = 1;
          a.accx = reinterpret_cast<const u64*>(accx.as<u32>() + (size_t)k2 * B * 2 * nt * N);
          a.accx32 = 1;
          a.out_bs = 2 * LN;
          if (add_pt && G == 1 && !rescale) {   // + plaintext on poly 0 in the ModDown epilogue
            a.addsrc = add_pt->d;
            a.add_bs = add_pt->B == 1 ? 0 : LN;
            a.add_parts = 1;
            a.add_gather = 0;
            add_pt = nullptr;   // done
          }
          if (rescale && G == 1 && ks_rescale_ok(a)) {
            inner[k2] = ct_new(c, B, 2, x->level - 1, x->scale * dscale / (double)c->hp.q[x->level]);
            ks_launch_rescale(c, a, inner[k2]->d, 2 * (LN - N), bias);
            rescale = false;   // done
          } else {
            inner[k2] = ct_new(c, B, 2, x->level, x->scale * dscale);
            a.out = inner[k2]->d;
            ks_launch(c, a);
          }
        }
      } catch (...) {
        dfree(c, ext);
        throw;
      }
      dfree(c, ext);
    } else {   // generic: one lazy accumulation per giant step (no sharing of the baby-step products)
      for (int k2 = 0; k2 < G; ++k2) {
        he_plaintext view{c, g, diags->level, diags->scale, diags->d + (size_t)k2 * g * nt * N, 1};
        inner[k2] = ct_vec_mat_lazy(c, x, &view, gals, step);
        dfree(c, view.dm);
      }
    }
    if (add_pt) {   // not merged into the ModDown: a separate add_plain
      if (G != 1 || rescale) throw HeError(HE_INVALID_ARGUMENT, "internal: epilogue add with several groups");
      he_ciphertext* r = ct_add_plain(c, inner[0], add_pt);
      ct_free(inner[0]);
      inner[0] = r;
    }
    if (rescale) {   // not merged into the ModDown (other contexts): a separate rescale
      if (G != 1) throw HeError(HE_INVALID_ARGUMENT, "internal: fused rescale with several giant-step groups");
      he_ciphertext* r = ct_rescale(c, inner[0], bias);
      ct_free(inner[0]);
      inner[0] = r;
    }
  } catch (...) {
    cleanup();
    throw;
  }
  pt_free(ones);
  return inner;
}

static he_ciphertext* ct_rot_sum(he_context* c, const he_ciphertext* x, int n, int step, bool rescale = false,
                                 const he_plaintext* bias = nullptr, const he_plaintext* add_pt = nullptr);

// diags->fold_n > 1 (he_vec_mat_encode_bsgs_fold, oracle vec_mat_bsgs_fold): the giant-step sum
// covers the first m = fold_step diagonals; the replicated-output fold sum_{t<fold_n} rot(., m t)
// (one hoisted unit-diagonal rotation sum) completes the n-term sum before the rescale.
he_ciphertext* ct_vec_mat_bsgs(he_context* c, const he_ciphertext* x, const he_plaintext* diags, int g,
                               const he_plaintext* bias, int fold_n, int fold_step) {
  if (fold_n < 0) {
    fold_n = diags->fold_n;
    fold_step = diags->fold_step;
  }
  const int G = diags->B / g;
  for (int k2 = 1; k2 < G; ++k2) {
    u32 gg;
    if (!has_galois_key(c, g * k2, &gg))
      throw HeError(HE_MISSING_GALOIS_KEY, "no Galois key for giant step " + std::to_string(g * k2));
  }
  if (G == 1 && fold_n <= 1) {   // one group, no fold: the rescale (+ bias) merged into the ModDown
    std::vector<he_ciphertext*> one = bsgs_inner(c, x, diags, g, 1, true, bias);
    return one[0];
  }
  std::vector<he_ciphertext*> inner = bsgs_inner(c, x, diags, g, 1);
  auto cleanup = [&] {
    for (auto* p : inner) ct_free(p);
  };
  try {
    // giant steps: acc = sum_k2 rot(inner_k2, g k2)
    he_ciphertext* acc = inner[0];
    inner[0] = nullptr;
    for (int k2 = 1; k2 < G; ++k2) {   // acc + rot(inner_k2, g k2), the add in the ModDown epilogue
      he_ciphertext* s2 = nullptr;
      try {
        s2 = ct_rotate_acc(c, inner[k2], g * k2, acc);
      } catch (...) {
        ct_free(acc);
        throw;
      }
      ct_free(inner[k2]);
      inner[k2] = nullptr;
      ct_free(acc);
      acc = s2;
    }
    if (fold_n > 1) {   // the fold's ModDown carries the rescale (+ bias)
      he_ciphertext* f = nullptr;
      try {
        f = ct_rot_sum(c, acc, fold_n, fold_step, true, bias);
      } catch (...) {
        ct_free(acc);
        throw;
      }
      ct_free(acc);
      return f;
    }
    he_ciphertext* res = ct_rescale(c, acc, bias);   // bias fused into the rescale's store
    ct_free(acc);
    return res;
  } catch (...) {
    cleanup();
    throw;
  }
}


// sum_{k < n} rot(x, k step) with ONE lazy ModDown: the baby-step machinery with unit
// diagonals (the plaintext polynomial 1, whose NTT words are all 1); scale unchanged.
static he_ciphertext* ct_rot_sum(he_context* c, const he_ciphertext* x, int n, int step, bool rescale,
                                 const he_plaintext* bias, const he_plaintext* add_pt) {
  if (n == 1) {
    if (rescale) return ct_rescale(c, x, bias);
    if (add_pt) return ct_add_plain(c, x, add_pt);
    he_ciphertext* o = ct_new(c, x->B, x->size, x->level, x->scale);
    HE_CK(cudaMemcpyAsync(o->d, x->d, ct_words(x) * 8, cudaMemcpyDeviceToDevice, c->stream));
    return o;
  }
  return bsgs_inner(c, x, nullptr, n, step, rescale, bias, add_pt)[0];
}

// im2col conv on the encrypted side (a15, C18/C19).  fold_n1 = 0: the paper's log2 rotate-and-add
// fold; fold_n1 > 0: the same sum as two hoisted lazy rotation sums (n1 x n2 chunks).
he_ciphertext* ct_conv(he_context* c, const he_ciphertext* x, const he_plaintext* kernels,
                       const he_plaintext* masks, const he_plaintext* bias, int chunk, int fold_n1) {
  const int Lc = x->level + 1, C = kernels->B, B = x->B;
  // t_c = rescale(ct (.) K_c) for all (b, c): the products are formed inside the rescale (C18)
  he_ciphertext* T = nullptr;
  he_ciphertext* t = ct_new(c, B * C, 2, x->level - 1, (x->scale * kernels->scale) / (double)c->hp.q[x->level]);
  try {
    RescaleSrc src{x->d, kernels->d, C, c->N, Lc};
    rescale_rows(c, src, (size_t)B * C * 2, x->level, t->d);
    const int ns = c->N / 2;
    if (fold_n1 > 0) {
      const int n_chunks = ns / chunk, n2 = n_chunks / fold_n1;
      he_ciphertext* t2 = ct_rot_sum(c, t, fold_n1, chunk);
      ct_free(t);
      t = t2;
      t2 = ct_rot_sum(c, t, n2, chunk * fold_n1);
      ct_free(t);
      t = t2;
    } else {
      for (int step = chunk; step < ns; step <<= 1) {
        he_ciphertext* t2 = ct_rotate(c, t, step, true);
        ct_free(t);
        t = t2;
      }
    }
    // sum_c t_c (.) Mask_c formed inside the second rescale (C19)
    he_ciphertext* r = ct_new(c, B, 2, t->level - 1, (t->scale * masks->scale) / (double)c->hp.q[t->level]);
    try {
      RescaleSrc src{t->d, masks->d, C, c->N, t->level + 1, 1};
      rescale_rows(c, src, (size_t)B * 2, t->level, r->d);
    } catch (...) {
      ct_free(r);
      throw;
    }
    ct_free(t);
    t = nullptr;
    if (bias) {
      he_ciphertext* r2 = ct_add_plain(c, r, bias);
      ct_free(r);
      r = r2;
    }
    return r;
  } catch (...) {
    ct_free(T);
    ct_free(t);
    throw;
  }
}

// One-level im2col conv (oracle circuits.im2col_conv_bsgs): v = rescale(ModDown(
// sum_{b<g} D_b (.) rot(x, chunk b))) with the g QP diagonals D_b = sum_c Mask_c (.) rot(K_c, chunk b)
// (the baby-step kernel, one group), then the giant steps sum_{a<n2} rot(v, chunk g a) as a
// unit-diagonal rotation sum, + bias.
he_ciphertext* ct_conv_bsgs(he_context* c, const he_ciphertext* x, const he_plaintext* diags,
                            const he_plaintext* bias, int chunk, int g) {
  std::vector<he_ciphertext*> inner = bsgs_inner(c, x, diags, g, chunk, true);   // rescale merged
  he_ciphertext* v = nullptr;
  he_ciphertext* r = inner[0];
  try {
    const int n2 = c->N / 2 / chunk / g;
    if (n2 > 1) {   // + bias in the rotation sum's ModDown epilogue
      he_ciphertext* r2 = ct_rot_sum(c, r, n2, chunk * g, false, nullptr, bias);
      ct_free(r);
      r = r2;
    } else if (bias) {
      he_ciphertext* r2 = ct_add_plain(c, r, bias);
      ct_free(r);
      r = r2;
    }
  } catch (...) {
    ct_free(v);
    ct_free(r);
    throw;
  }
  return r;
}

// ---- keygen (a2/a3, C9-C12) --------------------------------------------------
static void make_ksk(he_context* c, u64* key, u64 pur_a, u64 pur_e, u64 objbase, u32 gal) {
  const int L = c->L, NP = c->NP, N = c->N;
  // a_j[t] uniform (NTT words) straight into part 1
  {
    ProfScope ps_(c, "sample_uniform", 0.0, 0);
    k_sample_uniform<<<dim3((N + 255) / 256, std::min(L * NP, 65535)), 256, 0, c->stream>>>(
        key + (size_t)NP * N, (size_t)2 * NP * N, L, NP, N, c->seed, pur_a, objbase, c->d_primes);
  }
  check_launch(c);
  // e_j: one CDT polynomial per digit, NTT into every limb
  Scratch e(c, (size_t)L * N * 8), et(c, (size_t)L * NP * N * 8);
  {
    ProfScope ps_(c, "sample_small", 0.0, 0);
    k_sample_small<<<dim3((N + 255) / 256, std::min(L, 65535)), 256, 0, c->stream>>>(e.as<i64>(), N, L, c->seed,
                                                                                   pur_e, objbase, 1, c->d_cdt);
  }
  check_launch(c);
  signed_to_ntt(c, e.as<i64>(), et.as<u64>(), L, NP);
  {
    ProfScope ps_(c, "keygen_combine", 0.0, 0);
    k_ksk_combine<<<dim3((N + 255) / 256, std::min(L * NP, 65535)), 256, 0, c->stream>>>(
        key, et.as<u64>(), c->d_sk, c->d_P_mod, c->d_primes, N, c->logN, L, NP, gal);
  }
  check_launch(c);
}

// per-step device tables (Galois element and key pointers for every step 0..n_s)
void build_step_tables(he_context* c) {
  const int N = c->N;
  {
    const int ns = N / 2;
    std::vector<u32> sg(ns + 1);
    std::vector<const u64*> sk(ns + 1, nullptr);
    std::vector<const u32*> sk32(ns + 1, nullptr);
    for (int k = 0; k <= ns; ++k) {
      const u64 g = galois_element(N, k == 0 ? ns : k);
      sg[k] = (u32)g;
      auto it = c->gk.find(g);
      if (it != c->gk.end()) sk[k] = it->second;
      auto it32 = c->gk32.find(g);
      if (it32 != c->gk32.end()) sk32[k] = it32->second;
    }
    sg[0] = 1;
    HE_CK(cudaMalloc(&c->d_step_gal, sg.size() * 4));
    HE_CK(cudaMalloc(&c->d_step_key, sk.size() * sizeof(u64*)));
    HE_CK(cudaMalloc(&c->d_step_key32, sk32.size() * sizeof(u32*)));
    HE_CK(cudaMemcpy(c->d_step_gal, sg.data(), sg.size() * 4, cudaMemcpyHostToDevice));
    HE_CK(cudaMemcpy(c->d_step_key, sk.data(), sk.size() * sizeof(u64*), cudaMemcpyHostToDevice));
    HE_CK(cudaMemcpy(c->d_step_key32, sk32.data(), sk32.size() * sizeof(u32*), cudaMemcpyHostToDevice));
    c->owned.push_back(c->d_step_gal);
    c->owned.push_back((void*)c->d_step_key);
    c->owned.push_back((void*)c->d_step_key32);
  }
}

void keygen(he_context* c, const std::vector<int>& steps) {
  const int L = c->L, NP = c->NP, N = c->N;
  HE_CK(cudaMalloc(&c->d_sk, (size_t)NP * N * 8));
  {
    Scratch s(c, (size_t)N * 8);
    {
      ProfScope ps_(c, "sample_small", 0.0, 0);
      k_sample_small<<<dim3((N + 255) / 256, 1), 256, 0, c->stream>>>(s.as<i64>(), N, 1, c->seed, PUR_S, 0, 0,
                                                                     c->d_cdt);
    }
    check_launch(c);
    signed_to_ntt(c, s.as<i64>(), c->d_sk, 1, NP);
  }
  c->has_sk = true;
  HE_CK(cudaMalloc(&c->d_pk, (size_t)2 * L * N * 8));
  {
    {
      ProfScope ps_(c, "sample_uniform", 0.0, 0);
      k_sample_uniform<<<dim3((N + 255) / 256, L), 256, 0, c->stream>>>(c->d_pk + (size_t)L * N, 0, 1, L, N,
                                                                        c->seed, PUR_PK_A, 0, c->d_primes);
    }
    check_launch(c);
    Scratch e(c, (size_t)N * 8), et(c, (size_t)L * N * 8);
    {
      ProfScope ps_(c, "sample_small", 0.0, 0);
      k_sample_small<<<dim3((N + 255) / 256, 1), 256, 0, c->stream>>>(e.as<i64>(), N, 1, c->seed, PUR_PK_E, 0, 1,
                                                                     c->d_cdt);
    }
    check_launch(c);
    signed_to_ntt(c, e.as<i64>(), et.as<u64>(), 1, L);
    {
      ProfScope ps_(c, "keygen_combine", 0.0, 0);
      k_pk_combine<<<dim3((N + 255) / 256, L), 256, 0, c->stream>>>(c->d_pk, et.as<u64>(), c->d_sk, c->d_primes,
                                                                    N, L);
    }
    check_launch(c);
  }
  c->has_pk = true;
  if (c->K > 0) {
    const size_t kw = (size_t)L * 2 * NP * N;
    // Keys at rest: contexts on the fused small-prime key switch keep every switching
    // key as Montgomery-form u32 words only (4 bytes per residue instead of 8 + 4); the u64 form is
    // built in one reused scratch block here and, later, only on demand (galois_key / relin_key).
    const bool u32_only = fused_ks_ok(c);
    const size_t rows = (size_t)L * 2 * NP;
    u64* tmp64 = nullptr;
    if (u32_only) HE_CK(cudaMalloc(&tmp64, kw * 8));
    auto to32 = [&](const u64* key) {
      u32* k32 = nullptr;
      HE_CK(cudaMalloc(&k32, kw * 4));
      k_to_mont32<<<dim3((N + 255) / 256, (unsigned)std::min<size_t>(rows, 65535)), 256, 0, c->stream>>>(
          key, k32, c->d_primes, N, NP, NP, L, rows);
      check_launch(c);
      return k32;
    };
    try {
      if (!u32_only) HE_CK(cudaMalloc(&c->d_rlk, kw * 8));
      u64* rl = u32_only ? tmp64 : c->d_rlk;
      make_ksk(c, rl, PUR_RLK_A, PUR_RLK_E, 0, 0);
      c->has_rlk = true;
      if (c->small_primes) c->d_rlk32 = to32(rl);
      for (int st : steps) {
        const u64 g = galois_element(N, st);
        if (c->gk.count(g) || c->gk32.count(g)) continue;
        u64* key = tmp64;
        if (!u32_only) {
          HE_CK(cudaMalloc(&key, kw * 8));
          c->gk[g] = key;
        }
        make_ksk(c, key, PUR_GK_A, PUR_GK_E, g << 8, (u32)g);
        if (c->small_primes) c->gk32[g] = to32(key);
      }
    } catch (...) {
      if (tmp64) cudaFree(tmp64);
      throw;
    }
    if (tmp64) {
      HE_CK(cudaStreamSynchronize(c->stream));
      HE_CK(cudaFree(tmp64));
    }
  }
  build_step_tables(c);
  HE_CK(cudaStreamSynchronize(c->stream));
}

// he_make_public: a new context with the same parameters and seed holding copies of
// the public, relinearisation and Galois keys and no secret key.
he_context* context_make_public(he_context* c) {
  he_context* p = new he_context();
  try {
    context_init(p, c->hp, c->seed);
    p->stream = c->stream;
    p->pipe_grid_cap = c->pipe_grid_cap;
    const size_t N = c->N, L = c->L, NP = c->NP, kw = L * 2 * NP * N;
    auto dup = [&](const void* src, size_t bytes) -> void* {
      void* d = nullptr;
      HE_CK(cudaMalloc(&d, bytes));
      HE_CK(cudaMemcpyAsync(d, src, bytes, cudaMemcpyDeviceToDevice, c->stream));
      return d;
    };
    if (c->d_pk) p->d_pk = (u64*)dup(c->d_pk, 2 * L * N * 8);
    if (c->d_rlk) p->d_rlk = (u64*)dup(c->d_rlk, kw * 8);
    if (c->d_rlk32) p->d_rlk32 = (u32*)dup(c->d_rlk32, kw * 4);
    for (auto& kv : c->gk) p->gk[kv.first] = (u64*)dup(kv.second, kw * 8);
    for (auto& kv : c->gk32) p->gk32[kv.first] = (u32*)dup(kv.second, kw * 4);
    p->has_pk = c->has_pk;
    p->has_rlk = c->has_rlk;
    p->has_sk = false;
    if (c->d_step_gal) build_step_tables(p);
    HE_CK(cudaStreamSynchronize(c->stream));
  } catch (...) {
    context_destroy(p);
    delete p;
    throw;
  }
  return p;
}

// Signed integer coefficients of a plaintext (he_pt_to_int_coeffs): INTT, CRT compose, centre;
// fails with HE_SCALE_OVERFLOW when a centred coefficient is outside the int64 range.
void pt_to_int(he_context* c, const he_plaintext* pt, i64* out_dev) {
  const int N = c->N, Lc = pt->level + 1;
  const size_t B = pt->B;
  Scratch coef(c, B * Lc * N * 8), flag(c, 4);
  HE_CK(cudaMemsetAsync(flag.p, 0, 4, c->stream));
  const size_t pstride = (size_t)pt_limbs(pt) * N;
  ntt_rows(c, pt->d, coef.as<u64>(), B, Lc, pstride, (size_t)Lc * N, true);
  const size_t total = B * N;
  k_crt_compose<<<(unsigned)std::min<size_t>((total + 255) / 256, 148 * 16), 256, 0, c->stream>>>(
      coef.as<u64>(), nullptr, c->d_crt + c->hp.crt_off[pt->level], c->d_primes, N, Lc, total, out_dev,
      flag.as<int>());
  check_launch(c);
  int h = 0;
  HE_CK(cudaMemcpyAsync(&h, flag.p, 4, cudaMemcpyDeviceToHost, c->stream));
  HE_CK(cudaStreamSynchronize(c->stream));
  if (h) throw HeError(HE_SCALE_OVERFLOW, "pt_to_int_coeffs: a coefficient is outside the int64 range");
}

// ---- encode / decode / encrypt / decrypt --------------------------------------
// check_now: read the overflow flag back (stream sync) and fail here; otherwise the kernel ORs it
// into the context's sticky flag, reported by the next he_sync / host-output decode (take_err).
// k_encode_fft into m_dev [B][N] (int64); an overflow sets the context's sticky flag (he_sync reports it).
void encode_coeffs(he_context* c, const double* z_dev, size_t n, size_t B, double scale, i64* m_dev) {
  const int N = c->N, M = N / 2, logM = c->logN - 1;
  const bool in_smem = M <= 8192;
  Scratch g(c, in_smem ? 8 : B * M * 16);
  const int smem = in_smem ? M * 16 : 0;
  if (smem > 48 * 1024)
    smem_limit_once((const void*)k_encode_fft, smem);
  {
    ProfScope ps_(c, "encode_fft", 0.0, 0);
    k_encode_fft<<<(unsigned)B, 512, smem, c->stream>>>(z_dev, n, scale, m_dev, c->d_err, c->d_slot_index,
                                                        c->d_fft_w, c->d_zeta, N, logM,
                                                        in_smem ? nullptr : g.as<double2>());
  }
  check_launch(c);
}

he_plaintext* encode(he_context* c, const double* z_dev, size_t n, size_t B, double scale, int level, int qp,
                     bool check_now) {
  const int N = c->N, M = N / 2, logM = c->logN - 1;
  Scratch m(c, B * N * 8), flag(c, 4);
  if (check_now) HE_CK(cudaMemsetAsync(flag.p, 0, 4, c->stream));
  const bool in_smem = M <= 8192;
  Scratch g(c, in_smem ? 8 : B * M * 16);
  const int smem = in_smem ? M * 16 : 0;
  if (smem > 48 * 1024)
    smem_limit_once((const void*)k_encode_fft, smem);
  {
    ProfScope ps_(c, "encode_fft", 0.0, 0);
    k_encode_fft<<<(unsigned)B, 512, smem, c->stream>>>(z_dev, n, scale, m.as<i64>(),
                                                        check_now ? flag.as<int>() : c->d_err, c->d_slot_index,
                                                        c->d_fft_w, c->d_zeta, N, logM,
                                                        in_smem ? nullptr : g.as<double2>());
  }
  check_launch(c);
  if (check_now) {
    int hflag = 0;
    HE_CK(cudaMemcpyAsync(&hflag, flag.p, 4, cudaMemcpyDeviceToHost, c->stream));
    HE_CK(cudaStreamSynchronize(c->stream));
    if (hflag) throw HeError(HE_SCALE_OVERFLOW, "encode: |scale * z| >= 2^62");
  }
  he_plaintext* pt = pt_new(c, (int)B, level, scale, qp);
  signed_to_ntt(c, m.as<i64>(), pt->d, B, pt_limbs(pt), level + 1);
  return pt;
}

// The encode kernel's coefficient values before rounding (he_encode_unrounded).
void encode_unrounded(he_context* c, const double* z_dev, size_t n, size_t B, double scale, double* pre_dev) {
  const int N = c->N, M = N / 2, logM = c->logN - 1;
  Scratch m(c, B * N * 8), flag(c, 4);
  HE_CK(cudaMemsetAsync(flag.p, 0, 4, c->stream));
  const bool in_smem = M <= 8192;
  Scratch g(c, in_smem ? 8 : B * M * 16);
  const int smem = in_smem ? M * 16 : 0;
  if (smem > 48 * 1024)
    smem_limit_once((const void*)k_encode_fft, smem);
  k_encode_fft<<<(unsigned)B, 512, smem, c->stream>>>(z_dev, n, scale, m.as<i64>(), flag.as<int>(),
                                                      c->d_slot_index, c->d_fft_w, c->d_zeta, N, logM,
                                                      in_smem ? nullptr : g.as<double2>(), pre_dev);
  check_launch(c);
}

he_plaintext* pt_from_int(he_context* c, const i64* m_dev, size_t B, double scale, int level, int qp) {
  he_plaintext* pt = pt_new(c, (int)B, level, scale, qp);
  signed_to_ntt(c, m_dev, pt->d, B, pt_limbs(pt), level + 1);
  return pt;
}

void decode(he_context* c, const he_plaintext* pt, double* out_dev, size_t n) {
  const int N = c->N, M = N / 2, logM = c->logN - 1, Lc = pt->level + 1;
  const size_t B = pt->B;
  Scratch coef(c, B * Lc * N * 8), X(c, B * N * 8);
  ntt_rows(c, pt->d, coef.as<u64>(), B, Lc, (size_t)Lc * N, (size_t)Lc * N, true);
  const size_t total = B * N;
  {
    ProfScope ps_(c, "crt_compose", 0.0, 0);
    k_crt_compose<<<(unsigned)std::min<size_t>((total + 255) / 256, 148 * 16), 256, 0, c->stream>>>(
        coef.as<u64>(), X.as<double>(), c->d_crt + c->hp.crt_off[pt->level], c->d_primes, N, Lc, total);
  }
  check_launch(c);
  const bool in_smem = M <= 8192;
  Scratch g(c, in_smem ? 8 : B * M * 16);
  const int smem = in_smem ? M * 16 : 0;
  if (smem > 48 * 1024)
    smem_limit_once((const void*)k_decode_fft, smem);
  {
    ProfScope ps_(c, "decode_fft", 0.0, 0);
    k_decode_fft<<<(unsigned)B, 512, smem, c->stream>>>(X.as<double>(), n, pt->scale, out_dev, c->d_slot_index,
                                                        c->d_fft_w, c->d_zeta, N, logM,
                                                        in_smem ? nullptr : g.as<double2>());
  }
  check_launch(c);
}

he_ciphertext* encrypt(he_context* c, const he_plaintext* pt, u64 stream_id) {
  // three transforms with the Philox draws in their loads and the ciphertext
  // accumulation in their stores (JobEncrypt): v -> (v b + m, v a), + e0, + e1
  const int Lc = pt->level + 1, B = pt->B;
  he_ciphertext* ct = ct_new(c, B, 2, pt->level, pt->scale);
  try {
    for (int w = 0; w < 3; ++w) {
      JobEncrypt j{ct->d, c->d_pk, pt->d, pt->B == 1 ? 0 : (size_t)Lc * c->N, c->d_cdt, c->seed, stream_id,
                   c->N, Lc, c->L, w};
      launch_ntt<false>(c, j, B * Lc);
    }
  } catch (...) {
    ct_free(ct);
    throw;
  }
  return ct;
}

// Fused encode + public-key encryption (he_encode_encrypt): the canonical-embedding coefficients m
// (k_encode_fft, int64) feed the e0 pass directly, c0 = NTT(v) b + NTT(e0 + m), c1 = NTT(v) a + NTT(e1):
// the plaintext's own B * Lc transforms and its HBM round trip disappear; the words equal
// encrypt(encode(z)) exactly (the transform is linear mod q_i).
he_ciphertext* encode_encrypt(he_context* c, const double* z_dev, size_t n, size_t B, double scale, int level,
                              u64 stream_id) {
  const int Lc = level + 1;
  Scratch m(c, B * c->N * 8);
  encode_coeffs(c, z_dev, n, B, scale, m.as<i64>());
  he_ciphertext* ct = ct_new(c, (int)B, 2, level, scale);
  try {
    for (int w = 0; w < 3; ++w) {
      JobEncrypt j{ct->d, c->d_pk, nullptr, 0, c->d_cdt, c->seed, stream_id, c->N, Lc, c->L, w};
      j.mco = m.as<i64>();
      launch_ntt<false>(c, j, (int)B * Lc);
    }
  } catch (...) {
    ct_free(ct);
    throw;
  }
  return ct;
}

// Symmetric encryption (DESIGN.md §3 "seeded symmetric encryption"):
//   c1 = a,  a_i = Uniform(a_seed, (PUR_SYM_A, stream_id + b, i))  (NTT words, C13 sampler)
//   c0 = -a s + e + m,  e = CDT(seed, (PUR_SYM_E, stream_id + b, 0))  (C11)
__global__ void k_sym_combine(u64* __restrict__ ct, const u64* __restrict__ et, const u64* __restrict__ pt,
                              size_t pt_bs, const u64* __restrict__ sk, const PrimeD* __restrict__ primes, int N,
                              int Lc, size_t rows) {
  for (size_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const int b = (int)(r / Lc), i = (int)(r % Lc);
    const PrimeD P = load_prime(primes, i);
    const size_t LN = (size_t)Lc * N;
    u64* c0 = ct + (size_t)b * 2 * LN + (size_t)i * N;
    const u64* c1 = c0 + LN;
    for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
      const u64 as = mul_mod(c1[n], sk[(size_t)i * N + n], P);
      c0[n] = add_mod(sub_mod(et[r * N + n], as, P.q), pt[(size_t)b * pt_bs + (size_t)i * N + n], P.q);
    }
  }
}

void sym_regen_c1(he_context* c, he_ciphertext* ct) {
  const int Lc = ct->level + 1;
  const size_t LN = (size_t)Lc * c->N;
  ProfScope ps_(c, "sample_uniform", 0.0, 0);
  k_sample_uniform<<<dim3((c->N + 255) / 256, (unsigned)std::min<size_t>((size_t)ct->B * Lc, 65535)), 256, 0,
                     c->stream>>>(ct->d + LN, 2 * LN, ct->B, Lc, c->N, ct->a_seed, PUR_SYM_A, ct->stream0,
                                  c->d_primes);
  check_launch(c);
}

// c0 of every item to / from a dense [B][Lc][N] buffer (the seeded wire payload).
void ct_copy_c0(he_context* c, const he_ciphertext* ct, u64* dst, bool to_ct) {
  const size_t LN = (size_t)(ct->level + 1) * c->N;
  if (to_ct)
    HE_CK(cudaMemcpy2DAsync(ct->d, 2 * LN * 8, dst, LN * 8, LN * 8, ct->B, cudaMemcpyDeviceToDevice, c->stream));
  else
    HE_CK(cudaMemcpy2DAsync(dst, LN * 8, ct->d, 2 * LN * 8, LN * 8, ct->B, cudaMemcpyDeviceToDevice, c->stream));
}

he_ciphertext* encrypt_symmetric(he_context* c, const he_plaintext* pt, u64 stream_id, u64 a_seed) {
  const int Lc = pt->level + 1, B = pt->B;
  he_ciphertext* ct = ct_new(c, B, 2, pt->level, pt->scale);
  try {
    ct->seeded = 1;
    ct->a_seed = a_seed;
    ct->stream0 = stream_id;
    sym_regen_c1(c, ct);
    Scratch e(c, (size_t)B * c->N * 8), et(c, (size_t)B * Lc * c->N * 8);
    {
      ProfScope ps_(c, "sample_small", 0.0, 0);
      k_sample_small<<<dim3((c->N + 255) / 256, (unsigned)std::min(B, 65535)), 256, 0, c->stream>>>(
          e.as<i64>(), c->N, B, c->seed, PUR_SYM_E, stream_id, 1, c->d_cdt);
    }
    check_launch(c);
    signed_to_ntt(c, e.as<i64>(), et.as<u64>(), B, Lc);
    const size_t rows = (size_t)B * Lc;
    {
      ProfScope ps_(c, "sym_combine", 0.0, 0);
      k_sym_combine<<<rows_grid2(c, rows), 256, 0, c->stream>>>(ct->d, et.as<u64>(), pt->d,
                                                                pt->B == 1 ? 0 : (size_t)Lc * c->N, c->d_sk,
                                                                c->d_primes, c->N, Lc, rows);
    }
    check_launch(c);
  } catch (...) {
    ct_free(ct);
    throw;
  }
  return ct;
}

he_plaintext* decrypt(he_context* c, const he_ciphertext* ct) {
  const int Lc = ct->level + 1;
  he_plaintext* pt = pt_new(c, ct->B, ct->level, ct->scale);
  const size_t rows = (size_t)ct->B * Lc;
  {
    ProfScope ps_(c, "decrypt", 0.0, 0);
    k_decrypt<<<rows_grid2(c, rows), 256, 0, c->stream>>>(ct->d, c->d_sk, pt->d, c->d_primes, c->N, Lc, ct->size,
                                                         rows);
  }
  check_launch(c);
  return pt;
}

// Sticky asynchronous errors: read and clear (the caller has synchronized or is about to).
void take_err(he_context* c) {
  int h = 0;
  HE_CK(cudaMemcpyAsync(&h, c->d_err, 4, cudaMemcpyDeviceToHost, c->stream));
  HE_CK(cudaStreamSynchronize(c->stream));
  if (h) {
    HE_CK(cudaMemsetAsync(c->d_err, 0, 4, c->stream));
    HE_CK(cudaStreamSynchronize(c->stream));
    throw HeError(HE_SCALE_OVERFLOW, "an asynchronous he_encode_device saw |scale * z| >= 2^62");
  }
}

int check_words(he_context* c, const u64* w, size_t items, int Lc) {
  Scratch flag(c, 4);
  HE_CK(cudaMemsetAsync(flag.p, 0, 4, c->stream));
  const size_t rows = items * Lc;
  {
    ProfScope ps_(c, "check_words", 0.0, 0);
    k_check_words<<<rows_grid2(c, rows), 256, 0, c->stream>>>(w, c->d_primes, c->N, Lc, rows, flag.as<int>());
  }
  check_launch(c);
  int h = 0;
  HE_CK(cudaMemcpyAsync(&h, flag.p, 4, cudaMemcpyDeviceToHost, c->stream));
  HE_CK(cudaStreamSynchronize(c->stream));
  return h;
}

}  // namespace he
