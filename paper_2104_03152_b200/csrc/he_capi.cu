// he_capi.cu — the C-ABI of include/he_ckks.h: argument validation, status
// codes, host<->device marshalling and the host-side slot layouts of the
// composite ops (C17-C19).  All arithmetic is in he_ops.cu's kernels.
#include <cmath>
#include <cstring>
#include <new>

#include "he_ops.h"

using namespace he;

namespace {

thread_local std::string g_err;

template <class F>
he_status guard(F&& f) {
  try {
    f();
    return HE_OK;
  } catch (const HeError& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host out of memory";
    return HE_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HE_INVALID_ARGUMENT;
  }
}

void need(bool ok, he_status code, const char* msg) {
  if (!ok) throw HeError(code, msg);
}
void need_ctx(const he_context* c) { need(c != nullptr, HE_INVALID_ARGUMENT, "null context"); }
void need_ct(he_context* c, const he_ciphertext* a) {
  need(a != nullptr, HE_INVALID_ARGUMENT, "null ciphertext");
  need(a->ctx == c, HE_PARAM_MISMATCH, "ciphertext belongs to another context");
}
void need_pt(he_context* c, const he_plaintext* a) {
  need(a != nullptr, HE_INVALID_ARGUMENT, "null plaintext");
  need(a->ctx == c, HE_PARAM_MISMATCH, "plaintext belongs to another context");
}
void need_batch(int a, int b) {
  need(a == b || a == 1 || b == 1, HE_SHAPE_MISMATCH, "batch sizes differ (and neither is 1)");
}
void need_out(void* p) { need(p != nullptr, HE_INVALID_ARGUMENT, "null output pointer"); }

double shifted(u64 q, int shift) { return (double)q * std::ldexp(1.0, shift); }

// Upload host doubles into a device scratch buffer.
struct DevDoubles {
  he_context* c;
  double* d;
  DevDoubles(he_context* c_, const double* h, size_t n) : c(c_), d(dalloc_t<double>(c_, n)) {
    if (n) HE_CK(cudaMemcpyAsync(d, h, n * 8, cudaMemcpyHostToDevice, c->stream));
  }
  ~DevDoubles() { dfree(c, d); }
};

// A large host input of the encoder (a batch of slot vectors): uploaded on the context's copy stream
// into one of two context-owned buffers, so that the copy of this call runs while the kernels of the
// previous calls are still executing on c->stream (the host runs ahead of the device in a pipelined
// client loop; on c->stream the copy would queue behind them and the device would idle for its
// duration every step).  c->stream waits for the copy; the copy stream waits, before it refills a
// buffer, for the event recorded after the kernels that read it were enqueued.  Small inputs and
// calls recorded into a CUDA graph take the plain path (DevDoubles).
struct DevDoublesOverlap {
  he_context* c;
  double* d = nullptr;
  int k = -1;          // >= 0: upload buffer k; -1: a pool block (plain path)
  static constexpr size_t kMinBytes = 1u << 20;
  DevDoublesOverlap(he_context* c_, const double* h, size_t n) : c(c_) {
    const size_t bytes = n * 8;
    if (bytes < kMinBytes || c->rec) {
      d = dalloc_t<double>(c, n);
      if (n) HE_CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, c->stream));
      return;
    }
    auto& u = c->up;
    if (!u.stream) {
      HE_CK(cudaStreamCreateWithFlags(&u.stream, cudaStreamNonBlocking));
      for (int i = 0; i < 2; ++i) {
        HE_CK(cudaEventCreateWithFlags(&u.done[i], cudaEventDisableTiming));
        HE_CK(cudaEventCreateWithFlags(&u.free_[i], cudaEventDisableTiming));
      }
    }
    k = u.next;
    u.next ^= 1;
    if (u.cap[k] < bytes) {   // (re)size: the buffer's readers must have finished
      if (u.buf[k]) {
        HE_CK(cudaEventSynchronize(u.free_[k]));
        HE_CK(cudaFree(u.buf[k]));
        u.buf[k] = nullptr;
        u.cap[k] = 0;
      }
      HE_CK(cudaMalloc(&u.buf[k], bytes));
      u.cap[k] = bytes;
    } else {
      HE_CK(cudaStreamWaitEvent(u.stream, u.free_[k], 0));   // (never recorded: no-op)
    }
    d = u.buf[k];
    HE_CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, u.stream));
    HE_CK(cudaEventRecord(u.done[k], u.stream));
    HE_CK(cudaStreamWaitEvent(c->stream, u.done[k], 0));
  }
  ~DevDoublesOverlap() {
    if (k < 0) dfree(c, d);
    else cudaEventRecord(c->up.free_[k], c->stream);   // the readers of buffer k are enqueued
  }
};

struct PtGuard {
  he_plaintext* p = nullptr;
  ~PtGuard() { pt_free(p); }
};

// C17 diagonals: D_k[j] = W[(j+k) mod n][j'], j' = j mod m (replicated output)
// or j for j < m (zero beyond).
std::vector<double> vecmat_diagonals(const double* W, int n, int m, int ns, bool rep) {
  need(n >= 1 && m >= 1 && n <= ns && m <= ns, HE_SHAPE_MISMATCH, "vec_mat: n, m must be in [1, n_s]");
  if (rep) need(ns % n == 0 && ns % m == 0, HE_SHAPE_MISMATCH, "replicated output needs n | n_s and m | n_s");
  const int span = (ns / n) * n;
  std::vector<double> D((size_t)n * ns, 0.0);
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < ns; ++j) {
      const bool live = rep || j < m;
      if (!live) continue;
      if (ns % n && j + k >= span)
        throw HeError(HE_REPLICATION_EXHAUSTED, "vec_mat: diagonal reads past the replicated span");
      const int jp = rep ? j % m : j;
      D[(size_t)k * ns + j] = W[(size_t)((j + k) % n) * m + jp];
    }
  return D;
}

}  // namespace

extern "C" {

const char* he_last_error(void) { return g_err.c_str(); }

he_status he_context_create(const he_params* p, uint64_t seed, he_context** out) {
  return guard([&] {
    need(p != nullptr && out != nullptr && p->bits != nullptr, HE_INVALID_ARGUMENT, "null argument");
    need(p->n_primes >= 1 && p->n_primes <= 64, HE_INVALID_PARAMS, "n_primes out of range");
    const int L = p->n_primes - p->n_special;
    need(p->dnum == 0 || p->dnum == L, HE_INVALID_PARAMS, "only dnum = L (one prime per digit) is supported");
    HostParams hp;
    try {
      hp = make_params(p->log2N, std::vector<int>(p->bits, p->bits + p->n_primes), p->n_special);
    } catch (const std::runtime_error& e) {
      throw HeError(HE_INVALID_PARAMS, e.what());
    }
    he_context* c = new he_context();
    try {
      context_init(c, hp, seed);
    } catch (...) {
      context_destroy(c);
      delete c;
      throw;
    }
    *out = c;
  });
}

he_status he_context_free(he_context* ctx) {
  return guard([&] {
    if (!ctx) return;
    context_destroy(ctx);
    delete ctx;
  });
}

he_status he_context_info(const he_context* c, int* log2N, int* L, int* K) {
  return guard([&] {
    need_ctx(c);
    if (log2N) *log2N = c->logN;
    if (L) *L = c->L;
    if (K) *K = c->K;
  });
}

he_status he_context_primes(const he_context* c, uint64_t* primes_out, uint64_t* psi_out) {
  return guard([&] {
    need_ctx(c);
    for (int t = 0; t < c->NP; ++t) {
      if (primes_out) primes_out[t] = c->hp.q[t];
      if (psi_out) psi_out[t] = c->hp.psi[t];
    }
  });
}

he_status he_context_cdt(const he_context* c, uint64_t* table_out) {
  return guard([&] {
    need_ctx(c);
    need_out(table_out);
    for (size_t k = 0; k < c->hp.cdt.size(); ++k) table_out[k] = c->hp.cdt[k];
  });
}

he_status he_set_stream(he_context* c, void* stream) {
  return guard([&] {
    need_ctx(c);
    need(c->rec == nullptr, HE_INVALID_ARGUMENT, "he_set_stream while recording a graph");
    // cached scratch blocks were last used on the old stream
    if ((cudaStream_t)stream != c->stream) HE_CK(cudaStreamSynchronize(c->stream));
    c->stream = (cudaStream_t)stream;
  });
}

he_status he_sync(he_context* c) {
  return guard([&] {
    need_ctx(c);
    HE_CK(cudaStreamSynchronize(c->stream));
    take_err(c);
  });
}

uint64_t he_launch_count(const he_context* c) { return c ? c->launches : 0; }

// ---- CUDA-graph recording -------------------------------------------------------------------
static void graph_release(he_context* c, const std::vector<void*>& owned, const std::vector<void*>& deferred) {
  for (void* p : owned) {
    c->graph_owned.erase(p);
    c->live_bytes.erase(p);
    cudaFree(p);
  }
  for (void* p : deferred) {   // pre-existing blocks: back to their allocator now
    c->graph_owned.erase(p);
    dfree(c, p);
  }
}

he_status he_graph_begin(he_context* c) {
  return guard([&] {
    need_ctx(c);
    need(c->rec == nullptr, HE_INVALID_ARGUMENT, "already recording a graph");
    need(!c->prof_on, HE_INVALID_ARGUMENT, "he_graph_begin with the profiler enabled");
    auto* r = new he_context::GraphRec();
    try {
      HE_CK(cudaStreamCreateWithFlags(&r->cap, cudaStreamNonBlocking));
      cudaEvent_t ev;
      HE_CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      HE_CK(cudaEventRecord(ev, c->stream));
      HE_CK(cudaStreamWaitEvent(r->cap, ev, 0));
      HE_CK(cudaEventDestroy(ev));
      HE_CK(cudaStreamBeginCapture(r->cap, cudaStreamCaptureModeRelaxed));
    } catch (...) {
      if (r->cap) cudaStreamDestroy(r->cap);
      delete r;
      throw;
    }
    r->orig = c->stream;
    r->launches0 = c->launches;
    c->rec = r;
    c->stream = r->cap;
  });
}

he_status he_graph_end(he_context* c, he_graph** out) {
  return guard([&] {
    need_ctx(c);
    need_out(out);
    need(c->rec != nullptr, HE_INVALID_ARGUMENT, "not recording a graph");
    he_context::GraphRec* r = c->rec;
    c->rec = nullptr;
    c->stream = r->orig;
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(r->cap, &graph);
    cudaGraphExec_t exec = nullptr;
    if (e == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
    cudaStreamDestroy(r->cap);
    if (e != cudaSuccess) {
      cudaGetLastError();
      if (graph) cudaGraphDestroy(graph);
      HE_CK(cudaDeviceSynchronize());   // nothing recorded ran; the owned blocks are unreferenced
      graph_release(c, r->owned, r->deferred);
      delete r;
      throw HeError(HE_CUDA_ERROR, std::string("graph capture failed (a call synchronised or read back "
                                               "while recording?): ") + cudaGetErrorString(e));
    }
    auto* g = new he_graph();
    g->ctx = c;
    g->graph = graph;
    g->exec = exec;
    g->kernels = c->launches - r->launches0;
    c->launches = r->launches0;   // recorded, not launched
    g->owned = std::move(r->owned);
    g->deferred = std::move(r->deferred);
    delete r;
    *out = g;
  });
}

he_status he_graph_launch(he_graph* g) {
  return guard([&] {
    need(g != nullptr && g->ctx != nullptr, HE_INVALID_ARGUMENT, "null graph");
    need(g->ctx->rec == nullptr, HE_INVALID_ARGUMENT, "he_graph_launch while recording");
    HE_CK(cudaGraphLaunch(g->exec, g->ctx->stream));
    g->ctx->launches += g->kernels;
  });
}

uint64_t he_graph_kernels(const he_graph* g) { return g ? g->kernels : 0; }

he_status he_graph_free(he_graph* g) {
  return guard([&] {
    if (!g) return;
    he_context* c = g->ctx;
    // replays in flight on the context stream may still use the graph's memory
    HE_CK(cudaStreamSynchronize(c->stream));
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    graph_release(c, g->owned, g->deferred);
    delete g;
  });
}

he_status he_profile_enable(he_context* c, int on) {
  return guard([&] {
    need_ctx(c);
    c->prof_on = on != 0;
  });
}

he_status he_profile_read(he_context* c, char* buf, size_t len) {
  return guard([&] {
    need_ctx(c);
    need(buf != nullptr && len > 0, HE_INVALID_ARGUMENT, "null buffer");
    HE_CK(cudaStreamSynchronize(c->stream));
    struct Acc { long n = 0; double ms = 0, bytes = 0, blocks = 0, ops = 0; };
    std::map<std::string, Acc> acc;
    for (auto& r : c->prof) {
      float ms = 0;
      HE_CK(cudaEventElapsedTime(&ms, r.a, r.b));
      Acc& a = acc[r.tag];
      a.n++;
      a.ms += ms;
      a.bytes += r.bytes;
      a.blocks += r.blocks;
      a.ops += r.ops;
      c->ev_pool.push_back(r.a);
      c->ev_pool.push_back(r.b);
    }
    c->prof.clear();
    std::string js = "{";
    for (auto& kv : acc) {
      char tmp[256];
      snprintf(tmp, sizeof(tmp), "%s\"%s\": [%ld, %.6f, %.1f, %.0f, %.1f]", js.size() > 1 ? ", " : "",
               kv.first.c_str(), kv.second.n, kv.second.ms, kv.second.bytes, kv.second.blocks, kv.second.ops);
      js += tmp;
    }
    js += "}";
    strncpy(buf, js.c_str(), len - 1);
    buf[len - 1] = 0;
  });
}

he_status he_keygen(he_context* c, const int32_t* steps, size_t n_steps) {
  return guard([&] {
    need_ctx(c);
    need(!c->has_sk, HE_INVALID_ARGUMENT, "keys already generated for this context");
    need(n_steps == 0 || steps != nullptr, HE_INVALID_ARGUMENT, "null rotation steps");
    std::vector<int> st;
    for (size_t i = 0; i < n_steps; ++i) {
      need(steps[i] != 0 && std::abs(steps[i]) <= c->N / 2, HE_INVALID_ROTATION,
           "rotation steps must be nonzero with |step| <= n_s");
      st.push_back(steps[i]);
    }
    need(c->K > 0 || n_steps == 0, HE_INVALID_PARAMS, "rotation keys need at least one special prime");
    keygen(c, st);
  });
}

he_status he_drop_secret_key(he_context* c) {
  return guard([&] {
    need_ctx(c);
    if (c->d_sk) {
      HE_CK(cudaStreamSynchronize(c->stream));
      cudaFree(c->d_sk);
    }
    c->d_sk = nullptr;
    c->has_sk = false;
  });
}

he_status he_make_public(he_context* c, he_context** out) {
  return guard([&] {
    need_ctx(c);
    need_out(out);
    *out = context_make_public(c);
  });
}

he_status he_set_allocator(he_context* c, he_alloc_fn alloc, he_free_fn free_fn, void* user) {
  return guard([&] {
    need_ctx(c);
    need((alloc == nullptr) == (free_fn == nullptr), HE_INVALID_ARGUMENT, "alloc and free must both be set or both NULL");
    set_allocator(c, alloc, free_fn, user);
  });
}

// ---------------------------------------------------------------- encode ---
static void encode_common(he_context* c, const double* z_dev, size_t n, size_t B, double scale, int level,
                          he_plaintext** out, bool check_now = true) {
  need_ctx(c);
  need_out(out);
  need(B >= 1, HE_INVALID_ARGUMENT, "B must be >= 1");
  need(n <= (size_t)c->N / 2, HE_TOO_MANY_VALUES, "more values than slots");
  need(level >= 0 && level < c->L, HE_LEVEL_MISMATCH, "level out of range");
  need(scale > 0 && std::isfinite(scale), HE_INVALID_ARGUMENT, "scale must be positive");
  *out = encode(c, z_dev, n, B, scale, level, 0, check_now);
}

// C7 bound, checked on the host before anything is enqueued: |m_i| <= scale (2/N) sum_j |z_j|, so
// when that bound is below 2^62 (with a 2^-20 relative margin for the FFT's rounding) no
// coefficient can overflow and the encode needs no device-to-host readback.
static void host_overflow_check(const he_context* c, const double* z, size_t n, size_t B, double scale) {
  const double lim = 4611686018427387904.0 * (1.0 - 1.0 / 1048576.0);
  const double k = 2.0 * scale / (double)c->N;
  for (size_t b = 0; b < B; ++b) {
    double s = 0.0;
    const double* zb = z + b * n;
    for (size_t j = 0; j < n; ++j) s += std::fabs(zb[j]);
    need(std::isfinite(s) && k * s < lim, HE_SCALE_OVERFLOW,
         "encode: scale (2/N) sum |z| >= 2^62 (a coefficient may overflow), or a value is not finite");
  }
}

he_status he_encode(he_context* c, const double* z, size_t n, size_t B, double scale, int level,
                    he_plaintext** out) {
  return guard([&] {
    need_ctx(c);
    need(z != nullptr || n == 0, HE_INVALID_ARGUMENT, "null input");
    need(B >= 1, HE_INVALID_ARGUMENT, "B must be >= 1");
    need(n <= (size_t)c->N / 2, HE_TOO_MANY_VALUES, "more values than slots");
    need(scale > 0 && std::isfinite(scale), HE_INVALID_ARGUMENT, "scale must be positive");
    host_overflow_check(c, z, n, B, scale);
    // H2D on the context stream (asynchronous from pinned memory), then the encode kernels; the
    // host bound above already excludes an overflow, so nothing is read back
    DevDoublesOverlap d(c, z, n * B);
    encode_common(c, d.d, n, B, scale, level, out, false);
  });
}

he_status he_encode_unrounded(he_context* c, const double* z, size_t n, size_t B, double scale, double* out) {
  return guard([&] {
    need_ctx(c);
    need_out(out);
    need(z != nullptr || n == 0, HE_INVALID_ARGUMENT, "null input");
    need(B >= 1, HE_INVALID_ARGUMENT, "B must be >= 1");
    need(n <= (size_t)c->N / 2, HE_TOO_MANY_VALUES, "more values than slots");
    need(scale > 0 && std::isfinite(scale), HE_INVALID_ARGUMENT, "scale must be positive");
    DevDoubles d(c, z, n * B);
    Scratch pre(c, B * (size_t)c->N * 8);
    encode_unrounded(c, d.d, n, B, scale, pre.as<double>());
    HE_CK(cudaMemcpyAsync(out, pre.p, B * (size_t)c->N * 8, cudaMemcpyDeviceToHost, c->stream));
    HE_CK(cudaStreamSynchronize(c->stream));
  });
}

he_status he_encode_device(he_context* c, const double* z_dev, size_t n, size_t B, double scale, int level,
                           he_plaintext** out) {
  return guard([&] { encode_common(c, z_dev, n, B, scale, level, out, false); });
}

he_status he_decode(he_context* c, const he_plaintext* pt, double* out, size_t n) {
  return guard([&] {
    need_ctx(c);
    need_pt(c, pt);
    need_out(out);
    need(n <= (size_t)c->N / 2, HE_TOO_MANY_VALUES, "more values than slots");
    Scratch d(c, std::max<size_t>(1, (size_t)pt->B * n) * 8);
    decode(c, pt, d.as<double>(), n);
    take_err(c);   // (syncs) an asynchronous encode error fails the call before out is written
    HE_CK(cudaMemcpyAsync(out, d.p, (size_t)pt->B * n * 8, cudaMemcpyDeviceToHost, c->stream));
    HE_CK(cudaStreamSynchronize(c->stream));
  });
}

he_status he_decode_async(he_context* c, const he_plaintext* pt, double* out, size_t n) {
  return guard([&] {
    need_ctx(c);
    need_pt(c, pt);
    need_out(out);
    need(n <= (size_t)c->N / 2, HE_TOO_MANY_VALUES, "more values than slots");
    Scratch d(c, std::max<size_t>(1, (size_t)pt->B * n) * 8);
    decode(c, pt, d.as<double>(), n);
    HE_CK(cudaMemcpyAsync(out, d.p, (size_t)pt->B * n * 8, cudaMemcpyDeviceToHost, c->stream));
  });
}

he_status he_decode_device(he_context* c, const he_plaintext* pt, double* out_dev, size_t n) {
  return guard([&] {
    need_ctx(c);
    need_pt(c, pt);
    need_out(out_dev);
    need(n <= (size_t)c->N / 2, HE_TOO_MANY_VALUES, "more values than slots");
    decode(c, pt, out_dev, n);
  });
}

// -------------------------------------------------------- encrypt/decrypt ---
he_status he_encrypt(he_context* c, const he_plaintext* pt, uint64_t stream_id, he_ciphertext** out) {
  return guard([&] {
    need_ctx(c);
    need_pt(c, pt);
    need_out(out);
    need(c->has_pk, HE_MISSING_KEY, "no public key (call he_keygen)");
    *out = encrypt(c, pt, stream_id);
  });
}

static void encode_encrypt_common(he_context* c, const double* z_dev, size_t n, size_t B, double scale, int level,
                                  uint64_t stream_id, he_ciphertext** out) {
  need_ctx(c);
  need_out(out);
  need(B >= 1, HE_INVALID_ARGUMENT, "B must be >= 1");
  need(n <= (size_t)c->N / 2, HE_TOO_MANY_VALUES, "more values than slots");
  need(level >= 0 && level < c->L, HE_LEVEL_MISMATCH, "level out of range");
  need(scale > 0 && std::isfinite(scale), HE_INVALID_ARGUMENT, "scale must be positive");
  need(c->has_pk, HE_MISSING_KEY, "no public key (call he_keygen)");
  *out = encode_encrypt(c, z_dev, n, B, scale, level, stream_id);
}

he_status he_encode_encrypt(he_context* c, const double* z, size_t n, size_t B, double scale, int level,
                            uint64_t stream_id, he_ciphertext** out) {
  return guard([&] {
    need_ctx(c);
    need(z != nullptr || n == 0, HE_INVALID_ARGUMENT, "null input");
    need(B >= 1, HE_INVALID_ARGUMENT, "B must be >= 1");
    need(n <= (size_t)c->N / 2, HE_TOO_MANY_VALUES, "more values than slots");
    need(scale > 0 && std::isfinite(scale), HE_INVALID_ARGUMENT, "scale must be positive");
    host_overflow_check(c, z, n, B, scale);
    DevDoublesOverlap d(c, z, n * B);
    encode_encrypt_common(c, d.d, n, B, scale, level, stream_id, out);
  });
}

he_status he_encode_encrypt_device(he_context* c, const double* z_dev, size_t n, size_t B, double scale, int level,
                                   uint64_t stream_id, he_ciphertext** out) {
  return guard([&] { encode_encrypt_common(c, z_dev, n, B, scale, level, stream_id, out); });
}

he_status he_encrypt_symmetric(he_context* c, const he_plaintext* pt, uint64_t stream_id, uint64_t a_seed,
                               he_ciphertext** out) {
  return guard([&] {
    need_ctx(c);
    need_pt(c, pt);
    need_out(out);
    need(c->has_sk, HE_MISSING_KEY, "symmetric encryption needs the secret key");
    need(!pt->qp, HE_LAYOUT_MISMATCH, "plaintext must be on the data limbs only");
    *out = encrypt_symmetric(c, pt, stream_id, a_seed);
  });
}

he_status he_decrypt(he_context* c, const he_ciphertext* ct, he_plaintext** out) {
  return guard([&] {
    need_ctx(c);
    need_ct(c, ct);
    need_out(out);
    need(c->has_sk, HE_MISSING_KEY, "no secret key");
    *out = decrypt(c, ct);
  });
}

// ------------------------------------------------------------- arithmetic ---
static void need_same(const he_ciphertext* a, const he_ciphertext* b, bool scale_too) {
  need(a->level == b->level, HE_LEVEL_MISMATCH, "ciphertext levels differ");
  need(a->size == b->size, HE_SHAPE_MISMATCH, "ciphertext sizes differ");
  if (scale_too) need(a->scale == b->scale, HE_SCALE_MISMATCH, "ciphertext scales differ");
  need_batch(a->B, b->B);
}

he_status he_add(he_context* c, const he_ciphertext* a, const he_ciphertext* b, he_ciphertext** out) {
  return guard([&] {
    need_ctx(c); need_ct(c, a); need_ct(c, b); need_out(out);
    need_same(a, b, true);
    *out = ct_binop(c, 0, a, b);
  });
}

he_status he_sub(he_context* c, const he_ciphertext* a, const he_ciphertext* b, he_ciphertext** out) {
  return guard([&] {
    need_ctx(c); need_ct(c, a); need_ct(c, b); need_out(out);
    need_same(a, b, true);
    *out = ct_binop(c, 1, a, b);
  });
}

he_status he_negate(he_context* c, const he_ciphertext* a, he_ciphertext** out) {
  return guard([&] {
    need_ctx(c); need_ct(c, a); need_out(out);
    *out = ct_negate(c, a);
  });
}

static void need_plain_q(const he_plaintext* p) {
  need(!p->qp, HE_LAYOUT_MISMATCH, "QP plaintexts (with special limbs) are only accepted by he_vec_mat_pt");
}

he_status he_add_plain(he_context* c, const he_ciphertext* a, const he_plaintext* p, he_ciphertext** out) {
  return guard([&] {
    need_ctx(c); need_ct(c, a); need_pt(c, p); need_out(out);
    need_plain_q(p);
    need(a->level == p->level, HE_LEVEL_MISMATCH, "levels differ");
    need(a->scale == p->scale, HE_SCALE_MISMATCH, "scales differ");
    need_batch(a->B, p->B);
    *out = ct_add_plain(c, a, p);
  });
}

he_status he_mul_plain(he_context* c, const he_ciphertext* a, const he_plaintext* p, he_ciphertext** out) {
  return guard([&] {
    need_ctx(c); need_ct(c, a); need_pt(c, p); need_out(out);
    need_plain_q(p);
    need(a->level == p->level, HE_LEVEL_MISMATCH, "levels differ");
    need_batch(a->B, p->B);
    *out = ct_mul_plain(c, a, p);
  });
}

he_status he_mul(he_context* c, const he_ciphertext* a, const he_ciphertext* b, he_ciphertext** out) {
  return guard([&] {
    need_ctx(c); need_ct(c, a); need_ct(c, b); need_out(out);
    need(a->size == 2 && b->size == 2, HE_SHAPE_MISMATCH, "mul needs size-2 ciphertexts");
    need_same(a, b, false);
    *out = ct_tensor(c, a, b);
  });
}

he_status he_relinearize(he_context* c, const he_ciphertext* a, he_ciphertext** out) {
  return guard([&] {
    need_ctx(c); need_ct(c, a); need_out(out);
    need(a->size == 3, HE_SHAPE_MISMATCH, "relinearize needs a size-3 ciphertext");
    need(c->has_rlk, HE_MISSING_KEY, "no relinearisation key");
    *out = ct_relinearize(c, a);
  });
}

// ---- in-place forms (SURVEY 8(b) "_inplace variants exist for the hot loop") -------------------
// add / sub / add_plain / mul_plain write into a's storage (no allocation) when a holds the larger
// batch; rescale / rotate / square produce a new limb layout, so a's storage is replaced (the old
// block returns to the pool in stream order) and the handle stays the caller's.
static void adopt(he_ciphertext* a, he_ciphertext* r) {
  std::swap(a->B, r->B);
  std::swap(a->size, r->size);
  std::swap(a->level, r->level);
  std::swap(a->scale, r->scale);
  std::swap(a->d, r->d);
  a->seeded = 0;
  ct_free(r);
}

he_status he_add_inplace(he_context* c, he_ciphertext* a, const he_ciphertext* b) {
  return guard([&] {
    need_ctx(c); need_ct(c, a); need_ct(c, b);
    need_same(a, b, true);
    if (a->B >= b->B) ct_binop(c, 0, a, b, a);
    else adopt(a, ct_binop(c, 0, a, b));
    a->seeded = 0;
  });
}

he_status he_sub_inplace(he_context* c, he_ciphertext* a, const he_ciphertext* b) {
  return guard([&] {
    need_ctx(c); need_ct(c, a); need_ct(c, b);
    need_same(a, b, true);
    if (a->B >= b->B) ct_binop(c, 1, a, b, a);
    else adopt(a, ct_binop(c, 1, a, b));
    a->seeded = 0;
  });
}

he_status he_add_plain_inplace(he_context* c, he_ciphertext* a, const he_plaintext* p) {
  return guard([&] {
    need_ctx(c); need_ct(c, a); need_pt(c, p);
    need_plain_q(p);
    need(a->level == p->level, HE_LEVEL_MISMATCH, "levels differ");
    need(a->scale == p->scale, HE_SCALE_MISMATCH, "scales differ");
    need_batch(a->B, p->B);
    if (a->B >= p->B) ct_add_plain(c, a, p, a);
    else adopt(a, ct_add_plain(c, a, p));
    a->seeded = 0;
  });
}

he_status he_mul_plain_inplace(he_context* c, he_ciphertext* a, const he_plaintext* p) {
  return guard([&] {
    need_ctx(c); need_ct(c, a); need_pt(c, p);
    need_plain_q(p);
    need(a->level == p->level, HE_LEVEL_MISMATCH, "levels differ");
    need_batch(a->B, p->B);
    if (a->B >= p->B) ct_mul_plain(c, a, p, a);
    else adopt(a, ct_mul_plain(c, a, p));
    a->seeded = 0;
  });
}

he_status he_rescale_inplace(he_context* c, he_ciphertext* a) {
  he_ciphertext* r = nullptr;
  const he_status st = he_rescale(c, a, &r);
  if (st == HE_OK) adopt(a, r);
  return st;
}

he_status he_rotate_inplace(he_context* c, he_ciphertext* a, int32_t k) {
  he_ciphertext* r = nullptr;
  const he_status st = he_rotate(c, a, k, &r);
  if (st == HE_OK) adopt(a, r);
  return st;
}

he_status he_square_inplace(he_context* c, he_ciphertext* a) {
  he_ciphertext* r = nullptr;
  const he_status st = he_square(c, a, &r);
  if (st == HE_OK) adopt(a, r);
  return st;
}

he_status he_rescale(he_context* c, const he_ciphertext* a, he_ciphertext** out) {
  return guard([&] {
    need_ctx(c); need_ct(c, a); need_out(out);
    need(a->level >= 1, HE_LEVEL_EXHAUSTED, "rescale at level 0");
    *out = ct_rescale(c, a);
  });
}

he_status he_square(he_context* c, const he_ciphertext* a, he_ciphertext** out) {
  return guard([&] {
    need_ctx(c); need_ct(c, a); need_out(out);
    need(a->size == 2, HE_SHAPE_MISMATCH, "square needs a size-2 ciphertext");
    need(c->has_rlk, HE_MISSING_KEY, "no relinearisation key");
    need(a->level >= 1, HE_LEVEL_EXHAUSTED, "square needs a level to rescale");
    // tensor fused into the key switch and the rescale into its ModDown when available
    *out = ct_square_rescale(c, a);
  });
}

he_status he_rotate(he_context* c, const he_ciphertext* a, int32_t k, he_ciphertext** out) {
  return guard([&] {
    need_ctx(c); need_ct(c, a); need_out(out);
    need(a->size == 2, HE_SHAPE_MISMATCH, "rotate needs a size-2 ciphertext");
    const int ns = c->N / 2;
    need(std::abs(k) <= ns, HE_INVALID_ROTATION, "|k| must be <= n_s");
    u32 g;
    if (k % ns == 0 && !has_galois_key(c, k == 0 ? ns : k, &g)) {  // identity without a key: copy
      he_ciphertext* o = ct_new(c, a->B, a->size, a->level, a->scale);
      HE_CK(cudaMemcpyAsync(o->d, a->d, ct_words(a) * 8, cudaMemcpyDeviceToDevice, c->stream));
      *out = o;
      return;
    }
    *out = ct_rotate(c, a, k, false);
  });
}

// ------------------------------------------- level alignment + circuits ---
namespace {
struct CtGuard {
  he_ciphertext* p = nullptr;
  ~CtGuard() { ct_free(p); }
  he_ciphertext* release() {
    he_ciphertext* r = p;
    p = nullptr;
    return r;
  }
};

he_ciphertext* mod_switch(he_context* c, const he_ciphertext* a, int level) {
  he_ciphertext* o = ct_new(c, a->B, a->size, level, a->scale);
  const size_t N8 = (size_t)c->N * 8;
  HE_CK(cudaMemcpy2DAsync(o->d, (level + 1) * N8, a->d, (a->level + 1) * N8, (level + 1) * N8,
                          (size_t)a->B * a->size, cudaMemcpyDeviceToDevice, c->stream));
  return o;
}

// tensor -> relinearize -> rescale at the lower of the two levels (C14)
he_ciphertext* mul_relin_rescale(he_context* c, const he_ciphertext* a, const he_ciphertext* b) {
  const int lvl = std::min(a->level, b->level);
  need(lvl >= 1, HE_LEVEL_EXHAUSTED, "multiplication needs a level to rescale");
  CtGuard am, bm, t, r;
  if (a->level != lvl) am.p = mod_switch(c, a, lvl);
  if (b->level != lvl) bm.p = mod_switch(c, b, lvl);
  t.p = ct_tensor(c, am.p ? am.p : a, bm.p ? bm.p : b);
  r.p = ct_relinearize(c, t.p);
  return ct_rescale(c, r.p);
}

// rotate-and-add by 1, 2, 4, ... < n
he_ciphertext* fold_sum(he_context* c, he_ciphertext* t, int n) {
  for (int s = 1; s < n; s <<= 1) {
    he_ciphertext* u = ct_rotate(c, t, s, true);
    ct_free(t);
    t = u;
  }
  return t;
}

void need_fold_keys(he_context* c, int n) {
  for (int s = 1; s < n; s <<= 1) {
    u32 g;
    need(has_galois_key(c, s, &g), HE_MISSING_GALOIS_KEY, "dot needs Galois keys for powers of two below n");
  }
}

// x^1..x^d, depth-optimal (oracle circuits.powers)
std::map<int, he_ciphertext*> powers(he_context* c, const he_ciphertext* x, int d) {
  std::map<int, he_ciphertext*> P;
  P[1] = nullptr;   // x itself (not owned)
  auto get = [&](int i) -> const he_ciphertext* { return i == 1 ? x : P[i]; };
  try {
    for (int k = 1; 2 * k <= d; k *= 2) {
      const he_ciphertext* base = get(k);
      need(base->level >= 1, HE_LEVEL_EXHAUSTED, "power: levels exhausted");
      CtGuard t, r;
      t.p = ct_tensor(c, base, base);
      r.p = ct_relinearize(c, t.p);
      P[2 * k] = ct_rescale(c, r.p);
    }
    for (int i = 2; i <= d; ++i) {
      if (P.count(i)) continue;
      int hi = 1;
      while (2 * hi <= i) hi *= 2;
      P[i] = mul_relin_rescale(c, get(hi), get(i - hi));
    }
  } catch (...) {
    for (auto& kv : P) ct_free(kv.second);
    throw;
  }
  return P;
}
void free_powers(std::map<int, he_ciphertext*>& P) {
  for (auto& kv : P) ct_free(kv.second);
  P.clear();
}
}  // namespace

he_status he_mod_switch_to(he_context* c, const he_ciphertext* a, int level, he_ciphertext** out) {
  return guard([&] {
    need_ctx(c); need_ct(c, a); need_out(out);
    need(level >= 0 && level <= a->level, HE_LEVEL_MISMATCH, "target level must be in [0, ct level]");
    *out = mod_switch(c, a, level);
  });
}

he_status he_dot(he_context* c, const he_ciphertext* a, const he_ciphertext* b, int n, he_ciphertext** out) {
  return guard([&] {
    need_ctx(c); need_ct(c, a); need_ct(c, b); need_out(out);
    need(a->size == 2 && b->size == 2, HE_SHAPE_MISMATCH, "dot needs size-2 ciphertexts");
    need(n >= 1 && n <= c->N / 2, HE_SHAPE_MISMATCH, "1 <= n <= n_s");
    need_batch(a->B, b->B);
    need(c->has_rlk, HE_MISSING_KEY, "no relinearisation key");
    need_fold_keys(c, n);
    *out = fold_sum(c, mul_relin_rescale(c, a, b), n);
  });
}

he_status he_dot_plain(he_context* c, const he_ciphertext* a, const double* z, size_t nz, int n,
                       he_ciphertext** out) {
  return guard([&] {
    need_ctx(c); need_ct(c, a); need_out(out);
    need(z != nullptr && nz <= (size_t)c->N / 2, HE_TOO_MANY_VALUES, "z must hold <= n_s values");
    need(n >= 1 && n <= c->N / 2, HE_SHAPE_MISMATCH, "1 <= n <= n_s");
    need(a->level >= 1, HE_LEVEL_EXHAUSTED, "dot_plain consumes one level");
    need_fold_keys(c, n);
    PtGuard pz;
    {
      DevDoubles d(c, z, nz);
      pz.p = encode(c, d.d, nz, 1, (double)c->hp.q[a->level], a->level);
    }
    CtGuard m;
    m.p = ct_mul_plain(c, a, pz.p);
    he_ciphertext* t = ct_rescale(c, m.p);
    *out = fold_sum(c, t, n);
  });
}

he_status he_power(he_context* c, const he_ciphertext* x, int p, he_ciphertext** out) {
  return guard([&] {
    need_ctx(c); need_ct(c, x); need_out(out);
    need(x->size == 2, HE_SHAPE_MISMATCH, "power needs a size-2 ciphertext");
    need(p >= 1, HE_INVALID_ARGUMENT, "p >= 1");
    if (p == 1) {
      *out = mod_switch(c, x, x->level);
      return;
    }
    need(c->has_rlk, HE_MISSING_KEY, "no relinearisation key");
    int depth = 0;
    while ((1 << depth) < p) ++depth;
    need(x->level >= depth, HE_LEVEL_EXHAUSTED, "power: not enough levels");
    auto P = powers(c, x, p);
    he_ciphertext* r = P[p];
    P[p] = nullptr;
    free_powers(P);
    *out = r;
  });
}

he_status he_polyval(he_context* c, const he_ciphertext* x, const double* coeffs, int n_coeffs,
                     he_ciphertext** out) {
  return guard([&] {
    need_ctx(c); need_ct(c, x); need_out(out);
    need(coeffs != nullptr && n_coeffs >= 2, HE_INVALID_ARGUMENT, "need degree >= 1");
    need(x->size == 2, HE_SHAPE_MISMATCH, "polyval needs a size-2 ciphertext");
    const int d = n_coeffs - 1;
    int depth = 0;
    while ((1 << depth) < d) ++depth;
    need(x->level >= depth + 1, HE_LEVEL_EXHAUSTED, "polyval: not enough levels");
    need(d == 1 || c->has_rlk, HE_MISSING_KEY, "no relinearisation key");
    auto P = powers(c, x, d);
    CtGuard acc;
    try {
      const he_ciphertext* xd = d == 1 ? x : P[d];
      const int ld = xd->level;
      const double S = xd->scale;
      const int ns = c->N / 2;
      for (int i = 1; i <= d; ++i) {
        if (coeffs[i] == 0.0) continue;
        const he_ciphertext* xi = i == 1 ? x : P[i];
        CtGuard xm;
        if (xi->level != ld) xm.p = mod_switch(c, xi, ld);
        const he_ciphertext* xs = xm.p ? xm.p : xi;
        const double sc = S * (double)c->hp.q[ld] / xs->scale;
        std::vector<double> cv(ns, coeffs[i]);
        PtGuard pc;
        {
          DevDoubles dd(c, cv.data(), cv.size());
          pc.p = encode(c, dd.d, ns, 1, sc, ld);
        }
        CtGuard m;
        m.p = ct_mul_plain(c, xs, pc.p);
        he_ciphertext* t = ct_rescale(c, m.p);
        if (!acc.p) {
          acc.p = t;
        } else {   // equal scales up to double rounding: summed at acc's scale
          he_ciphertext* s2 = ct_binop(c, 0, acc.p, t);
          ct_free(t);
          ct_free(acc.p);
          acc.p = s2;
        }
      }
      need(acc.p != nullptr, HE_INVALID_ARGUMENT, "all non-constant coefficients are zero");
      if (coeffs[0] != 0.0) {
        std::vector<double> cv(ns, coeffs[0]);
        PtGuard pc;
        {
          DevDoubles dd(c, cv.data(), cv.size());
          pc.p = encode(c, dd.d, ns, 1, acc.p->scale, acc.p->level);
        }
        he_ciphertext* s2 = ct_add_plain(c, acc.p, pc.p);
        ct_free(acc.p);
        acc.p = s2;
      }
    } catch (...) {
      free_powers(P);
      throw;
    }
    free_powers(P);
    *out = acc.release();
  });
}

// ------------------------------------------------------------- composite ---
he_status he_im2col_encode(const double* img, int H, int W, int kh, int kw, int stride, size_t n_slots,
                           double* slots_out, int* windows, int* chunk) {
  return guard([&] {
    need(img && slots_out, HE_INVALID_ARGUMENT, "null argument");
    need(H >= kh && W >= kw && kh > 0 && kw > 0 && stride > 0, HE_SHAPE_MISMATCH, "bad conv geometry");
    const ConvGeom g = conv_geometry(H, W, kh, kw, stride);
    need((size_t)kh * kw * g.chunk <= n_slots, HE_LAYOUT_MISMATCH, "im2col matrix does not fit the slots");
    std::fill(slots_out, slots_out + n_slots, 0.0);
    for (int r = 0; r < g.oh; ++r)
      for (int cc = 0; cc < g.ow; ++cc) {
        const int w = r * g.ow + cc;
        for (int a = 0; a < kh; ++a)
          for (int b = 0; b < kw; ++b)
            slots_out[(size_t)(a * kw + b) * g.chunk + w] = img[(size_t)(r * stride + a) * W + cc * stride + b];
      }
    if (windows) *windows = g.windows;
    if (chunk) *chunk = g.chunk;
  });
}

he_status he_im2col_encode_batch(const double* imgs, size_t B, int H, int W, int kh, int kw, int stride,
                                 size_t n_slots, double* slots_out) {
  for (size_t b = 0; b < B; ++b) {
    he_status st = he_im2col_encode(imgs + b * (size_t)H * W, H, W, kh, kw, stride, n_slots, slots_out + b * n_slots,
                                    nullptr, nullptr);
    if (st != HE_OK) return st;
  }
  return HE_OK;
}

static void conv_checks(he_context* c, const he_ciphertext* ct, int C, int taps, int chunk) {
  const int ns = c->N / 2;
  need(ct->size == 2, HE_SHAPE_MISMATCH, "conv needs a size-2 ciphertext");
  need(ct->level >= 2, HE_LEVEL_EXHAUSTED, "conv consumes two levels");
  need(C >= 1, HE_SHAPE_MISMATCH, "need at least one channel");
  need(chunk >= 1 && (chunk & (chunk - 1)) == 0 && chunk <= ns && ns % chunk == 0, HE_LAYOUT_MISMATCH,
       "chunk must be a power of two dividing n_s");
  need((size_t)taps * chunk <= (size_t)ns, HE_LAYOUT_MISMATCH, "taps x chunk exceeds the slots");
}

static he_status conv_pt_impl(he_context* c, const he_ciphertext* ct, const he_plaintext* kernels,
                              const he_plaintext* masks, const he_plaintext* bias, int chunk, int fold_n1,
                              he_ciphertext** out);

he_status he_im2col_conv_pt(he_context* c, const he_ciphertext* ct, const he_plaintext* kernels,
                            const he_plaintext* masks, const he_plaintext* bias, int chunk, he_ciphertext** out) {
  return conv_pt_impl(c, ct, kernels, masks, bias, chunk, 0, out);
}

he_status he_im2col_conv_hoisted_pt(he_context* c, const he_ciphertext* ct, const he_plaintext* kernels,
                                    const he_plaintext* masks, const he_plaintext* bias, int chunk, int n1,
                                    he_ciphertext** out) {
  return guard([&] {
    need_ctx(c);
    need(n1 >= 1 && chunk >= 1 && (c->N / 2 / chunk) % n1 == 0, HE_LAYOUT_MISMATCH, "n1 must divide n_s / chunk");
    need(c->K > 0, HE_INVALID_PARAMS, "lazy ModDown needs special primes");
    const int nc = c->N / 2 / chunk, n2 = nc / n1;
    for (int b = 1; b < n1; ++b) {
      u32 g;
      need(has_galois_key(c, chunk * b, &g), HE_MISSING_GALOIS_KEY, "missing key for chunk * b");
    }
    for (int a = 1; a < n2; ++a) {
      u32 g;
      need(has_galois_key(c, chunk * n1 * a, &g), HE_MISSING_GALOIS_KEY, "missing key for chunk * n1 * a");
    }
    he_status st = conv_pt_impl(c, ct, kernels, masks, bias, chunk, n1, out);
    if (st != HE_OK) throw HeError(st, he_last_error());
  });
}

static he_status conv_pt_impl(he_context* c, const he_ciphertext* ct, const he_plaintext* kernels,
                              const he_plaintext* masks, const he_plaintext* bias, int chunk, int fold_n1,
                              he_ciphertext** out) {
  return guard([&] {
    need_ctx(c); need_ct(c, ct); need_pt(c, kernels); need_pt(c, masks); need_out(out);
    conv_checks(c, ct, kernels->B, 1, chunk);
    need_plain_q(kernels);
    need_plain_q(masks);
    if (bias) need_plain_q(bias);
    need(masks->B == kernels->B, HE_SHAPE_MISMATCH, "one mask per kernel");
    need(kernels->level == ct->level && masks->level == ct->level - 1, HE_LEVEL_MISMATCH,
         "kernels at the input level, masks one below");
    if (bias) {
      need_pt(c, bias);
      need(bias->B == 1, HE_SHAPE_MISMATCH, "bias is one plaintext");
      need(bias->level == ct->level - 2, HE_LEVEL_MISMATCH, "bias at the output level");
      const double s1 = ct->scale * kernels->scale / (double)c->hp.q[ct->level];
      const double s2 = s1 * masks->scale / (double)c->hp.q[ct->level - 1];
      need(bias->scale == s2, HE_SCALE_MISMATCH, "bias scale must equal the output scale");
    }
    if (fold_n1 == 0)
      for (int step = chunk; step < c->N / 2; step <<= 1) {
        u32 g;
        need(has_galois_key(c, step, &g), HE_MISSING_GALOIS_KEY, "missing Galois key for a fold step");
      }
    *out = ct_conv(c, ct, kernels, masks, bias, chunk, fold_n1);
  });
}

// C18/C19 plaintexts of the conv: kernels at q_l 2^kernel_shift (level l),
// masks at q_{l-1} 2^mask_shift (level l-1), bias at the output scale (l-2).
static void conv_encode(he_context* c, const double* kernels, int C, int kh, int kw, const double* bias,
                        int chunk, int kernel_shift, int mask_shift, int l, double in_scale,
                        he_plaintext** kp, he_plaintext** mp, he_plaintext** bp) {
  const int ns = c->N / 2, taps = kh * kw;
  need(kernels != nullptr, HE_INVALID_ARGUMENT, "null kernels");
  need(l >= 2 && l < c->L, HE_LEVEL_EXHAUSTED, "conv consumes two levels");
  need(C >= 1 && taps >= 1, HE_SHAPE_MISMATCH, "need at least one channel and tap");
  need(chunk >= 1 && (chunk & (chunk - 1)) == 0 && ns % chunk == 0, HE_LAYOUT_MISMATCH,
       "chunk must be a power of two dividing n_s");
  need((size_t)taps * chunk <= (size_t)ns, HE_LAYOUT_MISMATCH, "taps x chunk exceeds the slots");
  std::vector<double> K((size_t)C * ns, 0.0), M((size_t)C * ns, 0.0);
  for (int ch = 0; ch < C; ++ch) {
    for (int t = 0; t < taps; ++t)
      for (int w = 0; w < chunk; ++w) K[(size_t)ch * ns + (size_t)t * chunk + w] = kernels[(size_t)ch * taps + t];
    for (int s = 0; s < ns; ++s) M[(size_t)ch * ns + s] = ((s / chunk) % C == ch) ? 1.0 : 0.0;
  }
  PtGuard pk, pm, pb;
  {
    DevDoubles d(c, K.data(), K.size());
    pk.p = encode(c, d.d, ns, C, shifted(c->hp.q[l], kernel_shift), l);
  }
  {
    DevDoubles d(c, M.data(), M.size());
    pm.p = encode(c, d.d, ns, C, shifted(c->hp.q[l - 1], mask_shift), l - 1);
  }
  if (bias) {
    std::vector<double> bs(ns);
    for (int s = 0; s < ns; ++s) bs[s] = bias[(s / chunk) % C];
    const double s1 = in_scale * pk.p->scale / (double)c->hp.q[l];
    const double s2 = s1 * pm.p->scale / (double)c->hp.q[l - 1];
    DevDoubles d(c, bs.data(), bs.size());
    pb.p = encode(c, d.d, ns, 1, s2, l - 2);
  }
  *kp = pk.p;
  *mp = pm.p;
  *bp = pb.p;
  pk.p = pm.p = pb.p = nullptr;
}

he_status he_im2col_conv_encode(he_context* c, const double* kernels, int C, int kh, int kw, const double* bias,
                                int chunk, int kernel_shift, int mask_shift, int level, double in_scale,
                                he_plaintext** kp, he_plaintext** mp, he_plaintext** bp) {
  return guard([&] {
    need_ctx(c);
    need(kp && mp && bp, HE_INVALID_ARGUMENT, "null output pointer");
    conv_encode(c, kernels, C, kh, kw, bias, chunk, kernel_shift, mask_shift, level, in_scale, kp, mp, bp);
  });
}

// One-level conv plaintexts (oracle circuits.conv_bsgs_diagonals): D_b = sum_c Mask_c (.) rot(K_c, chunk b),
// b < g, as QP plaintexts at q_l 2^pt_shift (level l); bias at the output scale (level l-1).
static void conv_bsgs_encode(he_context* c, const double* kernels, int C, int kh, int kw, const double* bias,
                             int chunk, int g, int pt_shift, int l, double in_scale, he_plaintext** dp,
                             he_plaintext** bp) {
  const int ns = c->N / 2, taps = kh * kw;
  need(kernels != nullptr, HE_INVALID_ARGUMENT, "null kernels");
  need(c->K > 0, HE_INVALID_PARAMS, "the one-level conv needs special primes (lazy ModDown)");
  need(l >= 1 && l < c->L, HE_LEVEL_EXHAUSTED, "the one-level conv consumes one level");
  need(C >= 1 && taps >= 1, HE_SHAPE_MISMATCH, "need at least one channel and tap");
  need(chunk >= 1 && (chunk & (chunk - 1)) == 0 && ns % chunk == 0, HE_LAYOUT_MISMATCH,
       "chunk must be a power of two dividing n_s");
  need((size_t)taps * chunk <= (size_t)ns, HE_LAYOUT_MISMATCH, "taps x chunk exceeds the slots");
  const int nch = ns / chunk;
  need(g >= 1 && g % C == 0 && nch % g == 0, HE_LAYOUT_MISMATCH,
       "g must be a multiple of C dividing n_s / chunk (Mask_c has period C chunks)");
  // slot s of D_b: only channel c = (s / chunk) mod C has Mask_c[s] = 1; rot(K_c, chunk b)[s] =
  // K_c[s + chunk b] = kernel_c[tap] with tap = (s / chunk + b) mod n_chunks when tap < taps
  std::vector<double> D((size_t)g * ns, 0.0);
  for (int b = 0; b < g; ++b)
    for (int s = 0; s < ns; ++s) {
      const int ch = (s / chunk) % C, tap = (s / chunk + b) % nch;
      if (tap < taps) D[(size_t)b * ns + s] = kernels[(size_t)ch * taps + tap];
    }
  PtGuard pd, pb;
  {
    DevDoubles d(c, D.data(), D.size());
    pd.p = encode(c, d.d, ns, g, shifted(c->hp.q[l], pt_shift), l, 1);
  }
  if (bias) {
    std::vector<double> bs(ns);
    for (int s = 0; s < ns; ++s) bs[s] = bias[(s / chunk) % C];
    DevDoubles d(c, bs.data(), bs.size());
    pb.p = encode(c, d.d, ns, 1, in_scale * pd.p->scale / (double)c->hp.q[l], l - 1);
  }
  *dp = pd.p;
  *bp = pb.p;
  pd.p = pb.p = nullptr;
}

he_status he_im2col_conv_bsgs_encode(he_context* c, const double* kernels, int C, int kh, int kw,
                                     const double* bias, int chunk, int g, int pt_shift, int level,
                                     double in_scale, he_plaintext** diags, he_plaintext** bias_pt) {
  return guard([&] {
    need_ctx(c);
    need(diags && bias_pt, HE_INVALID_ARGUMENT, "null output pointer");
    conv_bsgs_encode(c, kernels, C, kh, kw, bias, chunk, g, pt_shift, level, in_scale, diags, bias_pt);
  });
}

he_status he_im2col_conv_bsgs_pt(he_context* c, const he_ciphertext* ct, const he_plaintext* diags,
                                 const he_plaintext* bias, int chunk, int g, he_ciphertext** out) {
  return guard([&] {
    need_ctx(c); need_ct(c, ct); need_pt(c, diags); need_out(out);
    need(ct->size == 2, HE_SHAPE_MISMATCH, "conv needs a size-2 ciphertext");
    need(ct->level >= 1, HE_LEVEL_EXHAUSTED, "the one-level conv consumes one level");
    need(diags->qp, HE_INVALID_ARGUMENT, "diagonals must come from he_im2col_conv_bsgs_encode (QP form)");
    need(diags->level == ct->level, HE_LEVEL_MISMATCH, "diagonals must be at the ciphertext level");
    const int ns = c->N / 2;
    need(chunk >= 1 && (chunk & (chunk - 1)) == 0 && ns % chunk == 0, HE_LAYOUT_MISMATCH,
         "chunk must be a power of two dividing n_s");
    need(g >= 1 && diags->B == g && (ns / chunk) % g == 0, HE_SHAPE_MISMATCH, "need g diagonals, g | n_s / chunk");
    const int n2 = ns / chunk / g;
    for (int b = 1; b < g; ++b) {
      u32 gg;
      need(has_galois_key(c, chunk * b, &gg), HE_MISSING_GALOIS_KEY, "missing key for chunk * b");
    }
    for (int a = 1; a < n2; ++a) {
      u32 gg;
      need(has_galois_key(c, chunk * g * a, &gg), HE_MISSING_GALOIS_KEY, "missing key for chunk * g * a");
    }
    if (bias) {
      need_pt(c, bias);
      need_plain_q(bias);
      need(bias->B == 1, HE_SHAPE_MISMATCH, "bias is one plaintext");
      need(bias->level == ct->level - 1, HE_LEVEL_MISMATCH, "bias at the rescaled level");
      need(bias->scale == ct->scale * diags->scale / (double)c->hp.q[ct->level], HE_SCALE_MISMATCH,
           "bias scale must equal the output scale");
    }
    *out = ct_conv_bsgs(c, ct, diags, bias, chunk, g);
  });
}

he_status he_im2col_conv(he_context* c, const he_ciphertext* ct, const double* kernels, int C, int kh, int kw,
                         const double* bias, int chunk, int kernel_shift, int mask_shift, he_ciphertext** out) {
  return guard([&] {
    need_ctx(c); need_ct(c, ct); need_out(out);
    conv_checks(c, ct, C, kh * kw, chunk);
    for (int step = chunk; step < c->N / 2; step <<= 1) {
      u32 g;
      need(has_galois_key(c, step, &g), HE_MISSING_GALOIS_KEY, "missing Galois key for a fold step");
    }
    PtGuard pk, pm, pb;
    conv_encode(c, kernels, C, kh, kw, bias, chunk, kernel_shift, mask_shift, ct->level, ct->scale, &pk.p, &pm.p,
                &pb.p);
    *out = ct_conv(c, ct, pk.p, pm.p, pb.p, chunk);
  });
}

static void need_vm_fold_keys(he_context* c, const he_plaintext* diags) {
  for (int t = 1; t < diags->fold_n; ++t) {
    u32 gg;
    need(has_galois_key(c, diags->fold_step * t, &gg), HE_MISSING_GALOIS_KEY,
         "missing Galois key for a fold step m t");
  }
}

he_status he_vec_mat_pt(he_context* c, const he_ciphertext* ct, const he_plaintext* diags,
                        const he_plaintext* bias_pt, he_ciphertext** out) {
  return guard([&] {
    need_ctx(c); need_ct(c, ct); need_pt(c, diags); need_out(out);
    need(ct->size == 2, HE_SHAPE_MISMATCH, "vec_mat needs a size-2 ciphertext");
    need(ct->level >= 1, HE_LEVEL_EXHAUSTED, "vec_mat consumes one level");
    need(diags->level == ct->level, HE_LEVEL_MISMATCH, "diagonals must be at the ciphertext level");
    need(diags->B >= 1 && diags->B <= c->N / 2, HE_SHAPE_MISMATCH, "1 <= n <= n_s diagonals");
    need(!diags->qp || c->K > 0, HE_MISSING_KEY, "lazy ModDown needs special primes");
    if (bias_pt) {
      need_pt(c, bias_pt);
      need_plain_q(bias_pt);
      need(bias_pt->B == 1, HE_SHAPE_MISMATCH, "bias is one plaintext");
      need(bias_pt->level == ct->level - 1, HE_LEVEL_MISMATCH, "bias at the rescaled level");
      need(bias_pt->scale == ct->scale * diags->scale / (double)c->hp.q[ct->level], HE_SCALE_MISMATCH,
           "bias scale must equal the output scale");
    }
    need_vm_fold_keys(c, diags);
    *out = ct_vec_mat(c, ct, diags, bias_pt);
  });
}

static void vecmat_encode(he_context* c, const double* W, int n, int m, const double* bias, int replicate_out,
                          int pt_scale_shift, int l, double in_scale, he_plaintext** dp, he_plaintext** bp,
                          int qp = 0, int g = 0, bool fold = false) {
  need(W != nullptr, HE_INVALID_ARGUMENT, "null matrix");
  need(l >= 1 && l < c->L, HE_LEVEL_EXHAUSTED, "vec_mat consumes one level");
  const int ns = c->N / 2;
  std::vector<double> D = vecmat_diagonals(W, n, m, ns, replicate_out != 0);
  // folded form: D_{k + m t} = rot(D_k, m t) for replicated output, keep the first m diagonals
  const int nd = fold ? m : n;
  if (fold) D.resize((size_t)m * ns);
  int items = nd;
  if (g > 0) {   // BSGS order: E[k2][k1] = rot(D_{k1 + g k2}, -g k2), zero past nd
    const int n2 = (nd + g - 1) / g;
    std::vector<double> E((size_t)n2 * g * ns, 0.0);
    for (int k2 = 0; k2 < n2; ++k2)
      for (int k1 = 0; k1 < g; ++k1) {
        const int k = k1 + g * k2;
        if (k >= nd) continue;
        for (int j = 0; j < ns; ++j) E[((size_t)k2 * g + k1) * ns + (j + g * k2) % ns] = D[(size_t)k * ns + j];
      }
    D.swap(E);
    items = n2 * g;
  }
  PtGuard pd, pb;
  {
    DevDoubles d(c, D.data(), D.size());
    pd.p = encode(c, d.d, ns, items, shifted(c->hp.q[l], -pt_scale_shift), l, qp);
    pd.p->bsgs_g = g;
    if (fold) {
      pd.p->fold_n = n / m;
      pd.p->fold_step = m;
    }
  }
  if (bias) {
    std::vector<double> bs(ns, 0.0);
    for (int j = 0; j < ns; ++j)
      if (replicate_out) bs[j] = bias[j % m];
      else if (j < m) bs[j] = bias[j];
    const double s = in_scale * pd.p->scale / (double)c->hp.q[l];
    DevDoubles d(c, bs.data(), bs.size());
    pb.p = encode(c, d.d, ns, 1, s, l - 1);
  }
  *dp = pd.p;
  *bp = pb.p;
  pd.p = pb.p = nullptr;
}

he_status he_vec_mat_encode(he_context* c, const double* W, int n, int m, const double* bias, int replicate_out,
                            int pt_scale_shift, int level, double in_scale, he_plaintext** diags,
                            he_plaintext** bias_pt) {
  return guard([&] {
    need_ctx(c);
    need(diags && bias_pt, HE_INVALID_ARGUMENT, "null output pointer");
    vecmat_encode(c, W, n, m, bias, replicate_out, pt_scale_shift, level, in_scale, diags, bias_pt);
  });
}

he_status he_vec_mat_encode_lazy(he_context* c, const double* W, int n, int m, const double* bias,
                                 int replicate_out, int pt_scale_shift, int level, double in_scale,
                                 he_plaintext** diags, he_plaintext** bias_pt) {
  return guard([&] {
    need_ctx(c);
    need(diags && bias_pt, HE_INVALID_ARGUMENT, "null output pointer");
    need(c->K > 0, HE_INVALID_PARAMS, "lazy ModDown needs special primes");
    vecmat_encode(c, W, n, m, bias, replicate_out, pt_scale_shift, level, in_scale, diags, bias_pt, 1);
  });
}

he_status he_vec_mat_encode_bsgs(he_context* c, const double* W, int n, int m, const double* bias,
                                 int replicate_out, int pt_scale_shift, int level, double in_scale, int g,
                                 he_plaintext** diags, he_plaintext** bias_pt) {
  return guard([&] {
    need_ctx(c);
    need(diags && bias_pt, HE_INVALID_ARGUMENT, "null output pointer");
    need(c->K > 0, HE_INVALID_PARAMS, "lazy ModDown needs special primes");
    need(g >= 1 && g <= n && (n + g - 1) / g <= 4, HE_SHAPE_MISMATCH, "baby step g: 1 <= g <= n, at most 4 giant steps");
    vecmat_encode(c, W, n, m, bias, replicate_out, pt_scale_shift, level, in_scale, diags, bias_pt, 1, g);
  });
}

he_status he_vec_mat_encode_bsgs_fold(he_context* c, const double* W, int n, int m, const double* bias,
                                      int pt_scale_shift, int level, double in_scale, int g, he_plaintext** diags,
                                      he_plaintext** bias_pt) {
  return guard([&] {
    need_ctx(c);
    need(diags && bias_pt, HE_INVALID_ARGUMENT, "null output pointer");
    need(c->K > 0, HE_INVALID_PARAMS, "lazy ModDown needs special primes");
    need(n >= 1 && m >= 1 && n % m == 0, HE_SHAPE_MISMATCH, "folded vec_mat needs m | n");
    need(g >= 1 && m % g == 0 && m / g <= 4, HE_SHAPE_MISMATCH, "baby step g: g | m, at most 4 giant steps");
    vecmat_encode(c, W, n, m, bias, 1, pt_scale_shift, level, in_scale, diags, bias_pt, 1, g, true);
  });
}

static void vec_mat_bsgs_checks(he_context* c, const he_ciphertext* ct, const he_plaintext* diags, int g,
                                const he_plaintext* bias_pt) {
  {
    need_ctx(c); need_ct(c, ct); need_pt(c, diags);
    need(diags->qp && c->K > 0, HE_LAYOUT_MISMATCH, "BSGS needs QP diagonals");
    need(ct->size == 2 && ct->level >= 1, HE_LEVEL_EXHAUSTED, "vec_mat needs a size-2 ciphertext with a level");
    need(diags->level == ct->level, HE_LEVEL_MISMATCH, "diagonals must be at the ciphertext level");
    need(g >= 1 && diags->B % g == 0 && diags->B / g <= 4, HE_SHAPE_MISMATCH, "diags must be G <= 4 groups of g");
    if (bias_pt) {
      need_pt(c, bias_pt);
      need_plain_q(bias_pt);
      need(bias_pt->B == 1 && bias_pt->level == ct->level - 1, HE_LEVEL_MISMATCH, "bias at the rescaled level");
      need(bias_pt->scale == ct->scale * diags->scale / (double)c->hp.q[ct->level], HE_SCALE_MISMATCH,
           "bias scale must equal the output scale");
    }
  }
}

he_status he_vec_mat_bsgs_pt(he_context* c, const he_ciphertext* ct, const he_plaintext* diags, int g,
                             const he_plaintext* bias_pt, he_ciphertext** out) {
  return guard([&] {
    need_out(out);
    vec_mat_bsgs_checks(c, ct, diags, g, bias_pt);
    need_vm_fold_keys(c, diags);
    *out = ct_vec_mat_bsgs(c, ct, diags, g, bias_pt);
  });
}

he_status he_vec_mat_bsgs_fold_pt(he_context* c, const he_ciphertext* ct, const he_plaintext* diags, int g, int n,
                                  int m, const he_plaintext* bias_pt, he_ciphertext** out) {
  return guard([&] {
    need_out(out);
    vec_mat_bsgs_checks(c, ct, diags, g, bias_pt);
    need(m >= 1 && n >= m && n % m == 0 && diags->B == ((m + g - 1) / g) * g, HE_SHAPE_MISMATCH,
         "folded vec_mat: m | n and the diagonals hold the first m in BSGS order");
    for (int t = 1; t < n / m; ++t) {
      u32 gg;
      need(has_galois_key(c, m * t, &gg), HE_MISSING_GALOIS_KEY, "missing Galois key for a fold step m t");
    }
    *out = ct_vec_mat_bsgs(c, ct, diags, g, bias_pt, n / m, m);
  });
}

he_status he_vec_mat(he_context* c, const he_ciphertext* ct, const double* W, int n, int m, const double* bias,
                     int replicate_out, int pt_scale_shift, he_ciphertext** out) {
  return guard([&] {
    need_ctx(c); need_ct(c, ct); need_out(out);
    need(ct->size == 2, HE_SHAPE_MISMATCH, "vec_mat needs a size-2 ciphertext");
    need(ct->level >= 1, HE_LEVEL_EXHAUSTED, "vec_mat consumes one level");
    for (int k = 1; k < n; ++k) {
      u32 g;
      need(has_galois_key(c, k, &g), HE_MISSING_GALOIS_KEY, "missing Galois key for a diagonal rotation");
    }
    PtGuard pd, pb;
    vecmat_encode(c, W, n, m, bias, replicate_out, pt_scale_shift, ct->level, ct->scale, &pd.p, &pb.p);
    *out = ct_vec_mat(c, ct, pd.p, pb.p);
  });
}

// ------------------------------------------------------ handles / words ---
he_status he_free_plaintext(he_plaintext* pt) {
  return guard([&] { pt_free(pt); });
}
he_status he_free_ciphertext(he_ciphertext* ct) {
  return guard([&] { ct_free(ct); });
}

he_status he_ct_info(const he_ciphertext* ct, size_t* B, int* size, int* level, double* scale) {
  return guard([&] {
    need(ct != nullptr, HE_INVALID_ARGUMENT, "null ciphertext");
    if (B) *B = ct->B;
    if (size) *size = ct->size;
    if (level) *level = ct->level;
    if (scale) *scale = ct->scale;
  });
}

he_status he_pt_info(const he_plaintext* pt, size_t* B, int* level, double* scale) {
  return guard([&] {
    need(pt != nullptr, HE_INVALID_ARGUMENT, "null plaintext");
    if (B) *B = pt->B;
    if (level) *level = pt->level;
    if (scale) *scale = pt->scale;
  });
}

he_status he_ct_device_ptr(const he_ciphertext* ct, uint64_t** words) {
  return guard([&] {
    need(ct && words, HE_INVALID_ARGUMENT, "null argument");
    *words = ct->d;
  });
}

he_status he_pt_device_ptr(const he_plaintext* pt, uint64_t** words) {
  return guard([&] {
    need(pt && words, HE_INVALID_ARGUMENT, "null argument");
    *words = pt->d;
  });
}

static void copy_out(he_context* c, const u64* src, size_t words, uint64_t* dst, int on_device) {
  HE_CK(cudaMemcpyAsync(dst, src, words * 8, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                        c->stream));
  if (!on_device) HE_CK(cudaStreamSynchronize(c->stream));
}

he_status he_ct_export_words(he_context* c, const he_ciphertext* ct, uint64_t* dst, int on_device) {
  return guard([&] {
    need_ctx(c); need_ct(c, ct); need_out(dst);
    copy_out(c, ct->d, ct_words(ct), dst, on_device);
  });
}

he_status he_pt_export_words(he_context* c, const he_plaintext* pt, uint64_t* dst, int on_device) {
  return guard([&] {
    need_ctx(c); need_pt(c, pt); need_out(dst);
    copy_out(c, pt->d, pt_words(pt), dst, on_device);
  });
}

he_status he_ct_import_words(he_context* c, const uint64_t* src, int on_device, size_t B, int size, int level,
                             double scale, he_ciphertext** out) {
  return guard([&] {
    need_ctx(c); need_out(out);
    need(src != nullptr && B >= 1, HE_INVALID_ARGUMENT, "bad source");
    need(size == 2 || size == 3, HE_SHAPE_MISMATCH, "size must be 2 or 3");
    need(level >= 0 && level < c->L, HE_LEVEL_MISMATCH, "level out of range");
    he_ciphertext* ct = ct_new(c, (int)B, size, level, scale);
    try {
      HE_CK(cudaMemcpyAsync(ct->d, src, ct_words(ct) * 8,
                            on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->stream));
      need(!check_words(c, ct->d, B * size, level + 1), HE_INVALID_ARGUMENT, "word not reduced mod its prime");
    } catch (...) {
      ct_free(ct);
      throw;
    }
    *out = ct;
  });
}

he_status he_pt_import_words(he_context* c, const uint64_t* src, int on_device, size_t B, int level, double scale,
                             he_plaintext** out) {
  return guard([&] {
    need_ctx(c); need_out(out);
    need(src != nullptr && B >= 1, HE_INVALID_ARGUMENT, "bad source");
    need(level >= 0 && level < c->L, HE_LEVEL_MISMATCH, "level out of range");
    he_plaintext* pt = pt_new(c, (int)B, level, scale);
    try {
      HE_CK(cudaMemcpyAsync(pt->d, src, pt_words(pt) * 8,
                            on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->stream));
      need(!check_words(c, pt->d, B, level + 1), HE_INVALID_ARGUMENT, "word not reduced mod its prime");
    } catch (...) {
      pt_free(pt);
      throw;
    }
    *out = pt;
  });
}

he_status he_pt_from_int_coeffs(he_context* c, const int64_t* m, size_t B, double scale, int level,
                                he_plaintext** out) {
  return guard([&] {
    need_ctx(c); need_out(out);
    need(m != nullptr && B >= 1, HE_INVALID_ARGUMENT, "bad source");
    need(level >= 0 && level < c->L, HE_LEVEL_MISMATCH, "level out of range");
    Scratch d(c, B * c->N * 8);
    HE_CK(cudaMemcpyAsync(d.p, m, B * c->N * 8, cudaMemcpyHostToDevice, c->stream));
    *out = pt_from_int(c, d.as<i64>(), B, scale, level);
  });
}

he_status he_pt_to_int_coeffs(he_context* c, const he_plaintext* pt, int64_t* m) {
  return guard([&] {
    need_ctx(c); need_pt(c, pt); need_out(m);
    Scratch d(c, (size_t)pt->B * c->N * 8);
    pt_to_int(c, pt, d.as<i64>());
    HE_CK(cudaMemcpyAsync(m, d.p, (size_t)pt->B * c->N * 8, cudaMemcpyDeviceToHost, c->stream));
    HE_CK(cudaStreamSynchronize(c->stream));
  });
}

he_status he_pt_from_int_coeffs_qp(he_context* c, const int64_t* m, size_t B, double scale, int level,
                                   he_plaintext** out) {
  return guard([&] {
    need_ctx(c); need_out(out);
    need(m != nullptr && B >= 1, HE_INVALID_ARGUMENT, "bad source");
    need(level >= 0 && level < c->L, HE_LEVEL_MISMATCH, "level out of range");
    need(c->K > 0, HE_INVALID_PARAMS, "no special primes");
    Scratch d(c, B * c->N * 8);
    HE_CK(cudaMemcpyAsync(d.p, m, B * c->N * 8, cudaMemcpyHostToDevice, c->stream));
    *out = pt_from_int(c, d.as<i64>(), B, scale, level, 1);
  });
}

he_status he_pt_limbs(const he_plaintext* pt, int* limbs) {
  return guard([&] {
    need(pt && limbs, HE_INVALID_ARGUMENT, "null argument");
    *limbs = pt_limbs(pt);
  });
}

size_t he_key_bytes(const he_context* c) { return c ? key_bytes(const_cast<he_context*>(c)) : 0; }

size_t he_key_words(const he_context* c, int kind) {
  if (!c) return 0;
  const size_t N = c->N;
  switch (kind) {
    case 0: return (size_t)c->NP * N;
    case 1: return (size_t)2 * c->L * N;
    case 2:
    case 3: return (size_t)c->L * 2 * c->NP * N;
    default: return 0;
  }
}

he_status he_key_export(he_context* c, int kind, int32_t step, uint64_t* dst) {
  return guard([&] {
    need_ctx(c); need_out(dst);
    const u64* src = nullptr;
    switch (kind) {
      case 0: src = c->d_sk; break;
      case 1: src = c->d_pk; break;
      case 2: src = relin_key(c); break;
      case 3: {
        u32 g;
        src = galois_key(c, step, &g);
        need(src != nullptr, HE_MISSING_GALOIS_KEY, "no Galois key for that step");
        break;
      }
      default: throw HeError(HE_INVALID_ARGUMENT, "unknown key kind");
    }
    need(src != nullptr, HE_MISSING_KEY, "key not present");
    copy_out(c, src, he_key_words(c, kind), dst, 0);
  });
}

// ------------------------------------------------------------ wire format ---
namespace {
struct WireHeader {
  char magic[8];
  uint32_t log2N, B, size, level;
  double scale;
  uint64_t payload_bytes;
  uint32_t n_limbs;
  char pad[20];   // seeded form: u64 a_seed, u64 stream0, 4 zero bytes (unaligned: memcpy)
};
static_assert(sizeof(WireHeader) == 64, "wire header is 64 bytes");
const char kMagic[8] = {'H', 'E', 'C', 'K', 'K', 'S', '0', '1'};
const char kMagicSeeded[8] = {'H', 'E', 'C', 'K', 'K', 'S', 'S', '1'};

size_t limb_bytes(he_context* c, int level) {
  size_t b = 0;
  for (int i = 0; i <= level; ++i) b += (size_t)c->N * c->hp.kbits[i] / 8;
  return b;
}
}  // namespace

he_status he_ct_serialized_size(he_context* c, const he_ciphertext* ct, size_t* bytes) {
  return guard([&] {
    need_ctx(c); need_ct(c, ct); need_out(bytes);
    *bytes = sizeof(WireHeader) + wire_payload_bytes(c, ct);
  });
}

he_status he_ct_serialize(he_context* c, const he_ciphertext* ct, void* dst, int on_device) {
  return guard([&] {
    need_ctx(c); need_ct(c, ct); need_out(dst);
    WireHeader h;
    memset(&h, 0, sizeof(h));
    memcpy(h.magic, kMagic, 8);
    h.log2N = c->logN;
    h.B = ct->B;
    h.size = ct->size;
    h.level = ct->level;
    h.scale = ct->scale;
    h.payload_bytes = wire_payload_bytes(c, ct);
    h.n_limbs = ct->level + 1;
    char* d = (char*)dst;
    if (on_device) {
      HE_CK(cudaMemcpyAsync(d, &h, sizeof(h), cudaMemcpyHostToDevice, c->stream));
      wire_pack(c, ct, (u64*)(d + sizeof(h)));
    } else {
      memcpy(d, &h, sizeof(h));
      Scratch buf(c, h.payload_bytes);
      wire_pack(c, ct, buf.as<u64>());
      HE_CK(cudaMemcpyAsync(d + sizeof(h), buf.p, h.payload_bytes, cudaMemcpyDeviceToHost, c->stream));
      HE_CK(cudaStreamSynchronize(c->stream));
    }
  });
}

he_status he_ct_serialized_size_seeded(he_context* c, const he_ciphertext* ct, size_t* bytes) {
  return guard([&] {
    need_ctx(c); need_ct(c, ct); need_out(bytes);
    need(ct->seeded, HE_INVALID_ARGUMENT, "only fresh symmetric ciphertexts have a seeded form");
    *bytes = sizeof(WireHeader) + limb_bytes(c, ct->level) * ct->B;
  });
}

he_status he_ct_serialize_seeded(he_context* c, const he_ciphertext* ct, void* dst, int on_device) {
  return guard([&] {
    need_ctx(c); need_ct(c, ct); need_out(dst);
    need(ct->seeded, HE_INVALID_ARGUMENT, "only fresh symmetric ciphertexts have a seeded form");
    WireHeader h;
    memset(&h, 0, sizeof(h));
    memcpy(h.magic, kMagicSeeded, 8);
    h.log2N = c->logN;
    h.B = ct->B;
    h.size = 2;
    h.level = ct->level;
    h.scale = ct->scale;
    h.payload_bytes = limb_bytes(c, ct->level) * ct->B;
    h.n_limbs = ct->level + 1;
    memcpy(h.pad, &ct->a_seed, 8);
    memcpy(h.pad + 8, &ct->stream0, 8);
    // c0 of every item as a size-1 batch, packed like he_ct_serialize
    he_ciphertext* c0 = ct_new(c, ct->B, 1, ct->level, ct->scale);
    try {
      ct_copy_c0(c, ct, c0->d, false);
      char* d = (char*)dst;
      if (on_device) {
        HE_CK(cudaMemcpyAsync(d, &h, sizeof(h), cudaMemcpyHostToDevice, c->stream));
        wire_pack(c, c0, (u64*)(d + sizeof(h)));
        HE_CK(cudaStreamSynchronize(c->stream));   // h is on this stack frame
      } else {
        memcpy(d, &h, sizeof(h));
        Scratch buf(c, h.payload_bytes);
        wire_pack(c, c0, buf.as<u64>());
        HE_CK(cudaMemcpyAsync(d + sizeof(h), buf.p, h.payload_bytes, cudaMemcpyDeviceToHost, c->stream));
        HE_CK(cudaStreamSynchronize(c->stream));
      }
    } catch (...) {
      ct_free(c0);
      throw;
    }
    ct_free(c0);
  });
}

he_status he_ct_deserialize(he_context* c, const void* src, int on_device, size_t len, he_ciphertext** out) {
  return guard([&] {
    need_ctx(c); need_out(out);
    need(src != nullptr && len >= sizeof(WireHeader), HE_INVALID_ARGUMENT, "truncated wire data");
    WireHeader h;
    if (on_device) {
      HE_CK(cudaMemcpyAsync(&h, src, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
      HE_CK(cudaStreamSynchronize(c->stream));
    } else {
      memcpy(&h, src, sizeof(h));
    }
    const bool seeded = memcmp(h.magic, kMagicSeeded, 8) == 0;
    need(seeded || memcmp(h.magic, kMagic, 8) == 0, HE_INVALID_ARGUMENT, "bad wire magic");
    need((int)h.log2N == c->logN, HE_PARAM_MISMATCH, "ring degree differs from the context's");
    need(h.size == 2 || (!seeded && h.size == 3), HE_SHAPE_MISMATCH, "size must be 2 or 3 (seeded: 2)");
    need((int)h.level < c->L && h.n_limbs == h.level + 1 && h.B >= 1, HE_INVALID_ARGUMENT, "bad header");
    // payload length implied by the context's primes must match the header and the buffer
    const size_t expect = limb_bytes(c, (int)h.level) * h.B * (seeded ? 1 : h.size);
    need(expect == h.payload_bytes && len == sizeof(h) + expect, HE_INVALID_ARGUMENT, "wire length mismatch");
    const char* s = (const char*)src + sizeof(h);
    if (seeded) {   // payload = c0 of every item; c1 regenerated from (a_seed, stream0)
      u64 a_seed, stream0;
      memcpy(&a_seed, h.pad, 8);
      memcpy(&stream0, h.pad + 8, 8);
      Scratch buf(c, expect);
      if (on_device) HE_CK(cudaMemcpyAsync(buf.p, s, expect, cudaMemcpyDeviceToDevice, c->stream));
      else HE_CK(cudaMemcpyAsync(buf.p, s, expect, cudaMemcpyHostToDevice, c->stream));
      he_ciphertext* c0 = wire_unpack(c, buf.as<u64>(), h.B, 1, (int)h.level, h.scale);
      he_ciphertext* ct = nullptr;
      try {
        ct = ct_new(c, h.B, 2, (int)h.level, h.scale);
        ct->seeded = 1;
        ct->a_seed = a_seed;
        ct->stream0 = stream0;
        ct_copy_c0(c, ct, c0->d, true);
        sym_regen_c1(c, ct);
      } catch (...) {
        ct_free(c0);
        ct_free(ct);
        throw;
      }
      ct_free(c0);
      *out = ct;
      return;
    }
    if (on_device) {
      *out = wire_unpack(c, (const u64*)s, h.B, (int)h.size, (int)h.level, h.scale);
    } else {
      Scratch buf(c, expect);
      HE_CK(cudaMemcpyAsync(buf.p, s, expect, cudaMemcpyHostToDevice, c->stream));
      *out = wire_unpack(c, buf.as<u64>(), h.B, (int)h.size, (int)h.level, h.scale);
    }
  });
}

// ------------------------------------------------------------ ring prims ---
static void ring_checks(he_context* c, const void* p, size_t B, int nl) {
  need_ctx(c);
  need(p != nullptr, HE_INVALID_ARGUMENT, "null buffer");
  need(B >= 1 && nl >= 1 && nl <= c->NP, HE_SHAPE_MISMATCH, "bad batch / limb count");
  need(B * nl < (1u << 31), HE_SHAPE_MISMATCH, "too many limbs in one call");
}

he_status he_ntt_forward(he_context* c, uint64_t* d, size_t B, int nl) {
  return guard([&] {
    ring_checks(c, d, B, nl);
    ntt_rows(c, d, d, B, nl, (size_t)nl * c->N, (size_t)nl * c->N, false);
  });
}

he_status he_ntt_inverse(he_context* c, uint64_t* d, size_t B, int nl) {
  return guard([&] {
    ring_checks(c, d, B, nl);
    ntt_rows(c, d, d, B, nl, (size_t)nl * c->N, (size_t)nl * c->N, true);
  });
}

he_status he_modmul(he_context* c, const uint64_t* a, const uint64_t* b, uint64_t* out, size_t B, int nl) {
  return guard([&] {
    ring_checks(c, a, B, nl);
    need(b && out, HE_INVALID_ARGUMENT, "null buffer");
    modmul_rows(c, a, b, out, B, nl);
  });
}

he_status he_ntt_mul_intt(he_context* c, const uint64_t* a, const uint64_t* b, uint64_t* out, size_t B, int nl) {
  return guard([&] {
    ring_checks(c, a, B, nl);
    need(b && out, HE_INVALID_ARGUMENT, "null buffer");
    ring_mul(c, a, b, out, B, nl);
  });
}

}  // extern "C"
