/*
 * he_ckks.h — C-ABI boundary of the B200 CKKS hot path (arXiv 2104.03152,
 * "TenSEAL: A Library for Encrypted Tensor Operations Using Homomorphic
 * Encryption").
 *
 * The paper's encrypted-inference method evaluates CKKSVector operations
 * on top of the CKKS scheme it takes from SEAL
 * ("relies on the implementation of the CKKS scheme").  This
 * header exposes exactly the calls of SURVEY.md §8(b): context/keygen
 * (PAPER.md:35), encode/encrypt, the op catalogue
 * (add, sub, negate, add_plain, mul_plain, mul, square),
 * rotation, relinearize/rescale ("automatic
 * relinearization and rescaling"), the im2col convolution (PAPER.md:57, 64,
 * 189-213) and the vector-plain-matrix product, decrypt /
 * decode; plus word import/export used by the parity tests.
 *
 * Every arithmetic step behind these calls runs in the library's own sm_100a
 * kernels (paper_2104_03152_b200/csrc).  There is no CPU fallback: a call that
 * needs the GPU and has none returns HE_CUDA_ERROR.
 *
 * Conventions (DESIGN.md §3 = SURVEY.md §8(c) C1-C20):
 *   - N = 2^log2N, slots n_s = N/2.  Data primes q_0..q_{L-1}, special primes
 *     p_0..p_{K-1} (the last K entries of he_params.bits), one uint64 word per
 *     residue.  Prime selection C2, primitive root C4.
 *   - A ciphertext handle is a BATCH of B ciphertexts sharing one level l,
 *     scale (double) and size (2 or 3).  Device layout, limb-major:
 *         words[b][poly][limb][n],  limb in 0..l, n in 0..N-1,
 *     always in the NTT (evaluation) domain, bit-reversed order C5:
 *         NTT(a)[j] = sum_i a_i psi^{(2 brv(j)+1) i}  (mod q_limb).
 *     Plaintexts are words[b][limb][n] in the same domain.
 *   - Rotation by k > 0 is a LEFT rotation of the slots, Galois
 *     element 5^k mod 2N; k < 0 uses 5^{n_s+k} (C6).
 *   - Hybrid key switching with one data prime per digit (dnum = L, C12),
 *     centered digit lift (C16), rounding DivRound (C15).
 *
 * Ownership: every handle is created by the library and released by the
 * caller with the matching he_free_* call.  Device memory is allocated
 * stream-ordered on the context's stream (cudaMallocAsync pool); calls are
 * asynchronous on that stream unless they read or write host memory, which
 * they do synchronously (they return after the host buffer is consumed /
 * filled).  Every operation is pure: it returns a fresh output handle and
 * never modifies its inputs.
 *
 * Errors: every function returns he_status (0 = HE_OK).  On failure nothing
 * is written to the output pointers and he_last_error() returns a
 * thread-local message.  No C++ exception crosses this boundary.
 *
 * Threads: a context (and the handles made from it) is used by one host thread
 * at a time; distinct contexts are independent.
 */
#ifndef HE_CKKS_H_
#define HE_CKKS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: SPEC taxonomy mapped by SURVEY.md §8(b). */
typedef int he_status;
enum {
  HE_OK = 0,
  HE_INVALID_PARAMS = 1,        /* bad he_params */
  HE_PARAM_MISMATCH = 2,        /* operands from different contexts */
  HE_DOMAIN_MISMATCH = 3,       /* reserved: all handles are NTT-domain */
  HE_LEVEL_MISMATCH = 4,        /* operand levels differ */
  HE_SCALE_MISMATCH = 5,        /* additive operands' scales differ bitwise */
  HE_LEVEL_EXHAUSTED = 6,       /* rescale at level 0 */
  HE_SCALE_OVERFLOW = 7,        /* |scale * z| >= 2^62 in encode */
  HE_MISSING_KEY = 8,           /* secret / relin key absent */
  HE_MISSING_GALOIS_KEY = 9,    /* rotation step without a key */
  HE_INVALID_ROTATION = 10,     /* step 0 or |step| >= n_s at keygen */
  HE_TOO_MANY_VALUES = 11,      /* more than n_s values to encode */
  HE_SHAPE_MISMATCH = 12,       /* batch sizes / ciphertext sizes disagree */
  HE_LAYOUT_MISMATCH = 13,      /* im2col geometry does not fit the slots */
  HE_REPLICATION_EXHAUSTED = 14,/* vec_mat diagonal reads past the replicated span */
  HE_CUDA_ERROR = 15,           /* a CUDA call failed (includes: no GPU present) */
  HE_OUT_OF_MEMORY = 16,        /* device allocation failed */
  HE_INVALID_ARGUMENT = 17      /* null pointer, bad size, etc. */
};

typedef struct he_context he_context;
typedef struct he_plaintext he_plaintext;
typedef struct he_ciphertext he_ciphertext;
typedef struct he_graph he_graph;

/* Parameters (SURVEY.md §8(b) "Context/keys").
 *   log2N      ring degree exponent, 10..15 (N = 1024..32768).
 *   n_primes   total number of primes L + K (<= 64).
 *   bits       n_primes prime bit sizes in [20, 60]; the LAST n_special are
 *              the special key-switching primes (C1: SEAL convention,
 *              PAPER.md:32).  Primes are chosen by rule C2.
 *   n_special  K in 0..2 (K = 0 disables key switching).
 *   scale_log2 informational default scale (encode takes an explicit scale).
 *   dnum       number of key-switching digits; must equal L or 0 (= L), C12. */
typedef struct he_params {
  int log2N;
  int n_primes;
  const int* bits;
  int n_special;
  double scale_log2;
  int dnum;
} he_params;

/* Last error message of the calling thread ("" if none). */
const char* he_last_error(void);

/* Create a context: prime search (C2), psi (C4), NTT twiddles with Shoup
 * companions, RNS constants, CDT table (C11), all uploaded once.  `seed` is
 * the Philox key of every draw the context makes (C9).  Fails with
 * HE_CUDA_ERROR when no CUDA device is usable. */
he_status he_context_create(const he_params* params, uint64_t seed, he_context** out);
he_status he_context_free(he_context* ctx);

/* Read back log2N, L (data primes), K (special primes). */
he_status he_context_info(const he_context* ctx, int* log2N, int* L, int* K);
/* Copy the L+K primes (data first, specials last) / psi values to host. */
he_status he_context_primes(const he_context* ctx, uint64_t* primes_out, uint64_t* psi_out);
/* Copy the C11 CDT table (20 words) to host. */
he_status he_context_cdt(const he_context* ctx, uint64_t* table_out);

/* Make all subsequent calls on ctx run on `stream` (a cudaStream_t, e.g. a
 * torch.cuda.Stream's cuda_stream).  NULL selects the legacy default stream. */
he_status he_set_stream(he_context* ctx, void* stream);
/* (Switching streams first synchronizes the old one: the context caches freed device
 * scratch blocks by size and hands them to later work in stream order.) */
/* Block until all work queued on the context's stream is done; reports (and
 * clears) an asynchronous he_encode_device overflow as HE_SCALE_OVERFLOW. */
he_status he_sync(he_context* ctx);

/* Device memory from the caller (SURVEY.md §8(b) "Creation/ownership": torch's
 * caching allocator in the Python binding).  After this call every ciphertext,
 * plaintext and scratch block of ctx is obtained as alloc(bytes, stream, user)
 * and returned as free(ptr, bytes, stream, user), where stream is the
 * context's cudaStream_t: a block freed on that stream may be reused by work
 * queued later on it (stream-ordered semantics, as torch's allocator gives).
 * alloc returns NULL on failure (-> HE_OUT_OF_MEMORY).  The context's cached
 * internal blocks are released first (synchronizes the stream).  Blocks that
 * were obtained before the call keep their origin and are returned to it.  The
 * parameter tables and keys stay library-owned (cudaMalloc at creation and
 * he_keygen).  alloc = free = NULL restores the internal pool. */
typedef void* (*he_alloc_fn)(size_t bytes, void* stream, void* user);
typedef void (*he_free_fn)(void* ptr, size_t bytes, void* stream, void* user);
he_status he_set_allocator(he_context* ctx, he_alloc_fn alloc, he_free_fn free, void* user);

/* Key generation on the device: ternary
 * secret s, public key (-a s + e, a) over the data limbs, relinearisation key
 * for s^2 and one Galois key per distinct element of `rot_steps` (each step
 * nonzero with |step| <= n_s; k = n_s gives the identity element, kept as a
 * real key per C20).  May be called once per context. */
he_status he_keygen(he_context* ctx, const int32_t* rot_steps, size_t n_steps);
/* Drop the secret key (the "public" context of S:311-318): decrypt then fails
 * with HE_MISSING_KEY. */
he_status he_drop_secret_key(he_context* ctx);
/* The "public" context a client hands to the server (PAPER.md:32,
 * 35): a NEW context with the same parameters and seed and device copies of
 * the public, relinearisation and Galois keys, without the secret key (decrypt
 * and symmetric encryption fail with HE_MISSING_KEY).  Free it with
 * he_context_free; ctx is unchanged.  The copy runs on ctx's stream. */
he_status he_make_public(he_context* ctx, he_context** out);

/* ---- encode / decode (C6/C7) -------------------------- */
/* Encode B real vectors of n_per_item <= n_s values each (host array
 * z[B][n_per_item], row-major) at `scale`, into a plaintext at `level`:
 * m_i = round_half_away(scale (2/N) Re sum_j z_j zeta^{-i 5^j}), reduced into
 * limbs 0..level and NTT'd.  Canonical-embedding IFFT in float64 on device. */
he_status he_encode(he_context* ctx, const double* z, size_t n_per_item, size_t B, double scale,
                    int level, he_plaintext** out);
/* (he_encode) The C7 bound is checked on the host before any work is queued:
 * HE_SCALE_OVERFLOW when scale (2/N) sum_j |z_j| >= 2^62 (1 - 2^-20) for some
 * item, or a value is not finite; the bound dominates every |m_i|, so no
 * device readback is needed and the call returns after enqueuing the H2D copy
 * and the encode kernels on the context's stream.  z is read by that copy:
 * pageable memory may be reused when the call returns; page-locked memory
 * (cudaHostAlloc, torch pin_memory) must stay unchanged until the stream has
 * passed the call (he_sync, or an event recorded on the stream).
 * Inputs of 1 MiB or more (a batch of slot vectors; he_encode and
 * he_encode_encrypt) are copied on a copy stream of the context's own into one
 * of two context-owned device buffers, and the context's stream waits for the
 * copy: in a pipelined client loop the upload of batch i+1 then overlaps the
 * kernels of batch i instead of queueing behind them.  Ordering as seen from
 * the context's stream is unchanged.  Smaller inputs, and calls recorded into
 * a CUDA graph, are copied on the context's stream itself. */
/* Same, with z already in device memory, and ASYNCHRONOUS: it only enqueues
 * work on the context's stream (a server pipeline never drains the device at
 * an encode).  A |scale z| >= 2^62 overflow is then reported as
 * HE_SCALE_OVERFLOW by the next he_sync or host-output he_decode on this
 * context (the affected plaintext is undefined); the other argument checks
 * still fail here. */
he_status he_encode_device(he_context* ctx, const double* z_dev, size_t n_per_item, size_t B,
                           double scale, int level, he_plaintext** out);
/* The float64 values he_encode rounds (a parity hook for C7: the canonical-
 * embedding IFFT's output before round_half_away), for host z[B][n_per_item]:
 * out[B][N] (host), out[b][i] = scale (2/N) Re(...) for i < N/2 and the
 * imaginary parts for i >= N/2, in the coefficient order of m.  Synchronous.
 * Same argument checks as he_encode except the 2^62 bound (values are
 * returned, not rounded). */
he_status he_encode_unrounded(he_context* ctx, const double* z, size_t n_per_item, size_t B, double scale,
                              double* out);
/* Decode the first n slots of every item into host out[B][n]: CRT compose,
 * centre, float64, FFT, divide by the plaintext's scale (C6). */
he_status he_decode(he_context* ctx, const he_plaintext* pt, double* out, size_t n);
/* Same, ASYNCHRONOUS: enqueues the decode and the device-to-host copy into
 * host out[B][n] on the context's stream and returns.  out is valid once the
 * stream has passed the call (he_sync, or an event recorded on the stream);
 * with page-locked out the copy overlaps later work (the e2e pipeline of
 * bench.py).  A pending he_encode_device overflow is reported by he_sync. */
he_status he_decode_async(he_context* ctx, const he_plaintext* pt, double* out, size_t n);
/* Same, writing device memory out_dev[B][n]. */
he_status he_decode_device(he_context* ctx, const he_plaintext* pt, double* out_dev, size_t n);

/* ---- encrypt / decrypt (C13) ----------------------------- */
/* Public-key encryption of every item of pt; item b draws its randomness
 * (v, e0, e1) from Philox stream `stream_id + b`.  Output scale/level = pt's. */
he_status he_encrypt(he_context* ctx, const he_plaintext* pt, uint64_t stream_id,
                     he_ciphertext** out);
/* Encode + public-key encryption in one call (a CKKSVector's creation,
 * PAPER.md:35, 57): the ciphertext words equal
 * he_encrypt(he_encode(z, scale, level), stream_id) exactly; the encoder's
 * integer coefficients m feed the transform of e0 (c0 = NTT(v) b + NTT(e0 + m),
 * the transform being linear mod q_i), so the plaintext's own transforms and
 * its HBM round trip are skipped.  Host z[B][n_per_item] with he_encode's
 * host-side C7 bound check and copy semantics; the _device form reads z_dev
 * and reports an overflow asynchronously like he_encode_device. */
he_status he_encode_encrypt(he_context* ctx, const double* z, size_t n_per_item, size_t B, double scale,
                            int level, uint64_t stream_id, he_ciphertext** out);
he_status he_encode_encrypt_device(he_context* ctx, const double* z_dev, size_t n_per_item, size_t B,
                                   double scale, int level, uint64_t stream_id, he_ciphertext** out);
/* Symmetric (secret-key) encryption (SURVEY 8(f) #3 "seeded symmetric
 * encryption halves the upload"): item b gets
 *   c1 = a,  a_i = Uniform(a_seed, stream (SYM_A, stream_id + b, i))   (C13 sampler)
 *   c0 = -a s + e + m,  e = CDT(context seed, stream (SYM_E, stream_id + b, 0))   (C11)
 * a_seed is PUBLIC (it travels in the seeded wire form; it must not be the
 * context seed, which also derives the secret key).  The result is marked
 * seeded: he_ct_serialize_seeded can omit c1.  Needs the secret key
 * (HE_MISSING_KEY).  Output scale/level = pt's. */
he_status he_encrypt_symmetric(he_context* ctx, const he_plaintext* pt, uint64_t stream_id, uint64_t a_seed,
                               he_ciphertext** out);
/* m = c0 + c1 s (+ c2 s^2).  Needs the secret key. */
he_status he_decrypt(he_context* ctx, const he_ciphertext* ct, he_plaintext** out);

/* ---- arithmetic ------------- */
/* Binary ops require equal level, equal size and (for add/sub) bitwise-equal
 * scale; B must match, or one side may have B = 1 (broadcast). */
he_status he_add(he_context* ctx, const he_ciphertext* a, const he_ciphertext* b, he_ciphertext** out);
he_status he_sub(he_context* ctx, const he_ciphertext* a, const he_ciphertext* b, he_ciphertext** out);
he_status he_negate(he_context* ctx, const he_ciphertext* a, he_ciphertext** out);
/* add_plain: level and scale must match the ciphertext's. */
he_status he_add_plain(he_context* ctx, const he_ciphertext* a, const he_plaintext* p, he_ciphertext** out);
/* mul_plain: level must match; output scale = scale_ct * scale_pt; no rescale (C14). */
he_status he_mul_plain(he_context* ctx, const he_ciphertext* a, const he_plaintext* p, he_ciphertext** out);
/* mul: tensor product, size-3 output, no relinearisation. */
he_status he_mul(he_context* ctx, const he_ciphertext* a, const he_ciphertext* b, he_ciphertext** out);
/* square = tensor(a, a) -> relinearize -> rescale (C14). */
he_status he_square(he_context* ctx, const he_ciphertext* a, he_ciphertext** out);
/* relinearize a size-3 ciphertext with the s^2 key. */
he_status he_relinearize(he_context* ctx, const he_ciphertext* a, he_ciphertext** out);
/* rescale: exact round(X / q_l) on every limb, level l -> l-1, scale / q_l (C15). */
he_status he_rescale(he_context* ctx, const he_ciphertext* a, he_ciphertext** out);
/* rotate left by k (Galois automorphism 5^k + key switch). */
he_status he_rotate(he_context* ctx, const he_ciphertext* a, int32_t k, he_ciphertext** out);

/* In-place forms for the hot loop: a <- op(a, ...), same
 * checks and results as the forms above.  add / sub / add_plain / mul_plain
 * write into a's storage (no allocation) when a's batch is the larger one;
 * rescale / rotate / square change the limb layout, so a's storage is
 * replaced (its old block returns to the pool in stream order).  On error a is
 * unchanged. */
he_status he_add_inplace(he_context* ctx, he_ciphertext* a, const he_ciphertext* b);
he_status he_sub_inplace(he_context* ctx, he_ciphertext* a, const he_ciphertext* b);
he_status he_add_plain_inplace(he_context* ctx, he_ciphertext* a, const he_plaintext* p);
he_status he_mul_plain_inplace(he_context* ctx, he_ciphertext* a, const he_plaintext* p);
he_status he_rescale_inplace(he_context* ctx, he_ciphertext* a);
he_status he_rotate_inplace(he_context* ctx, he_ciphertext* a, int32_t k);
he_status he_square_inplace(he_context* ctx, he_ciphertext* a);

/* Drop limbs above `level` (level <= ct level): the ciphertext mod Q_level
 * decrypts to the same message; scale unchanged.  Used to align levels. */
he_status he_mod_switch_to(he_context* ctx, const he_ciphertext* a, int level, he_ciphertext** out);

/* ---- composite ops ----------------------------------- */
/* Encrypted dot product (Table 5 "dot"): mul (at the lower
 * level) -> relinearize -> rescale, then rotate-and-add by 1, 2, 4, ... < n:
 * slot 0 holds sum_{i<n} a_i b_i (slots >= n must be zero).  Needs Galois keys
 * for the powers of two below n. */
he_status he_dot(he_context* ctx, const he_ciphertext* a, const he_ciphertext* b, int n, he_ciphertext** out);
/* Encrypted x plain dot product (Table 5 "dot_plain"): z[n_s] encoded at q_l,
 * mul_plain, rescale, the same rotate-and-add. */
he_status he_dot_plain(he_context* ctx, const he_ciphertext* a, const double* z, size_t nz, int n,
                       he_ciphertext** out);
/* x^p with depth ceil(log2 p) (PAPER.md:58 "depth-optimal", :166): squares for
 * x^(2^k), x^i = x^(2^k) x^(i-2^k) otherwise. */
he_status he_power(he_context* ctx, const he_ciphertext* x, int p, he_ciphertext** out);
/* sum_{i<=d} coeffs[i] x^i (Table 4 "polyval"); every term is
 * formed at the level of x^d and rescaled once; the terms' tracked scales agree
 * up to double rounding and are summed at the first term's scale. */
he_status he_polyval(he_context* ctx, const he_ciphertext* x, const double* coeffs, int n_coeffs,
                     he_ciphertext** out);

/* Client-side im2col + vertical scan (C18), host only, float64: image
 * img[H][W] -> slots[n_s] with slot = tap * chunk + window, chunk = next
 * power of two >= #windows.  Writes *windows / *chunk if non-NULL. */
he_status he_im2col_encode(const double* img, int H, int W, int kh, int kw, int stride,
                           size_t n_slots, double* slots_out, int* windows, int* chunk);
/* Batched form: imgs[B][H][W] -> slots_out[B][n_slots] (host, float64). */
he_status he_im2col_encode_batch(const double* imgs, size_t B, int H, int W, int kh, int kw, int stride,
                                 size_t n_slots, double* slots_out);
/* im2col convolution on the encrypted side (C18/C19): for every output
 * channel c: t_c = rescale(ct * K_c); log2(n_s/chunk) rounds t_c += rot(t_c,
 * chunk 2^r); then sum_c t_c * Mask_c, rescale, + bias.  kernels[C][kh*kw],
 * bias[C] (may be NULL).  Kernel plaintexts are encoded at scale
 * q_l * 2^kernel_shift, masks at q_{l-1} * 2^mask_shift.  Consumes 2 levels. */
he_status he_im2col_conv(he_context* ctx, const he_ciphertext* ct, const double* kernels,
                         int n_channels, int kh, int kw, const double* bias, int chunk,
                         int kernel_shift, int mask_shift, he_ciphertext** out);
/* Encrypted vector x plain matrix W[n][m] (in x out, row-major) by the
 * diagonal method (C17): y = sum_{k<n} rot(x, k) * D_k, one
 * rescale, + bias[m] (may be NULL).  The input must hold x replicated with
 * period n.  replicate_out != 0 makes D_k periodic in m (output replicated
 * with period m; needs n | n_s and m | n_s).  Diagonals are encoded at scale
 * q_l * 2^(-pt_scale_shift).  Consumes 1 level; n-1 rotations, hoisted. */
he_status he_vec_mat(he_context* ctx, const he_ciphertext* ct, const double* W, int n, int m,
                     const double* bias, int replicate_out, int pt_scale_shift, he_ciphertext** out);
/* Same with pre-encoded diagonals: diags is a plaintext batch of n items
 * (item k = D_k) at the ciphertext's level; bias_pt (may be NULL) at the
 * rescaled level and scale.  Used to inject oracle plaintexts (C7). */
he_status he_vec_mat_pt(he_context* ctx, const he_ciphertext* ct, const he_plaintext* diags,
                        const he_plaintext* bias_pt, he_ciphertext** out);
/* Same as he_im2col_conv with pre-encoded plaintexts: kernels (C items at
 * the input level), masks (C items at level-1), bias_pt (may be NULL). */
he_status he_im2col_conv_pt(he_context* ctx, const he_ciphertext* ct, const he_plaintext* kernels,
                            const he_plaintext* masks, const he_plaintext* bias_pt, int chunk,
                            he_ciphertext** out);

/* Same with the fold computed as two hoisted lazy-ModDown rotation sums:
 * u = sum_{b<n1} rot(t, chunk b), then sum_{a<n2} rot(u, chunk n1 a), n1 n2 =
 * n_s / chunk (the same sum as the log2 fold, rounded once per level; oracle
 * circuits.hoisted_fold).  Needs keys for chunk b and chunk n1 a. */
he_status he_im2col_conv_hoisted_pt(he_context* ctx, const he_ciphertext* ct, const he_plaintext* kernels,
                                    const he_plaintext* masks, const he_plaintext* bias_pt, int chunk, int n1,
                                    he_ciphertext** out);
/* One-level im2col conv (DESIGN.md §3 "conv as a baby-step/giant-step product";
 * oracle circuits.im2col_conv_bsgs).  The paper's conv (C18/C19)
 * is out = sum_c Mask_c (.) sum_{m < n_chunks} rot(ct (.) K_c, chunk m) + bias.
 * Slot products commute with rotations of both factors and Mask_c has period
 * C chunks, so with m = b + g a (C | g, g | n_chunks):
 *   out = sum_{a < n2} rot(v, chunk g a) + bias,  v = sum_{b < g} D_b (.) rot(ct, chunk b),
 *   D_b = sum_c Mask_c (.) rot(K_c, chunk b).
 * he_im2col_conv_bsgs_encode: kernels [C][kh][kw] row-major float64, bias [C]
 * (may be NULL); *diags = g QP plaintexts D_b at scale q_level 2^pt_shift,
 * *bias_pt at level-1 and the output scale in_scale * diags.scale / q_level.
 * he_im2col_conv_bsgs_pt: v by one lazy ModDown over the g baby steps, one
 * rescale, the n2 giant steps as one hoisted unit-diagonal rotation sum, +
 * bias.  Consumes ONE level (the paper's form consumes two).  Needs Galois
 * keys for chunk b (b < g) and chunk g a (a < n2); errors as he_vec_mat_pt,
 * HE_LAYOUT_MISMATCH if C does not divide g or g does not divide n_s / chunk. */
he_status he_im2col_conv_bsgs_encode(he_context* ctx, const double* kernels, int C, int kh, int kw,
                                     const double* bias, int chunk, int g, int pt_shift, int level,
                                     double in_scale, he_plaintext** diags, he_plaintext** bias_pt);
he_status he_im2col_conv_bsgs_pt(he_context* ctx, const he_ciphertext* ct, const he_plaintext* diags,
                                 const he_plaintext* bias_pt, int chunk, int g, he_ciphertext** out);
/* Encode-once forms of the two composite ops' plaintexts (weights stay
 * resident on the device across batches; PAPER.md:98 excludes weight
 * preparation from the timed forward).  `level` / `in_scale` describe the
 * ciphertext the op will be applied to.  vec_mat: *diags = n items at
 * `level`, *bias_pt (NULL if bias is NULL) at level-1 and the output scale.
 * conv: *kernels_pt = C items at `level`, *masks_pt = C items at level-1,
 * *bias_pt at level-2 and the output scale. */
he_status he_vec_mat_encode(he_context* ctx, const double* W, int n, int m, const double* bias,
                            int replicate_out, int pt_scale_shift, int level, double in_scale,
                            he_plaintext** diags, he_plaintext** bias_pt);
/* Lazy-ModDown form of he_vec_mat_encode: the n diagonals also carry the K
 * special limbs (a "QP" plaintext), and he_vec_mat_pt given such diagonals
 * sums every rotation's key-switch inner product, weighted by its diagonal, in
 * the extended basis Q_l P and applies ONE ModDown (DESIGN.md §3/§5; the
 * oracle's vec_mat_lazy).  Same scales, bias and level use as he_vec_mat_encode. */
he_status he_vec_mat_encode_lazy(he_context* ctx, const double* W, int n, int m, const double* bias,
                                 int replicate_out, int pt_scale_shift, int level, double in_scale,
                                 he_plaintext** diags, he_plaintext** bias_pt);
/* Baby-step/giant-step form: the QP diagonals are emitted in
 * the order E[k2][k1] = rot(D_{k1 + g k2}, -g k2) (zero past n), G = ceil(n/g)
 * <= 4 groups of g; he_vec_mat_pt (or he_vec_mat_bsgs_pt) then computes the
 * inner product of each baby step rot(x, k1), k1 < g, once for all groups
 * (one lazy ModDown per group) and adds rot(inner_k2, g k2) (oracle
 * vec_mat_bsgs).  Needs Galois keys for 1..g-1 and g, 2g, ... */
he_status he_vec_mat_encode_bsgs(he_context* ctx, const double* W, int n, int m, const double* bias,
                                 int replicate_out, int pt_scale_shift, int level, double in_scale, int g,
                                 he_plaintext** diags, he_plaintext** bias_pt);
he_status he_vec_mat_bsgs_pt(he_context* ctx, const he_ciphertext* ct, const he_plaintext* diags, int g,
                             const he_plaintext* bias_pt, he_ciphertext** out);
/* Folded baby-step/giant-step form for a replicated output (C17) with m | n
 * (oracle vec_mat_bsgs_fold; the rectangular "hybrid" diagonal method): the
 * replicated-output diagonals satisfy D_{k + m t} = rot(D_k, m t), so only the
 * first m diagonals are encoded (BSGS order, g | m, m/g <= 4 groups), and
 * he_vec_mat_pt / he_vec_mat_bsgs_pt finish the n-term sum with
 * sum_{t < n/m} rot(., m t) as one hoisted rotation sum before the rescale.
 * Needs Galois keys for 1..g-1, g k2 (k2 < m/g) and m t (t < n/m).  Same
 * scales, bias and level use as he_vec_mat_encode with replicate_out = 1. */
he_status he_vec_mat_encode_bsgs_fold(he_context* ctx, const double* W, int n, int m, const double* bias,
                                      int pt_scale_shift, int level, double in_scale, int g,
                                      he_plaintext** diags, he_plaintext** bias_pt);
/* The folded evaluation with the shape given explicitly (diags = the first m
 * diagonals in BSGS order, e.g. injected with he_pt_from_int_coeffs_qp). */
he_status he_vec_mat_bsgs_fold_pt(he_context* ctx, const he_ciphertext* ct, const he_plaintext* diags, int g,
                                  int n, int m, const he_plaintext* bias_pt, he_ciphertext** out);
he_status he_im2col_conv_encode(he_context* ctx, const double* kernels, int n_channels, int kh, int kw,
                                const double* bias, int chunk, int kernel_shift, int mask_shift,
                                int level, double in_scale, he_plaintext** kernels_pt,
                                he_plaintext** masks_pt, he_plaintext** bias_pt);

/* ---- handles, import / export (test injection; not in the paper) ------ */
he_status he_free_plaintext(he_plaintext* pt);
he_status he_free_ciphertext(he_ciphertext* ct);
he_status he_ct_info(const he_ciphertext* ct, size_t* B, int* size, int* level, double* scale);
he_status he_pt_info(const he_plaintext* pt, size_t* B, int* level, double* scale);
/* Device pointer of the words [B][size][level+1][N] (contiguous). */
he_status he_ct_device_ptr(const he_ciphertext* ct, uint64_t** words);
he_status he_pt_device_ptr(const he_plaintext* pt, uint64_t** words);
/* Copy words between host (or device when `on_device` != 0) memory and a
 * handle.  Import checks every word is < its prime (else HE_INVALID_ARGUMENT). */
he_status he_ct_export_words(he_context* ctx, const he_ciphertext* ct, uint64_t* dst, int on_device);
he_status he_ct_import_words(he_context* ctx, const uint64_t* src, int on_device, size_t B, int size,
                             int level, double scale, he_ciphertext** out);
he_status he_pt_export_words(he_context* ctx, const he_plaintext* pt, uint64_t* dst, int on_device);
he_status he_pt_import_words(he_context* ctx, const uint64_t* src, int on_device, size_t B, int level,
                             double scale, he_plaintext** out);
/* Plaintext from signed integer coefficients m[B][N] (host): reduce per limb
 * and NTT on device (C7 injection of an exactly-rounded encoding). */
he_status he_pt_from_int_coeffs(he_context* ctx, const int64_t* m, size_t B, double scale, int level,
                                he_plaintext** out);
/* The inverse of he_pt_from_int_coeffs (test/injection): the
 * plaintext's integer polynomials m[B][N] (host), i.e. INTT of the data limbs,
 * CRT composition mod Q_level and centring into (-Q/2, Q/2].  Fails with
 * HE_SCALE_OVERFLOW when a coefficient is outside the int64 range (then m is
 * not written).  For a QP plaintext the data limbs are used. */
he_status he_pt_to_int_coeffs(he_context* ctx, const he_plaintext* pt, int64_t* m);
/* Same with the K special limbs appended (a QP plaintext, limbs 0..level then
 * p_0..p_{K-1}), for he_vec_mat_pt's lazy-ModDown form. */
he_status he_pt_from_int_coeffs_qp(he_context* ctx, const int64_t* m, size_t B, double scale, int level,
                                   he_plaintext** out);
/* Number of limbs per item of a plaintext (level+1, or level+1+K for QP). */
he_status he_pt_limbs(const he_plaintext* pt, int* limbs);
/* Export keys as NTT words: kind 0 = secret [L+K][N], 1 = public [2][L][N],
 * 2 = relin [L][2][L+K][N], 3 = Galois key of rotation `step` (same shape). */
he_status he_key_export(he_context* ctx, int kind, int32_t step, uint64_t* dst);
/* Number of words he_key_export writes for `kind`. */
size_t he_key_words(const he_context* ctx, int kind);
/* Device bytes the context's public, relinearisation and Galois keys occupy right
 * now.  Keys at rest: a context whose primes are all < 2^31 (the
 * 32-bit engine, BASELINE config 4) keeps every switching key as 32-bit words in
 * Montgomery form only, 4 bytes per residue; the 64-bit words of a key are built
 * from them the first time something asks for them (he_key_export, the per-rotation
 * he_vec_mat_pt form and the other unfused paths) and then stay.  Other contexts
 * hold 64-bit words (8 bytes per residue).  0 for a null context. */
size_t he_key_bytes(const he_context* ctx);

/* ---- wire format ("427KB of communication") ----
 * A 64-byte header (magic "HECKKS01", u32 log2N, u32 B, u32 size, u32 level,
 * f64 scale, u64 payload_bytes, u32 n_limbs, 20 zero bytes) followed by, for
 * every item b, poly p and limb i, the N stored NTT-domain words of limb i
 * written with w_i = bit_length(q_i) bits each, least significant bit first,
 * as little-endian 64-bit words (N w_i is a multiple of 64, so each limb
 * segment is 64-bit aligned).  Packing and unpacking run on the device. */
/* Total serialized bytes (header + payload) of ct. */
he_status he_ct_serialized_size(he_context* ctx, const he_ciphertext* ct, size_t* bytes);
/* Write header + payload to dst (host, or device when on_device != 0). */
he_status he_ct_serialize(he_context* ctx, const he_ciphertext* ct, void* dst, int on_device);
/* Seeded form of a fresh he_encrypt_symmetric ciphertext (HE_INVALID_ARGUMENT
 * for any other ciphertext): magic "HECKKSS1", the same header fields with
 * size 2, the 20-byte tail holding u64 a_seed, u64 stream_id, 4 zero bytes;
 * the payload is c0 of every item only (half the bytes). */
he_status he_ct_serialized_size_seeded(he_context* ctx, const he_ciphertext* ct, size_t* bytes);
he_status he_ct_serialize_seeded(he_context* ctx, const he_ciphertext* ct, void* dst, int on_device);
/* Read a serialized ciphertext of len bytes (either form; a seeded one gets
 * its c1 regenerated on the device); rejects a bad header, a wrong
 * length or a residue >= its prime (HE_INVALID_ARGUMENT), other parameters
 * (HE_PARAM_MISMATCH). */
he_status he_ct_deserialize(he_context* ctx, const void* src, int on_device, size_t len, he_ciphertext** out);

/* ---- ring primitives (BASELINE config 2 microbench) ------ */
/* In-place batched forward / inverse negacyclic NTT (C5) of device words
 * d[B][n_limbs][N], limb i modulo prime i (n_limbs <= L+K). */
he_status he_ntt_forward(he_context* ctx, uint64_t* d, size_t B, int n_limbs);
he_status he_ntt_inverse(he_context* ctx, uint64_t* d, size_t B, int n_limbs);
/* out = a (.) b pointwise mod prime of the limb, device words [B][n_limbs][N]. */
he_status he_modmul(he_context* ctx, const uint64_t* a, const uint64_t* b, uint64_t* out, size_t B,
                    int n_limbs);
/* Fused: out = INTT(NTT(a) (.) b) for coefficient-domain a and NTT-domain b
 * (one kernel per limb: negacyclic ring product). */
he_status he_ntt_mul_intt(he_context* ctx, const uint64_t* a, const uint64_t* b, uint64_t* out,
                          size_t B, int n_limbs);

/* Opt-in profiler: with `on` != 0 every kernel launch of ctx is bracketed
 * by CUDA events recorded on the context stream.  he_profile_read
 * synchronises the stream and writes a JSON object into buf (NUL-terminated,
 * truncated to len):  {"<kernel tag>": [launches, total_ms, alg_bytes,
 * blocks, alg_ops], ...}  where alg_bytes / alg_ops are the algorithmic bytes
 * and modular operations (butterflies + multiply-accumulates) of those
 * launches (0 where not modelled).  Reading resets the records. */
he_status he_profile_enable(he_context* ctx, int on);
he_status he_profile_read(he_context* ctx, char* buf, size_t len);

/* Number of kernels this library has launched on ctx (for the bench's
 * gpu_launches claim; a he_graph_launch adds the kernels its graph holds). */
uint64_t he_launch_count(const he_context* ctx);

/* ---- CUDA-graph recording of a call sequence (batch-1 latency) --------- */
/* A batch-1 evaluation (e.g. BASELINE config 1: encode, encrypt, vec_mat,
 * decrypt, decode) is a few dozen short kernels whose launch overhead is most
 * of its latency.  he_graph_begin starts recording every library call made on
 * ctx (stream capture, relaxed mode, of a private stream that first waits for
 * ctx's stream); the calls then enqueue nothing and only record.  Device
 * memory any recorded call allocates (outputs and scratch) is owned by the
 * graph: it is never handed to other work while the graph exists, so every
 * replay writes the same addresses, and the handles returned during recording
 * stay valid and hold the last replay's results (freeing them is allowed and
 * deferred).  Blocks freed during recording that existed before it are
 * released at he_graph_free.  Inputs the sequence reads (device buffers such as
 * he_encode_device's z_dev, plaintexts, keys) must stay alive and may be
 * rewritten between replays.  A recorded he_encrypt draws the same Philox
 * stream on every replay (same randomness): record the server part only when
 * fresh encryption randomness matters.
 * Errors: he_graph_begin fails with HE_INVALID_ARGUMENT when ctx is already
 * recording or profiling; calls that read back to the host (host-output
 * decode, he_sync, exports) fail while recording (HE_CUDA_ERROR) and leave
 * the recording unusable: he_graph_end then fails and releases what was
 * recorded.  he_set_stream fails while recording. */
he_status he_graph_begin(he_context* ctx);
he_status he_graph_end(he_context* ctx, he_graph** out);
/* Enqueue one replay on ctx's current stream (asynchronous). */
he_status he_graph_launch(he_graph* g);
/* Number of kernel launches one replay performs. */
uint64_t he_graph_kernels(const he_graph* g);
/* Release the graph and the memory it owns (handles created during recording
 * must not be used afterwards; freeing them later is a no-op). */
he_status he_graph_free(he_graph* g);

#ifdef __cplusplus
}
#endif
#endif /* HE_CKKS_H_ */
