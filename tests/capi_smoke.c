/* capi_smoke.c — a plain-C client of include/he_ckks.h (no Python, no torch): the boundary a
 * user of the method calls (SURVEY.md §8(b); PAPER.md:35 context/keys, :57-58 encode/encrypt,
 * :61 rotations, :157-177 the op catalogue).  Built and run by tests/test_capi_c.py:
 *
 *   gcc -std=c99 -I include tests/capi_smoke.c -L paper_2104_03152_b200 -lhe_ckks \
 *       -L /usr/local/cuda/lib64 -lcudart -o capi_smoke
 *
 * Checks (decrypted values against the plaintext arithmetic, CKKS tolerance):
 *   keygen, host encode, encrypt, rotate (and the in-place form), square (in place), add_plain
 *   and mul_plain in place, rescale in place, decrypt, asynchronous host decode, he_make_public
 *   (decrypt must then fail with HE_MISSING_KEY), he_pt_to_int_coeffs / he_pt_from_int_coeffs
 *   round trip, and a caller-installed allocator (cudaMallocAsync / cudaFreeAsync) that must
 *   see every ciphertext allocation and get every block back.
 * Exit status 0 = all checks passed. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "he_ckks.h"

#define CK(call)                                                                  \
  do {                                                                            \
    he_status s_ = (call);                                                        \
    if (s_ != HE_OK) {                                                            \
      fprintf(stderr, "%s:%d %s -> %d (%s)\n", __FILE__, __LINE__, #call, s_,      \
              he_last_error());                                                   \
      return 1;                                                                   \
    }                                                                             \
  } while (0)
#define EXPECT(cond, msg)                                  \
  do {                                                     \
    if (!(cond)) {                                         \
      fprintf(stderr, "FAILED: %s (line %d)\n", msg, __LINE__); \
      return 1;                                            \
    }                                                      \
  } while (0)

static long n_alloc = 0, n_free = 0;
static void* my_alloc(size_t bytes, void* stream, void* user) {
  void* p = NULL;
  (void)user;
  if (cudaMallocAsync(&p, bytes, (cudaStream_t)stream) != cudaSuccess) return NULL;
  n_alloc++;
  return p;
}
static void my_free(void* p, size_t bytes, void* stream, void* user) {
  (void)bytes;
  (void)user;
  cudaFreeAsync(p, (cudaStream_t)stream);
  n_free++;
}

static double max_err(const double* a, const double* b, size_t n) {
  double m = 0;
  for (size_t i = 0; i < n; ++i) m = fmax(m, fabs(a[i] - b[i]));
  return m;
}

int main(void) {
  const int bits[] = {31, 26, 26, 26, 31};   /* config-4 style small primes, N = 2^12 */
  he_params prm = {12, 5, bits, 1, 26.0, 0};
  he_context* ctx = NULL;
  CK(he_context_create(&prm, 7, &ctx));
  int logN, L, K;
  CK(he_context_info(ctx, &logN, &L, &K));
  EXPECT(logN == 12 && L == 4 && K == 1, "context info");
  const size_t ns = (size_t)1 << (logN - 1);
  const int32_t steps[] = {1, 3};
  CK(he_keygen(ctx, steps, 2));
  CK(he_set_allocator(ctx, my_alloc, my_free, NULL));

  enum { B = 2 };
  double* z = (double*)malloc(B * ns * sizeof(double));
  double* out = (double*)malloc(B * ns * sizeof(double));
  double* ref = (double*)malloc(B * ns * sizeof(double));
  for (size_t b = 0; b < B; ++b)
    for (size_t j = 0; j < ns; ++j) z[b * ns + j] = sin(0.001 * (double)(j + 1) * (double)(b + 1));
  const double scale = ldexp(1.0, 26);
  he_plaintext* pt = NULL;
  CK(he_encode(ctx, z, ns, B, scale, L - 1, &pt));
  he_ciphertext* ct = NULL;
  CK(he_encrypt(ctx, pt, 100, &ct));

  /* rotate by 3 (out of place) and by 1 (in place) */
  he_ciphertext* r3 = NULL;
  CK(he_rotate(ctx, ct, 3, &r3));
  CK(he_rotate_inplace(ctx, r3, 1));
  he_plaintext* dec = NULL;
  CK(he_decrypt(ctx, r3, &dec));
  CK(he_decode_async(ctx, dec, out, ns));
  CK(he_sync(ctx));
  for (size_t b = 0; b < B; ++b)
    for (size_t j = 0; j < ns; ++j) ref[b * ns + j] = z[b * ns + (j + 4) % ns];
  EXPECT(max_err(out, ref, B * ns) < 5e-3, "rotate 3 then rotate_inplace 1 == roll by 4");  /* CKKS noise at 2^26, N = 4096: ~1e-3 */
  CK(he_free_plaintext(dec));
  CK(he_free_ciphertext(r3));

  /* (z^2 + 1/4) * 1/2 with in-place square, add_plain, mul_plain, rescale */
  CK(he_square_inplace(ctx, ct));
  int level = 0;
  double sc = 0;
  size_t bb = 0;
  int size = 0;
  CK(he_ct_info(ct, &bb, &size, &level, &sc));
  EXPECT(bb == B && size == 2 && level == L - 2, "square_inplace: batch, size, level");
  double* quarter = (double*)malloc(ns * sizeof(double));
  for (size_t j = 0; j < ns; ++j) quarter[j] = 0.25;
  he_plaintext* pq = NULL;
  CK(he_encode(ctx, quarter, ns, 1, sc, level, &pq));
  CK(he_add_plain_inplace(ctx, ct, pq));
  for (size_t j = 0; j < ns; ++j) quarter[j] = 0.5;
  he_plaintext* ph = NULL;
  CK(he_encode(ctx, quarter, ns, 1, scale, level, &ph));
  CK(he_mul_plain_inplace(ctx, ct, ph));
  CK(he_rescale_inplace(ctx, ct));
  CK(he_decrypt(ctx, ct, &dec));
  CK(he_decode(ctx, dec, out, ns));
  for (size_t i = 0; i < B * ns; ++i) ref[i] = (z[i] * z[i] + 0.25) * 0.5;
  EXPECT(max_err(out, ref, B * ns) < 1e-2, "in-place square / add_plain / mul_plain / rescale");

  /* integer coefficients round trip */
  int64_t* m = (int64_t*)malloc(B * ((size_t)1 << logN) * sizeof(int64_t));
  CK(he_pt_to_int_coeffs(ctx, pt, m));
  he_plaintext* pt2 = NULL;
  CK(he_pt_from_int_coeffs(ctx, m, B, scale, L - 1, &pt2));
  uint64_t* w1 = (uint64_t*)malloc((size_t)B * L * ((size_t)1 << logN) * 8);
  uint64_t* w2 = (uint64_t*)malloc((size_t)B * L * ((size_t)1 << logN) * 8);
  CK(he_pt_export_words(ctx, pt, w1, 0));
  CK(he_pt_export_words(ctx, pt2, w2, 0));
  EXPECT(memcmp(w1, w2, (size_t)B * L * ((size_t)1 << logN) * 8) == 0, "pt_to_int_coeffs -> pt_from_int_coeffs");

  /* public context: evaluates, cannot decrypt */
  he_context* pub = NULL;
  CK(he_make_public(ctx, &pub));
  he_plaintext* pt_pub = NULL;
  CK(he_encode(pub, z, ns, B, scale, L - 1, &pt_pub));
  he_ciphertext* ct_pub = NULL;
  CK(he_encrypt(pub, pt_pub, 5, &ct_pub));
  he_ciphertext* rot_pub = NULL;
  CK(he_rotate(pub, ct_pub, 1, &rot_pub));
  he_plaintext* nope = NULL;
  EXPECT(he_decrypt(pub, rot_pub, &nope) == HE_MISSING_KEY, "public context must not decrypt");
  /* the public keys are copies: a ciphertext of pub decrypts under ctx after export/import */
  uint64_t* cw = (uint64_t*)malloc((size_t)B * 2 * L * ((size_t)1 << logN) * 8);
  CK(he_ct_export_words(pub, rot_pub, cw, 0));
  he_ciphertext* back = NULL;
  CK(he_ct_import_words(ctx, cw, 0, B, 2, L - 1, scale, &back));
  CK(he_free_plaintext(dec));
  CK(he_decrypt(ctx, back, &dec));
  CK(he_decode(ctx, dec, out, ns));
  for (size_t b = 0; b < B; ++b)
    for (size_t j = 0; j < ns; ++j) ref[b * ns + j] = z[b * ns + (j + 1) % ns];
  EXPECT(max_err(out, ref, B * ns) < 5e-3, "public-context rotation decrypts under the secret context");

  CK(he_free_ciphertext(back));
  CK(he_free_ciphertext(rot_pub));
  CK(he_free_ciphertext(ct_pub));
  CK(he_free_plaintext(pt_pub));
  CK(he_context_free(pub));
  CK(he_free_plaintext(dec));
  CK(he_free_plaintext(pt2));
  CK(he_free_plaintext(ph));
  CK(he_free_plaintext(pq));
  CK(he_free_ciphertext(ct));
  CK(he_free_plaintext(pt));
  CK(he_sync(ctx));
  EXPECT(n_alloc > 0, "the installed allocator was used");
  CK(he_context_free(ctx));
  EXPECT(n_alloc == n_free, "every block returned to the installed allocator");
  printf("capi_smoke ok: %ld blocks through the caller's allocator\n", n_alloc);
  free(z); free(out); free(ref); free(quarter); free(m); free(w1); free(w2); free(cw);
  return 0;
}
