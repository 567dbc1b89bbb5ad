// he_ops.h — internal operations behind the C-ABI (he_capi.cu).  Product code.
#pragma once
#include <vector>

#include "he_internal.cuh"

namespace he {

inline size_t ct_words(const he_ciphertext* c) { return (size_t)c->B * c->size * (c->level + 1) * c->ctx->N; }
inline int pt_limbs(const he_plaintext* p) { return p->level + 1 + (p->qp ? p->ctx->K : 0); }
inline size_t pt_words(const he_plaintext* p) { return (size_t)p->B * pt_limbs(p) * p->ctx->N; }

void context_init(he_context* c, const HostParams& hp, u64 seed);
void context_destroy(he_context* c);
he_context* context_make_public(he_context* c);
void set_allocator(he_context* c, he_alloc_fn alloc, he_free_fn free_fn, void* user);
void build_step_tables(he_context* c);

he_ciphertext* ct_new(he_context* c, int B, int size, int level, double scale);
he_plaintext* pt_new(he_context* c, int B, int level, double scale, int qp = 0);
void ct_free(he_ciphertext* ct);
void pt_free(he_plaintext* pt);

// ring primitives on raw device words [items][nl][N]
void ntt_rows(he_context* c, const u64* src, u64* dst, size_t items, int nl, size_t src_bs, size_t dst_bs,
              bool inverse);
void modmul_rows(he_context* c, const u64* a, const u64* b, u64* out, size_t items, int nl);
void ring_mul(he_context* c, const u64* a, const u64* b, u64* out, size_t items, int nl);
void signed_to_ntt(he_context* c, const i64* poly, u64* dst, size_t items, int nl, int lc = -1);
int check_words(he_context* c, const u64* w, size_t items, int Lc);

// scheme
void keygen(he_context* c, const std::vector<int>& steps);
void encode_coeffs(he_context* c, const double* z_dev, size_t n, size_t B, double scale, i64* m_dev);
he_ciphertext* encode_encrypt(he_context* c, const double* z_dev, size_t n, size_t B, double scale, int level,
                              u64 stream_id);
void encode_unrounded(he_context* c, const double* z_dev, size_t n, size_t B, double scale, double* pre_dev);
he_plaintext* encode(he_context* c, const double* z_dev, size_t n, size_t B, double scale, int level, int qp = 0,
                     bool check_now = true);
void take_err(he_context* c);
he_plaintext* pt_from_int(he_context* c, const i64* m_dev, size_t B, double scale, int level, int qp = 0);
void decode(he_context* c, const he_plaintext* pt, double* out_dev, size_t n);
void pt_to_int(he_context* c, const he_plaintext* pt, i64* out_dev);
he_ciphertext* encrypt(he_context* c, const he_plaintext* pt, u64 stream_id);
he_ciphertext* encrypt_symmetric(he_context* c, const he_plaintext* pt, u64 stream_id, u64 a_seed);
void sym_regen_c1(he_context* c, he_ciphertext* ct);
void ct_copy_c0(he_context* c, const he_ciphertext* ct, u64* dst, bool to_ct);
he_plaintext* decrypt(he_context* c, const he_ciphertext* ct);

// into: write the result into that ciphertext (in-place forms; into == a with a->B >= the other batch)
he_ciphertext* ct_binop(he_context* c, int op, const he_ciphertext* a, const he_ciphertext* b,
                        he_ciphertext* into = nullptr);  // 0 add, 1 sub
he_ciphertext* ct_negate(he_context* c, const he_ciphertext* a);
he_ciphertext* ct_mul_plain(he_context* c, const he_ciphertext* a, const he_plaintext* p, he_ciphertext* into = nullptr);
he_ciphertext* ct_add_plain(he_context* c, const he_ciphertext* a, const he_plaintext* p, he_ciphertext* into = nullptr);
he_ciphertext* ct_tensor(he_context* c, const he_ciphertext* x, const he_ciphertext* y);
he_ciphertext* ct_rescale(he_context* c, const he_ciphertext* a, const he_plaintext* bias = nullptr);
he_ciphertext* ct_relinearize(he_context* c, const he_ciphertext* a);
he_ciphertext* ct_square_relin(he_context* c, const he_ciphertext* x);
he_ciphertext* ct_square_rescale(he_context* c, const he_ciphertext* x);
he_ciphertext* ct_rotate(he_context* c, const he_ciphertext* a, int step, bool add_input);
he_ciphertext* ct_vec_mat(he_context* c, const he_ciphertext* x, const he_plaintext* diags,
                          const he_plaintext* bias);
he_ciphertext* ct_vec_mat_bsgs(he_context* c, const he_ciphertext* x, const he_plaintext* diags, int g,
                               const he_plaintext* bias, int fold_n = -1, int fold_step = 0);
he_ciphertext* ct_conv(he_context* c, const he_ciphertext* x, const he_plaintext* kernels,
                       const he_plaintext* masks, const he_plaintext* bias, int chunk, int fold_n1 = 0);
he_ciphertext* ct_conv_bsgs(he_context* c, const he_ciphertext* x, const he_plaintext* diags,
                            const he_plaintext* bias, int chunk, int g);
bool has_galois_key(he_context* c, int step, u32* gal_out);       // either stored form
const u64* galois_key(he_context* c, int step, u32* gal_out);     // u64 form (materialised on demand)
const u64* relin_key(he_context* c);                              // u64 form (materialised on demand)
size_t key_bytes(he_context* c);                                  // device bytes held by pk / relin / Galois keys
size_t wire_payload_bytes(he_context* c, const he_ciphertext* ct);
void wire_pack(he_context* c, const he_ciphertext* ct, u64* out_dev);
he_ciphertext* wire_unpack(he_context* c, const u64* in_dev, size_t B, int size, int level, double scale);

}  // namespace he
