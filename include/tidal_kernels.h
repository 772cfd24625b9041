/* tidal_kernels.h — kernel-level C-ABI entry points (per-op parity tests).
 *
 * Each call launches exactly one of the library's sm_100a kernels on the
 * current device's default stream and synchronises; every pointer is DEVICE
 * memory owned by the caller; bf16 tensors are row-major.  They exist so the
 * tests can compare each op of the prefill path with
 * the oracle in isolation; tidal_invoke_prefill composes the same kernels.
 * Errors: TIDAL_ERR_CUDA (launch/sync failure), TIDAL_ERR_INVALID (shape).
 */
#ifndef TIDAL_KERNELS_H
#define TIDAL_KERNELS_H
#include <stdint.h>

#include "tidal.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Y[S,d] (bf16) = g * X / sqrt(mean(X^2) + eps), X fp32. d % 4 == 0. */
tidal_status tidal_k_rmsnorm(const float* X, const void* g, void* Y, int S, int d, float eps);
/* X[s,:] = E[tok[s]-row0,:] (fp32) if tok[s] in [row0,row0+rows) else 0.  d % 8 == 0. */
tidal_status tidal_k_embed(const int32_t* tok, const void* E, float* X, int S, int d, int row0,
                           int rows);
/* T[M,r] (bf16) = scale * X[M,K] A[r,K]^T, r in {8,16,32,64}, K % 8 == 0. */
tidal_status tidal_k_lora_shrink(const void* X, int M, int K, const void* A, void* T, int r,
                                 float scale);
/* O[S,H*hd] = causal GQA attention over QKV[S,(H+2KV)*hd]; hd in {64,128}. */
tidal_status tidal_k_attention(const void* qkv, void* O, int S, int H, int KV, int hd);
/* The tcgen05 attention used for hd = 128: Q, K from qkv[S,(H+2KV)*128]; V given
 * transposed, vt[KV*128][vt_ld] (vt_ld >= S, multiple of 8). */
tidal_status tidal_k_attention_tc(const void* qkv, const void* vt, int vt_ld, void* O, int S, int H,
                                  int KV);
/* logits[V] = W[V,d] . RMSNorm(xlast; g), *key = packed argmax (see tidal.h). */
tidal_status tidal_k_head(const float* xlast, const void* g, const void* W, int V, int d, float eps,
                          float* logits, unsigned long long* key);
/* tcgen05 GEMM out = A[M,K] . [W_0;W_1;W_2]^T (+ LoRA K-extension T_s . B_s^T).
 * epi: 0 store bf16, 1 store bf16 with RoPE on segments 0,1 (rope = float2
 * [M, head_dim/2] cos/sin), 2 SiLU(W_0 part) * (W_1 part) with seg_n[0] = F,
 * 3 fp32 out += acc.  T/B nullable (no LoRA).  K % 8 == 0, seg_n % 8 == 0 and
 * ldo (elements) keeps output rows 16-byte aligned, else TIDAL_ERR_INVALID.
 * Bits 8-16 of epi optionally force the N-tile width (128, 192 or 256) and
 * bits 20-21 the CTA group (1 single-SM, 2 CTA pair with cta_group::2);
 * 0 lets the library pick them as the runtime does. */
tidal_status tidal_k_gemm(int epi, const void* A, const void* const* W, const int* seg_n, int nseg,
                          void* out, int ldo, int M, int K, const void* const* T,
                          const void* const* B, int r, const void* rope, int head_dim);

#ifdef __cplusplus
}
#endif
#endif
