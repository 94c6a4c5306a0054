/*
 * spx.h — C-ABI of libspx.so, the B200 (sm_100a) compute library behind the SkipPipe
 * partial-pipeline executor.
 *
 * The reference (arxiv 2502.19913 "SkipPipe", /root/reference) ships no executor and no FFI:
 * its only execution seam is the simulator call `simulate(schedule, topology, sim_config)`
 * (SPEC.md:344), which *models* stage compute with `Topology.compute_fwd_ms` /
 * `compute_bwd_ms` (pkg/src/pipepath/topology.py:51,73-74) and path hops with
 * `comm_time = latency + bytes / bandwidth` (topology.py:128-136).  Every entry point below
 * replaces one of those modelled quantities with real work on a B200:
 *
 *   spx_gemm_bf16 / spx_rmsnorm_* / spx_rope / spx_attn_* / spx_swiglu_bwd / spx_embed_* /
 *   spx_xent_fwd_bwd        -> the stage compute modelled by compute_fwd_ms / compute_bwd_ms
 *                              (topology.py:51, :73-74); shapes from ModelPreset
 *                              (topology.py:150-180)
 *   spx_hop                 -> the per-hop transfer modelled by comm_time (topology.py:128-136),
 *                              message size activation_bytes (topology.py:190-194)
 *   spx_sumsq / spx_adamw   -> the synchronous once-per-iteration update,
 *                              which the reference omits
 *
 * Conventions (all functions):
 *   - return 0 (SPX_OK) on success, a negative SPX_ERR_* code otherwise; never throw.
 *     spx_last_error() returns a thread-local message for the last failure.
 *   - all tensor arguments are caller-owned device pointers; no function allocates.
 *   - shapes/strides are int64 element counts; `stream` is a cudaStream_t (may be NULL).
 *   - bf16 storage, fp32 accumulation; row-major unless stated.
 */
#ifndef SPX_H_
#define SPX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPX_ABI_VERSION 1
#define SPX_OK 0
#define SPX_ERR_ARG -1
#define SPX_ERR_CUDA -2

/* ---- runtime ---- */
int spx_abi_version(void);
const char* spx_last_error(void);
int spx_device_sm_count(void);
int spx_enable_peer_access(int32_t dev, int32_t peer);

/* Path hop: copy `bytes` from src (device src_dev) to dst (device dst_dev) on `stream`.
 * Cross-device copies go peer-to-peer over NVLink.  Replaces comm_time (topology.py:128-136). */
int spx_hop(int32_t dst_dev, void* dst, int32_t src_dev, const void* src, int64_t bytes, void* stream);

/* ---- GEMM (tcgen05 + TMEM + TMA) ----
 * D[m,n] = sum_k A(m,k) * B(n,k), fp32 accumulate.
 *   a_mn_major = 0: A stored [M][lda] (K contiguous); 1: A stored [K][lda] (M contiguous)
 *   b_mn_major = 0: B stored [N][ldb] (K contiguous); 1: B stored [K][ldb] (N contiguous)
 * epilogue:
 *   0  C bf16 [M][ldc]  = D
 *   1  C bf16 [M][ldc]  = D + R (R bf16 [M][ldc], may alias C)
 *   2  C f32  [M][ldc]  = D + beta * C   (beta in {0,1}; wgrad accumulation)
 *   3  SwiGLU: N = 2F with gate/up interleaved in 128-column blocks;
 *      C bf16 [M][ldc] = silu(gate) * up  (F columns), C2 bf16 [M][ldc2] = raw gate/up (N columns)
 * Requires N % 32 == 0, K, lda, ldb multiples of 8, 16-byte aligned A/B. */
int spx_gemm_bf16(const void* A, const void* B, void* C, const void* R, void* C2, int64_t M, int64_t N, int64_t K,
                  int64_t lda, int64_t ldb, int64_t ldc, int64_t ldc2, int32_t a_mn_major, int32_t b_mn_major,
                  int32_t epilogue, float beta, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SPX_H_ */
