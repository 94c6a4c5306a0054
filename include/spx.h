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
#define SPX_ERR_NCCL -3

/* element types for spx_allreduce */
#define SPX_DTYPE_F32 0
#define SPX_DTYPE_BF16 1

/* ---- runtime ---- */
int spx_abi_version(void);
const char* spx_last_error(void);
int spx_device_sm_count(void);

/* Number of kernels libspx has launched (or recorded into a CUDA graph under capture) in this
 * process; launch accounting for benchmarks. */
int64_t spx_launch_count(void);
int spx_enable_peer_access(int32_t dev, int32_t peer);

/* Path hop: copy `bytes` from src (device src_dev) to dst (device dst_dev) on `stream`.
 * Cross-device copies go peer-to-peer over NVLink.  Replaces comm_time (topology.py:128-136). */
int spx_hop(int32_t dst_dev, void* dst, int32_t src_dev, const void* src, int64_t bytes, void* stream);

/* Cross-process path hops over NVLink peer memory (one process per GPU).  Also replaces
 * comm_time (topology.py:128-136) for hops between logical nodes on different GPUs.
 *   spx_ipc_export: CUDA IPC handle (64 bytes into handle_out) of the allocation holding `ptr`,
 *                   and ptr's byte offset inside it;
 *   spx_ipc_open / spx_ipc_close: map / unmap a peer process's allocation (base pointer);
 *   spx_hop_push: `ctas` CTAs copy `bytes` (multiple of 16, 16-byte aligned) from local src to
 *                 the peer-mapped dst with 16-byte stores, then each CTA release-adds 1 to the
 *                 peer-mapped *flag (system scope) once its stores are visible (flag may be
 *                 NULL: an unsignalled copy, for bandwidth probes);
 *   spx_hop_push_ce: the same hop on the copy engine (cudaMemcpyAsync into the peer-mapped dst,
 *                 no SMs), then one thread fences and release-adds 1 to *flag (NULL: no flag);
 *   spx_hop_wait: the stream waits until *flag - target >= 0 (acquire, system scope); traps
 *                 after the hop timeout (default 120 s) so a lost hop fails loudly;
 *   spx_hop_set_timeout: process-wide hop_wait timeout in seconds (0 < s <= 86400), read at
 *                 each spx_hop_wait launch (executor: SPX_HOP_TIMEOUT_S). */
int spx_ipc_export(const void* ptr, void* handle_out, int64_t* offset_out);
int spx_ipc_open(const void* handle, void** base_out);
int spx_ipc_close(void* base);
int spx_hop_push(void* dst, const void* src, int64_t bytes, uint32_t* flag, int32_t ctas, void* stream);
int spx_hop_push_ce(void* dst, const void* src, int64_t bytes, uint32_t* flag, void* stream);
int spx_hop_wait(const uint32_t* flag, uint32_t target, void* stream);
int spx_hop_set_timeout(double seconds);

/* Stage-replica gradient aggregation (replaces the replica sync PAPER.md:97 describes; SURVEY.md
 * §8(b)).  NCCL communicators owned by libspx, one per replicated stage; NCCL is resolved at run
 * time (the process's libnccl.so.2), so these return SPX_ERR_NCCL on a box without it.
 *   spx_comm_unique_id: 128-byte ncclUniqueId into id_out (one rank creates it, the caller
 *                       broadcasts it to the group);
 *   spx_comm_init: join the group as `rank` of `nranks`, *comm_out = communicator handle;
 *   spx_allreduce: in-place sum of `count` elements (SPX_DTYPE_F32 / SPX_DTYPE_BF16) over the
 *                  group, enqueued on `stream`;
 *   spx_comm_destroy: free a communicator. */
int spx_comm_unique_id(void* id_out);
int spx_comm_init(const void* id, int32_t nranks, int32_t rank, void** comm_out);
int spx_allreduce(void* comm, void* buf, int64_t count, int32_t dtype, void* stream);
int spx_comm_destroy(void* comm);

/* ---- GEMM (tcgen05 + TMEM + TMA) ----
 * D[m,n] = sum_k A(m,k) * B(n,k), fp32 accumulate.
 *   a_mn_major = 0: A stored [M][lda] (K contiguous); 1: A stored [K][lda] (M contiguous)
 *   b_mn_major = 0: B stored [N][ldb] (K contiguous); 1: B stored [K][ldb] (N contiguous)
 * epilogue:
 *   0  C bf16 [M][ldc]  = D
 *   1  C bf16 [M][ldc]  = D + R (R bf16 [M][ldc], may alias C)
 *   2  C f32  [M][ldc]  = D + beta * C   (beta in {0,1}; wgrad accumulation)
 *   3  SwiGLU (forward layout: A and B K-major): N = 2F with gate/up interleaved in 128-column
 *      blocks; C bf16 [M][ldc] = silu(gate) * up  (F columns), C2 bf16 [M][ldc2] = raw gate/up
 *   6  SwiGLU backward fused into the down-projection dgrad (A K-major, B MN-major): D = dh [M][N=F]; R = gu [M][ldc2]
 *      (raw gate/up, 128-column interleave); C2 bf16 [M][ldc2] = dgu (dgate, dup interleaved)
 *   7  cross-entropy head (A and B K-major, N % 128 == 0): C bf16 [M][ldc] = D (logits) and
 *      C2 f32 [M][ldc2 >= 2*N/128] = per 128-column block (max, sum exp(z - max)) of the bf16
 *      logits, consumed by spx_xent_from_parts (replaces spx_head_xent_fwd_bwd's loss pass)
 * Requires N % 32 == 0, K, lda, ldb multiples of 8, 16-byte aligned A/B. */
int spx_gemm_bf16(const void* A, const void* B, void* C, const void* R, void* C2, int64_t M, int64_t N, int64_t K,
                  int64_t lda, int64_t ldb, int64_t ldc, int64_t ldc2, int32_t a_mn_major, int32_t b_mn_major,
                  int32_t epilogue, float beta, void* stream);

/* Register the split-K partials buffer of the current device (fp32, 16-byte aligned).  When set,
 * fp32-accumulating GEMMs (epilogue 2) with too few tiles for the SMs split K: each split stores its
 * partial product to the buffer and a reduce kernel adds the partials to C in split order
 * (deterministic).  Split counts are capped so the partials fit in n_floats.  NULL disables
 * split-K.  One split-K GEMM at a time may use the buffer on a device (the executor issues every
 * weight-gradient GEMM on one stream). */
int spx_gemm_set_workspace(float* partials, int64_t n_floats);

/* Weight-gradient group: C_i (+)= A_i . B_i^T for i < count (1..4), fp32 accumulation exactly as
 * epilogue 2 of spx_gemm_bf16 (beta_i != 0 adds into C_i), all problems sharing the operand majors,
 * in ONE persistent launch so their tiles fill the SMs together (the four wgrads of a decoder
 * layer).  Arrays are host arrays of length count.  No split-K. */
int spx_gemm_f32_group(int32_t count, const void* const* A, const void* const* B, float* const* C, const int64_t* M,
                       const int64_t* N, const int64_t* K, const int64_t* lda, const int64_t* ldb, const int64_t* ldc,
                       const float* beta, int32_t a_mn_major, int32_t b_mn_major, void* stream);

/* QKV projection with RoPE fused into the epilogue: C = A.B^T, then rotate-half RoPE (position =
 * row % T, cos_sin [hd/2][T][2], position-minor) on columns [0, rope_cols) (the q and k heads).  head_dim 64 or 128. */
int spx_gemm_bf16_rope(const void* A, const void* B, void* C, int64_t M, int64_t N, int64_t K, int64_t lda,
                       int64_t ldb, int64_t ldc, const float* cos_sin, int64_t rope_cols, int64_t T, int64_t head_dim,
                       void* stream);

/* Attention-output dgrad with the attention backward's D pass fused into its epilogue:
 * dO = A . B (A [M][K] K-major, B [K][N] MN-major: dO = dY . Wo), and for every (row, head) of the
 * [batch*T][H*head_dim] output D = sum over the head's columns of bf16(dO) * O, written with
 * lse*log2e into delta_ws (the [2][batch][H][T] prefix of spx_attn_bwd's workspace) -- then call
 * spx_attn_bwd_ex with SPX_ATTN_DELTA_READY.  head_dim 64 or 128, M = batch * T. */
int spx_gemm_bf16_attn_delta(const void* A, const void* B, void* dO, const void* O, int64_t ld_o, const float* lse,
                             float* delta_ws, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb, int64_t ldc,
                             int64_t batch, int64_t T, int64_t head_dim, void* stream);

/* ---- attention (causal, GQA; q/k/v read from the fused QKV buffer) ----
 * qkv [B*T][ld_qkv] bf16 with q heads at column h*hd, k heads at (H+j)*hd, v heads at (H+Hkv+j)*hd.
 * o [B*T][ld_o] bf16, lse [B][H][T] f32 (natural log).  T % 64 == 0, hd in {48, 64, 128}. */
int spx_attn_fwd(const void* qkv, void* o, float* lse, int64_t B, int64_t T, int64_t H, int64_t Hkv, int64_t hd,
                 int64_t ld_qkv, int64_t ld_o, float scale, void* stream);
/* Workspace of spx_attn_bwd in floats: D = rowsum(dO*O) and lse*log2e (B*H*T each) and, on the
 * tcgen05 path (hd 64/128, T % 128 == 0), the causal dS^T tiles the dQ GEMM reads. */
int64_t spx_attn_bwd_ws_floats(int64_t B, int64_t H, int64_t T, int64_t hd);
/* dqkv gets dq/dk/dv in the same layout as qkv.  delta_ws: spx_attn_bwd_ws_floats(B, H, T, hd)
 * floats (16-byte aligned).  rope_cos_sin (may be NULL): when given, dq and dk are written back
 * through the inverse RoPE rotation (the gradient w.r.t. the pre-RoPE projections). */
int spx_attn_bwd(const void* qkv, const void* o, const void* dout, const float* lse, float* delta_ws, void* dqkv,
                 int64_t B, int64_t T, int64_t H, int64_t Hkv, int64_t hd, int64_t ld_qkv, int64_t ld_o, float scale,
                 const float* rope_cos_sin, void* stream);
/* spx_attn_bwd with flags: SPX_ATTN_DELTA_READY = the first 2*B*H*T floats of delta_ws already hold
 * D = rowsum(dO*O) and lse*log2e (written by spx_gemm_bf16_attn_delta), so no D pass runs. */
#define SPX_ATTN_DELTA_READY 1
/* SPX_ATTN_WS_EX: delta_ws holds spx_attn_bwd_ws_floats_ex(B, H, Hkv, T, hd) floats; with GQA and fewer
 * (batch, kv head, 128-key block) items than SMs the dK/dV pass then splits each group over several
 * work items (fp32 partials, summed in a fixed order: still deterministic). */
#define SPX_ATTN_WS_EX 2
int64_t spx_attn_bwd_ws_floats_ex(int64_t B, int64_t H, int64_t Hkv, int64_t T, int64_t hd);
int spx_attn_bwd_ex(const void* qkv, const void* o, const void* dout, const float* lse, float* delta_ws, void* dqkv,
                    int64_t B, int64_t T, int64_t H, int64_t Hkv, int64_t hd, int64_t ld_qkv, int64_t ld_o, float scale,
                    const float* rope_cos_sin, int32_t flags, void* stream);

/* ---- RMSNorm ----
 * fwd: y = x * rsqrt(mean(x^2) + eps) * g ; rstd[rows] saved.
 * bwd: dx = dres + rstd*(g*dy - xhat*mean(xhat*g*dy)) (dres may be NULL); dg (f32) += sum_rows dy*xhat
 *      via ws (spx_rmsnorm_ws_floats(rows, d) floats), deterministic (fixed-order partials). */
int spx_rmsnorm_fwd(const void* x, const void* g, void* y, float* rstd, int64_t rows, int64_t d, float eps, void* stream);
int spx_rmsnorm_bwd(const void* x, const void* g, const float* rstd, const void* dy, const void* dres, void* dx,
                    float* dg, float* ws, int64_t rows, int64_t d, void* stream);
int64_t spx_rmsnorm_ws_floats(int64_t rows, int64_t d);

/* ---- RoPE (rotate-half), in place on the first n_heads heads of each row; position = row % T.
 * cos_sin [hd/2][T][2] f32 (position-minor).  inverse = 1 rotates by -theta (backward). */
int spx_rope(void* qkv, const float* cos_sin, int64_t rows, int64_t T, int64_t n_heads, int64_t hd, int64_t ld,
             int32_t inverse, void* stream);

/* ---- SwiGLU backward: gu [rows][2F] (gate/up interleaved per 128 columns), dh [rows][F] -> dgu [rows][2F] */
int spx_swiglu_bwd(const void* gu, const void* dh, void* dgu, int64_t rows, int64_t F, void* stream);

/* ---- embedding ----
 * fwd: out[r] = table[ids[r]].
 * bwd: deterministic scatter-add into the f32 table gradient; tokens grouped by id:
 *      perm = positions sorted by (id, position), seg_start[n+1], seg_id[n]; the segment count is read
 *      from device memory (*n_segments <= max_segments) so the call can sit inside a CUDA graph. */
int spx_embed_fwd(const int32_t* ids, const void* table, void* out, int64_t n, int64_t d, void* stream);
int spx_embed_bwd(const int32_t* perm, const int32_t* seg_start, const int32_t* seg_id, const int32_t* n_segments,
                  int64_t max_segments, const void* dout, float* dtable, int64_t d, void* stream);

/* ---- token batch preparation (the data format in front of S0): one microbatch's token block
 *      tokens[b][ld_tokens] (int64, T+1 used per row) -> ids[n] = tokens[r][t], targets[n] =
 *      tokens[r][t+1] (n = b*T, position r*T + t) and the embedding-backward grouping of
 *      spx_embed_bwd (perm, seg_start, seg_id, *n_segments), computed on the device so a step's
 *      only host->device input is the token block.  n <= 16384; ids must be < 2^31.  ids / targets
 *      may be NULL (grouping only); perm == NULL (with the other grouping outputs NULL) splits ids /
 *      targets only, with a fast many-CTA kernel -- the executor splits on the compute stream and
 *      sorts on a side stream, since only the embedding backward needs the grouping. */
int spx_token_prep(const int64_t* tokens, int64_t b, int64_t T, int64_t ld_tokens, int32_t* ids, int32_t* targets,
                   int32_t* perm, int32_t* seg_start, int32_t* seg_id, int32_t* n_segments, void* stream);

/* ---- softmax cross-entropy: row_loss[r] = lse(z_r) - z_r[t_r]; logits overwritten by
 *      (softmax - onehot) * scale (bf16).  One pass pair per row, logits never re-materialised. */
/* From the head GEMM's epilogue-7 partials (nb >= V/128 (max, sum) pairs per row): combine them
 * (fixed order), row_loss[r] = lse - z[t_r], and if scale != 0 rewrite the logits in place as
 * (softmax - onehot) * scale -- a single read and write of the logits. */
int spx_xent_from_parts(void* logits, const float* parts, int64_t nb, const int32_t* targets, float* row_loss,
                        int64_t n, int64_t V, int64_t ld, float scale, void* stream);
int spx_xent_fwd_bwd(void* logits, const int32_t* targets, float* row_loss, int64_t n, int64_t V, int64_t ld,
                     float scale, void* stream);

/* ---- reductions / optimizer ---- */
int spx_sum_f32(const float* x, int64_t n, float* out, float scale, int32_t accumulate, void* stream);
/* dst += src, fp32, n elements (16-byte aligned): merges the gradient buffers of co-resident
 * replicas of a stage before the replica all-reduce / optimizer. */
int spx_add_f32(float* dst, const float* src, int64_t n, void* stream);
/* dst += src, then src = 0 (merges a co-resident replica's gradient and leaves its buffer ready
 * for the next iteration) */
int spx_add_f32_clear(float* dst, float* src, int64_t n, void* stream);
int64_t spx_sumsq_ws_floats(void);
int spx_sumsq(const float* x, int64_t n, float* ws, float* out, void* stream);
/* scale[0] = min(1, max_norm / (sqrt(sum(sumsq[0:count])) + 1e-6))  (torch clip_grad_norm_) */
int spx_clip_scale(const float* sumsq, int32_t count, float max_norm, float* scale, float* norm_out, void* stream);
/* torch.optim.AdamW update over a flat f32 parameter set; decay applies to [0, n_decay);
 * gradients are multiplied by *grad_scale (may be NULL); p_bf16 receives the bf16 working copy. */
int spx_adamw(float* p, const float* g, float* m, float* v, void* p_bf16, int64_t n, int64_t n_decay, float lr,
              float beta1, float beta2, float eps, float weight_decay, int64_t step, const float* grad_scale,
              void* stream);
/* spx_adamw that also clears the gradient it consumed (g = 0), so the next iteration accumulates
 * from zero without a separate fill pass (bit-identical update) */
int spx_adamw_clear(float* p, float* g, float* m, float* v, void* p_bf16, int64_t n, int64_t n_decay, float lr,
                    float beta1, float beta2, float eps, float weight_decay, int64_t step, const float* grad_scale,
                    void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SPX_H_ */
