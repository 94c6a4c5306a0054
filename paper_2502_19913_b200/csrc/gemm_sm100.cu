// tcgen05 / TMEM / TMA bf16 GEMM for sm_100a with fused epilogues.
//
//   D[M,N] = sum_k A[m,k] * B[n,k]        (fp32 accumulation in TMEM)
//
// A and B may each be K-major (row-major [rows][K]) or MN-major ([K][rows]); this covers
// every GEMM of a LLaMA decoder stage without explicit transposes:
//   forward  Y  = X  . W^T   A=X  (K-major)  B=W (K-major)
//   dgrad    dX = dY . W     A=dY (K-major)  B=W (MN-major)
//   wgrad    dW = dY^T . X   A=dY (MN-major) B=X (MN-major)
//
// Persistent, warp-specialised kernel: one CTA per SM, warp 0 = TMA producer, warp 1 = MMA
// issuer (a single thread issues tcgen05.mma), warp 2 owns the TMEM allocation, warps 4-7 are
// the epilogue (tcgen05.ld -> registers -> fused op -> global).  The accumulator is double
// buffered in TMEM (2 x BN columns) so the epilogue of tile i overlaps the MMAs of tile i+1.
//
// The GEMM has no counterpart in the reference (the reference has no kernels);
// it realises the "stage compute" rows a15-a18 of SURVEY.md §8(a).
#include <cstdio>
#include <cstring>

#include "spx_common.cuh"
#include "spx_internal.h"

namespace spx {

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;
constexpr int GEMM_THREADS = 256;

enum GemmEpilogue : int {
  EPI_BF16 = 0,        // C(bf16) = acc
  EPI_BF16_RESID = 1,  // C(bf16) = acc + R(bf16)            (R may alias C)
  EPI_F32 = 2,         // C(f32)  = acc (+ C if beta != 0)   (wgrad accumulation)
  EPI_SWIGLU = 3,      // H(bf16)[m, N/2] = silu(g)*u ; GU(bf16)[m, N] = (g,u) raw, 128-col interleave
  EPI_ROPE64 = 4,      // C(bf16) = acc with rotate-half RoPE on columns < rope_cols (head dim 64)
  EPI_ROPE128 = 5,     // same, head dim 128
};

template <int EPI>
struct RopeHd {
  static constexpr int value = EPI == EPI_ROPE64 ? 64 : (EPI == EPI_ROPE128 ? 128 : 0);
};

template <int BN>
struct GemmCfg {
  static constexpr int A_BYTES = GEMM_BM * GEMM_BK * 2;
  static constexpr int B_BYTES = BN * GEMM_BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (BN == 256) ? 4 : 6;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align slack*/ + 256 /*barriers*/;
};

struct GemmArgs {
  int M, N, K;
  void* C;
  const void* R;
  void* C2;
  long long ldc, ldr, ldc2;
  float beta;
  const float* rope_cs;  // [T][hd/2][2] (cos, sin)
  int rope_cols, rope_T;
  int splits;            // split-K factor (EPI_F32 only); units = tiles * splits
  int* sem;              // per-tile split-order semaphores (zero between launches)
};

template <int BN, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const GemmArgs args) {
  using Cfg = GemmCfg<BN>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;   // [2]
  uint64_t* tempty_bar = tfull_bar + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_m = (args.M + GEMM_BM - 1) / GEMM_BM;
  const int num_n = (args.N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int num_kb = (args.K + GEMM_BK - 1) / GEMM_BK;
  // work unit u = split * num_tiles + tile: every CTA walks its units in increasing order, so a
  // split only ever waits for a lower unit (no deadlock with all CTAs resident)
  const int num_units = num_tiles * args.splits;
  const int kbs = (num_kb + args.splits - 1) / args.splits;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 4);
    }
    fence_barrier_init();
    fence_proxy_async();
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    int stage = 0;
    uint32_t phase = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
      const int tile = u % num_tiles, kb0 = (u / num_tiles) * kbs, kb1 = min(num_kb, kb0 + kbs);
      const int m0 = (tile % num_m) * GEMM_BM;
      const int n0 = (tile / num_m) * BN;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
        uint8_t* sb = sa + Cfg::A_BYTES;
        mbar_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
        const int k0 = kb * GEMM_BK;
        if (A_MN) {
#pragma unroll
          for (int a = 0; a < GEMM_BM / 64; ++a) tma_load_2d(sa + a * (GEMM_BK * 128), &tmA, &full_bar[stage], m0 + 64 * a, k0);
        } else {
          tma_load_2d(sa, &tmA, &full_bar[stage], k0, m0);
        }
        if (B_MN) {
#pragma unroll
          for (int a = 0; a < BN / 64; ++a) tma_load_2d(sb + a * (GEMM_BK * 128), &tmB, &full_bar[stage], n0 + 64 * a, k0);
        } else {
          tma_load_2d(sb, &tmB, &full_bar[stage], k0, n0);
        }
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer (single thread) ----------------
    constexpr uint32_t IDESC = umma_idesc_bf16(GEMM_BM, BN, A_MN, B_MN);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++it) {
      const int kb0 = (u / num_tiles) * kbs, kb1 = min(num_kb, kb0 + kbs);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + stage * Cfg::STAGE_BYTES);
        const uint32_t sb = sa + Cfg::A_BYTES;
#pragma unroll
        for (int kk = 0; kk < GEMM_BK / 16; ++kk) {
          const uint64_t ad = A_MN ? umma_desc_sw128(sa + kk * 2048, GEMM_BK * 128, 1024)
                                   : umma_desc_sw128(sa + kk * 32, 16, 1024);
          const uint64_t bd = B_MN ? umma_desc_sw128(sb + kk * 2048, GEMM_BK * 128, 1024)
                                   : umma_desc_sw128(sb + kk * 32, 16, 1024);
          mma_bf16_ss(d_tmem, ad, bd, IDESC, (kb != kb0) || (kk != 0));
        }
        mma_commit(&empty_bar[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      mma_commit(&tfull_bar[acc]);
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM -> registers -> global ----------------
    const int wq = warp & 3;
    const int row_in_tile = wq * 32 + lane;
    int it = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++it) {
      const int tile = u % num_tiles, split = u / num_tiles;
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int m0 = (tile % num_m) * GEMM_BM;
      const int n0 = (tile / num_m) * BN;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + ((uint32_t)(wq * 32) << 16) + acc * BN;
      const int row = m0 + row_in_tile;
      const bool row_ok = row < args.M;
      if constexpr (RopeHd<EPI>::value != 0) {
        // RoPE fused into the QKV projection: each thread owns one row, a head's hd columns sit
        // in one 256-wide tile, and the rotate-half pairs (j, j + hd/2) are both in registers.
        constexpr int HD = RopeHd<EPI>::value;
        const int t = row % args.rope_T;
        const bool rope_tile = n0 < args.rope_cols;  // rope_cols and n0 are multiples of 256 / HD
        // one row per thread, one position per row: the row's cos/sin are reused by every head of
        // the tile (kept in registers for HD=64, re-read from L1 for HD=128)
        float2 cs_reg[HD == 64 ? 32 : 1];
        const float2* cs_row = reinterpret_cast<const float2*>(args.rope_cs) + (size_t)t * (HD / 2);
        if constexpr (HD == 64) {
          if (rope_tile && row_ok) {
#pragma unroll
            for (int j = 0; j < 32; ++j) cs_reg[j] = cs_row[j];
          }
        }
#pragma unroll 1
        for (int hb = 0; hb < BN; hb += HD) {
          float f[HD];
#pragma unroll
          for (int c = 0; c < HD; c += 32) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(t_row + hb + c, v);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) f[c + j] = __uint_as_float(v[j]);
          }
          if (row_ok && n0 + hb < args.N) {
            if (n0 + hb < args.rope_cols) {
#pragma unroll
              for (int j = 0; j < HD / 2; ++j) {
                float2 w;
                if constexpr (HD == 64) w = cs_reg[j];
                else w = cs_row[j];
                const float a = f[j], b = f[j + HD / 2];
                f[j] = a * w.x - b * w.y;
                f[j + HD / 2] = b * w.x + a * w.y;
              }
            }
            uint4* C4 = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(args.C) + (size_t)row * args.ldc + n0 + hb);
#pragma unroll
            for (int q = 0; q < HD / 8; ++q)
              C4[q] = make_uint4(pack_bf16(f[8 * q], f[8 * q + 1]), pack_bf16(f[8 * q + 2], f[8 * q + 3]),
                                 pack_bf16(f[8 * q + 4], f[8 * q + 5]), pack_bf16(f[8 * q + 6], f[8 * q + 7]));
          }
        }
      } else if (EPI == EPI_SWIGLU) {
#pragma unroll 1
        for (int c = 0; c < BN / 2; c += 32) {
          uint32_t g[32], u[32];
          tmem_ld_32x32b_x32(t_row + c, g);
          tmem_ld_32x32b_x32(t_row + BN / 2 + c, u);
          tmem_ld_wait();
          if (row_ok && n0 + c < args.N) {
            __nv_bfloat16* H = reinterpret_cast<__nv_bfloat16*>(args.C) + (size_t)row * args.ldc + (n0 / 2 + c);
            __nv_bfloat16* GU = reinterpret_cast<__nv_bfloat16*>(args.C2) + (size_t)row * args.ldc2 + n0 + c;
            uint32_t hp[16], gp[16], up[16];
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              float g0 = __uint_as_float(g[j]), g1 = __uint_as_float(g[j + 1]);
              float u0 = __uint_as_float(u[j]), u1 = __uint_as_float(u[j + 1]);
              // silu computed from the bf16-rounded pre-activations the backward pass will see
              float2 gr = unpack_bf16(pack_bf16(g0, g1));
              float2 ur = unpack_bf16(pack_bf16(u0, u1));
              float h0 = gr.x / (1.f + __expf(-gr.x)) * ur.x;
              float h1 = gr.y / (1.f + __expf(-gr.y)) * ur.y;
              hp[j / 2] = pack_bf16(h0, h1);
              gp[j / 2] = pack_bf16(g0, g1);
              up[j / 2] = pack_bf16(u0, u1);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              reinterpret_cast<uint4*>(H)[q] = make_uint4(hp[4 * q], hp[4 * q + 1], hp[4 * q + 2], hp[4 * q + 3]);
              reinterpret_cast<uint4*>(GU)[q] = make_uint4(gp[4 * q], gp[4 * q + 1], gp[4 * q + 2], gp[4 * q + 3]);
              reinterpret_cast<uint4*>(GU + BN / 2)[q] =
                  make_uint4(up[4 * q], up[4 * q + 1], up[4 * q + 2], up[4 * q + 3]);
            }
          }
        }
      } else {
        const bool ordered = EPI == EPI_F32 && args.splits > 1;
        if (ordered) {
          // deterministic split-K: split s adds into C only after split s-1 of this tile did
          int v;
          do {
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(args.sem + tile) : "memory");
          } while (v != split);
        }
        const bool add = (split > 0) || (args.beta != 0.f);
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(t_row + c, v);
          tmem_ld_wait();
          if (row_ok && n0 + c < args.N) {
            if (EPI == EPI_F32) {
              float* C = reinterpret_cast<float*>(args.C) + (size_t)row * args.ldc + n0 + c;
              float4* C4 = reinterpret_cast<float4*>(C);
              if (add) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                  float4 o = C4[q];
                  o.x += __uint_as_float(v[4 * q]);
                  o.y += __uint_as_float(v[4 * q + 1]);
                  o.z += __uint_as_float(v[4 * q + 2]);
                  o.w += __uint_as_float(v[4 * q + 3]);
                  C4[q] = o;
                }
              } else {
#pragma unroll
                for (int q = 0; q < 8; ++q)
                  C4[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                      __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
              }
            } else {
              float f[32];
#pragma unroll
              for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
              if (EPI == EPI_BF16_RESID) {
                const uint4* R4 = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(args.R) +
                                                                 (size_t)row * args.ldr + n0 + c);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  uint4 r = R4[q];
                  float2 a = unpack_bf16(r.x), b = unpack_bf16(r.y), cc = unpack_bf16(r.z), d = unpack_bf16(r.w);
                  f[8 * q + 0] += a.x; f[8 * q + 1] += a.y; f[8 * q + 2] += b.x; f[8 * q + 3] += b.y;
                  f[8 * q + 4] += cc.x; f[8 * q + 5] += cc.y; f[8 * q + 6] += d.x; f[8 * q + 7] += d.y;
                }
              }
              uint4* C4 = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(args.C) + (size_t)row * args.ldc + n0 + c);
#pragma unroll
              for (int q = 0; q < 4; ++q)
                C4[q] = make_uint4(pack_bf16(f[8 * q], f[8 * q + 1]), pack_bf16(f[8 * q + 2], f[8 * q + 3]),
                                   pack_bf16(f[8 * q + 4], f[8 * q + 5]), pack_bf16(f[8 * q + 6], f[8 * q + 7]));
            }
          }
        }
        if (ordered) {
          __threadfence();
          asm volatile("bar.sync 1, 128;" ::: "memory");  // the 4 epilogue warps
          if (threadIdx.x == 128) atomicExch(args.sem + tile, split + 1 == args.splits ? 0 : split + 1);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
}

// ----------------------------------------------------------------------------
// host side
// ----------------------------------------------------------------------------
static int make_tmap_bf16_2d(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                             uint32_t box_inner, uint32_t box_outer) {
  auto encode = get_tensor_map_encoder();
  if (!encode) return set_error(SPX_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char msg[256];
    snprintf(msg, sizeof msg, "cuTensorMapEncodeTiled failed (%d): inner=%llu outer=%llu ld=%llu box=%ux%u", (int)r,
             (unsigned long long)inner, (unsigned long long)outer, (unsigned long long)ld_elems, box_inner, box_outer);
    return set_error(SPX_ERR_CUDA, msg);
  }
  return SPX_OK;
}

template <int BN, bool A_MN, bool B_MN, int EPI>
static int launch_gemm(const void* A, const void* B, long long lda, long long ldb, const GemmArgs& args,
                       cudaStream_t stream) {
  using Cfg = GemmCfg<BN>;
  CUtensorMap ta, tb;
  int rc;
  // A operand: rows = M, contraction = K
  if (A_MN) rc = make_tmap_bf16_2d(&ta, A, args.M, args.K, lda, 64, GEMM_BK);
  else rc = make_tmap_bf16_2d(&ta, A, args.K, args.M, lda, GEMM_BK, GEMM_BM);
  if (rc) return rc;
  if (B_MN) rc = make_tmap_bf16_2d(&tb, B, args.N, args.K, ldb, 64, GEMM_BK);
  else rc = make_tmap_bf16_2d(&tb, B, args.K, args.N, ldb, GEMM_BK, BN);
  if (rc) return rc;

  auto kern = gemm_bf16_kernel<BN, A_MN, B_MN, EPI>;
  static bool attr_set = false;  // one per template instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(gemm)");
    attr_set = true;
  }
  const int tiles = ((args.M + GEMM_BM - 1) / GEMM_BM) * ((args.N + BN - 1) / BN) * args.splits;
  const int grid = tiles < num_sms() ? tiles : num_sms();
  kern<<<grid, GEMM_THREADS, Cfg::SMEM_BYTES, stream>>>(ta, tb, args);
  return check_launch("gemm_bf16_kernel");
}

template <int BN, int EPI>
static int dispatch_major(const void* A, const void* B, long long lda, long long ldb, int a_mn, int b_mn,
                          const GemmArgs& args, cudaStream_t s) {
  if (!a_mn && !b_mn) return launch_gemm<BN, false, false, EPI>(A, B, lda, ldb, args, s);
  if (!a_mn && b_mn) return launch_gemm<BN, false, true, EPI>(A, B, lda, ldb, args, s);
  if (a_mn && b_mn) return launch_gemm<BN, true, true, EPI>(A, B, lda, ldb, args, s);
  return launch_gemm<BN, true, false, EPI>(A, B, lda, ldb, args, s);
}

// Per-device split-K semaphores, registered once by the caller (no allocation in the GEMM path).
static int* g_sem[64] = {nullptr};
static int64_t g_sem_n[64] = {0};

// Split-K factor for the fp32 (wgrad) epilogue: maximise wave efficiency of tiles x splits on the
// SMs, keeping >= 8 k-blocks per split; splits add into C in split order (deterministic).
static void pick_splits(GemmArgs& a, int bn) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int tiles = ((a.M + GEMM_BM - 1) / GEMM_BM) * ((a.N + bn - 1) / bn);
  const int num_kb = (a.K + GEMM_BK - 1) / GEMM_BK;
  if (dev < 0 || dev >= 64 || g_sem[dev] == nullptr || tiles > g_sem_n[dev]) return;
  const int sms = num_sms();
  double best = 0.0;
  int best_s = 1;
  for (int s = 1; s <= 8; ++s) {
    const int kbs = (num_kb + s - 1) / s;
    if (kbs < 8 && s > 1) break;
    const int s_eff = (num_kb + kbs - 1) / kbs;
    const long units = (long)tiles * s_eff;
    const double eff = (double)units / (double)(((units + sms - 1) / sms) * sms);
    if (eff > best + 0.05) {
      best = eff;
      best_s = s_eff;
    }
  }
  a.splits = best_s;
  a.sem = best_s > 1 ? g_sem[dev] : nullptr;
}

static int pick_bn(int M, int N) {
  auto eff = [&](int bn) {
    const long tiles = (long)((M + GEMM_BM - 1) / GEMM_BM) * ((N + bn - 1) / bn);
    const long w = (tiles + num_sms() - 1) / num_sms();
    return (double)tiles / (double)(w * num_sms());
  };
  return (eff(256) >= 0.9 * eff(128)) ? 256 : 128;
}

}  // namespace spx

using namespace spx;

extern "C" int spx_gemm_set_workspace(int32_t* sem, int64_t n_ints) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return set_error(SPX_ERR_ARG, "gemm workspace: bad device");
  if (sem == nullptr || n_ints <= 0) {
    g_sem[dev] = nullptr;
    g_sem_n[dev] = 0;
    return SPX_OK;
  }
  cudaError_t e = cudaMemset(sem, 0, (size_t)n_ints * sizeof(int32_t));
  if (e != cudaSuccess) return set_cuda_error(e, "gemm workspace memset");
  g_sem[dev] = sem;
  g_sem_n[dev] = n_ints;
  return SPX_OK;
}

extern "C" int spx_gemm_bf16_rope(const void* A, const void* B, void* C, int64_t M, int64_t N, int64_t K, int64_t lda,
                                  int64_t ldb, int64_t ldc, const float* cos_sin, int64_t rope_cols, int64_t T,
                                  int64_t head_dim, void* stream) {
  if (M <= 0 || N <= 0 || K <= 0) return set_error(SPX_ERR_ARG, "gemm_rope: non-positive shape");
  if (N % 32 != 0 || K % 8 != 0 || lda % 8 != 0 || ldb % 8 != 0)
    return set_error(SPX_ERR_ARG, "gemm_rope: N % 32, K/lda/ldb % 8 required");
  if (head_dim != 64 && head_dim != 128) return set_error(SPX_ERR_ARG, "gemm_rope: head_dim must be 64 or 128");
  if (rope_cols % head_dim || T <= 0) return set_error(SPX_ERR_ARG, "gemm_rope: rope_cols must be whole heads");
  GemmArgs args{(int)M, (int)N, (int)K, C, nullptr, nullptr, (long long)ldc, (long long)ldc, 0, 0.f,
                cos_sin, (int)rope_cols, (int)T, 1, nullptr};
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (head_dim == 64) return launch_gemm<256, false, false, EPI_ROPE64>(A, B, lda, ldb, args, s);
  return launch_gemm<256, false, false, EPI_ROPE128>(A, B, lda, ldb, args, s);
}

extern "C" int spx_gemm_bf16(const void* A, const void* B, void* C, const void* R, void* C2, int64_t M, int64_t N,
                             int64_t K, int64_t lda, int64_t ldb, int64_t ldc, int64_t ldc2, int32_t a_mn_major,
                             int32_t b_mn_major, int32_t epilogue, float beta, void* stream) {
  if (M <= 0 || N <= 0 || K <= 0) return set_error(SPX_ERR_ARG, "gemm: non-positive shape");
  if (N % 32 != 0) return set_error(SPX_ERR_ARG, "gemm: N must be a multiple of 32");
  if (K % 8 != 0 || lda % 8 != 0 || ldb % 8 != 0) return set_error(SPX_ERR_ARG, "gemm: K/lda/ldb must be multiples of 8");
  if (((uintptr_t)A | (uintptr_t)B) & 15) return set_error(SPX_ERR_ARG, "gemm: A/B must be 16-byte aligned");
  if (epilogue < 0 || epilogue > 3) return set_error(SPX_ERR_ARG, "gemm: bad epilogue");
  if (epilogue == EPI_SWIGLU && (N % 256 != 0 || C2 == nullptr))
    return set_error(SPX_ERR_ARG, "gemm: swiglu epilogue needs N % 256 == 0 and a GU output");
  if (epilogue == EPI_BF16_RESID && R == nullptr) return set_error(SPX_ERR_ARG, "gemm: residual epilogue needs R");
  GemmArgs args{(int)M, (int)N, (int)K, C, R, C2, (long long)ldc, (long long)ldc, (long long)ldc2, beta, nullptr, 0, 1,
                1, nullptr};
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int bn = (epilogue == EPI_SWIGLU || epilogue == EPI_F32) ? 256 : pick_bn((int)M, (int)N);
  if (epilogue == EPI_F32) pick_splits(args, bn);
  switch (epilogue) {
    case EPI_BF16:
      return bn == 256 ? dispatch_major<256, EPI_BF16>(A, B, lda, ldb, a_mn_major, b_mn_major, args, s)
                       : dispatch_major<128, EPI_BF16>(A, B, lda, ldb, a_mn_major, b_mn_major, args, s);
    case EPI_BF16_RESID:
      return bn == 256 ? dispatch_major<256, EPI_BF16_RESID>(A, B, lda, ldb, a_mn_major, b_mn_major, args, s)
                       : dispatch_major<128, EPI_BF16_RESID>(A, B, lda, ldb, a_mn_major, b_mn_major, args, s);
    case EPI_F32:
      return bn == 256 ? dispatch_major<256, EPI_F32>(A, B, lda, ldb, a_mn_major, b_mn_major, args, s)
                       : dispatch_major<128, EPI_F32>(A, B, lda, ldb, a_mn_major, b_mn_major, args, s);
    default:
      return dispatch_major<256, EPI_SWIGLU>(A, B, lda, ldb, a_mn_major, b_mn_major, args, s);
  }
}
