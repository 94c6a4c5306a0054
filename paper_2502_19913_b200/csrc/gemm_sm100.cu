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
#include <cstdlib>
#include <cstring>

#include "spx_common.cuh"
#include "spx_internal.h"

namespace spx {

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;
constexpr int GEMM_EPI_WARPS = 8;                          // 2 per TMEM lane quadrant
constexpr int GEMM_THREADS = 128 + 32 * GEMM_EPI_WARPS;   // + TMA, MMA, TMEM-alloc, spare warps

enum GemmEpilogue : int {
  EPI_BF16 = 0,        // C(bf16) = acc
  EPI_BF16_RESID = 1,  // C(bf16) = acc + R(bf16)            (R may alias C)
  EPI_F32 = 2,         // C(f32)  = acc (+ C if beta != 0)   (wgrad accumulation)
  EPI_SWIGLU = 3,      // H(bf16)[m, N/2] = silu(g)*u ; GU(bf16)[m, N] = (g,u) raw, 128-col interleave
  EPI_ROPE64 = 4,      // C(bf16) = acc with rotate-half RoPE on columns < rope_cols (head dim 64)
  EPI_ROPE128 = 5,     // same, head dim 128
  EPI_SWIGLU_BWD = 6,  // D = dh [M, F]; R = gu [M, 2F] (128-col gate/up interleave) -> C2 = dgu [M, 2F]
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
  static constexpr int STAGING_BYTES = GEMM_EPI_WARPS * 4096;  // one 32-row x 128-byte box per epilogue warp
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + STAGING_BYTES + 1024 /*align slack*/ + 256 /*barriers*/;
};

struct GemmArgs {
  int M, N, K;
  void* C;
  const void* R;
  void* C2;
  long long ldc, ldr, ldc2;
  float beta;
  const float* rope_cs;  // [hd/2][T][2] (cos, sin), position-minor
  int rope_cols, rope_T;
  int splits;            // split-K factor (EPI_F32 only); units = tiles * splits
  int* sem;              // per-tile split-order semaphores (zero between launches)
};

template <int BN, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmC2,
                     const GemmArgs args) {
  using Cfg = GemmCfg<BN>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES + Cfg::STAGING_BYTES);
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
    tma_prefetch_desc(&tmC);
    if (EPI == EPI_SWIGLU || EPI == EPI_SWIGLU_BWD) tma_prefetch_desc(&tmC2);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], GEMM_EPI_WARPS);
    }
    fence_barrier_init();
    fence_proxy_async();
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // upstream grid complete before any dependent global access

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
    pdl_trigger();  // all loads issued: let the next kernel launch and run its prologue
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
    // ---------------- epilogue: TMEM -> registers -> fused op -> swizzled smem box -> TMA ----------
    // 8 epilogue warps: warp w reads TMEM lanes (tile rows) 32*(w%4).. and the column half
    // (w-4)/4 of the tile.  A warp writes its rows as 32-row x 128-byte boxes through a private
    // 4 KB staging buffer (SWIZZLE_128B: its 16-byte smem stores are bank-conflict free) and one
    // lane issues the TMA store (or reduce-add for fp32 accumulation); the TMA unit clips rows and
    // columns outside the matrix.
    const int wq = warp & 3;
    const int half = (warp - 4) >> 2;
    const int cb = half * (BN / 2);  // this warp's first tile column
    uint8_t* box = smem + STAGES * Cfg::STAGE_BYTES + (warp - 4) * 4096;
    auto box_acquire = [&]() {
      if (lane == 0) bulk_wait_read<0>();  // the previous store from this buffer has read it
      __syncwarp();
    };
    auto box_put = [&](int r, int j, uint4 v) {
      *reinterpret_cast<uint4*>(box + r * 128 + ((j ^ (r & 7)) << 4)) = v;
    };
    auto box_get = [&](int r, int j) -> uint4 {
      return *reinterpret_cast<const uint4*>(box + r * 128 + ((j ^ (r & 7)) << 4));
    };
    auto box_issue = [&](const CUtensorMap* m, int c0, int c1, bool reduce) {
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        if (reduce) tma_reduce_add_2d(m, box, c0, c1);
        else tma_store_2d(m, box, c0, c1);
        bulk_commit();
      }
    };
    // 32 fp32 values -> 16-byte chunks j0..j0+3 of this lane's row (bf16)
    auto put32 = [&](int j0, const float* f) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        box_put(lane, j0 + j,
                make_uint4(pack_bf16(f[8 * j], f[8 * j + 1]), pack_bf16(f[8 * j + 2], f[8 * j + 3]),
                           pack_bf16(f[8 * j + 4], f[8 * j + 5]), pack_bf16(f[8 * j + 6], f[8 * j + 7])));
    };
    auto ld32 = [&](uint32_t taddr, float* f) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(taddr, v);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
    };
    int it = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++it) {
      const int tile = u % num_tiles, split = u / num_tiles;
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int m0 = (tile % num_m) * GEMM_BM;
      const int n0 = (tile / num_m) * BN;
      const int rbase = m0 + wq * 32;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + ((uint32_t)(wq * 32) << 16) + acc * BN;
      if constexpr (EPI == EPI_F32) {
        const bool ordered = args.splits > 1;
        if (ordered) {
          // deterministic split-K: split s adds into C only after split s-1 of this tile did
          int v;
          do {
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(args.sem + tile) : "memory");
          } while (v != split);
        }
        const bool add = (split > 0) || (args.beta != 0.f);
#pragma unroll 1
        for (int c = cb; c < cb + BN / 2 && n0 + c < args.N; c += 32) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(t_row + c, v);
          tmem_ld_wait();
          box_acquire();
#pragma unroll
          for (int j = 0; j < 8; ++j) box_put(lane, j, make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
          box_issue(&tmC, n0 + c, rbase, add);
        }
        if (ordered) {
          if (lane == 0) bulk_wait<0>();  // this warp's adds have landed in global memory
          __syncwarp();
          __threadfence();
          asm volatile("bar.sync 1, %0;" ::"n"(32 * GEMM_EPI_WARPS) : "memory");
          if (threadIdx.x == 128) atomicExch(args.sem + tile, split + 1 == args.splits ? 0 : split + 1);
        }
      } else if constexpr (EPI == EPI_SWIGLU) {
        // tile columns [0,128) are gate, [128,256) the matching up rows of the interleaved weight;
        // this warp handles gate/up columns [64*half, 64*half + 64)
        const int c = 64 * half;
        if (n0 + c < args.N) {
          float g[32], uu[32], h[32];
#pragma unroll 1
          for (int part = 0; part < 3; ++part) {  // 0: H, 1: gate, 2: up
            box_acquire();
#pragma unroll 1
            for (int q = 0; q < 2; ++q) {
              ld32(t_row + c + 32 * q, g);
              ld32(t_row + BN / 2 + c + 32 * q, uu);
              if (part == 0) {
#pragma unroll
                for (int j = 0; j < 32; j += 2) {
                  // silu from the bf16-rounded pre-activations the backward pass will see
                  const float2 gr = unpack_bf16(pack_bf16(g[j], g[j + 1]));
                  const float2 ur = unpack_bf16(pack_bf16(uu[j], uu[j + 1]));
                  h[j] = gr.x * __frcp_rn(1.f + __expf(-gr.x)) * ur.x;
                  h[j + 1] = gr.y * __frcp_rn(1.f + __expf(-gr.y)) * ur.y;
                }
                put32(4 * q, h);
              } else {
                put32(4 * q, part == 1 ? g : uu);
              }
            }
            if (part == 0) box_issue(&tmC, n0 / 2 + c, rbase, false);
            else if (part == 1) box_issue(&tmC2, n0 + c, rbase, false);
            else box_issue(&tmC2, n0 + BN / 2 + c, rbase, false);
          }
        }
      } else if constexpr (EPI == EPI_SWIGLU_BWD) {
        // dh tile columns [cb, cb+128) = one 128-column gate/up block of the interleaved layout:
        //   dgate = dh * up * sig(g) * (1 + g (1 - sig(g))),  dup = dh * silu(g)
        const int fc = n0 + cb;  // first dh column of this warp
        if (fc < args.N) {
          const int blk = fc >> 7;
          const int row = rbase + lane;
          const __nv_bfloat16* gur =
              reinterpret_cast<const __nv_bfloat16*>(args.R) + (size_t)(row < args.M ? row : 0) * args.ldr + blk * 256;
#pragma unroll 1
          for (int c = 0; c < 128; c += 64) {
#pragma unroll 1
            for (int part = 0; part < 2; ++part) {  // 0: dgate box, 1: dup box
              box_acquire();
#pragma unroll 1
              for (int q = 0; q < 2; ++q) {
                float dh[32], o[32];
                ld32(t_row + cb + c + 32 * q, dh);
#pragma unroll
                for (int j8 = 0; j8 < 4; ++j8) {
                  const uint4 g4 = *reinterpret_cast<const uint4*>(gur + c + 32 * q + 8 * j8);
                  const uint4 u4 = *reinterpret_cast<const uint4*>(gur + 128 + c + 32 * q + 8 * j8);
                  const uint32_t gw[4] = {g4.x, g4.y, g4.z, g4.w}, uw[4] = {u4.x, u4.y, u4.z, u4.w};
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    const float2 g2 = unpack_bf16(gw[e]), u2 = unpack_bf16(uw[e]);
                    const int j = 8 * j8 + 2 * e;
                    const float s0 = __frcp_rn(1.f + __expf(-g2.x)), s1 = __frcp_rn(1.f + __expf(-g2.y));
                    if (part == 0) {
                      o[j] = dh[j] * u2.x * s0 * (1.f + g2.x * (1.f - s0));
                      o[j + 1] = dh[j + 1] * u2.y * s1 * (1.f + g2.y * (1.f - s1));
                    } else {
                      o[j] = dh[j] * g2.x * s0;
                      o[j + 1] = dh[j + 1] * g2.y * s1;
                    }
                  }
                }
                put32(4 * q, o);
              }
              box_issue(&tmC2, blk * 256 + 128 * part + c, rbase, false);
            }
          }
        }
      } else if constexpr (RopeHd<EPI>::value != 0) {
        // RoPE fused into the QKV projection.  The table is position-minor ([hd/2][T] of
        // (cos, sin)), so for a pair index j the warp's 32 consecutive rows read one contiguous
        // 256-byte segment.  Output box b of a head holds columns [64b, 64b+64): for HD=64 the
        // rotated x1 (cols 0-31) and x2 (32-63) halves; for HD=128 box 0 is all x1' and box 1 x2'.
        constexpr int HD = RopeHd<EPI>::value;
        const int row = rbase + lane;
        const int t = (row < args.M ? row : 0) % args.rope_T;
        const float2* cs = reinterpret_cast<const float2*>(args.rope_cs) + t;
        const int T = args.rope_T;
#pragma unroll 1
        for (int hb = cb; hb < cb + BN / 2 && n0 + hb < args.N; hb += HD) {
          const bool rot = n0 + hb < args.rope_cols;
#pragma unroll 1
          for (int bx = 0; bx < HD / 64; ++bx) {
            box_acquire();
#pragma unroll 1
            for (int q = 0; q < 2; ++q) {
              // HD=64: q=0 -> x1' (pairs 0-31), q=1 -> x2' (pairs 0-31)
              // HD=128: bx selects x1'/x2', q selects pairs 32q..32q+31
              const int pair0 = (HD == 64) ? 0 : 32 * q;
              const bool second = (HD == 64) ? (q == 1) : (bx == 1);
              float x1[32], x2[32];
              ld32(t_row + hb + pair0, x1);
              ld32(t_row + hb + HD / 2 + pair0, x2);
              if (rot) {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                  const float2 w = cs[(size_t)(pair0 + j) * T];
                  const float a = x1[j], b = x2[j];
                  x1[j] = second ? (b * w.x + a * w.y) : (a * w.x - b * w.y);
                }
              } else if (second) {
#pragma unroll
                for (int j = 0; j < 32; ++j) x1[j] = x2[j];
              }
              put32(4 * q, x1);
            }
            box_issue(&tmC, n0 + hb + 64 * bx, rbase, false);
          }
        }
      } else {
        // plain bf16 store, optionally + residual R (read coalesced into the staging box first)
#pragma unroll 1
        for (int c = cb; c < cb + BN / 2 && n0 + c < args.N; c += 64) {
          box_acquire();
          if constexpr (EPI == EPI_BF16_RESID) {
            const __nv_bfloat16* R = reinterpret_cast<const __nv_bfloat16*>(args.R);
            uint4 rv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int r = (lane >> 3) + 4 * i, j = lane & 7;
              const int grow = rbase + r, gcol = n0 + c + 8 * j;
              rv[i] = make_uint4(0, 0, 0, 0);
              if (grow < args.M && gcol < args.N) rv[i] = *reinterpret_cast<const uint4*>(R + (size_t)grow * args.ldr + gcol);
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) box_put((lane >> 3) + 4 * i, lane & 7, rv[i]);
            __syncwarp();
          }
#pragma unroll 1
          for (int q = 0; q < 2; ++q) {
            float f[32];
            ld32(t_row + c + 32 * q, f);
            if constexpr (EPI == EPI_BF16_RESID) {
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const uint4 r4 = box_get(lane, 4 * q + j);
                const float2 a0 = unpack_bf16(r4.x), a1 = unpack_bf16(r4.y), a2 = unpack_bf16(r4.z),
                             a3 = unpack_bf16(r4.w);
                f[8 * j + 0] += a0.x; f[8 * j + 1] += a0.y; f[8 * j + 2] += a1.x; f[8 * j + 3] += a1.y;
                f[8 * j + 4] += a2.x; f[8 * j + 5] += a2.y; f[8 * j + 6] += a3.x; f[8 * j + 7] += a3.y;
              }
            }
            put32(4 * q, f);
          }
          box_issue(&tmC, n0 + c, rbase, false);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
    }
    if (lane == 0) bulk_wait<0>();  // staging smem must outlive the TMA reads
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
static int make_tmap_2d(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                        uint32_t box_inner, uint32_t box_outer, bool f32 = false) {
  auto encode = get_tensor_map_encoder();
  if (!encode) return set_error(SPX_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * (f32 ? 4 : 2)};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                      const_cast<void*>(ptr), dims, strides, box, estr,
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
  if (A_MN) rc = make_tmap_2d(&ta, A, args.M, args.K, lda, 64, GEMM_BK);
  else rc = make_tmap_2d(&ta, A, args.K, args.M, lda, GEMM_BK, GEMM_BM);
  if (rc) return rc;
  if (B_MN) rc = make_tmap_2d(&tb, B, args.N, args.K, ldb, 64, GEMM_BK);
  else rc = make_tmap_2d(&tb, B, args.K, args.N, ldb, GEMM_BK, BN);
  if (rc) return rc;

  // output boxes: 32 rows x 128 bytes (64 bf16 or 32 fp32 columns), SWIZZLE_128B
  CUtensorMap tc, tc2;
  memset(&tc2, 0, sizeof tc2);
  if (EPI == EPI_F32) rc = make_tmap_2d(&tc, args.C, args.N, args.M, args.ldc, 32, 32, true);
  else if (EPI == EPI_SWIGLU) rc = make_tmap_2d(&tc, args.C, args.N / 2, args.M, args.ldc, 64, 32);
  else if (EPI == EPI_SWIGLU_BWD) rc = make_tmap_2d(&tc, args.C2, 2 * args.N, args.M, args.ldc2, 64, 32);
  else rc = make_tmap_2d(&tc, args.C, args.N, args.M, args.ldc, 64, 32);
  if (rc) return rc;
  if (EPI == EPI_SWIGLU) {
    rc = make_tmap_2d(&tc2, args.C2, args.N, args.M, args.ldc2, 64, 32);
    if (rc) return rc;
  }
  if (EPI == EPI_SWIGLU_BWD) tc2 = tc;
  auto kern = gemm_bf16_kernel<BN, A_MN, B_MN, EPI>;
  static bool attr_set = false;  // one per template instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(gemm)");
    attr_set = true;
  }
  const int tiles = ((args.M + GEMM_BM - 1) / GEMM_BM) * ((args.N + BN - 1) / BN) * args.splits;
  const int grid = tiles < num_sms() ? tiles : num_sms();
  spx_launch_check(launch_k(kern, dim3(grid), dim3(GEMM_THREADS), Cfg::SMEM_BYTES, stream, ta, tb, tc, tc2, args));
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
  static const int enabled = [] {
    const char* e = getenv("SPX_SPLITK");
    return e ? atoi(e) : 0;
  }();
  if (!enabled) return;
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
  if (epilogue < 0 || epilogue > 6 || epilogue == 4 || epilogue == 5) return set_error(SPX_ERR_ARG, "gemm: bad epilogue");
  if (epilogue == EPI_SWIGLU_BWD && (N % 128 != 0 || C2 == nullptr || R == nullptr))
    return set_error(SPX_ERR_ARG, "gemm: swiglu-bwd epilogue needs N % 128 == 0, gu (R) and dgu (C2)");
  if (epilogue == EPI_SWIGLU && (N % 256 != 0 || C2 == nullptr))
    return set_error(SPX_ERR_ARG, "gemm: swiglu epilogue needs N % 256 == 0 and a GU output");
  if (epilogue == EPI_BF16_RESID && R == nullptr) return set_error(SPX_ERR_ARG, "gemm: residual epilogue needs R");
  GemmArgs args{(int)M, (int)N, (int)K, C, R, C2, (long long)ldc, (long long)(epilogue == EPI_SWIGLU_BWD ? ldc2 : ldc),
                (long long)ldc2, beta, nullptr, 0, 1, 1, nullptr};
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int bn = (epilogue == EPI_SWIGLU || epilogue == EPI_F32 || epilogue == EPI_SWIGLU_BWD) ? 256
                                                                                               : pick_bn((int)M, (int)N);
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
    case EPI_SWIGLU_BWD:
      return dispatch_major<256, EPI_SWIGLU_BWD>(A, B, lda, ldb, a_mn_major, b_mn_major, args, s);
    default:
      return dispatch_major<256, EPI_SWIGLU>(A, B, lda, ldb, a_mn_major, b_mn_major, args, s);
  }
}
