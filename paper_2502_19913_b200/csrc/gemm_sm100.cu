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
  EPI_XENT = 7,        // C(bf16) = acc (logits) and C2(f32)[m, 2*(N/128)] = per 128-column block
                       // (max, sum exp(x - max)) of the bf16-rounded logits (cross-entropy partials)
  EPI_ATTN_DELTA = 8,  // attention-output dgrad: C(bf16) = acc (dO), R = O (bf16, same layout), and per
                       // (row, head) D = sum_c bf16(acc) * O, written with lse*log2e in the [B, H, T]
                       // layout of the attention backward's workspace (spx_gemm_bf16_attn_delta)
};

template <int EPI>
struct RopeHd {
  static constexpr int value = EPI == EPI_ROPE64 ? 64 : (EPI == EPI_ROPE128 ? 128 : 0);
};

// CG = 2: a CTA pair (cluster of 2 on one TPC) computes a 256 x BN tile with cta_group::2 MMAs;
// each CTA stages its own 128 rows of A and half (BN/2 rows) of B, so per-SM operand traffic from
// L2 drops from 48 KB to 32 KB per 64-deep k-block (the 1-CTA kernel is L2->SM bandwidth bound).
// NBOX: 32-row x 128-byte staging boxes per epilogue warp (2 for the three-output SwiGLU epilogue).
template <int BN, int CG = 1, int NBOX = 1>
struct GemmCfg {
  static constexpr int A_BYTES = GEMM_BM * GEMM_BK * 2;
  static constexpr int B_BYTES = (BN / CG) * GEMM_BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGING_BYTES = GEMM_EPI_WARPS * 4096 * NBOX;
  static constexpr int FIT = (232448 - 1024 - 512 - STAGING_BYTES) / STAGE_BYTES;  // 227 KB opt-in limit
  static constexpr int STAGES = FIT < 6 ? FIT : 6;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + STAGING_BYTES + 1024 /*align slack*/ + 512 /*barriers, problem table*/;
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
  float* ws;             // split partials [splits][ws_rows][N] fp32 (tensor map tmC2)
  long long ws_rows;     // rows per split in ws (M rounded up to whole tiles)
  int probe;  // pipeline probe (SPX_GEMM_PROBE, benchmarking only): 1 no MMAs, 2 no loads, 3 no epilogue,
              // 4 MMAs only, 5 no output stores, 6 loads only
  int tma_store;  // bf16 outputs leave the staging box by TMA store (SPX_GEMM_TMA_STORE=1) instead of st.global
  int n_major;    // problem 0's tiles walk N first (consecutive units share an A row block; pick_raster)
  // EPI_ATTN_DELTA: lse [B, H, T] (natural log) in, delta [2][B, H, T] out (D, then lse*log2e)
  const float* lse;
  float* delta;
  int delta_hd, delta_T, delta_H;
  long long delta_total;  // B * H * T
};

// Grouped launch (EPI_F32 only, no split-K): up to GEMM_GROUP_MAX independent problems share one
// persistent launch -- the weight-gradient GEMMs of a decoder layer -- so their tiles fill the SMs
// together instead of each leaving a partial last wave.  Problem 0 is described by the kernel's
// own maps and GemmArgs; problems 1.. by this table.
constexpr int GEMM_GROUP_MAX = 4;
struct GemmProb {
  int M, N, K;
  float beta;
};
struct GemmGroup {
  CUtensorMap ta[GEMM_GROUP_MAX - 1], tb[GEMM_GROUP_MAX - 1], tc[GEMM_GROUP_MAX - 1];
  GemmProb prob[GEMM_GROUP_MAX - 1];
  int count;  // extra problems
};
// per-problem tile geometry, built in shared memory by thread 0
struct ProbInfo {
  int M, N, num_m, num_kb, unit_end;
  float beta;
};

template <int BN, bool A_MN, bool B_MN, int EPI, int CG>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmC2,
                     const GemmArgs args, const __grid_constant__ GemmGroup grp) {
  constexpr int NBOX = EPI == EPI_SWIGLU ? 2 : 1;
  using Cfg = GemmCfg<BN, CG, NBOX>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int PAIR_M = GEMM_BM * CG;  // rows per work unit
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES + Cfg::STAGING_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;   // [2]
  uint64_t* tempty_bar = tfull_bar + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  ProbInfo* probs = reinterpret_cast<ProbInfo*>(tmem_slot + 4);  // [1 + grp.count]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;  // CTA within the pair; rank 0 issues the MMAs
  const int unit0 = CG == 2 ? (int)cluster_id_x() : (int)blockIdx.x;
  const int ustep = CG == 2 ? (int)nclusters_x() : (int)gridDim.x;
  const int num_m = (args.M + PAIR_M - 1) / PAIR_M;
  const int num_n = (args.N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int num_kb = (args.K + GEMM_BK - 1) / GEMM_BK;
  // work unit u = split * num_tiles + tile (problem 0), then the grouped problems' tiles
  int num_units = num_tiles * args.splits;
  for (int q = 0; q < grp.count; ++q)
    num_units += ((grp.prob[q].M + PAIR_M - 1) / PAIR_M) * ((grp.prob[q].N + BN - 1) / BN);
  const int kbs = (num_kb + args.splits - 1) / args.splits;
  // unit -> problem index (0 unless grouped); problem geometry from the shared table
  auto prob_of = [&](int u) {
    int q = 0;
    while (u >= probs[q].unit_end) ++q;
    return q;
  };
  auto map_a = [&](int q) { return q == 0 ? &tmA : &grp.ta[q - 1]; };
  auto map_b = [&](int q) { return q == 0 ? &tmB : &grp.tb[q - 1]; };
  auto map_c = [&](int q) { return q == 0 ? &tmC : &grp.tc[q - 1]; };

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmC);
    if (EPI == EPI_SWIGLU || EPI == EPI_SWIGLU_BWD) tma_prefetch_desc(&tmC2);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    probs[0] = ProbInfo{args.M, args.N, num_m, num_kb, num_tiles * args.splits, args.beta};
    for (int q = 0; q < grp.count; ++q) {
      const GemmProb& g = grp.prob[q];
      const int nm = (g.M + PAIR_M - 1) / PAIR_M;
      probs[q + 1] = ProbInfo{g.M, g.N, nm, (g.K + GEMM_BK - 1) / GEMM_BK,
                              probs[q].unit_end + nm * ((g.N + BN - 1) / BN), g.beta};
      tma_prefetch_desc(&grp.ta[q]);
      tma_prefetch_desc(&grp.tb[q]);
      tma_prefetch_desc(&grp.tc[q]);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], CG * GEMM_EPI_WARPS);  // epilogue warps of both CTAs release an accumulator
    }
    fence_barrier_init();
    fence_proxy_async();
  }
  if (warp == 2) {
    if constexpr (CG == 2) tmem_alloc_pair(tmem_slot, Cfg::TMEM_COLS);
    else tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync();  // barrier inits visible to the peer before any remote arrive
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // upstream grid complete before any dependent global access

  if (warp == 0) {
    // ---------------- TMA producer (whole warp; one elected lane issues) ----------------
    int stage = 0;
    uint32_t phase = 0;
    // both CTAs of a pair count their bytes on the leader's full barrier
    const uint32_t full0 = CG == 2 ? mapa_shared(smem_u32(&full_bar[0]), 0) : smem_u32(&full_bar[0]);
    auto load = [&](void* dst, const CUtensorMap* m, int st, int c0, int c1) {
      if constexpr (CG == 2) tma_load_2d_pair(dst, m, full0 + 8 * st, c0, c1);
      else tma_load_2d(dst, m, &full_bar[st], c0, c1);
    };
    for (int u = unit0; u < num_units; u += ustep) {
      const int q = prob_of(u);
      const ProbInfo pi = probs[q];
      const CUtensorMap* mA = map_a(q);
      const CUtensorMap* mB = map_b(q);
      const int lu = q == 0 ? u : u - probs[q - 1].unit_end;
      const int tile = q == 0 ? u % num_tiles : lu;
      const int kb0 = q == 0 ? (u / num_tiles) * kbs : 0;
      const int kb1 = q == 0 ? min(num_kb, kb0 + kbs) : pi.num_kb;
      const bool nmaj = q == 0 && args.n_major;
      const int m0 = (nmaj ? tile / num_n : tile % pi.num_m) * PAIR_M + (int)rank * GEMM_BM;
      const int nb = (nmaj ? tile % num_n : tile / pi.num_m) * BN + (int)rank * (BN / CG);  // this CTA's B rows
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
        uint8_t* sb = sa + Cfg::A_BYTES;
        if (args.probe == 2 || args.probe == 4) {
          if (rank == 0 && elect_one()) mbar_arrive(&full_bar[stage]);
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
          continue;
        }
        const int k0 = kb * GEMM_BK;
        if (elect_one()) {
          if (rank == 0) mbar_expect_tx(&full_bar[stage], CG * Cfg::STAGE_BYTES);
          if (A_MN) {
#pragma unroll
            for (int a = 0; a < GEMM_BM / 64; ++a) load(sa + a * (GEMM_BK * 128), mA, stage, m0 + 64 * a, k0);
          } else {
            load(sa, mA, stage, k0, m0);
          }
          if (B_MN) {
#pragma unroll
            for (int a = 0; a < BN / CG / 64; ++a) load(sb + a * (GEMM_BK * 128), mB, stage, nb + 64 * a, k0);
          } else {
            load(sb, mB, stage, k0, nb);
          }
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
    pdl_trigger();  // all loads issued: let the next kernel launch and run its prologue
  } else if (warp == 1 && rank == 0) {
    // ---------------- MMA issuer (the pair's leader CTA for CG = 2) ----------------
    // the whole warp runs the loop (descriptors stay in uniform registers); one elected lane
    // issues the tcgen05 instructions
    constexpr uint32_t IDESC = umma_idesc_bf16(PAIR_M, BN, A_MN, B_MN);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int u = unit0; u < num_units; u += ustep, ++it) {
      const int q = prob_of(u);
      const int kb0 = q == 0 ? (u / num_tiles) * kbs : 0;
      const int kb1 = q == 0 ? min(num_kb, kb0 + kbs) : probs[q].num_kb;
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      if constexpr (CG == 2) mbar_wait_cluster(&tempty_bar[acc], acc_phase ^ 1);
      else mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + stage * Cfg::STAGE_BYTES);
        const uint32_t sb = sa + Cfg::A_BYTES;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < GEMM_BK / 16; ++kk) {
            if (args.probe == 1 || args.probe == 6) break;
            const uint64_t ad = A_MN ? umma_desc_sw128(sa + kk * 2048, GEMM_BK * 128, 1024)
                                     : umma_desc_sw128(sa + kk * 32, 16, 1024);
            const uint64_t bd = B_MN ? umma_desc_sw128(sb + kk * 2048, GEMM_BK * 128, 1024)
                                     : umma_desc_sw128(sb + kk * 32, 16, 1024);
            if constexpr (CG == 2) mma_bf16_ss_pair(d_tmem, ad, bd, IDESC, (kb != kb0) || (kk != 0));
            else mma_bf16_ss(d_tmem, ad, bd, IDESC, (kb != kb0) || (kk != 0));
          }
          if constexpr (CG == 2) mma_commit_pair(&empty_bar[stage]);
          else mma_commit(&empty_bar[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (elect_one()) {
        if constexpr (CG == 2) mma_commit_pair(&tfull_bar[acc]);
        else mma_commit(&tfull_bar[acc]);
      }
      __syncwarp();
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
    uint8_t* const box0 = smem + STAGES * Cfg::STAGE_BYTES + (warp - 4) * 4096 * NBOX;
    uint8_t* box = box0;  // the box the helpers below write / issue
    auto box_acquire = [&]() {
      if (lane == 0) bulk_wait_read<0>();  // the previous store from this buffer has read it
      __syncwarp();
    };
    auto box_put = [&](int r, int j, uint4 v) { sts128(smem_u32(box) + r * 128 + ((j ^ (r & 7)) << 4), v); };
    auto box_get = [&](int r, int j) -> uint4 { return lds128(smem_u32(box) + r * 128 + ((j ^ (r & 7)) << 4)); };
    auto box_issue = [&](const CUtensorMap* m, int c0, int c1, bool reduce) {
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        if (args.probe == 5) {
          // probe: output store skipped
        } else if (reduce) tma_reduce_add_2d(m, box, c0, c1);
        else tma_store_2d(m, box, c0, c1);
        bulk_commit();
      }
    };
    // bf16 box -> global with coalesced 16-byte stores (8 lanes per 128-byte row); keeps the
    // epilogue's output off the TMA unit, which the producer's operand loads keep busy
    auto box_store = [&](void* base, long long ld, int ncols, int c0, int r0) {
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = i * 4 + (lane >> 3), j = lane & 7;
        const int grow = r0 + r, gcol = c0 + 8 * j;
        const uint4 v = box_get(r, j);
        if (grow < args.M && gcol < ncols)
          *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(base) + (size_t)grow * ld + gcol) = v;
      }
      __syncwarp();
    };
    // output 0 = C (ncols0 columns), 1 = C2 (ncols1 columns)
    const int ncols0 = EPI == EPI_SWIGLU ? args.N / 2 : args.N;
    const int ncols1 = EPI == EPI_SWIGLU_BWD ? 2 * args.N : args.N;
    auto box_out = [&](int which, int c0, int r0) {
      if (args.tma_store || args.probe == 5) box_issue(which ? &tmC2 : &tmC, c0, r0, false);
      else if (which == 0) box_store(args.C, args.ldc, ncols0, c0, r0);
      else box_store(args.C2, args.ldc2, ncols1, c0, r0);
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
    const uint32_t tempty0 = CG == 2 ? mapa_shared(smem_u32(&tempty_bar[0]), 0) : 0;
    for (int u = unit0; u < num_units; u += ustep, ++it) {
      const int q = prob_of(u);
      const ProbInfo pi = probs[q];
      const int tile = q == 0 ? u % num_tiles : u - probs[q - 1].unit_end;
      const int split = q == 0 ? u / num_tiles : 0;
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const bool nmaj = q == 0 && args.n_major;
      const int m0 = (nmaj ? tile / num_n : tile % pi.num_m) * PAIR_M + (int)rank * GEMM_BM;
      const int n0 = (nmaj ? tile % num_n : tile / pi.num_m) * BN;
      const int rbase = m0 + wq * 32;
      // residual / attention-delta epilogues: this warp's R rows (32 x BN/2; O for the delta) are
      // loaded before the accumulator is ready, so their latency hides under the tile's MMAs
      // instead of lengthening the exposed epilogue
      constexpr int RCH = (EPI == EPI_BF16_RESID || EPI == EPI_ATTN_DELTA) ? BN / 128 : 0;  // 64-col chunks per warp
      uint4 rpre[RCH > 0 ? RCH : 1][8];
      if constexpr (RCH > 0) {
        const __nv_bfloat16* R = reinterpret_cast<const __nv_bfloat16*>(args.R);
#pragma unroll
        for (int ch = 0; ch < RCH; ++ch)
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = (lane >> 3) + 4 * i, j = lane & 7;
            const int grow = rbase + r, gcol = n0 + cb + 64 * ch + 8 * j;
            rpre[ch][i] = make_uint4(0, 0, 0, 0);
            if (grow < args.M && gcol < args.N)
              rpre[ch][i] = *reinterpret_cast<const uint4*>(R + (size_t)grow * args.ldr + gcol);
          }
      }
      // RoPE (head dim 64): the row's 32 (cos, sin) pairs serve every head of the tile; loaded
      // once, before the accumulator is ready
      constexpr int RPP = RopeHd<EPI>::value == 64 ? 32 : 1;
      float2 wpre[RPP];
      if constexpr (RopeHd<EPI>::value == 64) {
        const int row = rbase + lane;
        const float2* cs = reinterpret_cast<const float2*>(args.rope_cs) + (row < args.M ? row : 0) % args.rope_T;
        if (n0 + cb < args.rope_cols) {
#pragma unroll
          for (int j = 0; j < 32; ++j) wpre[j] = cs[(size_t)j * args.rope_T];
        }
      }
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + ((uint32_t)(wq * 32) << 16) + acc * BN;
      if (args.probe == 3 || args.probe == 4 || args.probe == 6) {
        // probe: accumulator released without reading it
      } else if constexpr (EPI == EPI_F32) {
        if (args.splits == 1) {
          const bool add = pi.beta != 0.f;
          const CUtensorMap* mC = map_c(q);
#pragma unroll 1
          for (int c = cb; c < cb + BN / 2 && n0 + c < pi.N; c += 32) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(t_row + c, v);
            tmem_ld_wait();
            box_acquire();
#pragma unroll
            for (int j = 0; j < 8; ++j) box_put(lane, j, make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
            box_issue(mC, n0 + c, rbase, add);
          }
        } else {
          // split-K: this split's partial goes to the workspace (plain store); splitk_reduce_kernel
          // then adds the partials to C in split order (deterministic)
#pragma unroll 1
          for (int c = cb; c < cb + BN / 2 && n0 + c < args.N; c += 32) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(t_row + c, v);
            tmem_ld_wait();
            box_acquire();
#pragma unroll
            for (int j = 0; j < 8; ++j) box_put(lane, j, make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
            box_issue(&tmC2, n0 + c, (int)(split * args.ws_rows) + rbase, false);
          }
        }
      } else if constexpr (EPI == EPI_SWIGLU) {
        // tile columns [0,128) are gate, [128,256) the matching up rows of the interleaved weight;
        // this warp handles gate/up columns [64*half, 64*half + 64).  Each accumulator column is
        // read from TMEM once: the raw gate and up values go to boxes A and B, H = silu(g) * u is
        // kept in registers and written through box A once the gate store has read it.
        const int c = 64 * half;
        if (n0 + c < args.N) {
          uint8_t* const boxA = box0;
          uint8_t* const boxB = box0 + 4096;
          float h[2][32];
          if (lane == 0) bulk_wait_read<0>();  // both boxes free (previous tile's stores have read them)
          __syncwarp();
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            float g[32], uu[32];
            ld32(t_row + c + 32 * q, g);
            ld32(t_row + BN / 2 + c + 32 * q, uu);
            box = boxA;
            put32(4 * q, g);
            box = boxB;
            put32(4 * q, uu);
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              // silu from the bf16-rounded pre-activations the backward pass will see
              const float2 gr = unpack_bf16(pack_bf16(g[j], g[j + 1]));
              const float2 ur = unpack_bf16(pack_bf16(uu[j], uu[j + 1]));
              h[q][j] = gr.x * fast_sigmoid(gr.x) * ur.x;
              h[q][j + 1] = gr.y * fast_sigmoid(gr.y) * ur.y;
            }
          }
          box = boxA;
          box_out(1, n0 + c, rbase);           // gate
          box = boxB;
          box_out(1, n0 + BN / 2 + c, rbase);  // up
          if (lane == 0) bulk_wait_read<1>();                // the gate store has read box A
          __syncwarp();
          box = boxA;
          put32(0, h[0]);
          put32(4, h[1]);
          box_out(0, n0 / 2 + c, rbase);       // H
          box = box0;
        }
      } else if constexpr (EPI == EPI_SWIGLU_BWD) {
        // dh tile columns [cb, cb+128) = one 128-column gate/up block of the interleaved layout:
        //   dgate = dh * up * sig(g) * (1 + g (1 - sig(g))),  dup = dh * silu(g)
        // Per 32-column slice the warp stages gate and up (32 rows x 64 B each) through its
        // swizzled box with coalesced 16-byte loads (8 lanes per 128-byte box row: chunks 0-3
        // gate, 4-7 up), computes in place (lane = row) and writes dgate/dup back the same way;
        // the next slice's gate/up loads are in flight while this one computes.
        const int fc = n0 + cb;  // first dh column of this warp
        if (fc < args.N) {
          const int blk = fc >> 7;
          const __nv_bfloat16* GU = reinterpret_cast<const __nv_bfloat16*>(args.R);
          __nv_bfloat16* DGU = reinterpret_cast<__nv_bfloat16*>(args.C2);
          const int j = lane & 7;            // 16-byte chunk of a box row this lane moves
          const int col_off = (j < 4 ? 0 : 128) + 8 * (j & 3);  // gate / up column within the block
          auto load_slice = [&](int q, uint4 (&rv)[8]) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int r = (lane >> 3) + 4 * i, grow = rbase + r;
              rv[i] = grow < args.M
                          ? *reinterpret_cast<const uint4*>(GU + (size_t)grow * args.ldr + blk * 256 + 32 * q + col_off)
                          : make_uint4(0, 0, 0, 0);
            }
          };
          uint4 rv[8];
          load_slice(0, rv);
          box_acquire();
#pragma unroll 1
          for (int q = 0; q < 4; ++q) {
#pragma unroll
            for (int i = 0; i < 8; ++i) box_put((lane >> 3) + 4 * i, j, rv[i]);
            __syncwarp();
            if (q + 1 < 4) load_slice(q + 1, rv);
            float dh[32];
            ld32(t_row + cb + 32 * q, dh);
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
              const uint4 g4 = box_get(lane, c4), u4 = box_get(lane, 4 + c4);
              const uint32_t gw[4] = {g4.x, g4.y, g4.z, g4.w}, uw[4] = {u4.x, u4.y, u4.z, u4.w};
              uint32_t og[4], ou[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 g2 = unpack_bf16(gw[e]), u2 = unpack_bf16(uw[e]);
                const float d0 = dh[8 * c4 + 2 * e], d1 = dh[8 * c4 + 2 * e + 1];
                const float s0 = fast_sigmoid(g2.x), s1 = fast_sigmoid(g2.y);
                og[e] = pack_bf16(d0 * u2.x * s0 * (1.f + g2.x * (1.f - s0)), d1 * u2.y * s1 * (1.f + g2.y * (1.f - s1)));
                ou[e] = pack_bf16(d0 * g2.x * s0, d1 * g2.y * s1);
              }
              box_put(lane, c4, make_uint4(og[0], og[1], og[2], og[3]));
              box_put(lane, 4 + c4, make_uint4(ou[0], ou[1], ou[2], ou[3]));
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int r = (lane >> 3) + 4 * i, grow = rbase + r;
              const uint4 v = box_get(r, j);
              if (grow < args.M)
                *reinterpret_cast<uint4*>(DGU + (size_t)grow * args.ldc2 + blk * 256 + 32 * q + col_off) = v;
            }
            __syncwarp();
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
              // HD=128: this slice's (cos, sin) pairs are requested before the TMEM loads (whose
              // wait would otherwise serialise them)
              float2 wq[HD == 64 ? 1 : 32];
              if constexpr (HD != 64) {
                if (rot) {
#pragma unroll
                  for (int j = 0; j < 32; ++j) wq[j] = cs[(size_t)(pair0 + j) * T];
                }
              }
              float x1[32], x2[32];
              ld32(t_row + hb + pair0, x1);
              ld32(t_row + hb + HD / 2 + pair0, x2);
              if (rot) {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                  const float2 w = HD == 64 ? wpre[j % RPP] : wq[j % (HD == 64 ? 1 : 32)];
                  const float a = x1[j], b = x2[j];
                  x1[j] = second ? (b * w.x + a * w.y) : (a * w.x - b * w.y);
                }
              } else if (second) {
#pragma unroll
                for (int j = 0; j < 32; ++j) x1[j] = x2[j];
              }
              put32(4 * q, x1);
            }
            box_out(0, n0 + hb + 64 * bx, rbase);
          }
        }
      } else {
        // plain bf16 store, optionally + residual R (read coalesced into the staging box first);
        // EPI_XENT also folds the row's 128 rounded logits into (max, sum exp) partials
        float xm = -INFINITY, xs = 0.f;
        float dsum = 0.f;  // EPI_ATTN_DELTA: this row's dO . O over the current head
#pragma unroll 1
        for (int c = cb; c < cb + BN / 2 && n0 + c < args.N; c += 64) {
          box_acquire();
          if constexpr (RCH > 0) {  // the prefetched R / O chunk into the swizzled box
            const int ch = (c - cb) >> 6;
#pragma unroll
            for (int cc = 0; cc < RCH; ++cc)
              if (cc == ch)
#pragma unroll
                for (int i = 0; i < 8; ++i) box_put((lane >> 3) + 4 * i, lane & 7, rpre[cc][i]);
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
            if constexpr (EPI == EPI_ATTN_DELTA) {
              // D from dO as stored (bf16-rounded), in column order
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const uint4 r4 = box_get(lane, 4 * q + j);
                const uint32_t ow[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float2 o2 = unpack_bf16(ow[e]);
                  const float2 d2 = unpack_bf16(pack_bf16(f[8 * j + 2 * e], f[8 * j + 2 * e + 1]));
                  dsum = fmaf(d2.x, o2.x, dsum);
                  dsum = fmaf(d2.y, o2.y, dsum);
                }
              }
            }
            if constexpr (EPI == EPI_XENT) {
              // statistics of the values as stored (bf16), online over the 32-column chunks
              float cm = -INFINITY;
#pragma unroll
              for (int j = 0; j < 32; j += 2) {
                const float2 r2 = unpack_bf16(pack_bf16(f[j], f[j + 1]));
                f[j] = r2.x;
                f[j + 1] = r2.y;
                cm = fmaxf(cm, fmaxf(r2.x, r2.y));
              }
              if (cm > xm) {
                xs *= exp2f((xm - cm) * 1.4426950408889634f);
                xm = cm;
              }
              const float nm = -xm * 1.4426950408889634f;
              float sk[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
              for (int j = 0; j < 32; ++j) sk[j & 3] += exp2f(fmaf(f[j], 1.4426950408889634f, nm));
              xs += (sk[0] + sk[1]) + (sk[2] + sk[3]);
            }
            put32(4 * q, f);
          }
          box_out(0, n0 + c, rbase);
          if constexpr (EPI == EPI_ATTN_DELTA) {
            if ((n0 + c + 64) % args.delta_hd == 0) {  // the head ends with this 64-column box
              const int row = rbase + lane;
              if (row < args.M) {
                const int b = row / args.delta_T, t = row - b * args.delta_T;
                const int h = (n0 + c + 64) / args.delta_hd - 1;
                const long long idx = ((long long)b * args.delta_H + h) * args.delta_T + t;
                args.delta[idx] = dsum;
                args.delta[args.delta_total + idx] = args.lse[idx] * 1.4426950408889634f;
              }
              dsum = 0.f;
            }
          }
        }
        if constexpr (EPI == EPI_XENT) {
          const int row = rbase + lane;
          if (row < args.M && n0 + cb < args.N)
            *reinterpret_cast<float2*>(reinterpret_cast<float*>(args.C2) + (size_t)row * args.ldc2 + 2 * ((n0 + cb) >> 7)) =
                make_float2(xm, xs);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2) mbar_arrive_cluster_relaxed(tempty0 + 8 * acc);
        else mbar_arrive_relaxed(&tempty_bar[acc]);
      }
    }
    if (lane == 0) bulk_wait<0>();  // staging smem must outlive the TMA reads
  }
  __syncwarp();
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync();  // the peer's TMEM / smem / barriers are in use until both finish
  else __syncthreads();
  tc_fence_after();
  if (warp == 2) {
    if constexpr (CG == 2) tmem_dealloc_pair(tmem_base, Cfg::TMEM_COLS);
    else tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

// C (+)= sum_s ws[s] over the split partials, in split order (deterministic); 4 columns per thread.
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float* __restrict__ ws, float* __restrict__ C,
                                                            int M, int N, long long ldc, long long ws_rows,
                                                            int splits, int accumulate) {
  pdl_wait();
  const long long n4 = N / 4;
  const long long total = (long long)M * n4;
  const long long split_stride = ws_rows * N;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / n4, c = (i % n4) * 4;
    const float* src = ws + r * N + c;
    float4 acc = __ldcs(reinterpret_cast<const float4*>(src));
    for (int sp = 1; sp < splits; ++sp) {
      const float4 t = __ldcs(reinterpret_cast<const float4*>(src + sp * split_stride));
      acc.x += t.x; acc.y += t.y; acc.z += t.z; acc.w += t.w;
    }
    float4* dst = reinterpret_cast<float4*>(C + r * ldc + c);
    if (accumulate) {
      const float4 o = *dst;
      acc.x = o.x + acc.x; acc.y = o.y + acc.y; acc.z = o.z + acc.z; acc.w = o.w + acc.w;
    }
    *dst = acc;
  }
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

static const GemmGroup kNoGroup{};

template <int BN, bool A_MN, bool B_MN, int EPI, int CG = 1>
static int launch_gemm(const void* A, const void* B, long long lda, long long ldb, const GemmArgs& args,
                       cudaStream_t stream, const GemmGroup& grp = kNoGroup) {
  using Cfg = GemmCfg<BN, CG, EPI == EPI_SWIGLU ? 2 : 1>;
  CUtensorMap ta, tb;
  int rc;
  // A operand: rows = M, contraction = K
  if (A_MN) rc = make_tmap_2d(&ta, A, args.M, args.K, lda, 64, GEMM_BK);
  else rc = make_tmap_2d(&ta, A, args.K, args.M, lda, GEMM_BK, GEMM_BM);
  if (rc) return rc;
  if (B_MN) rc = make_tmap_2d(&tb, B, args.N, args.K, ldb, 64, GEMM_BK);
  else rc = make_tmap_2d(&tb, B, args.K, args.N, ldb, GEMM_BK, BN / CG);
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
  if (EPI == EPI_F32 && args.splits > 1) {
    rc = make_tmap_2d(&tc2, args.ws, args.N, (uint64_t)args.splits * args.ws_rows, args.N, 32, 32, true);
    if (rc) return rc;
  }
  auto kern = gemm_bf16_kernel<BN, A_MN, B_MN, EPI, CG>;
  static int max_units = 0;  // co-resident CTAs (CG = 1) or CTA pairs (CG = 2); one per template instantiation
  if (!max_units) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(gemm)");
    int n = num_sms();
    if (CG == 2) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(2 * (num_sms() / 2));
      cfg.blockDim = dim3(GEMM_THREADS);
      cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      n = 0;
      e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
      if (e != cudaSuccess || n <= 0) return set_cuda_error(e, "cudaOccupancyMaxActiveClusters(gemm)");
    }
    max_units = n;
  }
  int units = ((args.M + GEMM_BM * CG - 1) / (GEMM_BM * CG)) * ((args.N + BN - 1) / BN) * args.splits;
  for (int q = 0; q < grp.count; ++q)
    units += ((grp.prob[q].M + GEMM_BM * CG - 1) / (GEMM_BM * CG)) * ((grp.prob[q].N + BN - 1) / BN);
  const int g = units < max_units ? units : max_units;
  if (CG == 2)
    spx_launch_check(launch_k_cluster(kern, 2, dim3(2 * g), dim3(GEMM_THREADS), Cfg::SMEM_BYTES, stream, ta, tb, tc, tc2, args, grp));
  else
    spx_launch_check(launch_k(kern, dim3(g), dim3(GEMM_THREADS), Cfg::SMEM_BYTES, stream, ta, tb, tc, tc2, args, grp));
  rc = check_launch("gemm_bf16_kernel");
  if (rc || EPI != EPI_F32 || args.splits == 1) return rc;
  const long long work = (long long)args.M * (args.N / 4);
  const long long want = (work + 255) / 256;
  const int rg = (int)(want < 8LL * num_sms() ? want : 8LL * num_sms());
  spx_launch_check(launch_k(splitk_reduce_kernel, dim3(rg), dim3(256), 0, stream, (const float*)args.ws, (float*)args.C,
                            args.M, args.N, args.ldc, args.ws_rows, args.splits, args.beta != 0.f ? 1 : 0));
  return check_launch("splitk_reduce_kernel");
}

template <int BN, int EPI, int CG = 1>
static int dispatch_major(const void* A, const void* B, long long lda, long long ldb, int a_mn, int b_mn,
                          const GemmArgs& args, cudaStream_t s) {
  if (!a_mn && !b_mn) return launch_gemm<BN, false, false, EPI, CG>(A, B, lda, ldb, args, s);
  if (!a_mn && b_mn) return launch_gemm<BN, false, true, EPI, CG>(A, B, lda, ldb, args, s);
  if (a_mn && b_mn) return launch_gemm<BN, true, true, EPI, CG>(A, B, lda, ldb, args, s);
  return launch_gemm<BN, true, false, EPI, CG>(A, B, lda, ldb, args, s);
}

// Per-device split-K partials buffer, registered once by the caller (no allocation in the GEMM path).
static float* g_ws[64] = {nullptr};
static int64_t g_ws_n[64] = {0};

static int tma_store_mode() {
  static const int t = [] {
    const char* e = getenv("SPX_GEMM_TMA_STORE");
    return e ? atoi(e) : 0;
  }();
  return t;
}

static int probe_mode() {
  static const int p = [] {
    const char* e = getenv("SPX_GEMM_PROBE");
    return e ? atoi(e) : 0;
  }();
  return p;
}

// 256-row CTA-pair tiles (cta_group::2) for BN = 256 whenever M spans at least two 128-row
// tiles; SPX_GEMM_PAIR=0 forces single-CTA tiles.
static bool use_pair(int M) {
  static const int enabled = [] {
    const char* e = getenv("SPX_GEMM_PAIR");
    return e ? atoi(e) : 1;
  }();
  return enabled && M > GEMM_BM;
}

// Split-K factor for the fp32 (wgrad) epilogue: the smallest split count within 5 % of the best
// wave efficiency of tiles x splits on the SMs (CTA pairs), keeping >= 8 k-blocks per split and
// the partials within the registered workspace (no workspace registered: no split-K).
static void pick_splits(GemmArgs& a, int bn) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || g_ws[dev] == nullptr) return;
  if ((a.ldc & 3) || (reinterpret_cast<uintptr_t>(a.C) & 15)) return;  // the reduce kernel stores float4
  const int cg = (bn == 256 && use_pair(a.M)) ? 2 : 1;
  const int num_m = (a.M + GEMM_BM * cg - 1) / (GEMM_BM * cg);
  const int tiles = num_m * ((a.N + bn - 1) / bn);
  const long long ws_rows = (long long)num_m * GEMM_BM * cg;
  const int num_kb = (a.K + GEMM_BK - 1) / GEMM_BK;
  const int slots = num_sms() / cg;
  double eff[9] = {0};
  double best = 0.0;
  for (int sp = 1; sp <= 8; ++sp) {
    if (sp > 1 && (num_kb / sp < 8 || (long long)sp * ws_rows * a.N > g_ws_n[dev])) break;
    const long units = (long)tiles * sp;
    eff[sp] = (double)units / (double)(((units + slots - 1) / slots) * slots);
    if (eff[sp] > best) best = eff[sp];
  }
  int pick = 1;
  while (pick < 8 && eff[pick] < best - 0.05) ++pick;
  a.splits = pick;
  if (pick > 1) {
    a.ws = g_ws[dev];
    a.ws_rows = ws_rows;
  }
}

template <int EPI>
static int dispatch_256(const void* A, const void* B, long long lda, long long ldb, int a_mn, int b_mn,
                        const GemmArgs& args, cudaStream_t s) {
  if (use_pair(args.M)) return dispatch_major<256, EPI, 2>(A, B, lda, ldb, a_mn, b_mn, args, s);
  return dispatch_major<256, EPI, 1>(A, B, lda, ldb, a_mn, b_mn, args, s);
}

// epilogues that exist for one operand layout only (fewer template instantiations)
template <int EPI, bool A_MN, bool B_MN>
static int dispatch_256_fixed(const void* A, const void* B, long long lda, long long ldb, const GemmArgs& args,
                              cudaStream_t s) {
  if (use_pair(args.M)) return launch_gemm<256, A_MN, B_MN, EPI, 2>(A, B, lda, ldb, args, s);
  return launch_gemm<256, A_MN, B_MN, EPI, 1>(A, B, lda, ldb, args, s);
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

extern "C" int spx_gemm_set_workspace(float* partials, int64_t n_floats) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return set_error(SPX_ERR_ARG, "gemm workspace: bad device");
  if (partials == nullptr || n_floats <= 0) {
    g_ws[dev] = nullptr;
    g_ws_n[dev] = 0;
    return SPX_OK;
  }
  if (((uintptr_t)partials) & 15) return set_error(SPX_ERR_ARG, "gemm workspace: partials must be 16-byte aligned");
  g_ws[dev] = partials;
  g_ws_n[dev] = n_floats;
  return SPX_OK;
}

// Weight-gradient group: C_i (+)= A_i . B_i^T (fp32 accumulate, epilogue 2) for up to four
// independent problems in one persistent launch.  All share the operand majors.
extern "C" int spx_gemm_f32_group(int32_t count, const void* const* A, const void* const* B, float* const* C,
                                  const int64_t* M, const int64_t* N, const int64_t* K, const int64_t* lda,
                                  const int64_t* ldb, const int64_t* ldc, const float* beta, int32_t a_mn_major,
                                  int32_t b_mn_major, void* stream) {
  if (count < 1 || count > GEMM_GROUP_MAX) return set_error(SPX_ERR_ARG, "gemm_f32_group: 1..4 problems");
  int min_m = 1 << 30;
  for (int i = 0; i < count; ++i) {
    if (M[i] <= 0 || N[i] <= 0 || K[i] <= 0) return set_error(SPX_ERR_ARG, "gemm_f32_group: non-positive shape");
    if (N[i] % 32 != 0 || K[i] % 8 != 0 || lda[i] % 8 != 0 || ldb[i] % 8 != 0)
      return set_error(SPX_ERR_ARG, "gemm_f32_group: N % 32, K/lda/ldb % 8 required");
    if (((uintptr_t)A[i] | (uintptr_t)B[i]) & 15) return set_error(SPX_ERR_ARG, "gemm_f32_group: A/B must be 16-byte aligned");
    if (M[i] < min_m) min_m = (int)M[i];
  }
  GemmArgs args{(int)M[0], (int)N[0], (int)K[0], C[0], nullptr, nullptr, (long long)ldc[0], (long long)ldc[0], 0,
                beta[0], nullptr, 0, 1, 1, nullptr};
  args.probe = probe_mode();
  args.tma_store = tma_store_mode();
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const bool pair = use_pair(min_m);
  GemmGroup grp{};
  grp.count = count - 1;
  for (int i = 1; i < count; ++i) {
    GemmProb& g = grp.prob[i - 1];
    g.M = (int)M[i];
    g.N = (int)N[i];
    g.K = (int)K[i];
    g.beta = beta[i];
    int rc;
    if (a_mn_major) rc = make_tmap_2d(&grp.ta[i - 1], A[i], M[i], K[i], lda[i], 64, GEMM_BK);
    else rc = make_tmap_2d(&grp.ta[i - 1], A[i], K[i], M[i], lda[i], GEMM_BK, GEMM_BM);
    if (rc) return rc;
    const uint32_t bbox = pair ? 128 : 256;
    if (b_mn_major) rc = make_tmap_2d(&grp.tb[i - 1], B[i], N[i], K[i], ldb[i], 64, GEMM_BK);
    else rc = make_tmap_2d(&grp.tb[i - 1], B[i], K[i], N[i], ldb[i], GEMM_BK, bbox);
    if (rc) return rc;
    rc = make_tmap_2d(&grp.tc[i - 1], C[i], N[i], M[i], ldc[i], 32, 32, true);
    if (rc) return rc;
  }
  const int am = a_mn_major ? 1 : 0, bm = b_mn_major ? 1 : 0;
#define SPX_GRP(AM, BM)                                                                                     \
  if (am == AM && bm == BM)                                                                                 \
    return pair ? launch_gemm<256, AM, BM, EPI_F32, 2>(A[0], B[0], lda[0], ldb[0], args, s, grp)            \
                : launch_gemm<256, AM, BM, EPI_F32, 1>(A[0], B[0], lda[0], ldb[0], args, s, grp);
  SPX_GRP(true, true)
  SPX_GRP(false, false)
  SPX_GRP(false, true)
  SPX_GRP(true, false)
#undef SPX_GRP
  return set_error(SPX_ERR_ARG, "gemm_f32_group: bad majors");
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
  args.probe = probe_mode();
  args.tma_store = tma_store_mode();
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (head_dim == 64) return dispatch_256_fixed<EPI_ROPE64, false, false>(A, B, lda, ldb, args, s);
  return dispatch_256_fixed<EPI_ROPE128, false, false>(A, B, lda, ldb, args, s);
}

// Tile raster of a single-problem launch.  M-first (default): concurrent units share a B column
// block and stream all of A once per column of tiles; N-first: they share an A row block and
// stream B once per row.  When the grid takes more than one wave, pick the order whose re-streamed
// operand fits L2 (or costs fewer DRAM bytes) -- e.g. the LM-head weight gradient (M = V = 32000,
// N = d, K = tokens) re-read its 262 MB A operand once per N tile in M-first order.
static int pick_raster(long long M, long long N, long long K, int bn, int cg) {
  const long long nm = (M + 128LL * cg - 1) / (128LL * cg), nn = (N + bn - 1) / bn;
  if (nm * nn <= num_sms() / cg) return 0;  // a single wave: all reuse is concurrent anyway
  const double l2 = 40e6;                    // L2 bytes a wave can keep resident (two 63 MB halves)
  const double a = 2.0 * M * K, b = 2.0 * N * K;
  const double cost_m = (a > l2 ? a * nn : a) + b;
  const double cost_n = (b > l2 ? b * nm : b) + a;
  return cost_n < cost_m ? 1 : 0;
}

extern "C" int spx_gemm_bf16_attn_delta(const void* A, const void* B, void* dO, const void* O, int64_t ld_o,
                                        const float* lse, float* delta_ws, int64_t M, int64_t N, int64_t K, int64_t lda,
                                        int64_t ldb, int64_t ldc, int64_t batch, int64_t T, int64_t head_dim,
                                        void* stream) {
  if (M <= 0 || N <= 0 || K <= 0 || batch <= 0 || T <= 0) return set_error(SPX_ERR_ARG, "gemm_attn_delta: non-positive shape");
  if (K % 8 != 0 || lda % 8 != 0 || ldb % 8 != 0 || ldc % 8 != 0 || ld_o % 8 != 0)
    return set_error(SPX_ERR_ARG, "gemm_attn_delta: K/lda/ldb/ldc/ld_o must be multiples of 8");
  if (head_dim != 64 && head_dim != 128) return set_error(SPX_ERR_ARG, "gemm_attn_delta: head_dim must be 64 or 128");
  if (N % head_dim != 0 || M != batch * T) return set_error(SPX_ERR_ARG, "gemm_attn_delta: N = H*head_dim and M = batch*T");
  if (((uintptr_t)A | (uintptr_t)B | (uintptr_t)O) & 15) return set_error(SPX_ERR_ARG, "gemm_attn_delta: 16-byte alignment");
  GemmArgs args{(int)M, (int)N, (int)K, dO, O, nullptr, (long long)ldc, (long long)ld_o, 0, 0.f,
                nullptr, 0, 1, 1, nullptr};
  args.probe = probe_mode();
  args.tma_store = tma_store_mode();
  args.n_major = pick_raster(M, N, K, 256, use_pair((int)M) ? 2 : 1);
  args.lse = lse;
  args.delta = delta_ws;
  args.delta_hd = (int)head_dim;
  args.delta_T = (int)T;
  args.delta_H = (int)(N / head_dim);
  args.delta_total = (long long)M * (N / head_dim);
  return dispatch_256_fixed<EPI_ATTN_DELTA, false, true>(A, B, lda, ldb, args, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int spx_gemm_bf16(const void* A, const void* B, void* C, const void* R, void* C2, int64_t M, int64_t N,
                             int64_t K, int64_t lda, int64_t ldb, int64_t ldc, int64_t ldc2, int32_t a_mn_major,
                             int32_t b_mn_major, int32_t epilogue, float beta, void* stream) {
  if (M <= 0 || N <= 0 || K <= 0) return set_error(SPX_ERR_ARG, "gemm: non-positive shape");
  if (N % 32 != 0) return set_error(SPX_ERR_ARG, "gemm: N must be a multiple of 32");
  if (K % 8 != 0 || lda % 8 != 0 || ldb % 8 != 0) return set_error(SPX_ERR_ARG, "gemm: K/lda/ldb must be multiples of 8");
  if (((uintptr_t)A | (uintptr_t)B) & 15) return set_error(SPX_ERR_ARG, "gemm: A/B must be 16-byte aligned");
  if (epilogue < 0 || epilogue > 7 || epilogue == 4 || epilogue == 5) return set_error(SPX_ERR_ARG, "gemm: bad epilogue");
  if (epilogue == EPI_XENT && (N % 128 != 0 || C2 == nullptr || ldc2 < 2 * (N / 128)))
    return set_error(SPX_ERR_ARG, "gemm: xent epilogue needs N % 128 == 0 and a partials output C2 with ldc2 >= 2*N/128");
  if (epilogue == EPI_SWIGLU_BWD && (N % 128 != 0 || C2 == nullptr || R == nullptr))
    return set_error(SPX_ERR_ARG, "gemm: swiglu-bwd epilogue needs N % 128 == 0, gu (R) and dgu (C2)");
  if (epilogue == EPI_SWIGLU && (N % 256 != 0 || C2 == nullptr))
    return set_error(SPX_ERR_ARG, "gemm: swiglu epilogue needs N % 256 == 0 and a GU output");
  if (epilogue == EPI_BF16_RESID && R == nullptr) return set_error(SPX_ERR_ARG, "gemm: residual epilogue needs R");
  GemmArgs args{(int)M, (int)N, (int)K, C, R, C2, (long long)ldc, (long long)(epilogue == EPI_SWIGLU_BWD ? ldc2 : ldc),
                (long long)ldc2, beta, nullptr, 0, 1, 1, nullptr};
  args.probe = probe_mode();
  args.tma_store = tma_store_mode();
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int bn = (epilogue == EPI_SWIGLU || epilogue == EPI_F32 || epilogue == EPI_SWIGLU_BWD || epilogue == EPI_XENT) ? 256
                 : (use_pair((int)M) ? 256 : pick_bn((int)M, (int)N));  // CTA pairs need 256-col tiles
  if (epilogue == EPI_F32) pick_splits(args, bn);
  args.n_major = pick_raster(M, N, K, bn, (bn == 256 && use_pair((int)M)) ? 2 : 1);
  switch (epilogue) {
    case EPI_BF16:
      return bn == 256 ? dispatch_256<EPI_BF16>(A, B, lda, ldb, a_mn_major, b_mn_major, args, s)
                       : dispatch_major<128, EPI_BF16>(A, B, lda, ldb, a_mn_major, b_mn_major, args, s);
    case EPI_BF16_RESID:
      return bn == 256 ? dispatch_256<EPI_BF16_RESID>(A, B, lda, ldb, a_mn_major, b_mn_major, args, s)
                       : dispatch_major<128, EPI_BF16_RESID>(A, B, lda, ldb, a_mn_major, b_mn_major, args, s);
    case EPI_F32:
      return bn == 256 ? dispatch_256<EPI_F32>(A, B, lda, ldb, a_mn_major, b_mn_major, args, s)
                       : dispatch_major<128, EPI_F32>(A, B, lda, ldb, a_mn_major, b_mn_major, args, s);
    case EPI_XENT:
      if (a_mn_major || b_mn_major) return set_error(SPX_ERR_ARG, "gemm: xent epilogue needs K-major A and B (forward)");
      return dispatch_256_fixed<EPI_XENT, false, false>(A, B, lda, ldb, args, s);
    case EPI_SWIGLU_BWD:
      if (a_mn_major || !b_mn_major) return set_error(SPX_ERR_ARG, "gemm: swiglu-bwd epilogue needs K-major A, MN-major B (dgrad)");
      return dispatch_256_fixed<EPI_SWIGLU_BWD, false, true>(A, B, lda, ldb, args, s);
    default:
      if (a_mn_major || b_mn_major) return set_error(SPX_ERR_ARG, "gemm: swiglu epilogue needs K-major A and B (forward)");
      return dispatch_256_fixed<EPI_SWIGLU, false, false>(A, B, lda, ldb, args, s);
  }
}
