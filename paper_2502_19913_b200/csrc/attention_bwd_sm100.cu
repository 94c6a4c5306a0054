// tcgen05 flash-attention backward for sm_100a (causal, GQA, head_dim 64/128), deterministic.
//
// Two kernels, no atomics (every output element is written by exactly one CTA):
//   dkdv: CTA = 128 keys of one (batch, kv-head); loops over the GQA group and the query blocks
//         at or after it.  Per step: S^T = K Q^T and dP^T = V dO^T (M=128 keys, N=128 queries) in
//         TMEM; 8 elementwise warps (thread = key row, half the query columns each) form
//         P^T = exp2(S^T*scale*log2e - lse*log2e) and dS^T = P^T (dP^T - D) as bf16 swizzled
//         smem tiles; then dV += P^T dO and dK += dS^T Q accumulate in TMEM (dO and Q tiles are
//         re-used as MN-major B operands).
//         The dK/dV kernel also stores each dS^T tile (bf16) to the workspace.
//   dq:   dQ = dS K as a GEMM over those tiles (CTA = 128 queries of one head, key blocks
//         0..its own), so S, dP and the softmax are computed once.
// Both write bf16 gradients into the dQKV buffer (same layout as QKV) with the inverse RoPE
// applied to dq/dk when a table is given, scale folded in.  D = rowsum(dO*O) comes from
// attn_bwd_delta_kernel (attention.cu).
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "spx_common.cuh"
#include "spx_internal.h"

namespace spx {
namespace fab {

// benchmarking hooks (tools/ubench/attn_main.cu builds variants; libspx uses the defaults)
#ifndef SPX_FAB_NST64
#define SPX_FAB_NST64 3
#endif
#ifndef SPX_FAB_KVS64
#define SPX_FAB_KVS64 2
#endif
#ifndef SPX_FAB_HS
#define SPX_FAB_HS 1
#endif
#ifndef SPX_FAB_PT128
#define SPX_FAB_PT128 1
#endif
#ifndef SPX_FAB_PT_TMEM
#define SPX_FAB_PT_TMEM 1
#endif
#ifdef SPX_FAB_PROBE
// per-step clock64 stamps of CTA 0: [event][step]
__device__ long long g_fab_probe[8][256];
#define FAB_PROBE(ev, step) \
  do { if (blockIdx.x == 0 && (step) < 256) g_fab_probe[ev][step] = clock64(); } while (0)
#else
#define FAB_PROBE(ev, step) do { } while (0)
#endif

constexpr int BLK = 128;                 // rows per block (queries and keys)
constexpr int EW_WARPS = 8;              // elementwise warps: 2 per TMEM lane quadrant
constexpr int THREADS = 128 + 32 * EW_WARPS;
constexpr float LOG2E = 1.4426950408889634f;
constexpr int ATOM = BLK * 128;          // 128 rows x 128 B swizzle atom block

// Heavy-first item lists are dealt to CTAs in boustrophedon order (round k: CTA c takes item
// k*G + c for even k, k*G + G-1-c for odd k), pairing heavy and light items per CTA.
SPX_DEVICE int snake(int k, int c, int G) { return k * G + ((k & 1) ? (G - 1 - c) : c); }

SPX_DEVICE float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

SPX_DEVICE void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
SPX_DEVICE void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
SPX_DEVICE void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
SPX_DEVICE void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

SPX_DEVICE void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

struct BwdParams {
  __nv_bfloat16* dqkv;   // [B*T, ld]
  const float* lse;      // [B, H, T] (dQ kernel; the dK/dV kernel reads lse*log2e from the workspace)
  const float* delta;    // [B, H, T]
  const float* rope_cs;  // [hd/2][T][2] or null
  __nv_bfloat16* ds;     // dS^T tiles [B*H][tri(nqb)][128 keys][128 queries] (workspace)
  long long ld;
  int B, T, H, Hkv;
  float scale;
  int gsplit;            // dK/dV items per (batch, kv head, key block): 1, or the GQA group size
  float* part;           // gsplit > 1: fp32 dV/dK partials [B*Hkv*nqb][gsplit][2][hd][128] (workspace)
};

// store one 128-column bf16 tile row of P^T / dS^T / dS (K-major SWIZZLE_128B, two 64-col atoms)
SPX_DEVICE void put_row8(uint8_t* tile, int r, int c8, const float* v) {
  const int atom = c8 >> 3, chunk = c8 & 7;
  *reinterpret_cast<uint4*>(tile + atom * ATOM + r * 128 + ((chunk ^ (r & 7)) << 4)) =
      make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]), pack_bf16(v[6], v[7]));
}

SPX_DEVICE void put_row8p(uint8_t* tile, int r, int c8, const uint32_t* v) {
  const int atom = c8 >> 3, chunk = c8 & 7;
  *reinterpret_cast<uint4*>(tile + atom * ATOM + r * 128 + ((chunk ^ (r & 7)) << 4)) = make_uint4(v[0], v[1], v[2], v[3]);
}

// write a 128 x HD accumulator row (TMEM lane) as bf16 into this warp's 32-row SWIZZLE_128B
// staging box(es) -- box a holds columns [64a, 64a+64) -- for a TMA store: one coalesced bulk
// write per box instead of 32 scattered rows per st.global
template <int HD>
SPX_DEVICE void stage_grad_row(uint32_t taddr, uint8_t* box0, uint8_t* box1, int row, float scale, const float* cs,
                               int T, int pos, int only = -1) {
  // only >= 0: write just the columns of box `only` (into box0); the others are skipped
  auto put = [&](int col, const float* v) {  // 8 columns starting at col (multiple of 8)
    if (only >= 0 && (col >> 6) != only) return;
    uint8_t* box = (only >= 0 || col < 64) ? box0 : box1;
    const int chunk = (col & 63) >> 3;
    *reinterpret_cast<uint4*>(box + row * 128 + ((chunk ^ (row & 7)) << 4)) =
        make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]), pack_bf16(v[6], v[7]));
  };
  if (cs) {
    const float2* c2 = reinterpret_cast<const float2*>(cs);
#pragma unroll 1
    for (int j0 = 0; j0 < HD / 2; j0 += 32) {
      float2 w[32];  // requested before the TMEM loads, whose wait would serialise them
#pragma unroll
      for (int j = 0; j < 32; ++j) w[j] = c2[(size_t)(j0 + j) * T + pos];
      uint32_t a[32], b[32];
      tmem_ld_32x32b_x32(taddr + j0, a);
      tmem_ld_32x32b_x32(taddr + HD / 2 + j0, b);
      tmem_ld_wait();
      float o1[32], o2[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float x1 = __uint_as_float(a[j]) * scale, x2 = __uint_as_float(b[j]) * scale;
        o1[j] = x1 * w[j].x + x2 * w[j].y;
        o2[j] = x2 * w[j].x - x1 * w[j].y;
      }
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        put(j0 + j, o1 + j);
        put(HD / 2 + j0 + j, o2 + j);
      }
    }
  } else {
#pragma unroll 1
    for (int c = 0; c < HD; c += 32) {
      uint32_t a[32];
      tmem_ld_32x32b_x32(taddr + c, a);
      tmem_ld_wait();
      float o[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) o[j] = __uint_as_float(a[j]) * scale;
#pragma unroll
      for (int j = 0; j < 32; j += 8) put(c + j, o + j);
    }
  }
}

// ------------------------------------------------------------------------------------------
// dK / dV (persistent: one CTA per SM walks heavy-first items (batch, kv-head, key block))
// ------------------------------------------------------------------------------------------
template <int HD>
struct DkdvSmem {
  // hd=128 (ALIAS): P^T / dS^T are written into the TMEM columns of S^T / dP^T once those are read
  // (TMEM holds S^T, dP^T, dV, dK = 512 columns, nothing spare), which frees the P^T smem tile for a
  // second Q/dO stage: the next step's loads then overlap this step
  static constexpr bool ALIAS = HD == 128 && SPX_FAB_PT128;
  static constexpr int NST = HD == 64 ? SPX_FAB_NST64 : (ALIAS ? 2 : 1);  // Q/dO ring depth
  static constexpr int TILE = (HD / 64) * ATOM;     // 128 x HD bf16
  // hd=64: K/V double-buffered across items, so the next item's K/V load and its first S/dP
  // MMAs overlap the current item's last step and dV/dK epilogue (hd=128 has no smem for it)
  static constexpr int KVS = HD == 64 ? SPX_FAB_KVS64 : 1;
  static constexpr int OFF_K = 0;                   // [KVS]
  static constexpr int OFF_V = OFF_K + KVS * TILE;  // [KVS]
  static constexpr int OFF_Q = OFF_V + KVS * TILE;  // [NST]
  static constexpr int OFF_DO = OFF_Q + NST * TILE; // [NST]
  // hd=64: P^T and dS^T are A operands straight from TMEM (TS MMAs), only dS^T is also staged in
  // shared memory for its TMA store; hd=128 has no spare TMEM columns and stages both in smem
  static constexpr bool PT_TMEM = (HD == 64 && SPX_FAB_PT_TMEM) || ALIAS;
  static constexpr int OFF_PT = OFF_DO + NST * TILE;
  static constexpr int OFF_DST = OFF_PT + (PT_TMEM ? 0 : 2 * ATOM);
  static constexpr int OFF_LSE = OFF_DST + 2 * ATOM;  // [NST][128] f32
  static constexpr int OFF_D = OFF_LSE + NST * 512;   // [NST][128] f32
  static constexpr int OFF_BAR = OFF_D + NST * 512;
  static constexpr int BYTES = OFF_BAR + 256;         // base is __align__(1024)
  static_assert(BYTES <= 232448, "dK/dV shared memory exceeds the 227 KB opt-in limit");
};

template <int HD>
__global__ void __launch_bounds__(THREADS, 1)
    attn_bwd_dkdv_tc_kernel(const __grid_constant__ CUtensorMap tmQKV, const __grid_constant__ CUtensorMap tmDO,
                            const __grid_constant__ CUtensorMap tmDS, const __grid_constant__ CUtensorMap tmOut,
                            const BwdParams p) {
  using L = DkdvSmem<HD>;
  constexpr int NST = L::NST;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  static_assert(NST <= 4, "barrier layout holds up to 4 ring stages");
  uint64_t* full = bars + 0;      // [NST]
  uint64_t* empty = bars + 4;     // [NST]
  constexpr int KVS = L::KVS;
  uint64_t* kv_full = bars + 8;     // [KVS]
  uint64_t* kv_empty = bars + 10;   // [KVS]
  uint64_t* sdp_full = bars + 12;
  uint64_t* p_ready = bars + 13;
  uint64_t* mma2_done = bars + 14;
  uint64_t* tmem_free = bars + 15;  // S / dP of the current step copied to registers
  uint64_t* acc_free = bars + 16;   // dV / dK of the previous item read out of TMEM
  uint64_t* ds_read = bars + 17;    // the dS^T tile of the step has been read by its TMA store
  uint64_t* sdp_full_b = bars + 18;  // HS: S/dP of the second query half (sdp_full = first half)
  uint64_t* p_ready_b = bars + 19;   // HS: P^T/dS^T of the second half written (p_ready = first)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = p.T / BLK;
  const int group = p.H / p.Hkv;
  const int hpi = group / p.gsplit;  // query heads per item (GQA split: p.gsplit items per key block)
  const int BHk = p.B * p.Hkv * p.gsplit;
  const int n_items = nqb * BHk;
  // item w: key block jb = w / (B*Hkv*gsplit) (early key blocks see the most query blocks: heavy
  // first), then (batch, kv head, head subset gs)
  auto item = [&](int w, int& b, int& kvh, int& jb, int& gs) {
    jb = w / BHk;
    const int bk = (w % BHk) / p.gsplit;
    gs = (w % BHk) % p.gsplit;
    b = bk / p.Hkv;
    kvh = bk % p.Hkv;
  };

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmQKV);
    tma_prefetch_desc(&tmDO);
    for (int i = 0; i < KVS; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < NST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(sdp_full, 1);
    mbar_init(p_ready, EW_WARPS);
    mbar_init(mma2_done, 1);
    mbar_init(tmem_free, EW_WARPS);
    mbar_init(acc_free, EW_WARPS);
    mbar_init(ds_read, 1);
    mbar_init(sdp_full_b, 1);
    mbar_init(p_ready_b, EW_WARPS);
    tma_prefetch_desc(&tmDS);
    tma_prefetch_desc(&tmOut);
    fence_barrier_init();
    fence_proxy_async();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // upstream grid complete before any dependent global access
  constexpr uint32_t TM_S = 0, TM_DP = 128, TM_DV = 256, TM_DK = 256 + HD;
  constexpr bool PT_TMEM = L::PT_TMEM, ALIAS = L::ALIAS;
  // HS (hd=128): each step runs as two 64-query halves, software-pipelined -- the softmax of one
  // half overlaps the MMAs of the other (dV/dK of the previous half, S/dP of the next)
  constexpr bool HS = ALIAS && SPX_FAB_HS;
  // P^T, dS^T (bf16 pairs along queries): hd=64 in spare columns, hd=128 over S^T / dP^T
  constexpr uint32_t TM_PT = ALIAS ? TM_S : 384, TM_DST = ALIAS ? TM_DP : 448;

  if (warp == 0 && lane == 0) {
    // ---------------- producer ----------------
    int gi = 0, n = 0;
    for (int k = 0, w = snake(0, blockIdx.x, gridDim.x); k * (int)gridDim.x < n_items; ++k, w = snake(k, blockIdx.x, gridDim.x), ++n) {
      if (w >= n_items) continue;
      int b, kvh, jb, gs;
      item(w, b, kvh, jb, gs);
      const int row0 = b * p.T, nq = nqb - jb;
      const int kv = n % KVS;
      mbar_wait(&kv_empty[kv], ((n / KVS) & 1) ^ 1);
      mbar_expect_tx(&kv_full[kv], 2 * L::TILE);
      for (int a = 0; a < HD / 64; ++a) {
        tma_load_2d(smem + L::OFF_K + kv * L::TILE + a * ATOM, &tmQKV, &kv_full[kv], (p.H + kvh) * HD + 64 * a,
                    row0 + jb * BLK);
        tma_load_2d(smem + L::OFF_V + kv * L::TILE + a * ATOM, &tmQKV, &kv_full[kv],
                    (p.H + p.Hkv + kvh) * HD + 64 * a, row0 + jb * BLK);
      }
      for (int it = 0; it < hpi * nq; ++it, ++gi) {
        const int s = gi % NST;
        const int h = kvh * group + gs * hpi + it / nq, qb = jb + it % nq;
        mbar_wait(&empty[s], ((gi / NST) & 1) ^ 1);
        FAB_PROBE(0, gi);
        mbar_expect_tx(&full[s], 2 * L::TILE + 1024);
        for (int a = 0; a < HD / 64; ++a) {
          tma_load_2d(smem + L::OFF_Q + s * L::TILE + a * ATOM, &tmQKV, &full[s], h * HD + 64 * a, row0 + qb * BLK);
          tma_load_2d(smem + L::OFF_DO + s * L::TILE + a * ATOM, &tmDO, &full[s], h * HD + 64 * a, row0 + qb * BLK);
        }
        const size_t off = ((size_t)b * p.H + h) * p.T + qb * BLK;
        bulk_load(smem + L::OFF_LSE + s * 512, p.delta + (size_t)p.B * p.H * p.T + off, 512, &full[s]);  // lse*log2e
        bulk_load(smem + L::OFF_D + s * 512, p.delta + off, 512, &full[s]);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (whole warp; one elected lane issues) ----------------
    constexpr uint32_t ID_S = umma_idesc_bf16(BLK, BLK, false, false);   // K.Q^T, V.dO^T
    constexpr uint32_t ID_G = umma_idesc_bf16(BLK, HD, false, true);     // P^T.dO, dS^T.Q
    const uint32_t sPT = smem_u32(smem + L::OFF_PT), sDST = smem_u32(smem + L::OFF_DST);
    auto issue_sdp = [&](int gi, int kv) {
      const uint32_t sK = smem_u32(smem + L::OFF_K + kv * L::TILE), sV = smem_u32(smem + L::OFF_V + kv * L::TILE);
      const int s = gi % NST;
      mbar_wait(&full[s], (gi / NST) & 1);
      tc_fence_after();
      const uint32_t sQ = smem_u32(smem + L::OFF_Q + s * L::TILE), sDO = smem_u32(smem + L::OFF_DO + s * L::TILE);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t ko = (kk >> 2) * ATOM + (kk & 3) * 32;
          mma_bf16_ss(tmem + TM_S, umma_desc_sw128(sK + ko, 16, 1024), umma_desc_sw128(sQ + ko, 16, 1024), ID_S,
                      kk > 0);
          mma_bf16_ss(tmem + TM_DP, umma_desc_sw128(sV + ko, 16, 1024), umma_desc_sw128(sDO + ko, 16, 1024), ID_S,
                      kk > 0);
        }
        mma_commit(sdp_full);
      }
      __syncwarp();
    };
    if constexpr (HS) {
      constexpr uint32_t ID_SH = umma_idesc_bf16(BLK, 64, false, false);  // half the queries
      // S^T / dP^T of query half hf of step gi -> TMEM columns [64 hf, 64 hf + 64) of S / dP
      auto issue_sdp_half = [&](int gi, int kv, int hf) {
        const uint32_t sK = smem_u32(smem + L::OFF_K + kv * L::TILE), sV = smem_u32(smem + L::OFF_V + kv * L::TILE);
        const int s = gi % NST;
        mbar_wait(&full[s], (gi / NST) & 1);
        tc_fence_after();
        const uint32_t sQ = smem_u32(smem + L::OFF_Q + s * L::TILE) + hf * 64 * 128;
        const uint32_t sDO = smem_u32(smem + L::OFF_DO + s * L::TILE) + hf * 64 * 128;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint32_t ko = (kk >> 2) * ATOM + (kk & 3) * 32;
            mma_bf16_ss(tmem + TM_S + 64 * hf, umma_desc_sw128(sK + ko, 16, 1024), umma_desc_sw128(sQ + ko, 16, 1024),
                        ID_SH, kk > 0);
            mma_bf16_ss(tmem + TM_DP + 64 * hf, umma_desc_sw128(sV + ko, 16, 1024),
                        umma_desc_sw128(sDO + ko, 16, 1024), ID_SH, kk > 0);
          }
          mma_commit(hf ? sdp_full_b : sdp_full);
        }
        __syncwarp();
      };
      int gi = 0, n = 0;
      for (int k = 0, w = snake(0, blockIdx.x, gridDim.x); k * (int)gridDim.x < n_items; ++k, w = snake(k, blockIdx.x, gridDim.x), ++n) {
        if (w >= n_items) continue;
        int b, kvh, jb, gs;
        item(w, b, kvh, jb, gs);
        const int n_it = hpi * (nqb - jb);
        const int kv = n % KVS;
        mbar_wait(&kv_full[kv], (n / KVS) & 1);
        for (int it = 0; it < n_it; ++it, ++gi) {
          const int s = gi % NST;
          if (it == 0) {
            issue_sdp_half(gi, kv, 0);
            issue_sdp_half(gi, kv, 1);
          }
          const uint32_t sQ = smem_u32(smem + L::OFF_Q + s * L::TILE), sDO = smem_u32(smem + L::OFF_DO + s * L::TILE);
#pragma unroll 1
          for (int hf = 0; hf < 2; ++hf) {
            mbar_wait(hf ? p_ready_b : p_ready, gi & 1);
            if (it == 0 && hf == 0) mbar_wait(acc_free, (n & 1) ^ 1);  // previous item's dV/dK read out
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
              for (int kq = 0; kq < 4; ++kq) {  // the half's 64 queries, 16 per MMA
                const int kk = 4 * hf + kq;
                const uint32_t bo = kk * 2048;
                const uint32_t acc = (it > 0) || (kk > 0);
                mma_bf16_ts(tmem + TM_DV, tmem + TM_S + 64 * hf + kq * 8, umma_desc_sw128(sDO + bo, ATOM, 1024), ID_G,
                            acc);
                mma_bf16_ts(tmem + TM_DK, tmem + TM_DP + 64 * hf + kq * 8, umma_desc_sw128(sQ + bo, ATOM, 1024),
                            ID_G, acc);
              }
              if (hf == 1) {
                mma_commit(mma2_done);
                mma_commit(&empty[s]);
                if (it + 1 == n_it) mma_commit(&kv_empty[kv]);
              }
            }
            __syncwarp();
            // the same half of the next step, in issue order after the MMAs that read its P^T / dS^T
            if (it + 1 < n_it) issue_sdp_half(gi + 1, kv, hf);
          }
        }
      }
    } else {
    int gi = 0, n = 0;
    bool issued = false;  // S/dP of step gi already issued (look-ahead from the previous step)
    for (int k = 0, w = snake(0, blockIdx.x, gridDim.x); k * (int)gridDim.x < n_items; ++k, w = snake(k, blockIdx.x, gridDim.x), ++n) {
      if (w >= n_items) continue;
      int b, kvh, jb, gs;
      item(w, b, kvh, jb, gs);
      const int n_it = hpi * (nqb - jb);
      const int kv = n % KVS;
      // the CTA's next item (rounds past the last valid one hold none)
      const int w_next = snake(k + 1, blockIdx.x, gridDim.x);
      const bool has_next = w_next < n_items;
      mbar_wait(&kv_full[kv], (n / KVS) & 1);
      for (int it = 0; it < n_it; ++it, ++gi) {
        const int s = gi % NST;
        if (!issued) issue_sdp(gi, kv);
        // S/dP of this step are in registers: with a 2-deep Q/dO ring the next step's S/dP
        // overlap the elementwise math -- within the item (K/V stay), and with double-buffered
        // K/V also across items; otherwise they follow this step's dV/dK
        mbar_wait(tmem_free, gi & 1);
        if (lane == 0) FAB_PROBE(1, gi);
        tc_fence_after();
        issued = false;
        if (ALIAS) {
          // S/dP of the next step overwrite P^T / dS^T: issued after this step's dV/dK (below)
        } else if (NST > 1 && it + 1 < n_it) {
          issue_sdp(gi + 1, kv);
          issued = true;
        } else if (NST > 1 && KVS > 1 && has_next) {
          const int kv1 = (n + 1) % KVS;
          mbar_wait(&kv_full[kv1], ((n + 1) / KVS) & 1);
          tc_fence_after();
          issue_sdp(gi + 1, kv1);
          issued = true;
        }
        mbar_wait(p_ready, gi & 1);
        if (lane == 0) FAB_PROBE(2, gi);
        if (it == 0) mbar_wait(acc_free, (n & 1) ^ 1);  // previous item's dV/dK read out
        tc_fence_after();
        const uint32_t sQ = smem_u32(smem + L::OFF_Q + s * L::TILE), sDO = smem_u32(smem + L::OFF_DO + s * L::TILE);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BLK / 16; ++kk) {
            const uint32_t ao = (kk >> 2) * ATOM + (kk & 3) * 32;
            const uint32_t bo = kk * 2048;
            const uint32_t acc = (it > 0) || (kk > 0);
            if constexpr (PT_TMEM) {
              mma_bf16_ts(tmem + TM_DV, tmem + TM_PT + kk * 8, umma_desc_sw128(sDO + bo, ATOM, 1024), ID_G, acc);
              mma_bf16_ts(tmem + TM_DK, tmem + TM_DST + kk * 8, umma_desc_sw128(sQ + bo, ATOM, 1024), ID_G, acc);
            } else {
              mma_bf16_ss(tmem + TM_DV, umma_desc_sw128(sPT + ao, 16, 1024), umma_desc_sw128(sDO + bo, ATOM, 1024),
                          ID_G, acc);
              mma_bf16_ss(tmem + TM_DK, umma_desc_sw128(sDST + ao, 16, 1024), umma_desc_sw128(sQ + bo, ATOM, 1024),
                          ID_G, acc);
            }
          }
          mma_commit(mma2_done);
          mma_commit(&empty[s]);
          if (it + 1 == n_it) mma_commit(&kv_empty[kv]);
        }
        __syncwarp();
        if (ALIAS && it + 1 < n_it) {  // in issue order after the dV/dK MMAs that read P^T / dS^T
          issue_sdp(gi + 1, kv);
          issued = true;
        }
      }
    }
    }  // !HS
  } else if (warp == 3 && lane == 0) {
    // ---------------- dS^T tile -> workspace (b, h, qb, jb) for the dQ GEMM ----------------
    int gi = 0;
    const int ntri = nqb * (nqb + 1) / 2;
    for (int k = 0, w = snake(0, blockIdx.x, gridDim.x); k * (int)gridDim.x < n_items; ++k, w = snake(k, blockIdx.x, gridDim.x)) {
      if (w >= n_items) continue;
      int b, kvh, jb, gs;
      item(w, b, kvh, jb, gs);
      const int nq = nqb - jb, n_it = hpi * nq;
      for (int it = 0; it < n_it; ++it, ++gi) {
        const int h = kvh * group + gs * hpi + it / nq, qb = jb + it % nq;
        mbar_wait(HS ? p_ready_b : p_ready, gi & 1);
        const int row = ((b * p.H + h) * ntri + qb * (qb + 1) / 2 + jb) * BLK;
        for (int a = 0; a < 2; ++a) tma_store_2d(&tmDS, smem + L::OFF_DST + a * ATOM, 64 * a, row);
        bulk_commit();
        bulk_wait_read<0>();
        mbar_arrive(ds_read);
      }
    }
    bulk_wait<0>();
  } else if (warp >= 4) {
    // ---------------- elementwise: thread = key row, 64 query columns ----------------
    const int quad = warp & 3, half = (warp - 4) >> 2;
    const int r = quad * 32 + lane;  // key row within the block
    const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
    const float sl2 = p.scale * LOG2E;
    uint8_t* sPT = smem + L::OFF_PT;
    uint8_t* sDST = smem + L::OFF_DST;
    int gi = 0;
    for (int k = 0, w = snake(0, blockIdx.x, gridDim.x); k * (int)gridDim.x < n_items; ++k, w = snake(k, blockIdx.x, gridDim.x)) {
      if (w >= n_items) continue;
      int b, kvh, jb, gs;
      item(w, b, kvh, jb, gs);
      const int nq = nqb - jb, n_it = hpi * nq;
      for (int it = 0; it < n_it; ++it, ++gi) {
        const int s = gi % NST;
        const bool diag = (it % nq) == 0;  // query block == key block
        if constexpr (HS) {
          // two 64-query halves; this warp takes 32 query columns of each (half selects which)
          mbar_wait(&full[s], (gi / NST) & 1);  // lse / D of this step are in smem
          const float* lse = reinterpret_cast<const float*>(smem + L::OFF_LSE + s * 512);
          const float* dd = reinterpret_cast<const float*>(smem + L::OFF_D + s * 512);
#pragma unroll 1
          for (int hf = 0; hf < 2; ++hf) {
            mbar_wait(hf ? sdp_full_b : sdp_full, gi & 1);
            tc_fence_after();
            const int c0 = 64 * hf + 32 * half;
            uint32_t sv[32], dv[32];
            tmem_ld_32x32b_x32(lane_base + TM_S + c0, sv);
            tmem_ld_32x32b_x32(lane_base + TM_DP + c0, dv);
            tmem_ld_wait();
            uint32_t pk[16], dk[16];
            auto body = [&](auto diag_c) {
              constexpr bool DIAG = decltype(diag_c)::value;
#pragma unroll
              for (int c8 = 0; c8 < 4; ++c8) {
                float pv[8], ds[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                  const int c = c0 + 8 * c8 + j;
                  float pp = ex2(fmaf(__uint_as_float(sv[8 * c8 + j]), sl2, -lse[c]));
                  if (DIAG && c < r) pp = 0.f;  // query before key
                  pv[j] = pp;
                  ds[j] = pp * (__uint_as_float(dv[8 * c8 + j]) - dd[c]);
                }
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  pk[4 * c8 + e] = pack_bf16(pv[2 * e], pv[2 * e + 1]);
                  dk[4 * c8 + e] = pack_bf16(ds[2 * e], ds[2 * e + 1]);
                }
              }
            };
            if (diag) body(std::true_type{});
            else body(std::false_type{});
            if (hf == 0 && gi > 0) {
              mbar_wait(ds_read, (gi - 1) & 1);  // the previous dS^T tile store has read smem
              if (it == 0) {                     // this warp's dV/dK store has read its staging box
                if (lane == 0) bulk_wait_read<0>();
                __syncwarp();
              }
            }
            // P^T / dS^T over the half's S^T / dP^T columns: both warps of the quadrant have read them
            named_bar_sync(1 + quad, 64);
            tmem_st_32x32b_x16(lane_base + TM_S + 64 * hf + 16 * half, pk);
            tmem_st_32x32b_x16(lane_base + TM_DP + 64 * hf + 16 * half, dk);
#pragma unroll
            for (int c8 = 0; c8 < 4; ++c8) put_row8p(sDST, r, (c0 >> 3) + c8, dk + 4 * c8);
            tmem_st_wait();
            tc_fence_before();
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(hf ? p_ready_b : p_ready);
          }
          continue;
        }
        mbar_wait(&full[s], (gi / NST) & 1);  // lse / D of this step are in smem
        mbar_wait(sdp_full, gi & 1);
        if (warp == 4 && lane == 0) FAB_PROBE(3, gi);
        tc_fence_after();
        const float* lse = reinterpret_cast<const float*>(smem + L::OFF_LSE + s * 512);
        const float* dd = reinterpret_cast<const float*>(smem + L::OFF_D + s * 512);
        const int cb = 64 * half;
        // P^T and dS^T are formed in registers (bf16 pairs, 32 columns at a time) while the
        // previous step's dV/dK MMAs still read the tiles; only the stores wait for them
        uint32_t pk[32], dk[32];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t sv[32], dv[32];
          tmem_ld_32x32b_x32(lane_base + TM_S + cb + 32 * hh, sv);
          tmem_ld_32x32b_x32(lane_base + TM_DP + cb + 32 * hh, dv);
          tmem_ld_wait();
          if (hh == 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tmem_free);
          }
          // lse2 = lse * log2e (precomputed by the delta kernel); the causal mask only on the
          // diagonal block (separate code path: no per-element compare elsewhere)
          auto body = [&](auto diag_c) {
            constexpr bool DIAG = decltype(diag_c)::value;
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
              const int c8 = 4 * hh + c4;
              float pv[8], ds[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const int c = cb + 8 * c8 + j;
                float pp = ex2(fmaf(__uint_as_float(sv[8 * c4 + j]), sl2, -lse[c]));
                if (DIAG && c < r) pp = 0.f;  // query before key
                pv[j] = pp;
                ds[j] = pp * (__uint_as_float(dv[8 * c4 + j]) - dd[c]);
              }
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                pk[4 * c8 + e] = pack_bf16(pv[2 * e], pv[2 * e + 1]);
                dk[4 * c8 + e] = pack_bf16(ds[2 * e], ds[2 * e + 1]);
              }
            }
          };
          if (diag) body(std::true_type{});
          else body(std::false_type{});
        }
        if (warp == 4 && lane == 0) FAB_PROBE(4, gi);
        if (gi > 0) {
          mbar_wait(mma2_done, (gi - 1) & 1);  // P^T / dS^T tiles free
          mbar_wait(ds_read, (gi - 1) & 1);    // the dS^T store has read its tile
          if (it == 0) {                       // this warp's dV/dK store has read its staging boxes
            if (lane == 0) bulk_wait_read<0>();
            __syncwarp();
          }
        }
        if (warp == 4 && lane == 0) FAB_PROBE(5, gi);
        if constexpr (PT_TMEM) {
          // P^T / dS^T of this thread's key row and 64 query columns -> TMEM (A of the TS MMAs).
          // ALIAS: the two warps of a lane quadrant both finished reading S^T / dP^T first (half 1
          // writes columns half 0 reads)
          if constexpr (ALIAS) named_bar_sync(1 + quad, 64);
          tmem_st_32x32b_x32(lane_base + TM_PT + (cb >> 1), pk);
          tmem_st_32x32b_x32(lane_base + TM_DST + (cb >> 1), dk);
#pragma unroll
          for (int c8 = 0; c8 < 8; ++c8) put_row8p(sDST, r, (cb >> 3) + c8, dk + 4 * c8);
          tmem_st_wait();
          tc_fence_before();
        } else {
#pragma unroll
          for (int c8 = 0; c8 < 8; ++c8) {
            put_row8p(sPT, r, (cb >> 3) + c8, pk + 4 * c8);
            put_row8p(sDST, r, (cb >> 3) + c8, dk + 4 * c8);
          }
        }

        fence_proxy_async();
        __syncwarp();
        if (warp == 4 && lane == 0) FAB_PROBE(6, gi);
        if (lane == 0) mbar_arrive(p_ready);
      }
      // item outputs: half 0 writes dV, half 1 writes dK (scaled, inverse RoPE), staged in the
      // warp's own quarter of the P^T / dS^T tiles (free once the last dV/dK MMAs and the last
      // dS^T store are done; the warp writes the same bytes again first at its next step) and
      // written by TMA
      mbar_wait(mma2_done, (gi - 1) & 1);
      mbar_wait(ds_read, (gi - 1) & 1);
      tc_fence_after();
      if (p.gsplit > 1) {
        // GQA split: this item's fp32 dV / dK partial (raw: unscaled, no RoPE) to the workspace,
        // [tile][gs][dV|dK][column][row] so a warp's 32 rows are one 128-byte store per column;
        // dkdv_reduce_kernel sums the partials in gs order
        const size_t tile = ((size_t)(b * p.Hkv + kvh) * nqb + jb) * p.gsplit + gs;
        float* dst = p.part + (tile * 2 + half) * HD * BLK;
        const uint32_t ta = lane_base + (half == 0 ? TM_DV : TM_DK);
#pragma unroll 1
        for (int c = 0; c < HD; c += 32) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(ta + c, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) dst[(size_t)(c + j) * BLK + r] = __uint_as_float(v[j]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_free);
        continue;
      }
      const int key = jb * BLK + r;
      if constexpr (ALIAS) {
        // one 4 KB box per warp (its quarter of the dS^T tile): the two 64-column halves in turn
        uint8_t* box = smem + L::OFF_DST + half * ATOM + quad * 4096;
        const int col = (half == 0 ? p.H + p.Hkv + kvh : p.H + kvh) * HD, row = b * p.T + jb * BLK + quad * 32;
#pragma unroll 1
        for (int a = 0; a < 2; ++a) {
          if (a == 1) {
            if (lane == 0) bulk_wait_read<0>();
            __syncwarp();
          }
          if (half == 0) stage_grad_row<HD>(lane_base + TM_DV, box, box, lane, 1.f, nullptr, p.T, key, a);
          else stage_grad_row<HD>(lane_base + TM_DK, box, box, lane, p.scale, p.rope_cs, p.T, key, a);
          tc_fence_before();
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            if (a == 1) mbar_arrive(acc_free);
            tma_store_2d(&tmOut, box, col + 64 * a, row);
            bulk_commit();
          }
        }
        continue;
      }
      uint8_t* box0 = smem + (L::PT_TMEM ? L::OFF_DST : L::OFF_PT) + half * ATOM + quad * 4096;
      uint8_t* box1 = smem + L::OFF_DST + half * ATOM + quad * 4096;
      if (half == 0) stage_grad_row<HD>(lane_base + TM_DV, box0, box1, lane, 1.f, nullptr, p.T, key);
      else stage_grad_row<HD>(lane_base + TM_DK, box0, box1, lane, p.scale, p.rope_cs, p.T, key);
      tc_fence_before();
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(acc_free);
        const int col = (half == 0 ? p.H + p.Hkv + kvh : p.H + kvh) * HD, row = b * p.T + jb * BLK + quad * 32;
        tma_store_2d(&tmOut, box0, col, row);
        if (HD == 128) tma_store_2d(&tmOut, box1, col + 64, row);
        bulk_commit();
      }
    }
    if (lane == 0) bulk_wait<0>();
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

// ------------------------------------------------------------------------------------------
// dQ = dS K as a GEMM over the dS^T tiles the dK/dV kernel stored (no recomputation of S, dP or
// the softmax).  Persistent, heavy-first items (batch, head, query block ib); per key block j <= ib
// the producer stages the dS^T tile (A, MN-major: rows = keys, columns = queries) and K_j (B,
// MN-major); dQ accumulates in TMEM (double-buffered across items) and 4 epilogue warps write it
// (scaled, inverse RoPE) while the next item accumulates.
// ------------------------------------------------------------------------------------------
template <int HD>
struct DqmSmem {
  static constexpr int DS_BYTES = 2 * ATOM;                 // 128 keys x 128 queries bf16
  static constexpr int K_BYTES = (HD / 64) * ATOM;          // 128 keys x HD
  static constexpr int STAGE = DS_BYTES + K_BYTES;
  static constexpr int STAGES = HD == 64 ? 4 : 3;
  static constexpr int OFF_STG = STAGES * STAGE;            // dQ staging: [HD/64][128 rows][128 B]
  static constexpr int OFF_BAR = OFF_STG + (HD / 64) * ATOM;
  static constexpr int BYTES = OFF_BAR + 256;
  static constexpr int THREADS = 256;                       // producer, MMA, TMEM, spare, 4 epilogue warps
};

template <int HD>
__global__ void __launch_bounds__(DqmSmem<HD>::THREADS, 1)
    attn_bwd_dq_mma_kernel(const __grid_constant__ CUtensorMap tmQKV, const __grid_constant__ CUtensorMap tmDS,
                           const __grid_constant__ CUtensorMap tmOut, const BwdParams p) {
  using L = DqmSmem<HD>;
  constexpr int STAGES = L::STAGES;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* full = bars;                // [STAGES]
  uint64_t* empty = bars + STAGES;      // [STAGES]
  uint64_t* acc_full = bars + 2 * STAGES;       // [2]
  uint64_t* acc_empty = bars + 2 * STAGES + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = p.T / BLK;
  const int ntri = nqb * (nqb + 1) / 2;
  const int BH = p.B * p.H;
  const int n_items = nqb * BH;
  const int group = p.H / p.Hkv;
  auto item = [&](int w, int& b, int& h, int& ib) {
    ib = nqb - 1 - w / BH;  // late query blocks see the most key blocks: heavy first
    b = (w % BH) / p.H;
    h = (w % BH) % p.H;
  };

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmQKV);
    tma_prefetch_desc(&tmDS);
    tma_prefetch_desc(&tmOut);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 4);
    }
    fence_barrier_init();
    fence_proxy_async();
  }
  constexpr uint32_t TMEM_COLS = 2 * HD;
  if (warp == 2) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // the dK/dV kernel's dS^T tiles are complete

  if (warp == 0 && lane == 0) {
    int g = 0;
    for (int k = 0, w = snake(0, blockIdx.x, gridDim.x); k * (int)gridDim.x < n_items; ++k, w = snake(k, blockIdx.x, gridDim.x)) {
      if (w >= n_items) continue;
      int b, h, ib;
      item(w, b, h, ib);
      const int kvh = h / group;
      const int tile0 = (b * p.H + h) * ntri + ib * (ib + 1) / 2;
      for (int j = 0; j <= ib; ++j, ++g) {
        const int st = g % STAGES;
        mbar_wait(&empty[st], ((g / STAGES) & 1) ^ 1);
        mbar_expect_tx(&full[st], L::STAGE);
        uint8_t* sd = smem + st * L::STAGE;
        for (int a = 0; a < 2; ++a) tma_load_2d(sd + a * ATOM, &tmDS, &full[st], 64 * a, (tile0 + j) * BLK);
        for (int a = 0; a < HD / 64; ++a)
          tma_load_2d(sd + L::DS_BYTES + a * ATOM, &tmQKV, &full[st], (p.H + kvh) * HD + 64 * a, b * p.T + j * BLK);
      }
    }
  } else if (warp == 1) {  // MMA issuer: whole warp, one elected lane issues
    constexpr uint32_t ID = umma_idesc_bf16(BLK, HD, true, true);  // dS (MN-major) . K (MN-major)
    int g = 0, n = 0;
    for (int k = 0, w = snake(0, blockIdx.x, gridDim.x); k * (int)gridDim.x < n_items; ++k, w = snake(k, blockIdx.x, gridDim.x), ++n) {
      if (w >= n_items) continue;
      int b, h, ib;
      item(w, b, h, ib);
      const int acc = n & 1;
      mbar_wait(&acc_empty[acc], ((n >> 1) & 1) ^ 1);
      tc_fence_after();
      for (int j = 0; j <= ib; ++j, ++g) {
        const int st = g % STAGES;
        mbar_wait(&full[st], (g / STAGES) & 1);
        tc_fence_after();
        const uint32_t sd = smem_u32(smem + st * L::STAGE), sk = sd + L::DS_BYTES;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BLK / 16; ++kk)
            mma_bf16_ss(tmem + acc * HD, umma_desc_sw128(sd + kk * 2048, ATOM, 1024),
                        umma_desc_sw128(sk + kk * 2048, ATOM, 1024), ID, (j > 0) || (kk > 0));
          mma_commit(&empty[st]);
        }
        __syncwarp();
      }
      if (elect_one()) mma_commit(&acc_full[acc]);
      __syncwarp();
    }
  } else if (warp >= 4) {
    const int quad = warp - 4;
    const int r = quad * 32 + lane;
    int n = 0;
    for (int k = 0, w = snake(0, blockIdx.x, gridDim.x); k * (int)gridDim.x < n_items; ++k, w = snake(k, blockIdx.x, gridDim.x), ++n) {
      if (w >= n_items) continue;
      int b, h, ib;
      item(w, b, h, ib);
      const int acc = n & 1;
      mbar_wait(&acc_full[acc], (n >> 1) & 1);
      tc_fence_after();
      if (lane == 0) bulk_wait_read<0>();  // the previous item's store has read the staging boxes
      __syncwarp();
      const int t = ib * BLK + r;
      uint8_t* box0 = smem + L::OFF_STG + quad * 4096;
      stage_grad_row<HD>(tmem + ((uint32_t)(quad * 32) << 16) + acc * HD, box0, box0 + ATOM, lane, p.scale,
                         p.rope_cs, p.T, t);
      tc_fence_before();
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&acc_empty[acc]);
        const int row = b * p.T + ib * BLK + quad * 32;
        tma_store_2d(&tmOut, box0, h * HD, row);
        if (HD == 128) tma_store_2d(&tmOut, box0 + ATOM, h * HD + 64, row);
        bulk_commit();
      }
    }
    if (lane == 0) bulk_wait<0>();
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, TMEM_COLS);
}

// GQA split: dK / dV of one (batch, kv head, key block) tile = the sum of its gsplit fp32 partials
// in gs order (deterministic), scaled (dK), inverse RoPE (dK, when a table is given), bf16 into
// dQKV.  Block = (tile, dV|dK, 16 rotation pairs (c, c + hd/2)), thread = key row: every partial
// load is coalesced along the rows and all of a thread's loads are in flight together.
template <int HD>
__global__ void __launch_bounds__(BLK) dkdv_reduce_kernel(const BwdParams p) {
  pdl_wait();
  constexpr int NP = 16;  // pairs per block
  const int nqb = p.T / BLK;
  const int tile = blockIdx.x, which = blockIdx.y, j0 = blockIdx.z * NP;  // which: 0 = dV, 1 = dK
  const int jb = tile % nqb, kvh = (tile / nqb) % p.Hkv, b = tile / (nqb * p.Hkv);
  const int r = threadIdx.x, pos = jb * BLK + r;
  const float* src = p.part + (size_t)tile * p.gsplit * 2 * HD * BLK + (size_t)which * HD * BLK + r;
  const size_t gstride = (size_t)2 * HD * BLK;
  float x1[NP], x2[NP];
#pragma unroll
  for (int j = 0; j < NP; ++j) x1[j] = x2[j] = 0.f;
  for (int g = 0; g < p.gsplit; ++g) {
    const float* sg = src + g * gstride;
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      x1[j] += sg[(size_t)(j0 + j) * BLK];
      x2[j] += sg[(size_t)(HD / 2 + j0 + j) * BLK];
    }
  }
  const float scale = which == 1 ? p.scale : 1.f;
  float o1[NP], o2[NP];
  if (which == 1 && p.rope_cs) {
    const float2* cs = reinterpret_cast<const float2*>(p.rope_cs);
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const float a = x1[j] * scale, c = x2[j] * scale;
      const float2 w = cs[(size_t)(j0 + j) * p.T + pos];
      o1[j] = a * w.x + c * w.y;
      o2[j] = c * w.x - a * w.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      o1[j] = x1[j] * scale;
      o2[j] = x2[j] * scale;
    }
  }
  __nv_bfloat16* dst = p.dqkv + (size_t)(b * p.T + pos) * p.ld + (which == 0 ? p.H + p.Hkv + kvh : p.H + kvh) * HD;
#pragma unroll
  for (int j = 0; j < NP; j += 8) {
    *reinterpret_cast<uint4*>(dst + j0 + j) = make_uint4(pack_bf16(o1[j], o1[j + 1]), pack_bf16(o1[j + 2], o1[j + 3]),
                                                         pack_bf16(o1[j + 4], o1[j + 5]), pack_bf16(o1[j + 6], o1[j + 7]));
    *reinterpret_cast<uint4*>(dst + HD / 2 + j0 + j) =
        make_uint4(pack_bf16(o2[j], o2[j + 1]), pack_bf16(o2[j + 2], o2[j + 3]), pack_bf16(o2[j + 4], o2[j + 5]),
                   pack_bf16(o2[j + 6], o2[j + 7]));
  }
}

static int make_map(CUtensorMap* m, const void* ptr, long long ld, long long rows, int box_rows = 128) {
  // 2D bf16 [rows][ld], 64 x box_rows boxes, SWIZZLE_128B
  auto encode = get_tensor_map_encoder();
  if (!encode) return set_error(SPX_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? SPX_OK : set_error(SPX_ERR_CUDA, "attn_bwd_tc: tensor map encode failed");
}

template <int HD>
static int launch(const void* qkv, const void* dout, long long ld_o, const BwdParams& p, cudaStream_t s) {
  CUtensorMap mq, md;
  int rc = make_map(&mq, qkv, p.ld, (long long)p.B * p.T);
  if (rc) return rc;
  rc = make_map(&md, dout, ld_o, (long long)p.B * p.T);
  if (rc) return rc;
  CUtensorMap mo;  // dQKV, 32-row boxes (one per epilogue warp)
  rc = make_map(&mo, p.dqkv, p.ld, (long long)p.B * p.T, 32);
  if (rc) return rc;
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_dkdv_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         DkdvSmem<HD>::BYTES);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_bwd_dq_mma_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               DqmSmem<HD>::BYTES);
    if (e != cudaSuccess) return set_cuda_error(e, "attn_bwd_tc attr");
    set = true;
  }
  const int nqb = p.T / BLK;
  CUtensorMap mds;  // dS^T tiles [B*H*tri(nqb)*128][128] bf16
  const long long ntiles = (long long)p.B * p.H * (nqb * (nqb + 1) / 2);
  rc = make_map(&mds, p.ds, BLK, ntiles * BLK);
  if (rc) return rc;
  const int items_kv = nqb * p.Hkv * p.B * p.gsplit, items_q = nqb * p.H * p.B;
  const int g1 = items_kv < num_sms() ? items_kv : num_sms(), g2 = items_q < num_sms() ? items_q : num_sms();
  spx_launch_check(launch_k(attn_bwd_dkdv_tc_kernel<HD>, dim3(g1), dim3(THREADS), DkdvSmem<HD>::BYTES, s, mq, md, mds, mo, p));
  rc = check_launch("attn_bwd_dkdv_tc_kernel");
  if (rc) return rc;
  if (p.gsplit > 1) {
    spx_launch_check(launch_k(dkdv_reduce_kernel<HD>, dim3(p.B * p.Hkv * nqb, 2, HD / 32), dim3(BLK), 0, s, p));
    rc = check_launch("dkdv_reduce_kernel");
    if (rc) return rc;
  }
  spx_launch_check(launch_k(attn_bwd_dq_mma_kernel<HD>, dim3(g2), dim3(DqmSmem<HD>::THREADS), DqmSmem<HD>::BYTES, s,
                            mq, mds, mo, p));
  return check_launch("attn_bwd_dq_mma_kernel");
}

}  // namespace fab

// used by spx_attn_bwd (attention.cu) for head_dim 64/128, T % 128 == 0; delta must be computed
int attn_bwd_tcgen05(const void* qkv, const void* dout, const float* lse, const float* delta, void* dqkv, int64_t B,
                     int64_t T, int64_t H, int64_t Hkv, int64_t hd, int64_t ld_qkv, int64_t ld_o, float scale,
                     const float* rope_cs, bool gqa_split, cudaStream_t s) {
  // workspace: delta [BHT] | lse*log2e [BHT] | dS^T tiles (bf16) | GQA-split dV/dK partials (fp32)
  __nv_bfloat16* ds = reinterpret_cast<__nv_bfloat16*>(const_cast<float*>(delta) + 2 * B * H * T);
  const int64_t nqb = T / fab::BLK;
  float* part = const_cast<float*>(delta) + 2 * B * H * T + B * H * (nqb * (nqb + 1) / 2) * fab::BLK * fab::BLK / 2;
  fab::BwdParams p{reinterpret_cast<__nv_bfloat16*>(dqkv), lse, delta, rope_cs, ds, (long long)ld_qkv,
                   (int)B, (int)T, (int)H, (int)Hkv, scale, gqa_split ? (int)(H / Hkv) : 1, part};
  if (hd == 64) return fab::launch<64>(qkv, dout, ld_o, p, s);
  return fab::launch<128>(qkv, dout, ld_o, p, s);
}

}  // namespace spx
