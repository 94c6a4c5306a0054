// tcgen05 flash-attention forward for sm_100a (causal, GQA, head_dim 64 or 128).
//
// Persistent kernel: one CTA per SM walks a heavy-first list of work items (128 query rows of one
// (batch, head)); TMEM is allocated once and every mbarrier keeps its phase across items, so the
// pipeline never drains between items.  Warp roles:
//   warp 0      TMA producer: Q per item, then K_j / V_j (128 keys) into a 2-stage ring, read in
//               place from the fused QKV buffer with one SWIZZLE_128B tensor map
//   warp 1      single-thread tcgen05.mma issuer:  S_j = Q K_j^T  (M=128, N=128, K=hd) into one of
//               two TMEM buffers, then O += P_j V_j (M=128, N=hd, K=128; V as an MN-major operand)
//   warp 2      TMEM allocation (512 columns: S0, S1, O)
//   warps 4-11  softmax: thread = query row (its TMEM lane), two warps per lane quadrant splitting
//               the 128 keys of a block.  Reads S_j, keeps running max/sum in the exp2 domain
//               (split accumulators: no long dependent chains; lazy rescaling), rescales O in TMEM
//               when the max grows by more than 2^8, writes P_j (bf16 pairs) into TMEM (A of the PV
//               MMA), and at the end of an item writes O / l and the LSE.
// S_{j+1} overlaps the softmax of block j; the next item's S MMAs overlap the previous item's
// epilogue.  O and LSE match attn_fwd_kernel (attention.cu).
#include <cmath>

#include "spx_common.cuh"
#include "spx_internal.h"

namespace spx {
namespace fa {

constexpr int BM = 128;    // query rows per work item
constexpr int BN = 128;    // keys per block
constexpr int THREADS = 384;  // 4 role warps + 8 softmax warps (2 per TMEM lane quadrant)
constexpr float LOG2E = 1.4426950408889634f;
constexpr float RESCALE_LOG2 = 8.f;  // lazy-rescale threshold (log2 domain)

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
SPX_DEVICE void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// named barrier over the two softmax warps that share a TMEM lane quadrant
SPX_DEVICE void pair_bar(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }

// Heavy-first item lists are dealt to CTAs in boustrophedon order (round k: CTA c takes item
// k*G + c for even k, k*G + G-1-c for odd k), pairing heavy and light items per CTA.
SPX_DEVICE int snake(int k, int c, int G) { return k * G + ((k & 1) ? (G - 1 - c) : c); }

SPX_DEVICE float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

#ifdef SPX_FA_PROBE
__device__ long long g_fa_probe[8][256];
#define FA_PROBE(ev, step) \
  do { if (blockIdx.x == 0 && (step) < 256) g_fa_probe[ev][step] = clock64(); } while (0)
#else
#define FA_PROBE(ev, step) do { } while (0)
#endif

constexpr float EXTREME_LOG2 = 64.f;  // lagged-max overflow guard (P <= 2^64)

// tcgen05.wait::ld that the compiler sees as redefining the loaded registers, so no use of them
// is scheduled before the wait
SPX_DEVICE void tmem_ld_wait_dep(uint32_t (&a)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7]),
                 "+r"(a[8]), "+r"(a[9]), "+r"(a[10]), "+r"(a[11]), "+r"(a[12]), "+r"(a[13]), "+r"(a[14]),
                 "+r"(a[15]), "+r"(a[16]), "+r"(a[17]), "+r"(a[18]), "+r"(a[19]), "+r"(a[20]), "+r"(a[21]),
                 "+r"(a[22]), "+r"(a[23]), "+r"(a[24]), "+r"(a[25]), "+r"(a[26]), "+r"(a[27]), "+r"(a[28]),
                 "+r"(a[29]), "+r"(a[30]), "+r"(a[31])::"memory");
}
SPX_DEVICE void tmem_ld_wait_dep(uint32_t (&a)[32], uint32_t (&b)[32]) {
  tmem_ld_wait_dep(a);
  // b completed with a (wait::ld covers every outstanding load); pin it after the wait as well
  asm volatile(""
               : "+r"(b[0]), "+r"(b[1]), "+r"(b[2]), "+r"(b[3]), "+r"(b[4]), "+r"(b[5]), "+r"(b[6]), "+r"(b[7]),
                 "+r"(b[8]), "+r"(b[9]), "+r"(b[10]), "+r"(b[11]), "+r"(b[12]), "+r"(b[13]), "+r"(b[14]),
                 "+r"(b[15]), "+r"(b[16]), "+r"(b[17]), "+r"(b[18]), "+r"(b[19]), "+r"(b[20]), "+r"(b[21]),
                 "+r"(b[22]), "+r"(b[23]), "+r"(b[24]), "+r"(b[25]), "+r"(b[26]), "+r"(b[27]), "+r"(b[28]),
                 "+r"(b[29]), "+r"(b[30]), "+r"(b[31])::"memory");
}

SPX_DEVICE float max3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// causal mask on the diagonal block: scores of keys after query row r -> -inf
SPX_DEVICE void mask_chunk(uint32_t (&v)[32], int col0, int r) {
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (col0 + i > r) v[i] = 0xff800000u;
}

// raw (unscaled) maximum of 32 scores
SPX_DEVICE float chunk_max(const uint32_t (&v)[32]) {
  float mk[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) mk[k] = -INFINITY;
#pragma unroll
  for (int i = 0; i < 32; i += 2) mk[(i >> 1) & 3] = max3(mk[(i >> 1) & 3], __uint_as_float(v[i]), __uint_as_float(v[i + 1]));
  return fmaxf(fmaxf(mk[0], mk[1]), fmaxf(mk[2], mk[3]));
}

// P = 2^(s * sl2 - m) for 32 scores -> 16 bf16 pairs; adds to sum and tracks the raw maximum.
// Scale-and-shift as packed FFMA2, sums as packed FADD2, maxima as 3-input FMNMX.
#ifndef SPX_FA_POLY
#define SPX_FA_POLY 1  // quarters of the exponentials computed by ex2_poly2 (0..4)
#endif
// 2^x for two arguments on the FMA / integer pipes (FA4-style MUFU relief): x = j + f with
// j = round(x) from the 1.5*2^23 magic add, 2^f on [-0.5, 0.5] by a cubic with p(0) = 1 (max
// relative error 1.0e-4, below bf16's 3.9e-3 half-ulp), 2^j added to the exponent bits.  x is
// clamped at -127, where the result is exactly 0 (masked scores).
SPX_DEVICE void ex2_poly2(float& ya, float& yb) {
  constexpr float C1 = 0.693282932425875f, C2 = 0.24221100073552806f, C3 = 0.05500892622514074f;
  const float xa = fmaxf(ya, -127.f), xb = fmaxf(yb, -127.f);
  float ta, tb, fa, fb, pa, pb;
  asm("{\n\t.reg .b64 x, m, t, j, f;\n\t"
      "mov.b64 x, {%6, %7};\n\tmov.b64 m, {%8, %8};\n\t"
      "add.rn.f32x2 t, x, m;\n\tsub.rn.f32x2 j, t, m;\n\tsub.rn.f32x2 f, x, j;\n\t"
      "mov.b64 {%0, %1}, t;\n\tmov.b64 {%2, %3}, f;\n\t}"
      : "=f"(ta), "=f"(tb), "=f"(fa), "=f"(fb), "=f"(pa), "=f"(pb)
      : "f"(xa), "f"(xb), "f"(12582912.f));
  asm("{\n\t.reg .b64 f, p, c;\n\t"
      "mov.b64 f, {%2, %3};\n\t"
      "mov.b64 c, {%5, %5};\n\tmov.b64 p, {%4, %4};\n\tfma.rn.f32x2 p, p, f, c;\n\t"
      "mov.b64 c, {%6, %6};\n\tfma.rn.f32x2 p, p, f, c;\n\t"
      "mov.b64 c, {%7, %7};\n\tfma.rn.f32x2 p, p, f, c;\n\t"
      "mov.b64 {%0, %1}, p;\n\t}"
      : "=f"(pa), "=f"(pb)
      : "f"(fa), "f"(fb), "f"(C3), "f"(C2), "f"(C1), "f"(1.f));
  ya = __int_as_float(__float_as_int(pa) + (__float_as_int(ta) << 23));
  yb = __int_as_float(__float_as_int(pb) + (__float_as_int(tb) << 23));
}

SPX_DEVICE void exp_chunk(const uint32_t (&v)[32], float sl2, float m, uint32_t* pk, float& sum, float& bmax) {
  float s2[4][2] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
  float mk[2] = {bmax, -INFINITY};
  const float nm = -m;
#pragma unroll
  for (int i = 0; i < 32; i += 2) {
    const float a = __uint_as_float(v[i]), b = __uint_as_float(v[i + 1]);
    mk[(i >> 1) & 1] = max3(mk[(i >> 1) & 1], a, b);
    float ya, yb;
    asm("{\n\t.reg .b64 x, k, c, y;\n\t"
        "mov.b64 x, {%2, %3};\n\tmov.b64 k, {%4, %4};\n\tmov.b64 c, {%5, %5};\n\t"
        "fma.rn.f32x2 y, x, k, c;\n\tmov.b64 {%0, %1}, y;\n\t}"
        : "=f"(ya), "=f"(yb)
        : "f"(a), "f"(b), "f"(sl2), "f"(nm));
    if (((i >> 1) & 3) >= 4 - SPX_FA_POLY) {
      ex2_poly2(ya, yb);  // a quarter of the exponentials on the FMA pipe (MUFU relief)
    } else {
      ya = ex2(ya);
      yb = ex2(yb);
    }
    float* acc = s2[(i >> 1) & 3];
    asm("{\n\t.reg .b64 x, y;\n\t"
        "mov.b64 x, {%0, %1};\n\tmov.b64 y, {%2, %3};\n\t"
        "add.rn.f32x2 x, x, y;\n\tmov.b64 {%0, %1}, x;\n\t}"
        : "+f"(acc[0]), "+f"(acc[1])
        : "f"(ya), "f"(yb));
    pk[i >> 1] = pack_bf16(ya, yb);
  }
  bmax = fmaxf(mk[0], mk[1]);
  sum += ((s2[0][0] + s2[0][1]) + (s2[1][0] + s2[1][1])) + ((s2[2][0] + s2[2][1]) + (s2[3][0] + s2[3][1]));
}

struct FwdParams {
  __nv_bfloat16* out;  // O [B*T, ldo]
  float* lse;          // [B, H, T]
  long long ldo;
  int B, T, H, Hkv;
  float scale;
};

// work item w (heavy first): query block qb = nqb-1 - w / (B*H), (b, h) = w % (B*H)
struct Item {
  int b, h, qb;
};
SPX_DEVICE Item item_of(int w, int nqb, int BH, int H) {
  Item it;
  it.qb = nqb - 1 - w / BH;
  const int bh = w % BH;
  it.b = bh / H;
  it.h = bh % H;
  return it;
}

template <int HD>
struct FwdSmem {
  static constexpr int ATOM = BM * 128;              // 128 rows x 128 B (64 bf16) swizzle atom block
  static constexpr int Q_BYTES = (HD / 64) * ATOM;   // same for one K or V tile (128 rows)
  // K and V have separate rings: a K tile is released as soon as its S MMA completes, a V tile
  // only after its PV MMA, so K prefetch runs ahead of the softmax
  static constexpr int NK = HD == 64 ? 3 : 2;
  static constexpr int NV = HD == 64 ? 3 : 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;        // [NK]
  static constexpr int OFF_V = OFF_K + NK * Q_BYTES;   // [NV]
  static constexpr int OFF_BAR = OFF_V + NV * Q_BYTES;
  // row-max exchange between the two column halves of a row: [block parity][half][row], then the
  // row-sum exchange at the end of an item: [half][row]
  static constexpr int OFF_RED = OFF_BAR + 256;
  // >= 116 KB: one CTA per SM (it owns all 512 TMEM columns)
  // hd=128: O staging for the TMA store, one 32-row x 64-column box per softmax warp
  static constexpr bool STG = HD == 128;
  static constexpr int OFF_STG = (OFF_RED + 6 * BM * 4 + 1023) / 1024 * 1024;
  static constexpr int RAW = OFF_STG + (STG ? 2 * ATOM : 0);
  static constexpr int BYTES = RAW > 116 * 1024 ? RAW : 116 * 1024;
};

// 32 fp32 accumulator values (columns c0 .. c0+31 of a 64-column box row) * inv -> bf16, into a
// 32-row SWIZZLE_128B box (the TMA store's layout; conflict-free 16-byte writes)
SPX_DEVICE void box_put32(uint8_t* box, int row, int c0, const uint32_t* v, float inv) {
#pragma unroll
  for (int i = 0; i < 32; i += 8) {
    const int chunk = (c0 + i) >> 3;
    *reinterpret_cast<uint4*>(box + row * 128 + ((chunk ^ (row & 7)) << 4)) =
        make_uint4(pack_bf16(__uint_as_float(v[i]) * inv, __uint_as_float(v[i + 1]) * inv),
                   pack_bf16(__uint_as_float(v[i + 2]) * inv, __uint_as_float(v[i + 3]) * inv),
                   pack_bf16(__uint_as_float(v[i + 4]) * inv, __uint_as_float(v[i + 5]) * inv),
                   pack_bf16(__uint_as_float(v[i + 6]) * inv, __uint_as_float(v[i + 7]) * inv));
  }
}

template <int HD>
__global__ void __launch_bounds__(THREADS, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmQKV, const __grid_constant__ CUtensorMap tmO,
                       const FwdParams p) {
  using L = FwdSmem<HD>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  constexpr int NK = L::NK, NV = L::NV;
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* s_full = bars + 2;   // [2]
  uint64_t* p_full = bars + 4;   // [2] by block parity (P is double-buffered in TMEM)
  uint64_t* o_free = bars + 6;
  uint64_t* pv_done = bars + 14 + 2 * NK + 2 * NV;  // [2] by block parity
  uint64_t* k_full = bars + 8;            // [NK]
  uint64_t* k_empty = bars + 8 + NK;      // [NK]
  uint64_t* v_full = bars + 8 + 2 * NK;   // [NV]
  uint64_t* v_empty = bars + 8 + 2 * NK + NV;  // [NV]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8 + 2 * NK + 2 * NV);  // (+ 6 words spare)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = p.T / BM;
  const int BH = p.B * p.H;
  const int n_items = nqb * BH;
  const int group = p.H / p.Hkv;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmQKV);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < 2; ++i) mbar_init(&s_full[i], 1);
    for (int i = 0; i < NK; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < NV; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&p_full[i], 8);
      mbar_init(&pv_done[i], 1);
    }
    mbar_init(o_free, 8);
    fence_barrier_init();
    fence_proxy_async();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // upstream grid complete before any dependent global access
  // TMEM: S0 [0,128), S1 [128,256), O [256, 256+HD), P double buffer [384,448), [448,512): P
  // (bf16 pairs, row = query) is the A operand of the PV MMA straight from TMEM, so it never
  // touches shared memory (the kernel is otherwise shared-memory-bandwidth bound at hd=64)
  constexpr uint32_t TM_O = 256, TM_P = 384;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer: Q and K ----------------
    int g = 0, n = 0;  // global key-block counter, item counter
    for (int k = 0, w = snake(0, blockIdx.x, gridDim.x); k * (int)gridDim.x < n_items; ++k, w = snake(k, blockIdx.x, gridDim.x), ++n) {
      if (w >= n_items) continue;
      const Item it = item_of(w, nqb, BH, p.H);
      const int row0 = it.b * p.T, kvh = it.h / group;
      mbar_wait(q_empty, (n & 1) ^ 1);
      mbar_expect_tx(q_full, L::Q_BYTES);
      for (int a = 0; a < HD / 64; ++a)
        tma_load_2d(smem + L::OFF_Q + a * L::ATOM, &tmQKV, q_full, it.h * HD + 64 * a, row0 + it.qb * BM);
      for (int j = 0; j <= it.qb; ++j, ++g) {
        const int s = g % NK;
        mbar_wait(&k_empty[s], ((g / NK) & 1) ^ 1);
        mbar_expect_tx(&k_full[s], L::Q_BYTES);
        for (int a = 0; a < HD / 64; ++a)
          tma_load_2d(smem + L::OFF_K + s * L::Q_BYTES + a * L::ATOM, &tmQKV, &k_full[s], (p.H + kvh) * HD + 64 * a,
                      row0 + j * BN);
      }
    }
  } else if (warp == 3 && lane == 0) {
    // ---------------- TMA producer: V ----------------
    int g = 0;
    for (int k = 0, w = snake(0, blockIdx.x, gridDim.x); k * (int)gridDim.x < n_items; ++k, w = snake(k, blockIdx.x, gridDim.x)) {
      if (w >= n_items) continue;
      const Item it = item_of(w, nqb, BH, p.H);
      const int row0 = it.b * p.T, kvh = it.h / group;
      for (int j = 0; j <= it.qb; ++j, ++g) {
        const int s = g % NV;
        mbar_wait(&v_empty[s], ((g / NV) & 1) ^ 1);
        mbar_expect_tx(&v_full[s], L::Q_BYTES);
        for (int a = 0; a < HD / 64; ++a)
          tma_load_2d(smem + L::OFF_V + s * L::Q_BYTES + a * L::ATOM, &tmQKV, &v_full[s],
                      (p.H + p.Hkv + kvh) * HD + 64 * a, row0 + j * BN);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (whole warp; one elected lane issues) ----------------
    constexpr uint32_t IDESC_S = umma_idesc_bf16(BM, BN, false, false);
    constexpr uint32_t IDESC_O = umma_idesc_bf16(BM, HD, false, true);
    const uint32_t sQ = smem_u32(smem + L::OFF_Q);
    int g = 0, n = 0;
    // PV of block (global index gb, item-local j); the first PV of an item overwrites O, which
    // the softmax warps must have read out for the previous item
    auto issue_pv = [&](int gb, int j, int item_n) {
      const int s = gb % NV;
      if (j == 0) mbar_wait(o_free, (item_n & 1) ^ 1);
      mbar_wait(&p_full[gb & 1], (gb >> 1) & 1);
      mbar_wait(&v_full[s], (gb / NV) & 1);
      if (lane == 0) FA_PROBE(7, gb);
      tc_fence_after();
      const uint32_t sV = smem_u32(smem + L::OFF_V + s * L::Q_BYTES);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk) {
          const uint64_t bd = umma_desc_sw128(sV + kk * 2048, L::ATOM, 1024);
          mma_bf16_ts(tmem + TM_O, tmem + TM_P + (gb & 1) * 64 + kk * 8, bd, IDESC_O, (j > 0) || (kk > 0));
        }
        mma_commit(&pv_done[gb & 1]);
        mma_commit(&v_empty[s]);
      }
      __syncwarp();
    };
    int pend_g = -1, pend_j = 0, pend_n = 0;  // the PV lagging one block behind S
    for (int k = 0, w = snake(0, blockIdx.x, gridDim.x); k * (int)gridDim.x < n_items; ++k, w = snake(k, blockIdx.x, gridDim.x), ++n) {
      if (w >= n_items) continue;
      const Item it = item_of(w, nqb, BH, p.H);
      mbar_wait(q_full, n & 1);
      for (int j = 0; j <= it.qb; ++j, ++g) {
        const int s = g & 1;  // S buffer
        const int sk = g % NK;
        mbar_wait(&k_full[sk], (g / NK) & 1);
        if (lane == 0) FA_PROBE(6, g);
        tc_fence_after();
        const uint32_t sK = smem_u32(smem + L::OFF_K + sk * L::Q_BYTES);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint64_t ad = umma_desc_sw128(sQ + (kk >> 2) * L::ATOM + (kk & 3) * 32, 16, 1024);
            const uint64_t bd = umma_desc_sw128(sK + (kk >> 2) * L::ATOM + (kk & 3) * 32, 16, 1024);
            mma_bf16_ss(tmem + s * BN, ad, bd, IDESC_S, kk > 0);
          }
          mma_commit(&s_full[s]);
          mma_commit(&k_empty[sk]);
          if (j == it.qb) mma_commit(q_empty);  // last S of this item issued: Q reusable
        }
        __syncwarp();
        if (pend_g >= 0) issue_pv(pend_g, pend_j, pend_n);
        pend_g = g;
        pend_j = j;
        pend_n = n;
      }
    }
    if (pend_g >= 0) issue_pv(pend_g, pend_j, pend_n);
  } else if (warp >= 4) {
    // ---------------- softmax (thread = query row, warp pair = column halves) ----------------
    // warps 4-7 take keys [0, 64) of each block, warps 8-11 keys [64, 128), for the rows of TMEM
    // lane quadrant warp % 4: two warps per SM sub-partition interleave their ex2 / FMA chains.
    // The halves exchange their row maxima through shared memory each block (same running max m
    // and rescale factor in both), keep separate row sums (added at the end of an item) and each
    // rescales / normalises its own half of O's columns.
    constexpr int HB = BN / 2;   // keys per half
    constexpr int HO = HD / 2;   // O columns per half
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    const int r = q * 32 + lane;  // row within the block
    const int bar_id = 1 + q;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    float* red = reinterpret_cast<float*>(smem + L::OFF_RED);  // [2][2][BM] maxima, then [2][BM] sums
    const float sl2 = p.scale * LOG2E;
    int g = 0;
    for (int k = 0, w = snake(0, blockIdx.x, gridDim.x); k * (int)gridDim.x < n_items; ++k, w = snake(k, blockIdx.x, gridDim.x)) {
      if (w >= n_items) continue;
      const Item it = item_of(w, nqb, BH, p.H);
      float m = -INFINITY, l = 0.f;
      float alpha_pend = 1.f;  // O rescale owed before the next PV (the running max moved)
      for (int j = 0; j <= it.qb; ++j, ++g) {
        const int s = g & 1;
        const bool diag = j == it.qb;
        mbar_wait(&s_full[s], (g >> 1) & 1);
        if (warp == 4 && lane == 0) FA_PROBE(0, g);
        tc_fence_after();
        const uint32_t sb = lane_base + s * BN + half * HB;
        uint32_t va[32], vb[32], pk[32];
        float sum = 0.f, bmax = -INFINITY;
        if (j == 0) {
          // first block of an item: the running max must exist before any exponential
          tmem_ld_32x32b_x32(sb, va);
          tmem_ld_32x32b_x32(sb + 32, vb);
          tmem_ld_wait_dep(va, vb);
          if (diag) {
            mask_chunk(va, half * HB, r);
            mask_chunk(vb, half * HB + 32, r);
          }
          float mraw = fmaxf(chunk_max(va), chunk_max(vb));
          red[(s * 2 + half) * BM + r] = mraw;
          pair_bar(bar_id);
          mraw = fmaxf(mraw, red[(s * 2 + (half ^ 1)) * BM + r]);
          m = mraw * sl2;
        }
        // Later blocks use the lagged max: exponentiate with the running max of the previous blocks
        // (no max pass and no exchange before the exponentials) while the second chunk streams out
        // of TMEM; the block maximum is tracked on the side and agreed with the other half after.
        // Pass 1 (rare) redoes the block after an extreme max growth (P could overflow).  One copy
        // of the exponential code serves every case (instruction-cache footprint).
#pragma unroll 1
        for (int pass = 0; pass < 2; ++pass) {
          sum = 0.f;
          bmax = -INFINITY;
          tmem_ld_32x32b_x32(sb, va);
          tmem_ld_wait_dep(va);
          tmem_ld_32x32b_x32(sb + 32, vb);
          if (diag) mask_chunk(va, half * HB, r);
          exp_chunk(va, sl2, m, pk, sum, bmax);
          tmem_ld_wait_dep(vb);
          if (diag) mask_chunk(vb, half * HB + 32, r);
          exp_chunk(vb, sl2, m, pk + 16, sum, bmax);
          if (warp == 4 && lane == 0) FA_PROBE(1, g);
          if (j == 0 || pass == 1) break;
          red[(s * 2 + half) * BM + r] = bmax;
          pair_bar(bar_id);
          bmax = fmaxf(bmax, red[(s * 2 + (half ^ 1)) * BM + r]);
          const float mx = bmax * sl2;
          const bool extreme = mx > m + EXTREME_LOG2;
          if (warp == 4 && lane == 0) FA_PROBE(2, g);
          if (!__any_sync(0xffffffffu, extreme)) break;
          if (extreme) {  // rescale O (before this block's PV) and l, then redo the block
            const float a = ex2(m - mx);
            m = mx;
            l *= a;
            alpha_pend *= a;
          }
        }
        l += sum;
        // O rescale owed by the previous block (its PV used the old max; this block's P uses the
        // new one): wait for that PV, then scale this half's O columns
        if (__any_sync(0xffffffffu, alpha_pend != 1.f)) {
          mbar_wait(&pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < HO; c += 32) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(lane_base + TM_O + half * HO + c, v);
            tmem_ld_wait_dep(v);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha_pend);
            tmem_st_32x32b_x32(lane_base + TM_O + half * HO + c, v);
          }
          tmem_st_wait();
          alpha_pend = 1.f;
        }
        // P (bf16 pairs along the keys) into TMEM buffer g & 1, last read by the PV of block g-2
        if (g >= 2) {
          mbar_wait(&pv_done[g & 1], ((g - 2) >> 1) & 1);
          tc_fence_after();
        }
        if (warp == 4 && lane == 0) FA_PROBE(4, g);
        tmem_st_32x32b_x32(lane_base + TM_P + (g & 1) * 64 + 32 * half, pk);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (warp == 4 && lane == 0) FA_PROBE(5, g);
        if (lane == 0) mbar_arrive(&p_full[g & 1]);
        // lazy rescaling: the running max only moves when a block's max exceeds it by more than
        // 2^8 (P <= 256 is exact enough in bf16; O / l is invariant to the choice of m); O owes
        // the factor until the next block (or the item epilogue)
        if (j > 0) {
          const float mx = bmax * sl2;
          if (mx > m + RESCALE_LOG2) {
            const float a = ex2(m - mx);
            m = mx;
            l *= a;
            alpha_pend = a;
          }
        }
      }
      // item epilogue: O / l -> bf16 (each half its columns), LSE; then hand O back to the MMA warp
      red[(4 + half) * BM + r] = l;
      pair_bar(bar_id);
      l += red[(4 + (half ^ 1)) * BM + r];
      mbar_wait(&pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1);
      tc_fence_after();
      const float inv = alpha_pend * __frcp_rn(l);
      const int t = it.qb * BM + r;
      if constexpr (L::STG) {
        // hd=128: this warp's 32 rows x 64 columns through its staging box and one TMA store
        uint8_t* box = smem + L::OFF_STG + half * L::ATOM + q * 4096;
        if (lane == 0) bulk_wait_read<0>();  // the previous item's store has read the box
        __syncwarp();
#pragma unroll
        for (int c = 0; c < HO; c += 32) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(lane_base + TM_O + half * HO + c, v);
          tmem_ld_wait();
          box_put32(box, lane, c, v, inv);
        }
        if (half == 0) p.lse[((size_t)it.b * p.H + it.h) * p.T + t] = (m + __log2f(l)) * (1.f / LOG2E);
        tc_fence_before();
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(o_free);
          tma_store_2d(&tmO, box, it.h * HD + half * HO, it.b * p.T + it.qb * BM + q * 32);
          bulk_commit();
        }
      } else {
        __nv_bfloat16* orow = p.out + (size_t)(it.b * p.T + t) * p.ldo + it.h * HD + half * HO;
#pragma unroll
        for (int c = 0; c < HO; c += 32) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(lane_base + TM_O + half * HO + c, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            *reinterpret_cast<uint4*>(orow + c + i) =
                make_uint4(pack_bf16(__uint_as_float(v[i]) * inv, __uint_as_float(v[i + 1]) * inv),
                           pack_bf16(__uint_as_float(v[i + 2]) * inv, __uint_as_float(v[i + 3]) * inv),
                           pack_bf16(__uint_as_float(v[i + 4]) * inv, __uint_as_float(v[i + 5]) * inv),
                           pack_bf16(__uint_as_float(v[i + 6]) * inv, __uint_as_float(v[i + 7]) * inv));
          }
        }
        if (half == 0) p.lse[((size_t)it.b * p.H + it.h) * p.T + t] = (m + __log2f(l)) * (1.f / LOG2E);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(o_free);
      }
    }
    if (L::STG && lane == 0) bulk_wait<0>();
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

// ------------------------------------------------------------------------------------------
// hd = 64, T % 256 == 0: two query tiles per work item (query blocks 2i and 2i+1 of one (b, h))
// with one softmax warpgroup each (warps 4-7 tile 0, warps 8-11 tile 1; thread = a full
// 128-column query row, its own lagged running max, sum and O accumulator -- no exchange between
// warps).  The groups work on different rows, so nothing is merged; each key / value block is
// loaded once for both tiles; one group's TMEM reads, P stores and waits overlap the other's
// exponentials.
//   TMEM: S0 [0,128)  S1 [128,256)  O0 [256,320)  O1 [320,384)  P0 [384,448)  P1 [448,512)
// ------------------------------------------------------------------------------------------
struct Q2Smem {
  static constexpr int ATOM = BM * 128;
  static constexpr int TILE = ATOM;  // 128 x 64 bf16
  static constexpr int NK = 3, NV = 3;
  static constexpr int OFF_Q = 0;                       // [2]
  static constexpr int OFF_K = OFF_Q + 2 * TILE;        // [NK]
  static constexpr int OFF_V = OFF_K + NK * TILE;       // [NV]
  static constexpr int OFF_STG = OFF_V + NV * TILE;     // [tile] O staging, a 32-row box per warp
  static constexpr int OFF_BAR = OFF_STG + 2 * TILE;
  static constexpr int RAW = OFF_BAR + 256;
  static constexpr int BYTES = RAW > 116 * 1024 ? RAW : 116 * 1024;
};

// O row (64 fp32 columns in TMEM) *= a
SPX_DEVICE void q2_scale_o(uint32_t taddr, float a) {
#pragma unroll 1
  for (int c = 0; c < 64; c += 32) {
    uint32_t v[32];
    tmem_ld_32x32b_x32(taddr + c, v);
    tmem_ld_wait_dep(v);
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * a);
    tmem_st_32x32b_x32(taddr + c, v);
  }
  tmem_st_wait();
}

SPX_DEVICE void q2_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

// exponentiate one 128-column row of S (4 chunks of 32, the next loading while one is processed)
// with max m and store P (bf16 pairs) to TMEM at pdst; returns the row sum, tracks the raw max
SPX_DEVICE float q2_exp_row(uint32_t sb, uint32_t pdst, int r, bool diag, float sl2, float m, float& bmax) {
  uint32_t va[32], vb[32], pk[16];
  float sum = 0.f;
  tmem_ld_32x32b_x32(sb, va);
  tmem_ld_wait_dep(va);
#pragma unroll
  for (int c = 0; c < 4; c += 2) {
    tmem_ld_32x32b_x32(sb + 32 * (c + 1), vb);
    if (diag) mask_chunk(va, 32 * c, r);
    exp_chunk(va, sl2, m, pk, sum, bmax);
    q2_st16(pdst + 16 * c, pk);
    tmem_ld_wait_dep(vb);
    if (c + 2 < 4) tmem_ld_32x32b_x32(sb + 32 * (c + 2), va);
    if (diag) mask_chunk(vb, 32 * (c + 1), r);
    exp_chunk(vb, sl2, m, pk, sum, bmax);
    q2_st16(pdst + 16 * (c + 1), pk);
    if (c + 2 < 4) tmem_ld_wait_dep(va);
  }
  return sum;
}

// work item w (heavy first): query-block pair pi = npair-1 - w / (B*H)
SPX_DEVICE Item q2_item_of(int w, int npair, int BH, int H) {
  Item it;
  it.qb = npair - 1 - w / BH;  // pair index
  const int bh = w % BH;
  it.b = bh / H;
  it.h = bh % H;
  return it;
}

__global__ void __launch_bounds__(THREADS, 1)
    attn_fwd_q2_kernel(const __grid_constant__ CUtensorMap tmQKV, const __grid_constant__ CUtensorMap tmO,
                       const FwdParams p) {
  using L = Q2Smem;
  constexpr int HD = 64;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  constexpr int NK = L::NK, NV = L::NV;
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* s_full = bars + 2;   // [tile]
  uint64_t* p_full = bars + 4;   // [tile], 4 arrivals
  uint64_t* pv_done = bars + 6;  // [tile]
  uint64_t* o_free = bars + 8;   // [tile], 4 arrivals
  uint64_t* k_full = bars + 10;            // [NK]
  uint64_t* k_empty = bars + 10 + NK;      // [NK]
  uint64_t* v_full = bars + 10 + 2 * NK;   // [NV]
  uint64_t* v_empty = bars + 10 + 2 * NK + NV;  // [NV]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10 + 2 * NK + 2 * NV);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int npair = p.T / (2 * BM);
  const int BH = p.B * p.H;
  const int n_items = npair * BH;
  const int group = p.H / p.Hkv;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmQKV);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&pv_done[i], 1);
      mbar_init(&o_free[i], 4);
    }
    for (int i = 0; i < NK; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < NV; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    fence_barrier_init();
    fence_proxy_async();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  constexpr uint32_t TM_O = 256, TM_P = 384;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer: the two Q tiles, then K_j ----------------
    int g = 0, n = 0;
    for (int k = 0, w = snake(0, blockIdx.x, gridDim.x); k * (int)gridDim.x < n_items; ++k, w = snake(k, blockIdx.x, gridDim.x), ++n) {
      if (w >= n_items) continue;
      const Item it = q2_item_of(w, npair, BH, p.H);
      const int row0 = it.b * p.T, kvh = it.h / group, nb = 2 * it.qb + 2;
      mbar_wait(q_empty, (n & 1) ^ 1);
      mbar_expect_tx(q_full, 2 * L::TILE);
      tma_load_2d(smem + L::OFF_Q, &tmQKV, q_full, it.h * HD, row0 + 2 * it.qb * BM);
      tma_load_2d(smem + L::OFF_Q + L::TILE, &tmQKV, q_full, it.h * HD, row0 + (2 * it.qb + 1) * BM);
      for (int j = 0; j < nb; ++j, ++g) {
        const int s = g % NK;
        mbar_wait(&k_empty[s], ((g / NK) & 1) ^ 1);
        mbar_expect_tx(&k_full[s], L::TILE);
        tma_load_2d(smem + L::OFF_K + s * L::TILE, &tmQKV, &k_full[s], (p.H + kvh) * HD, row0 + j * BN);
      }
    }
  } else if (warp == 3 && lane == 0) {
    // ---------------- TMA producer: V_j ----------------
    int g = 0;
    for (int k = 0, w = snake(0, blockIdx.x, gridDim.x); k * (int)gridDim.x < n_items; ++k, w = snake(k, blockIdx.x, gridDim.x)) {
      if (w >= n_items) continue;
      const Item it = q2_item_of(w, npair, BH, p.H);
      const int row0 = it.b * p.T, kvh = it.h / group, nb = 2 * it.qb + 2;
      for (int j = 0; j < nb; ++j, ++g) {
        const int s = g % NV;
        mbar_wait(&v_empty[s], ((g / NV) & 1) ^ 1);
        mbar_expect_tx(&v_full[s], L::TILE);
        tma_load_2d(smem + L::OFF_V + s * L::TILE, &tmQKV, &v_full[s], (p.H + p.Hkv + kvh) * HD, row0 + j * BN);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: per key block j, for each tile t: S_t(j), then PV_t(j-1) ----------------
    constexpr uint32_t IDESC_S = umma_idesc_bf16(BM, BN, false, false);
    constexpr uint32_t IDESC_O = umma_idesc_bf16(BM, HD, false, true);
    int g = 0, n = 0;
    int cs0 = 0, cs1 = 0;  // S MMAs issued per tile (p_full phases)
    auto issue_s = [&](int t, uint32_t sK) {
      const uint32_t sQ = smem_u32(smem + L::OFF_Q + t * L::TILE);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          mma_bf16_ss(tmem + t * BN, umma_desc_sw128(sQ + kk * 32, 16, 1024), umma_desc_sw128(sK + kk * 32, 16, 1024),
                      IDESC_S, kk > 0);
        mma_commit(&s_full[t]);
      }
      __syncwarp();
    };
    // PV of tile t for the block whose V sits in ring slot vs; acc = 0 for the tile's first block
    auto issue_pv = [&](int t, int vs, bool acc) {
      tc_fence_after();
      const uint32_t sV = smem_u32(smem + L::OFF_V + vs * L::TILE);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk)
          mma_bf16_ts(tmem + TM_O + t * HD, tmem + TM_P + t * 64 + kk * 8, umma_desc_sw128(sV + kk * 2048, L::ATOM, 1024),
                      IDESC_O, acc || (kk > 0));
        mma_commit(&pv_done[t]);
      }
      __syncwarp();
    };
    for (int k = 0, w = snake(0, blockIdx.x, gridDim.x); k * (int)gridDim.x < n_items; ++k, w = snake(k, blockIdx.x, gridDim.x), ++n) {
      if (w >= n_items) continue;
      const Item it = q2_item_of(w, npair, BH, p.H);
      const int last0 = 2 * it.qb, nb = 2 * it.qb + 2;
      mbar_wait(q_full, n & 1);
      for (int j = 0; j <= nb; ++j, ++g) {
        const int sk = g % NK;
        const int gp = g - 1;  // global index of block j-1 (V ring slot)
        if (j < nb) {
          mbar_wait(&k_full[sk], (g / NK) & 1);
          tc_fence_after();
        }
        const uint32_t sK = smem_u32(smem + L::OFF_K + sk * L::TILE);
        // tile 0
        if (j > 0 && j - 1 <= last0) {
          mbar_wait(&p_full[0], (cs0 - 1) & 1);  // softmax of S0(j-1) done: S0 free, P0(j-1) ready
          if (j - 1 == 0) mbar_wait(&o_free[0], (n & 1) ^ 1);
          mbar_wait(&v_full[gp % NV], (gp / NV) & 1);
        }
        if (j <= last0) {
          issue_s(0, sK);
          ++cs0;
        }
        if (j > 0 && j - 1 <= last0) issue_pv(0, gp % NV, j - 1 > 0);
        // tile 1
        if (j > 0) {
          mbar_wait(&p_full[1], (cs1 - 1) & 1);
          if (j - 1 == 0) mbar_wait(&o_free[1], (n & 1) ^ 1);
          mbar_wait(&v_full[gp % NV], (gp / NV) & 1);
        }
        if (j < nb) {
          issue_s(1, sK);
          ++cs1;
          if (elect_one()) {
            mma_commit(&k_empty[sk]);
            if (j == nb - 1) mma_commit(q_empty);
          }
          __syncwarp();
        }
        if (j > 0) {
          issue_pv(1, gp % NV, j - 1 > 0);
          if (elect_one()) mma_commit(&v_empty[gp % NV]);
          __syncwarp();
        }
      }
      --g;  // the j = nb pass only drained the last PVs
    }
  } else if (warp >= 4) {
    // ---------------- softmax: tile t = (warp - 4) / 4, thread = query row ----------------
    const int t = (warp - 4) >> 2;
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    const float sl2 = p.scale * LOG2E;
    int cx = 0;  // this tile's blocks so far (s_full / pv_done phases)
    for (int k = 0, w = snake(0, blockIdx.x, gridDim.x); k * (int)gridDim.x < n_items; ++k, w = snake(k, blockIdx.x, gridDim.x)) {
      if (w >= n_items) continue;
      const Item it = q2_item_of(w, npair, BH, p.H);
      const int lastb = 2 * it.qb + t;  // this tile's diagonal block
      float m = -INFINITY, l = 0.f, alpha_pend = 1.f;
      for (int j = 0; j <= lastb; ++j, ++cx) {
        const bool diag = j == lastb;
        mbar_wait(&s_full[t], cx & 1);
        const uint32_t sb = lane_base + t * BN, pdst = lane_base + TM_P + t * 64;
        // the tile's previous PV has read P_t and finished O_t
        if (cx > 0) mbar_wait(&pv_done[t], (cx - 1) & 1);
        tc_fence_after();
        if (j > 0 && __any_sync(0xffffffffu, alpha_pend != 1.f)) {
          q2_scale_o(lane_base + TM_O + t * HD, alpha_pend);
          alpha_pend = 1.f;
        }
        if (j == 0) {
          float mraw = -INFINITY;
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(sb + 32 * c, v);
            tmem_ld_wait_dep(v);
            if (diag) mask_chunk(v, 32 * c, r);
            mraw = fmaxf(mraw, chunk_max(v));
          }
          m = mraw * sl2;
        }
        float bmax, sum;
#pragma unroll 1
        for (int pass = 0; pass < 2; ++pass) {
          bmax = -INFINITY;
          sum = q2_exp_row(sb, pdst, r, diag, sl2, m, bmax);
          if (j == 0 || pass == 1) break;
          const float mx = bmax * sl2;
          const bool extreme = mx > m + EXTREME_LOG2;
          if (!__any_sync(0xffffffffu, extreme)) break;
          const float a = extreme ? ex2(m - mx) : 1.f;
          if (extreme) {
            m = mx;
            l *= a;
          }
          tmem_st_wait();
          q2_scale_o(lane_base + TM_O + t * HD, a);
        }
        l += sum;
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[t]);
        if (j > 0) {
          const float mx = bmax * sl2;
          if (mx > m + RESCALE_LOG2) {
            const float a = ex2(m - mx);
            m = mx;
            l *= a;
            alpha_pend = a;
          }
        }
      }
      // item epilogue: this tile's O / l -> bf16, LSE; then O_t back to the MMA warp
      mbar_wait(&pv_done[t], (cx - 1) & 1);
      tc_fence_after();
      const float inv = alpha_pend * __frcp_rn(l);
      const int tq = (2 * it.qb + t) * BM + r;
      // this warp's 32 rows through its staging box and one TMA store
      uint8_t* box = smem + L::OFF_STG + t * L::TILE + q * 4096;
      if (lane == 0) bulk_wait_read<0>();  // the previous item's store has read the box
      __syncwarp();
#pragma unroll 1
      for (int c = 0; c < HD; c += 32) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(lane_base + TM_O + t * HD + c, v);
        tmem_ld_wait_dep(v);
        box_put32(box, lane, c, v, inv);
      }
      p.lse[((size_t)it.b * p.H + it.h) * p.T + tq] = (m + __log2f(l)) * (1.f / LOG2E);
      tc_fence_before();
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&o_free[t]);
        tma_store_2d(&tmO, box, it.h * HD, it.b * p.T + (2 * it.qb + t) * BM + q * 32);
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

// hd=64 with T % 256 == 0: the two-query-tile kernel when it has at least one work item per SM
// (its items are twice as coarse, so fewer of them balance worse: with B=4, T=1024, H=16 it is
// 3 % faster, at T=4096 9 %, but with 128 items 50 % slower).  SPX_ATTN_Q2=0 / 1 forces it off / on.
static bool fwd_q2(int items) {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("SPX_ATTN_Q2");
    v = e ? (e[0] == '1' ? 1 : 0) : -1;
  }
  return v == 1 || (v == -1 && items >= num_sms());
}

template <int HD>
int launch_fwd(const void* qkv, const FwdParams& p, long long ld_qkv, cudaStream_t s) {
  auto encode = get_tensor_map_encoder();
  if (!encode) return set_error(SPX_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)ld_qkv, (cuuint64_t)p.B * p.T};
  cuuint64_t strides[1] = {(cuuint64_t)ld_qkv * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(qkv), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(SPX_ERR_CUDA, "attn_fwd_tc: tensor map encode failed");
  CUtensorMap omap;  // O [B*T][ldo], 64 x 32 boxes (one per softmax warp)
  cuuint64_t odims[2] = {(cuuint64_t)p.ldo, (cuuint64_t)p.B * p.T};
  cuuint64_t ostrides[1] = {(cuuint64_t)p.ldo * 2};
  cuuint32_t obox[2] = {64, 32};
  r = encode(&omap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p.out, odims, ostrides, obox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(SPX_ERR_CUDA, "attn_fwd_tc: output tensor map encode failed");
  if (HD == 64 && p.T % (2 * BM) == 0 && fwd_q2((p.T / (2 * BM)) * p.B * p.H)) {
    static bool setq2 = false;
    if (!setq2) {
      cudaError_t e = cudaFuncSetAttribute(attn_fwd_q2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, Q2Smem::BYTES);
      if (e != cudaSuccess) return set_cuda_error(e, "attn_fwd_q2 attr");
      setq2 = true;
    }
    const int items2 = (p.T / (2 * BM)) * p.B * p.H;
    const int grid2 = items2 < num_sms() ? items2 : num_sms();
    spx_launch_check(launch_k(attn_fwd_q2_kernel, dim3(grid2), dim3(THREADS), Q2Smem::BYTES, s, map, omap, p));
    return check_launch("attn_fwd_q2_kernel");
  }
  auto k = attn_fwd_tc_kernel<HD>;
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdSmem<HD>::BYTES);
    if (e != cudaSuccess) return set_cuda_error(e, "attn_fwd_tc attr");
    set = true;
  }
  const int items = (p.T / BM) * p.B * p.H;
  const int grid = items < num_sms() ? items : num_sms();
  spx_launch_check(launch_k(k, dim3(grid), dim3(THREADS), FwdSmem<HD>::BYTES, s, map, omap, p));
  return check_launch("attn_fwd_tc_kernel");
}

}  // namespace fa

// used by spx_attn_fwd (attention.cu) for head_dim 64/128 and T % 128 == 0
int attn_fwd_tcgen05(const void* qkv, void* o, float* lse, int64_t B, int64_t T, int64_t H, int64_t Hkv, int64_t hd,
                     int64_t ld_qkv, int64_t ld_o, float scale, cudaStream_t s) {
  fa::FwdParams p{reinterpret_cast<__nv_bfloat16*>(o), lse, (long long)ld_o, (int)B, (int)T, (int)H, (int)Hkv, scale};
  if (hd == 64) return fa::launch_fwd<64>(qkv, p, ld_qkv, s);
  return fa::launch_fwd<128>(qkv, p, ld_qkv, s);
}

}  // namespace spx
