// Causal flash attention (forward + deterministic backward) for LLaMA decoder stages.
//
// Q/K/V are read in place from the fused QKV projection output [B*T, ld] (q heads at
// column h*hd, k heads at (H + kv)*hd, v heads at (H + Hkv + kv)*hd, GQA when Hkv < H) and the
// gradients are written into a buffer of the same layout, so the QKV dgrad / wgrad GEMMs
// consume them without any transpose.  Softmax statistics are kept in the exp2 domain; the
// saved log-sum-exp is natural-log.
//
// Round-1 implementation: warp-level mma.sync m16n8k16 (bf16 in, fp32 accumulate) with
// ldmatrix-fed operands and cp.async double-buffered K/V tiles.  The backward splits into a
// dK/dV kernel (one CTA per 64-key block, loops over query blocks and over the GQA group) and
// a dQ kernel (one CTA per 64-query block), so no atomics are needed and results are
// bit-reproducible run to run.
#include <cmath>
#include <cstdlib>

#include "spx_common.cuh"
#include "spx_internal.h"

namespace spx {
namespace attn {

constexpr int WARPS = 4;
constexpr int THREADS = WARPS * 32;
constexpr int BQ = 64;   // query rows per CTA (16 per warp)
constexpr int BK = 64;   // keys per CTA tile
constexpr float LOG2E = 1.4426950408889634f;

SPX_DEVICE void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

SPX_DEVICE void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

SPX_DEVICE void ldsm_x4_t(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

SPX_DEVICE void ldsm_x2(uint32_t& r0, uint32_t& r1, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}

SPX_DEVICE void ldsm_x2_t(uint32_t& r0, uint32_t& r1, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}

SPX_DEVICE void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
SPX_DEVICE void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
SPX_DEVICE void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// smem tile of ROWS x HD bf16 with a 16-byte row pad (ldmatrix bank-conflict free)
template <int HD>
struct Tile {
  static constexpr int LD = HD + 8;
};

// Load ROWS rows of HD bf16 (global row stride ld elements) into a padded smem tile.
template <int ROWS, int HD>
SPX_DEVICE void load_tile_async(__nv_bfloat16* s, const __nv_bfloat16* g, long long ld) {
  constexpr int CH = HD / 8;  // 16-byte chunks per row
  for (int i = threadIdx.x; i < ROWS * CH; i += THREADS) {
    const int r = i / CH, c = i % CH;
    cp_async16(s + r * Tile<HD>::LD + c * 8, g + (long long)r * ld + c * 8);
  }
}

// A fragments (16 rows x HD) of a row-major smem tile starting at row r0.
template <int HD>
SPX_DEVICE void load_a_frags(uint32_t (&a)[HD / 16][4], const __nv_bfloat16* s, int r0) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int kc = 0; kc < HD / 16; ++kc) {
    const __nv_bfloat16* p = s + (r0 + (lane & 15)) * Tile<HD>::LD + kc * 16 + (lane >> 4) * 8;
    ldsm_x4(a[kc], smem_u32(p));
  }
}

// B fragments for an n-tile pair (16 n-rows) x 16 k taken from an smem tile stored [n][k]
// (non-transposed load): gives b0,b1 of n-tile n0 and of n-tile n0+8.
template <int HD>
SPX_DEVICE void load_b_nk(uint32_t (&b)[4], const __nv_bfloat16* s, int n0, int k0) {
  const int lane = threadIdx.x & 31;
  const __nv_bfloat16* p = s + (n0 + (lane & 7) + ((lane >> 4) << 3)) * Tile<HD>::LD + k0 + ((lane >> 3) & 1) * 8;
  ldsm_x4(b, smem_u32(p));
}

// B fragments for 16 k x (two n-tiles) from an smem tile stored [k][n] (transposed load).
template <int HD>
SPX_DEVICE void load_b_kn(uint32_t (&b)[4], const __nv_bfloat16* s, int k0, int n0) {
  const int lane = threadIdx.x & 31;
  const __nv_bfloat16* p = s + (k0 + (lane & 7) + (((lane >> 3) & 1) << 3)) * Tile<HD>::LD + n0 + (lane >> 4) * 8;
  ldsm_x4_t(b, smem_u32(p));
}

// Inverse rotate-half RoPE on a thread's accumulator fragments: the thread holds columns
// 8i + 2t4 + {0,1} of rows r and r+8; column j and j + HD/2 sit in n-tiles i and i + HD/16.
template <int HD>
SPX_DEVICE void unrope_frags(float (&acc)[HD / 8][4], const float* cs, int T, int pos0, int pos1, int t4) {
  // cs: [hd/2][T][2] position-minor (cos, sin)
  const float2* c = reinterpret_cast<const float2*>(cs);
#pragma unroll
  for (int i = 0; i < HD / 16; ++i) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int j = 8 * i + 2 * t4 + (e & 1);
      const float2 w = c[(size_t)j * T + ((e >> 1) ? pos1 : pos0)];
      const float a = acc[i][e], b = acc[i + HD / 16][e];
      acc[i][e] = a * w.x + b * w.y;
      acc[i + HD / 16][e] = b * w.x - a * w.y;
    }
  }
}

struct Params {
  const __nv_bfloat16* qkv;
  __nv_bfloat16* out;   // fwd: O [B*T, H*hd]; bwd: dQKV [B*T, ld]
  const __nv_bfloat16* o;
  const __nv_bfloat16* dout;
  float* lse;           // [B, H, T]
  float* delta;         // [B, H, T]
  const float* rope_cs; // bwd: [hd/2][T][2] cos/sin -> dq, dk written un-rotated (inverse RoPE)
  long long ld;         // qkv / dqkv row stride
  long long ldo;        // O / dO row stride
  int B, T, H, Hkv;
  float scale;
  int delta_ready;      // bwd: the workspace already holds D and lse*log2e (spx_gemm_bf16_attn_delta)
  int ws_ex;            // bwd: the workspace is sized by spx_attn_bwd_ws_floats_ex (GQA split allowed)
};

// ----------------------------------------------------------------------------------------
// forward
// ----------------------------------------------------------------------------------------
template <int HD>
__global__ void __launch_bounds__(THREADS) attn_fwd_kernel(const Params p) {
  pdl_wait();
  extern __shared__ __align__(16) uint8_t smem_raw[];
  constexpr int LD = Tile<HD>::LD;
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __nv_bfloat16* sK = sQ + BQ * LD;       // [2][BK][LD]
  __nv_bfloat16* sV = sK + 2 * BK * LD;   // [2][BK][LD]

  const int qb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int kvh = h / (p.H / p.Hkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const long long row0 = (long long)b * p.T;
  const __nv_bfloat16* Qg = p.qkv + (row0 + qb * BQ) * p.ld + h * HD;
  const __nv_bfloat16* Kg = p.qkv + row0 * p.ld + (p.H + kvh) * HD;
  const __nv_bfloat16* Vg = p.qkv + row0 * p.ld + (p.H + p.Hkv + kvh) * HD;

  load_tile_async<BQ, HD>(sQ, Qg, p.ld);
  load_tile_async<BK, HD>(sK, Kg, p.ld);
  load_tile_async<BK, HD>(sV, Vg, p.ld);
  cp_async_commit();

  float acc[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const float sl2 = p.scale * LOG2E;
  uint32_t qf[HD / 16][4];
  const int nkb = qb + 1;  // causal: key blocks 0..qb (BQ == BK)
  for (int kb = 0; kb < nkb; ++kb) {
    const int buf = kb & 1;
    if (kb + 1 < nkb) {
      load_tile_async<BK, HD>(sK + (buf ^ 1) * BK * LD, Kg + (long long)(kb + 1) * BK * p.ld, p.ld);
      load_tile_async<BK, HD>(sV + (buf ^ 1) * BK * LD, Vg + (long long)(kb + 1) * BK * p.ld, p.ld);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (kb == 0) load_a_frags<HD>(qf, sQ, warp * 16);
    const __nv_bfloat16* k_s = sK + buf * BK * LD;
    const __nv_bfloat16* v_s = sV + buf * BK * LD;
    float s[BK / 8][4];
#pragma unroll
    for (int j = 0; j < BK / 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int kc = 0; kc < HD / 16; ++kc) {
#pragma unroll
      for (int j = 0; j < BK / 16; ++j) {
        uint32_t bb[4];
        load_b_nk<HD>(bb, k_s, j * 16, kc * 16);
        mma16816(s[2 * j], qf[kc], bb[0], bb[1]);
        mma16816(s[2 * j + 1], qf[kc], bb[2], bb[3]);
      }
    }
    // scale (log2 domain) + causal mask on the diagonal block
    const int qrow0 = qb * BQ + warp * 16 + g;
    float mx0 = m0, mx1 = m1;
#pragma unroll
    for (int j = 0; j < BK / 8; ++j) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = kb * BK + j * 8 + 2 * t4 + (e & 1);
        const int q = qrow0 + ((e >> 1) << 3);
        float v = s[j][e] * sl2;
        if (kb == qb && key > q) v = -INFINITY;
        s[j][e] = v;
      }
      mx0 = fmaxf(mx0, fmaxf(s[j][0], s[j][1]));
      mx1 = fmaxf(mx1, fmaxf(s[j][2], s[j][3]));
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float c0 = exp2f(m0 - mx0), c1 = exp2f(m1 - mx1);
    m0 = mx0;
    m1 = mx1;
    float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
    for (int j = 0; j < BK / 8; ++j) {
      s[j][0] = exp2f(s[j][0] - m0);
      s[j][1] = exp2f(s[j][1] - m0);
      s[j][2] = exp2f(s[j][2] - m1);
      s[j][3] = exp2f(s[j][3] - m1);
      rs0 += s[j][0] + s[j][1];
      rs1 += s[j][2] + s[j][3];
    }
    l0 = l0 * c0 + rs0;
    l1 = l1 * c1 + rs1;
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      acc[i][0] *= c0; acc[i][1] *= c0; acc[i][2] *= c1; acc[i][3] *= c1;
    }
    // O += P V
#pragma unroll
    for (int kc = 0; kc < BK / 16; ++kc) {
      uint32_t a[4];
      a[0] = pack_bf16(s[2 * kc][0], s[2 * kc][1]);
      a[1] = pack_bf16(s[2 * kc][2], s[2 * kc][3]);
      a[2] = pack_bf16(s[2 * kc + 1][0], s[2 * kc + 1][1]);
      a[3] = pack_bf16(s[2 * kc + 1][2], s[2 * kc + 1][3]);
#pragma unroll
      for (int nt = 0; nt < HD / 16; ++nt) {
        uint32_t bb[4];
        load_b_kn<HD>(bb, v_s, kc * 16, nt * 16);
        mma16816(acc[2 * nt], a, bb[0], bb[1]);
        mma16816(acc[2 * nt + 1], a, bb[2], bb[3]);
      }
    }
    __syncthreads();
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float inv0 = 1.f / l0, inv1 = 1.f / l1;
  const int qr = qb * BQ + warp * 16 + g;
  __nv_bfloat16* O0 = p.out + (row0 + qr) * p.ldo + h * HD;
  __nv_bfloat16* O1 = O0 + 8 * p.ldo;
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) {
    *reinterpret_cast<uint32_t*>(O0 + i * 8 + 2 * t4) = pack_bf16(acc[i][0] * inv0, acc[i][1] * inv0);
    *reinterpret_cast<uint32_t*>(O1 + i * 8 + 2 * t4) = pack_bf16(acc[i][2] * inv1, acc[i][3] * inv1);
  }
  if (t4 == 0) {
    float* L = p.lse + ((long long)b * p.H + h) * p.T;
    L[qr] = (m0 + log2f(l0)) / LOG2E;
    L[qr + 8] = (m1 + log2f(l1)) / LOG2E;
  }
}

// ----------------------------------------------------------------------------------------
// backward: delta = rowsum(dO * O)
// ----------------------------------------------------------------------------------------
template <int HD>
__global__ void attn_bwd_delta_kernel(const Params p) {
  pdl_wait();
  // 8 lanes per (row, head); lane j sums the 16-byte vectors j, j+8, ... of that head's row.
  // Groups are numbered in the [B, H, T] order of the outputs (position fastest), so the D and
  // lse*log2e stores of a warp's four groups are contiguous; each thread takes DG groups a grid
  // apart with all their loads in flight (the kernel is load-latency bound at one group each).
  constexpr int DG = 4;
  const long long rows = (long long)p.B * p.T;
  const long long total = rows * p.H;
  const long long stride = ((long long)gridDim.x * blockDim.x) >> 3;
  const long long g0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const int j = threadIdx.x & 7;
  constexpr int NV = (HD / 8 + 7) / 8;  // 16-byte vectors per lane (hd 48: lanes 6, 7 idle)
  uint4 a[DG][NV], c[DG][NV];
#pragma unroll
  for (int k = 0; k < DG; ++k) {
    const long long gg = g0 + k * stride < total ? g0 + k * stride : 0;
    const int t_ = (int)(gg % p.T);
    const long long bh = gg / p.T;
    const int h = (int)(bh % p.H);
    const long long r = (bh / p.H) * p.T + t_;
    const __nv_bfloat16* o = p.o + r * p.ldo + h * HD;
    const __nv_bfloat16* d = p.dout + r * p.ldo + h * HD;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const bool in = j + 8 * v < HD / 8;
      a[k][v] = in ? *reinterpret_cast<const uint4*>(o + (j + 8 * v) * 8) : make_uint4(0, 0, 0, 0);
      c[k][v] = in ? *reinterpret_cast<const uint4*>(d + (j + 8 * v) * 8) : make_uint4(0, 0, 0, 0);
    }
  }
#pragma unroll
  for (int k = 0; k < DG; ++k) {
    float s = 0.f;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a[k][v]);
      const __nv_bfloat162* c2 = reinterpret_cast<const __nv_bfloat162*>(&c[k][v]);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 fa = __bfloat1622float2(a2[i]), fc = __bfloat1622float2(c2[i]);
        s += fa.x * fc.x + fa.y * fc.y;
      }
    }
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    const long long idx = g0 + k * stride;  // ((b * H + h) * T + t)
    if (j == 0 && idx < total) {
      p.delta[idx] = s;
      // second half of the workspace: lse in the exp2 domain for the tcgen05 dK/dV kernel
      p.delta[total + idx] = p.lse[idx] * 1.4426950408889634f;
    }
  }
}

// ----------------------------------------------------------------------------------------
// backward: dK, dV (one CTA per 64-key block of one kv head; warps own 16 keys each)
// ----------------------------------------------------------------------------------------
template <int HD>
__global__ void __launch_bounds__(THREADS) attn_bwd_dkdv_kernel(const Params p) {
  pdl_wait();
  constexpr int LD = Tile<HD>::LD;
  constexpr int BQI = (HD > 64) ? 32 : 64;  // query rows per inner step
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __nv_bfloat16* sK = reinterpret_cast<__nv_bfloat16*>(smem_raw);  // [BK][LD]
  __nv_bfloat16* sV = sK + BK * LD;                                // [BK][LD]
  __nv_bfloat16* sQ = sV + BK * LD;                                // [BQI][LD]
  __nv_bfloat16* sdO = sQ + BQI * LD;                              // [BQI][LD]
  float* sL = reinterpret_cast<float*>(sdO + BQI * LD);            // [BQI]
  float* sD = sL + BQI;                                            // [BQI]

  const int kb = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
  const int group = p.H / p.Hkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const long long row0 = (long long)b * p.T;
  load_tile_async<BK, HD>(sK, p.qkv + (row0 + kb * BK) * p.ld + (p.H + kvh) * HD, p.ld);
  load_tile_async<BK, HD>(sV, p.qkv + (row0 + kb * BK) * p.ld + (p.H + p.Hkv + kvh) * HD, p.ld);
  cp_async_commit();

  float dk[HD / 8][4], dv[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;
  const float sl2 = p.scale * LOG2E;
  const int key_w = kb * BK + warp * 16;  // first key of this warp

  for (int hq = 0; hq < group; ++hq) {
    const int h = kvh * group + hq;
    const float* Lh = p.lse + ((long long)b * p.H + h) * p.T;
    const float* Dh = p.delta + ((long long)b * p.H + h) * p.T;
    for (int q0 = kb * BK; q0 < p.T; q0 += BQI) {
      __syncthreads();  // previous step's smem reads done
      load_tile_async<BQI, HD>(sQ, p.qkv + (row0 + q0) * p.ld + h * HD, p.ld);
      load_tile_async<BQI, HD>(sdO, p.dout + (row0 + q0) * p.ldo + h * HD, p.ldo);
      cp_async_commit();
      for (int i = threadIdx.x; i < BQI; i += THREADS) {
        sL[i] = Lh[q0 + i] * LOG2E;
        sD[i] = Dh[q0 + i];
      }
      cp_async_wait<0>();
      __syncthreads();
      if (q0 + BQI <= key_w) continue;  // whole step masked for this warp (warp-uniform)
      uint32_t kf[HD / 16][4], vf[HD / 16][4];
      load_a_frags<HD>(kf, sK, warp * 16);
      load_a_frags<HD>(vf, sV, warp * 16);
      // S^T (16 keys x BQI queries) and dP^T
      float s[BQI / 8][4], dp[BQI / 8][4];
#pragma unroll
      for (int j = 0; j < BQI / 8; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) s[j][e] = dp[j][e] = 0.f;
#pragma unroll
      for (int kc = 0; kc < HD / 16; ++kc) {
#pragma unroll
        for (int j = 0; j < BQI / 16; ++j) {
          uint32_t bb[4];
          load_b_nk<HD>(bb, sQ, j * 16, kc * 16);
          mma16816(s[2 * j], kf[kc], bb[0], bb[1]);
          mma16816(s[2 * j + 1], kf[kc], bb[2], bb[3]);
          load_b_nk<HD>(bb, sdO, j * 16, kc * 16);
          mma16816(dp[2 * j], vf[kc], bb[0], bb[1]);
          mma16816(dp[2 * j + 1], vf[kc], bb[2], bb[3]);
        }
      }
      // P^T = exp2(S*scale*log2e - lse*log2e), dS^T = P^T (dP^T - D)
#pragma unroll
      for (int j = 0; j < BQI / 8; ++j) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int qi = j * 8 + 2 * t4 + (e & 1);
          const int key = key_w + g + ((e >> 1) << 3);
          float pv = exp2f(s[j][e] * sl2 - sL[qi]);
          if (q0 + qi < key) pv = 0.f;
          s[j][e] = pv;
          dp[j][e] = pv * (dp[j][e] - sD[qi]);
        }
      }
      // dV += P^T dO ; dK += dS^T Q
#pragma unroll
      for (int kc = 0; kc < BQI / 16; ++kc) {
        uint32_t ap[4], ad[4];
        ap[0] = pack_bf16(s[2 * kc][0], s[2 * kc][1]);
        ap[1] = pack_bf16(s[2 * kc][2], s[2 * kc][3]);
        ap[2] = pack_bf16(s[2 * kc + 1][0], s[2 * kc + 1][1]);
        ap[3] = pack_bf16(s[2 * kc + 1][2], s[2 * kc + 1][3]);
        ad[0] = pack_bf16(dp[2 * kc][0], dp[2 * kc][1]);
        ad[1] = pack_bf16(dp[2 * kc][2], dp[2 * kc][3]);
        ad[2] = pack_bf16(dp[2 * kc + 1][0], dp[2 * kc + 1][1]);
        ad[3] = pack_bf16(dp[2 * kc + 1][2], dp[2 * kc + 1][3]);
#pragma unroll
        for (int nt = 0; nt < HD / 16; ++nt) {
          uint32_t bb[4];
          load_b_kn<HD>(bb, sdO, kc * 16, nt * 16);
          mma16816(dv[2 * nt], ap, bb[0], bb[1]);
          mma16816(dv[2 * nt + 1], ap, bb[2], bb[3]);
          load_b_kn<HD>(bb, sQ, kc * 16, nt * 16);
          mma16816(dk[2 * nt], ad, bb[0], bb[1]);
          mma16816(dk[2 * nt + 1], ad, bb[2], bb[3]);
        }
      }
    }
  }
  const int kr = kb * BK + warp * 16 + g;
  if (p.rope_cs) unrope_frags<HD>(dk, p.rope_cs, p.T, kr, kr + 8, t4);
  __nv_bfloat16* dK0 = p.out + (row0 + kr) * p.ld + (p.H + kvh) * HD;
  __nv_bfloat16* dV0 = p.out + (row0 + kr) * p.ld + (p.H + p.Hkv + kvh) * HD;
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) {
    const int c = i * 8 + 2 * t4;
    *reinterpret_cast<uint32_t*>(dK0 + c) = pack_bf16(dk[i][0] * p.scale, dk[i][1] * p.scale);
    *reinterpret_cast<uint32_t*>(dK0 + 8 * p.ld + c) = pack_bf16(dk[i][2] * p.scale, dk[i][3] * p.scale);
    *reinterpret_cast<uint32_t*>(dV0 + c) = pack_bf16(dv[i][0], dv[i][1]);
    *reinterpret_cast<uint32_t*>(dV0 + 8 * p.ld + c) = pack_bf16(dv[i][2], dv[i][3]);
  }
}

// ----------------------------------------------------------------------------------------
// backward: dQ (one CTA per 64-query block; warps own 16 queries)
// ----------------------------------------------------------------------------------------
template <int HD>
__global__ void __launch_bounds__(THREADS) attn_bwd_dq_kernel(const Params p) {
  pdl_wait();
  constexpr int LD = Tile<HD>::LD;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem_raw);  // [BQ][LD]
  __nv_bfloat16* sdO = sQ + BQ * LD;                               // [BQ][LD]
  __nv_bfloat16* sK = sdO + BQ * LD;                               // [2][BK][LD]
  __nv_bfloat16* sV = sK + 2 * BK * LD;                            // [2][BK][LD]

  const int qb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int kvh = h / (p.H / p.Hkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const long long row0 = (long long)b * p.T;
  const __nv_bfloat16* Kg = p.qkv + row0 * p.ld + (p.H + kvh) * HD;
  const __nv_bfloat16* Vg = p.qkv + row0 * p.ld + (p.H + p.Hkv + kvh) * HD;
  load_tile_async<BQ, HD>(sQ, p.qkv + (row0 + qb * BQ) * p.ld + h * HD, p.ld);
  load_tile_async<BQ, HD>(sdO, p.dout + (row0 + qb * BQ) * p.ldo + h * HD, p.ldo);
  load_tile_async<BK, HD>(sK, Kg, p.ld);
  load_tile_async<BK, HD>(sV, Vg, p.ld);
  cp_async_commit();

  const int qr = qb * BQ + warp * 16 + g;
  const float* Lh = p.lse + ((long long)b * p.H + h) * p.T;
  const float* Dh = p.delta + ((long long)b * p.H + h) * p.T;
  const float sl2 = p.scale * LOG2E;
  const float lse0 = Lh[qr] * LOG2E, lse1 = Lh[qr + 8] * LOG2E;
  const float d0 = Dh[qr], d1 = Dh[qr + 8];

  float dq[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;
  uint32_t qf[HD / 16][4], of[HD / 16][4];
  const int nkb = qb + 1;
  for (int kb = 0; kb < nkb; ++kb) {
    const int buf = kb & 1;
    if (kb + 1 < nkb) {
      load_tile_async<BK, HD>(sK + (buf ^ 1) * BK * LD, Kg + (long long)(kb + 1) * BK * p.ld, p.ld);
      load_tile_async<BK, HD>(sV + (buf ^ 1) * BK * LD, Vg + (long long)(kb + 1) * BK * p.ld, p.ld);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (kb == 0) {
      load_a_frags<HD>(qf, sQ, warp * 16);
      load_a_frags<HD>(of, sdO, warp * 16);
    }
    const __nv_bfloat16* k_s = sK + buf * BK * LD;
    const __nv_bfloat16* v_s = sV + buf * BK * LD;
    float s[BK / 8][4], dp[BK / 8][4];
#pragma unroll
    for (int j = 0; j < BK / 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[j][e] = dp[j][e] = 0.f;
#pragma unroll
    for (int kc = 0; kc < HD / 16; ++kc) {
#pragma unroll
      for (int j = 0; j < BK / 16; ++j) {
        uint32_t bb[4];
        load_b_nk<HD>(bb, k_s, j * 16, kc * 16);
        mma16816(s[2 * j], qf[kc], bb[0], bb[1]);
        mma16816(s[2 * j + 1], qf[kc], bb[2], bb[3]);
        load_b_nk<HD>(bb, v_s, j * 16, kc * 16);
        mma16816(dp[2 * j], of[kc], bb[0], bb[1]);
        mma16816(dp[2 * j + 1], of[kc], bb[2], bb[3]);
      }
    }
#pragma unroll
    for (int j = 0; j < BK / 8; ++j) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = kb * BK + j * 8 + 2 * t4 + (e & 1);
        const bool hi = e >> 1;
        float pv = exp2f(s[j][e] * sl2 - (hi ? lse1 : lse0));
        if (kb == qb && key > qr + (hi ? 8 : 0)) pv = 0.f;
        dp[j][e] = pv * (dp[j][e] - (hi ? d1 : d0));
      }
    }
#pragma unroll
    for (int kc = 0; kc < BK / 16; ++kc) {
      uint32_t a[4];
      a[0] = pack_bf16(dp[2 * kc][0], dp[2 * kc][1]);
      a[1] = pack_bf16(dp[2 * kc][2], dp[2 * kc][3]);
      a[2] = pack_bf16(dp[2 * kc + 1][0], dp[2 * kc + 1][1]);
      a[3] = pack_bf16(dp[2 * kc + 1][2], dp[2 * kc + 1][3]);
#pragma unroll
      for (int nt = 0; nt < HD / 16; ++nt) {
        uint32_t bb[4];
        load_b_kn<HD>(bb, k_s, kc * 16, nt * 16);
        mma16816(dq[2 * nt], a, bb[0], bb[1]);
        mma16816(dq[2 * nt + 1], a, bb[2], bb[3]);
      }
    }
    __syncthreads();
  }
  if (p.rope_cs) unrope_frags<HD>(dq, p.rope_cs, p.T, qr, qr + 8, t4);
  __nv_bfloat16* dQ0 = p.out + (row0 + qr) * p.ld + h * HD;
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) {
    const int c = i * 8 + 2 * t4;
    *reinterpret_cast<uint32_t*>(dQ0 + c) = pack_bf16(dq[i][0] * p.scale, dq[i][1] * p.scale);
    *reinterpret_cast<uint32_t*>(dQ0 + 8 * p.ld + c) = pack_bf16(dq[i][2] * p.scale, dq[i][3] * p.scale);
  }
}

template <int HD>
static int run_fwd(const Params& p, cudaStream_t s) {
  constexpr int LD = Tile<HD>::LD;
  const int smem = (BQ + 4 * BK) * LD * 2;
  auto k = attn_fwd_kernel<HD>;
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_cuda_error(e, "attn_fwd attr");
    set = true;
  }
  spx_launch_check(launch_k(k, dim3(dim3(p.T / BQ, p.H, p.B)), dim3(THREADS), smem, s, p));
  return check_launch("attn_fwd_kernel");
}

template <int HD>
static int run_bwd(const Params& p, cudaStream_t s) {
  constexpr int LD = Tile<HD>::LD;
  constexpr int BQI = (HD > 64) ? 32 : 64;
  if (!p.delta_ready) {
    const long long groups = (long long)p.B * p.T * p.H;  // 8 threads each, 4 groups per thread
    const int threads = 256;
    const long long per_block = threads / 8 * 4;
    spx_launch_check(launch_k(attn_bwd_delta_kernel<HD>, dim3((unsigned)((groups + per_block - 1) / per_block)), dim3(threads), 0, s, p));
    int rc = check_launch("attn_bwd_delta_kernel");
    if (rc) return rc;
  }
  if ((HD == 64 || HD == 128) && p.T % 128 == 0 && !attn_use_legacy())
    return attn_bwd_tcgen05(p.qkv, p.dout, p.lse, p.delta, p.out, p.B, p.T, p.H, p.Hkv, HD, p.ld, p.ldo, p.scale,
                            p.rope_cs, p.ws_ex && attn_gqa_split(p.B, p.H, p.Hkv, p.T, HD), s);
  {
    const int smem = (2 * BK + 2 * BQI) * LD * 2 + 2 * BQI * 4;
    auto k = attn_bwd_dkdv_kernel<HD>;
    static bool set = false;
    if (!set) {
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return set_cuda_error(e, "attn_bwd_dkdv attr");
      set = true;
    }
    spx_launch_check(launch_k(k, dim3(dim3(p.T / BK, p.Hkv, p.B)), dim3(THREADS), smem, s, p));
    int rc = check_launch("attn_bwd_dkdv_kernel");
    if (rc) return rc;
  }
  {
    const int smem = (2 * BQ + 4 * BK) * LD * 2;
    auto k = attn_bwd_dq_kernel<HD>;
    static bool set = false;
    if (!set) {
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return set_cuda_error(e, "attn_bwd_dq attr");
      set = true;
    }
    spx_launch_check(launch_k(k, dim3(dim3(p.T / BQ, p.H, p.B)), dim3(THREADS), smem, s, p));
    return check_launch("attn_bwd_dq_kernel");
  }
}

static int check_args(int64_t B, int64_t T, int64_t H, int64_t Hkv, int64_t hd) {
  if (B <= 0 || T <= 0 || H <= 0 || Hkv <= 0) return set_error(SPX_ERR_ARG, "attn: non-positive shape");
  if (T % 64) return set_error(SPX_ERR_ARG, "attn: T must be a multiple of 64");
  if (H % Hkv) return set_error(SPX_ERR_ARG, "attn: H must be a multiple of Hkv");
  if (hd != 48 && hd != 64 && hd != 128) return set_error(SPX_ERR_ARG, "attn: head_dim must be 48, 64 or 128");
  return SPX_OK;
}

}  // namespace attn
}  // namespace spx

using namespace spx;

extern "C" int spx_attn_fwd(const void* qkv, void* o, float* lse, int64_t B, int64_t T, int64_t H, int64_t Hkv,
                            int64_t hd, int64_t ld_qkv, int64_t ld_o, float scale, void* stream) {
  int rc = attn::check_args(B, T, H, Hkv, hd);
  if (rc) return rc;
  attn::Params p{};
  p.qkv = reinterpret_cast<const __nv_bfloat16*>(qkv);
  p.out = reinterpret_cast<__nv_bfloat16*>(o);
  p.lse = lse;
  p.ld = ld_qkv;
  p.ldo = ld_o;
  p.B = (int)B; p.T = (int)T; p.H = (int)H; p.Hkv = (int)Hkv;
  p.scale = scale;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if ((hd == 64 || hd == 128) && T % 128 == 0 && !attn_use_legacy())
    return attn_fwd_tcgen05(qkv, o, lse, B, T, H, Hkv, hd, ld_qkv, ld_o, scale, s);
  if (hd == 48) return attn::run_fwd<48>(p, s);
  if (hd == 64) return attn::run_fwd<64>(p, s);
  return attn::run_fwd<128>(p, s);
}

namespace spx {
// SPX_ATTN_LEGACY=1 forces the mma.sync forward (A/B comparisons; the tests check both agree).
bool attn_use_legacy() {
  static const bool legacy = [] {
    const char* e = getenv("SPX_ATTN_LEGACY");
    return e && atoi(e) != 0;
  }();
  return legacy;
}

// SPX_ATTN_GQA_SPLIT=0 disables the split (A/B comparisons)
bool attn_gqa_split(int64_t B, int64_t H, int64_t Hkv, int64_t T, int64_t hd) {
  static const bool enabled = [] {
    const char* e = getenv("SPX_ATTN_GQA_SPLIT");
    return !(e && atoi(e) == 0);
  }();
  if (!enabled || H <= Hkv || Hkv <= 0 || H % Hkv || (hd != 64 && hd != 128) || T % 128 || attn_use_legacy())
    return false;
  return B * Hkv * (T / 128) < num_sms();
}
}  // namespace spx

extern "C" int64_t spx_attn_bwd_ws_floats(int64_t B, int64_t H, int64_t T, int64_t hd) {
  int64_t n = 2 * B * H * T;  // D and lse*log2e
  if ((hd == 64 || hd == 128) && T % 128 == 0 && !attn_use_legacy()) {
    const int64_t nqb = T / 128;
    n += B * H * (nqb * (nqb + 1) / 2) * 128 * 128 / 2;  // dS^T tiles, bf16
  }
  return n;
}

extern "C" int64_t spx_attn_bwd_ws_floats_ex(int64_t B, int64_t H, int64_t Hkv, int64_t T, int64_t hd) {
  int64_t n = spx_attn_bwd_ws_floats(B, H, T, hd);
  if (attn_gqa_split(B, H, Hkv, T, hd)) n += B * H * (T / 128) * 2 * hd * 128;  // dV/dK partials, fp32
  return n;
}

extern "C" int spx_attn_bwd(const void* qkv, const void* o, const void* dout, const float* lse, float* delta_ws,
                            void* dqkv, int64_t B, int64_t T, int64_t H, int64_t Hkv, int64_t hd, int64_t ld_qkv,
                            int64_t ld_o, float scale, const float* rope_cos_sin, void* stream) {
  return spx_attn_bwd_ex(qkv, o, dout, lse, delta_ws, dqkv, B, T, H, Hkv, hd, ld_qkv, ld_o, scale, rope_cos_sin, 0,
                         stream);
}

extern "C" int spx_attn_bwd_ex(const void* qkv, const void* o, const void* dout, const float* lse, float* delta_ws,
                               void* dqkv, int64_t B, int64_t T, int64_t H, int64_t Hkv, int64_t hd, int64_t ld_qkv,
                               int64_t ld_o, float scale, const float* rope_cos_sin, int32_t flags, void* stream) {
  if (flags & ~(SPX_ATTN_DELTA_READY | SPX_ATTN_WS_EX)) return set_error(SPX_ERR_ARG, "attn_bwd: unknown flags");
  int rc = attn::check_args(B, T, H, Hkv, hd);
  if (rc) return rc;
  if (ld_o % 8 != 0 || (((uintptr_t)o | (uintptr_t)dout) & 15))
    return set_error(SPX_ERR_ARG, "attn_bwd: O/dO must be 16-byte aligned with ld_o % 8 == 0");
  attn::Params p{};
  p.qkv = reinterpret_cast<const __nv_bfloat16*>(qkv);
  p.out = reinterpret_cast<__nv_bfloat16*>(dqkv);
  p.o = reinterpret_cast<const __nv_bfloat16*>(o);
  p.dout = reinterpret_cast<const __nv_bfloat16*>(dout);
  p.lse = const_cast<float*>(lse);
  p.delta = delta_ws;
  p.rope_cs = rope_cos_sin;
  p.ld = ld_qkv;
  p.ldo = ld_o;
  p.B = (int)B; p.T = (int)T; p.H = (int)H; p.Hkv = (int)Hkv;
  p.scale = scale;
  p.delta_ready = (flags & SPX_ATTN_DELTA_READY) ? 1 : 0;
  p.ws_ex = (flags & SPX_ATTN_WS_EX) ? 1 : 0;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (hd == 48) return attn::run_bwd<48>(p, s);
  if (hd == 64) return attn::run_bwd<64>(p, s);
  return attn::run_bwd<128>(p, s);
}
