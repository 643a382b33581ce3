// tcgen05 / TMEM / TMA GEMM for the decoder projections (sm_100a).
//
//   out[t, n] = epilogue( sum_k X[t, k] * W[n, k] )      X: [T, K] bf16, W: [N, K] bf16
//
// Both operands are K-major, staged by TMA into 128-byte-swizzled shared
// memory, multiplied by tcgen05.mma (kind::f16, fp32 accumulator in TMEM) and
// drained by tcgen05.ld in the epilogue.  Two operand orientations:
//
//   SWAP  (decode, T <= 256): the weight tile is the MMA "A" operand (M = 128
//          output features per CTA) and the tokens are the MMA N dimension
//          (16..256).  Weight bytes dominate, so the kernel is an HBM stream of
//          W with split-K chosen from (N, K) only -- never from T -- so among
//          decode (SWAP) batches a token's result does not depend on the batch it
//          rides in.  The orientation itself switches at T = 256 (SWAP above has
//          split-K, !SWAP does not), so prefill rows may round differently in a
//          <= 256-token micro-batch than in a larger one.
//   !SWAP (prefill): tokens are the A operand (M = 128 rows), features are N = 256;
//          at T >= 512 gemm_pair_kernel (CTA pairs, cta_group::2, 256 x 256 tiles).
//
// Persistent and warp-specialized (256 threads): warp 0 lane 0 = weight TMA
// producer, warp 6 lane 0 = activation TMA producer (each runs its smem ring
// continuously across work items), warp 1 = TMEM allocator + MMA issuer (lane 0),
// warps 2-5 = epilogue, warp w owning TMEM lanes [32(w%4), +32); in a single-item
// CTA's decode epilogue warps 0, 1, 6 and 7 take the second half of the columns.  The accumulator
// is double-buffered in TMEM so the epilogue of item i overlaps the main loop of
// item i+1.  Decode split-K: partials + a reduce kernel, or (cluster split-K) a
// DSMEM reduction inside the launch.
//
// Epilogues (rounding points follow HF modeling_llama.py: every bf16 tensor op
// rounds its fp32 result to bf16):
//   STORE     out = bf16(acc)
//   BIAS      out = bf16(acc + bias[n])                 (Qwen2 qkv bias, modeling_qwen2.py:200-203)
//   RESIDUAL  out = bf16(bf16(acc) + residual[t, n])     (o_proj / down_proj + residual, :313-331)
//   SWIGLU    W rows interleaved in 64-row blocks [gate 64 | up 64]:
//             out[t, j] = bf16(bf16(silu(bf16(g))) * bf16(u))   (LlamaMLP, :182-184)
//   split-K   token-contiguous fp32 partials per split, summed in split order by
//             gemm_splitk_reduce_kernel, which applies the epilogue
//   ARGMAX    per token (max logit, index) over this CTA's 128 vocabulary rows
#include <cudaTypedefs.h>

#include <array>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "pl_internal.h"

namespace pl {

constexpr int BK = 64;          // bf16 elements per 128-byte swizzle row
constexpr int GEMM_THREADS = 224;  // pair kernel: warp 0 weight producer, 1 MMA, 2-5 epilogue, 6 activation producer
constexpr int GEMM_ACT_WARP = 6;
// gemm_tc_kernel adds warp 7: with warps 0, 1 and 6 (done with their roles by then) it
// takes the second half of the accumulator columns of a single-item CTA's decode
// epilogue, two warps per TMEM lane quarter (warp w reads lanes [32 (w % 4), +32))
// (profiles/r2/decode/epilogue_helpers_ab.log: epilogue phases -1 to -1.5 us per GEMM,
// -3.5 us per layer at T = 32)
constexpr int TC_THREADS = 256;
constexpr int BM = 128;         // MMA M (A-operand rows per CTA)
constexpr int A_TILE_BYTES = BM * BK * 2;

struct GemmArgs {
  int T;             // tokens (logical rows of out)
  int N;             // output features of the GEMM (rows of W)
  int num_kb;        // K / 64
  int kb_per_split;
  int splits;
  int tiles_m;       // 128-row tiles of the A operand
  int num_items;     // tiles_m * tiles_n * splits
  int epi;
  __nv_bfloat16* C;
  int64_t ldc;
  const __nv_bfloat16* bias;
  const __nv_bfloat16* residual;
  int64_t ldr;
  __nv_bfloat16* C2;  // fused transport: a second copy of every final output row (ldc), or null
  float* partial;     // split-K partials, fp32: pmode 0 [splits][N][Tp], pmode 1 [splits][T][N]
  int Tp;             // T rounded up to the BN tile
  int pmode;
  float2* argmax_ws;  // [N/128 tiles][T] (value, index-as-float-bits)
  const uint8_t* wp;  // pre-packed weights (pl_pack_weight): 16 KB SW128 tile images, [N/128][K/64]
  int swiglu_il;      // packed gate_up: rows alternate gate_j, up_j inside each 128-row tile
  int raster_m;       // > 0: grouped tile raster, bands of raster_m row tiles (prefill)
  // cluster split-K (decode / SWAP): the `splits` CTAs of one weight tile form a cluster,
  // each parks its fp32 partial in its own (idle) ring memory and the cluster reduces
  // over distributed shared memory -- no partial round trip through HBM/L2, no reduce
  // kernel.  rope: the reduction also applies RoPE + the paged K/V append
  // (reduce_qkv_rope_kernel's math; a 128-feature tile is one head).
  int csk;
  int rope;
  const int32_t* pos;
  const int32_t* slot;
  const __nv_bfloat16* cos_sin;
  int max_pos;
  __nv_bfloat16* k_cache;
  __nv_bfloat16* v_cache;
  int block_size, Hq, Hkv;
};

// One unit of work: k-blocks [kb0, kb0 + nkb) of output tile (m_tile, n_tile).
struct Piece {
  int m_tile, n_tile, split, kb0, nkb;
};

// Walks this CTA's pieces (identical in the producer, MMA and epilogue roles):
// items blockIdx.x, blockIdx.x + gridDim.x, ...
struct PieceWalk {
  int it, end;
  PL_DEV void init(const GemmArgs& a) {
    it = blockIdx.x;
    end = a.num_items;
  }
  PL_DEV bool next(const GemmArgs& a, Piece& p) {
    if (it >= end) return false;
    p.split = it % a.splits;
    const int tile = it / a.splits;
    if (a.raster_m > 0) {
      // grouped raster (prefill): bands of raster_m row tiles walk all column tiles, so
      // the CTAs in flight share a few MB of A rows and B columns in L2 instead of
      // cycling every A row tile per B column tile (measured: 11 GB of DRAM reads for a
      // 369 MB gate_up at T = 16384 without it)
      const int tiles_n = a.num_items / (a.tiles_m * a.splits);
      const int band = tile / (a.raster_m * tiles_n);
      const int gm = min(a.raster_m, a.tiles_m - band * a.raster_m);
      const int idx = tile - band * a.raster_m * tiles_n;
      p.m_tile = band * a.raster_m + idx % gm;
      p.n_tile = idx / gm;
    } else {
      p.m_tile = tile % a.tiles_m;
      p.n_tile = tile / a.tiles_m;
    }
    p.kb0 = p.split * a.kb_per_split;
    p.nkb = min(a.num_kb, p.kb0 + a.kb_per_split) - p.kb0;
    it += gridDim.x;
    return true;
  }
};

// Decode tiles (BN <= 128) run 2 CTAs per SM with a shallower ring each (two
// independent epilogues per SM); BN = 256 tiles run one CTA per SM.
//
// Two rings: A tiles and B tiles have their own depth.  In the decode (SWAP)
// orientation A = weights streamed once from HBM and B = the activations,
// re-read per weight tile from L2 (short latency): the activation ring is 3
// deep and every other byte of shared memory holds weights in flight -- the
// kernel is latency-bound on HBM, so weight bytes in flight set its speed.
// The producer issues B block k only (AS - BS) blocks behind A block k.
// Ring split (SWAP): the producer issues B block k (L2 hit, latency ~Ll) only
// (AS - BS) blocks behind A block k (HBM, ~Ld ~ 2 Ll), so each ring bounds the
// k-block rate: rate <= min(AS / Ld, BS / Ll).  Pick the split maximizing
// min(AS, 2 BS) within the budget (measured: a 3-deep B ring capped one CTA at
// ~48 GB/s however deep the A ring was).
#ifndef PL_RING_RATIO
#define PL_RING_RATIO 1
#endif
constexpr int ring_bs(int budget, int a_bytes, int b_bytes) {
  int best_bs = 2, best = 0;
  for (int bs = 2; bs <= 16; ++bs) {
    const int as = (budget - bs * b_bytes) / a_bytes;
    if (as < 2) break;
    const int v = as < PL_RING_RATIO * bs ? as : PL_RING_RATIO * bs;
    if (v > best || (v == best && as > (budget - best_bs * b_bytes) / a_bytes)) best = v, best_bs = bs;
  }
  return best_bs;
}

template <int BN, bool SWAP, int CTAS>
struct GemmSmem {
  static constexpr int B_TILE_BYTES = BN * BK * 2;
  static constexpr int BUDGET = CTAS == 2 ? 104 * 1024 : 200 * 1024;
  static constexpr int BS0 = SWAP ? ring_bs(BUDGET, A_TILE_BYTES, B_TILE_BYTES)
                                  : BUDGET / (A_TILE_BYTES + B_TILE_BYTES);
  static constexpr int AS = SWAP ? (BUDGET - BS0 * B_TILE_BYTES) / A_TILE_BYTES : BS0;
  // left-over budget deepens the activation ring (its L2 latency caps the k-block rate too)
  static constexpr int BS_FILL = SWAP ? (BUDGET - AS * A_TILE_BYTES) / B_TILE_BYTES : BS0;
  static constexpr int BS = BS_FILL > 16 ? 16 : BS_FILL;
  static constexpr int B_OFFSET = AS * A_TILE_BYTES;
  static constexpr int BAR_OFFSET = B_OFFSET + BS * B_TILE_BYTES;
  // fullA[AS], emptyA[AS], fullB[BS], emptyB[BS], tmem_full[2], tmem_empty[2], tmem slot + flag
  static constexpr int SCRATCH_OFFSET = BAR_OFFSET + 8 * (2 * AS + 2 * BS + 4) + 16;
  static constexpr int SCRATCH_BYTES = 64 * 16 * 4;  // swiglu exchange / argmax partials
  static constexpr int TOTAL = SCRATCH_OFFSET + SCRATCH_BYTES + 1024;  // + alignment slack
  static_assert(AS >= 2 && BS >= 2, "ring too shallow");
};

PL_DEV float silu_f(float x) { return x / (1.0f + expf(-x)); }
PL_DEV void epi_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Final (non-partial) epilogue for one accumulator element.
PL_DEV void store_out(const GemmArgs& a, int epi, int t, int n, float acc) {
  __nv_bfloat16 v;
  if (epi == EPI_RESIDUAL)
    v = f2bf(rbf(acc) + bf2f(a.residual[(int64_t)t * a.ldr + n]));
  else if (epi == EPI_BIAS)
    v = f2bf(acc + bf2f(a.bias[n]));
  else
    v = f2bf(acc);
  a.C[(int64_t)t * a.ldc + n] = v;
  if (a.C2) a.C2[(int64_t)t * a.ldc + n] = v;  // the next stage's receive buffer (peer memory)
}

// Cluster split-K QKV epilogue (RoPE + K/V append), vectorised: thread q = ep & 15 owns
// features [4q, 4q + 4) of both rotary halves of the head, column group g = ep >> 4
// (0..7) owns token columns c_begin + g + 8u; the splits' DSMEM partials come as 16-byte
// loads.  The position / RoPE-table / KV-slot metadata of a thread's first CSK_COLS
// columns is loaded by the epilogue warps while the main loop streams (they are idle
// then; the predecessor completed at their griddepcontrol.wait) and kept as packed bf16.
// Against one feature per thread with the metadata loaded after the main loop: -3.8 us
// per layer at T = 64, -2.5 at T = 32 (profiles/r2/decode/csk_v4_preload_ab.log).
constexpr int CSK_COLS = 2;
struct CskMeta {
  uint2 cs[CSK_COLS], sn[CSK_COLS];  // bf16 x4: cos / sin of features [4q, 4q + 4)
  int sl[CSK_COLS];
};

PL_DEV void csk_rope_meta(const GemmArgs& args, int c_end, int f1, bool roped, int cb, uint2* cs, uint2* sn,
                          int* sl) {
  constexpr int HDIM = 128, HALF = 64;
  int pp[CSK_COLS];
#pragma unroll
  for (int u = 0; u < CSK_COLS; ++u) {
    const int c = max(0, min(cb + 8 * u, c_end - 1));  // clamped: duplicates are never stored
    pp[u] = roped ? args.pos[c] : 0;
    sl[u] = args.slot ? args.slot[c] : -1;
  }
#pragma unroll
  for (int u = 0; u < CSK_COLS; ++u) {
    const int p = pp[u] < 0 ? 0 : (pp[u] >= args.max_pos ? args.max_pos - 1 : pp[u]);
    cs[u] = sn[u] = make_uint2(0, 0);
    if (roped) {
      cs[u] = *reinterpret_cast<const uint2*>(args.cos_sin + static_cast<int64_t>(p) * HDIM + f1);
      sn[u] = *reinterpret_cast<const uint2*>(args.cos_sin + static_cast<int64_t>(p) * HDIM + HALF + f1);
    }
  }
}

PL_DEV void csk_preload(const GemmArgs& args, int ep, int BN, CskMeta& m) {
  const int s = args.splits;
  const int rank = static_cast<int>(cluster_ctarank());
  const int ncols = min(args.T, BN);
  const int per = (ncols + s - 1) / s;
  const int c_begin = rank * per, c_end = min(ncols, c_begin + per);
  const bool roped = static_cast<int>(blockIdx.x) / s < args.Hq + args.Hkv;
  csk_rope_meta(args, c_end, 4 * (ep & 15), roped, c_begin + (ep >> 4), m.cs, m.sn, m.sl);
}

// Cluster split-K reduction (SWAP, one weight tile per cluster, cluster rank = split):
// CTA r finalises token columns [r * per, +per) of the tile, summing the splits' parked
// partials over DSMEM in split order (the order of gemm_splitk_reduce_kernel /
// reduce_qkv_rope_kernel, so results are bit-identical to the two-kernel path).
PL_DEV void csk_reduce(const GemmArgs& args, const uint8_t* smem, int ep, int BN, const CskMeta& pre) {
  const int s = args.splits;
  const int rank = static_cast<int>(cluster_ctarank());
  const int m_tile = static_cast<int>(blockIdx.x) / s;
  const int ncols = min(args.T, BN);
  const int per = (ncols + s - 1) / s;
  const int c_begin = rank * per, c_end = min(ncols, c_begin + per);
  if (!args.rope) {
    // vectorised like the RoPE path: thread q = ep & 31 owns features [4q, 4q + 4) of the
    // tile, column group g = ep >> 5 owns columns c_begin + g + 4u; residual / bias /
    // output move as bf16 x4
    const int q = ep & 31, g = ep >> 5;
    const int n0 = m_tile * BM + 4 * q;
    if (n0 >= args.N) return;  // N % 4 == 0 on this path (csk needs tiles_n == 1 and N % 128 == 0)
    const int epi = args.epi;
    float bb[4] = {0.f, 0.f, 0.f, 0.f};
    if (epi == EPI_BIAS) {
      const uint2 u = *reinterpret_cast<const uint2*>(args.bias + n0);
      const float2 a0 = unpack_bf16x2(u.x), a1 = unpack_bf16x2(u.y);
      bb[0] = a0.x, bb[1] = a0.y, bb[2] = a1.x, bb[3] = a1.y;
    }
    constexpr int CC = 4;  // columns per batch
    for (int cb = c_begin + g; cb < c_end; cb += 4 * CC) {
      uint2 res[CC];
#pragma unroll
      for (int u = 0; u < CC; ++u) {
        const int c = min(cb + 4 * u, c_end - 1);  // clamped: duplicates are never stored
        res[u] = epi == EPI_RESIDUAL ? *reinterpret_cast<const uint2*>(args.residual + (int64_t)c * args.ldr + n0)
                                     : make_uint2(0, 0);
      }
      float4 acc[CC];
#pragma unroll
      for (int u = 0; u < CC; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int j0 = 0; j0 < s; j0 += 4) {  // split order, 4 splits' loads per round in flight
        float4 x[4][CC];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
#pragma unroll
          for (int u = 0; u < CC; ++u) {
            const int c = min(cb + 4 * u, c_end - 1);
            x[jj][u] = ld_dsmem_f32x4(mapa_shared(smem, min(j0 + jj, s - 1)) +
                                      static_cast<uint32_t>((c * BM + 4 * q) * 4));
          }
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
          if (j0 + jj < s)
#pragma unroll
            for (int u = 0; u < CC; ++u)
              acc[u].x += x[jj][u].x, acc[u].y += x[jj][u].y, acc[u].z += x[jj][u].z, acc[u].w += x[jj][u].w;
      }
#pragma unroll
      for (int u = 0; u < CC; ++u) {
        const int t = cb + 4 * u;
        if (t >= c_end) break;
        const float av[4] = {acc[u].x, acc[u].y, acc[u].z, acc[u].w};
        const float2 r01 = unpack_bf16x2(res[u].x), r23 = unpack_bf16x2(res[u].y);
        const float rv[4] = {r01.x, r01.y, r23.x, r23.y};
        float o[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)  // store_out's rounding points
          o[e] = epi == EPI_RESIDUAL ? rbf(av[e]) + rv[e] : epi == EPI_BIAS ? av[e] + bb[e] : av[e];
        const uint2 w = make_uint2(pack_bf16x2(o[0], o[1]), pack_bf16x2(o[2], o[3]));
        *reinterpret_cast<uint2*>(args.C + (int64_t)t * args.ldc + n0) = w;
        if (args.C2) *reinterpret_cast<uint2*>(args.C2 + (int64_t)t * args.ldc + n0) = w;
      }
    }
    return;
  }
  constexpr int HDIM = 128, HALF = 64;
  const int hh = m_tile;  // a 128-feature tile is one q / k / v head
  {
    const int q = ep & 15, g = ep >> 4;
    const int f1 = 4 * q, f2 = HALF + 4 * q;
    const int n1 = hh * HDIM + f1, n2 = hh * HDIM + f2;
    float b1[4] = {0.f, 0.f, 0.f, 0.f}, b2[4] = {0.f, 0.f, 0.f, 0.f};
    if (args.bias) {
      const uint2 u1 = *reinterpret_cast<const uint2*>(args.bias + n1);
      const uint2 u2 = *reinterpret_cast<const uint2*>(args.bias + n2);
      const float2 a0 = unpack_bf16x2(u1.x), a1 = unpack_bf16x2(u1.y);
      const float2 c0 = unpack_bf16x2(u2.x), c1 = unpack_bf16x2(u2.y);
      b1[0] = a0.x, b1[1] = a0.y, b1[2] = a1.x, b1[3] = a1.y;
      b2[0] = c0.x, b2[1] = c0.y, b2[2] = c1.x, b2[3] = c1.y;
    }
    const bool roped = hh < args.Hq + args.Hkv;
    for (int cb = c_begin + g, k = 0; cb < c_end; cb += 8 * CSK_COLS, ++k) {
      uint2 cs[CSK_COLS], sn[CSK_COLS];
      int sl[CSK_COLS];
      if (k == 0) {
#pragma unroll
        for (int u = 0; u < CSK_COLS; ++u) cs[u] = pre.cs[u], sn[u] = pre.sn[u], sl[u] = pre.sl[u];
      } else {  // T > 16 * splits: later columns load theirs here
        csk_rope_meta(args, c_end, f1, roped, cb, cs, sn, sl);
      }
      // split-ordered sums (0 + x0 + x1 + ..., the order of reduce_qkv_rope_kernel, so the
      // result is bit-identical to the two-kernel path), 4 splits' loads per round in flight
      float4 a1[CSK_COLS], a2[CSK_COLS];
#pragma unroll
      for (int u = 0; u < CSK_COLS; ++u) a1[u] = a2[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int j0 = 0; j0 < s; j0 += 4) {
        float4 x1[4][CSK_COLS], x2[4][CSK_COLS];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
#pragma unroll
          for (int u = 0; u < CSK_COLS; ++u) {
            const int j = min(j0 + jj, s - 1);
            const int c = min(cb + 8 * u, c_end - 1);
            const uint32_t addr = mapa_shared(smem, j) + static_cast<uint32_t>((c * BM + f1) * 4);
            x1[jj][u] = ld_dsmem_f32x4(addr);
            x2[jj][u] = ld_dsmem_f32x4(addr + HALF * 4);
          }
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
          if (j0 + jj < s)
#pragma unroll
            for (int u = 0; u < CSK_COLS; ++u) {
              a1[u].x += x1[jj][u].x, a1[u].y += x1[jj][u].y, a1[u].z += x1[jj][u].z, a1[u].w += x1[jj][u].w;
              a2[u].x += x2[jj][u].x, a2[u].y += x2[jj][u].y, a2[u].z += x2[jj][u].z, a2[u].w += x2[jj][u].w;
            }
      }
#pragma unroll
      for (int u = 0; u < CSK_COLS; ++u) {
        const int t = cb + 8 * u;
        if (t >= c_end) break;
        const float s1[4] = {a1[u].x, a1[u].y, a1[u].z, a1[u].w};
        const float s2[4] = {a2[u].x, a2[u].y, a2[u].z, a2[u].w};
        const float2 c01 = unpack_bf16x2(cs[u].x), c23 = unpack_bf16x2(cs[u].y);
        const float2 n01 = unpack_bf16x2(sn[u].x), n23 = unpack_bf16x2(sn[u].y);
        const float cv[4] = {c01.x, c01.y, c23.x, c23.y}, sv[4] = {n01.x, n01.y, n23.x, n23.y};
        float o1[4], o2[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float v1 = rbf(s1[e] + b1[e]), v2 = rbf(s2[e] + b2[e]);
          o1[e] = v1, o2[e] = v2;
          if (roped) {
            const float c_ = cv[e], s_ = sv[e];
            o1[e] = rbf(rbf(v1 * c_) + rbf(-v2 * s_));
            o2[e] = rbf(rbf(v2 * c_) + rbf(v1 * s_));
          }
        }
        const uint2 w1 = make_uint2(pack_bf16x2(o1[0], o1[1]), pack_bf16x2(o1[2], o1[3]));
        const uint2 w2 = make_uint2(pack_bf16x2(o2[0], o2[1]), pack_bf16x2(o2[2], o2[3]));
        __nv_bfloat16* row = args.C + static_cast<int64_t>(t) * args.ldc;
        *reinterpret_cast<uint2*>(row + n1) = w1;
        *reinterpret_cast<uint2*>(row + n2) = w2;
        if (hh >= args.Hq && sl[u] >= 0) {
          const bool is_k = roped;
          const int kh = is_k ? hh - args.Hq : hh - args.Hq - args.Hkv;
          __nv_bfloat16* cache = is_k ? args.k_cache : args.v_cache;
          __nv_bfloat16* dst = cache + ((static_cast<int64_t>(sl[u] / args.block_size) * args.Hkv + kh) *
                                            args.block_size + sl[u] % args.block_size) * HDIM;
          *reinterpret_cast<uint2*>(dst + f1) = w1;
          *reinterpret_cast<uint2*>(dst + f2) = w2;
        }
      }
    }
    return;
  }
}

// Decode (SWAP) epilogues over accumulator columns [c_lo, c_hi) (multiples of 16), two
// TMEM loads (32 columns) per tcgen05.wait::ld (batched waits:
// profiles/r2/decode/epilogue_x4_ab.log; 32 keeps the 256-thread kernel within 128 registers).
// SwiGLU on interleaved rows: lane pairs (gate_j, up_j) meet by one shuffle; the pair
// splits each 16-token chunk (even lane tokens 0-7, odd lane 8-15) so both lanes evaluate
// SiLU (instruction-bound: one lane per pair doing all 64 tokens took ~9 us).
PL_DEV void epi_swiglu_cols(const GemmArgs& args, uint32_t tcol, int row, int m_tile, int t_base, int c_lo,
                            int c_hi) {
  const int j = m_tile * 64 + (row >> 1);
  const bool odd = row & 1;
  for (int g0 = c_lo; g0 < c_hi; g0 += 32) {
    const int nch = min(2, (c_hi - g0) / 16);
    uint32_t rr[2][16];
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (h < nch) tmem_ld16(tcol + g0 + 16 * h, rr[h]);
    tmem_ld_wait();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h >= nch) break;
      const int c0 = g0 + 16 * h;
      float v[16], other[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) v[c] = __uint_as_float(rr[h][c]);
#pragma unroll
      for (int c = 0; c < 16; ++c) other[c] = __shfl_xor_sync(0xffffffffu, v[c], 1);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float g = odd ? other[k + 8] : v[k];
        const float u = odd ? v[k + 8] : other[k];
        const int t = t_base + c0 + k + (odd ? 8 : 0);
        if (t < args.T) args.C[(int64_t)t * args.ldc + j] = f2bf(rbf(silu_f(rbf(g))) * rbf(u));
      }
    }
  }
}

// feature-contiguous split-K partials [split][T][N] (per-token fused reductions)
PL_DEV void epi_partial_cols(const GemmArgs& args, uint32_t tcol, int n, int split, int t_base, int c_lo,
                             int c_hi) {
  for (int g0 = c_lo; g0 < c_hi; g0 += 32) {
    const int nch = min(2, (c_hi - g0) / 16);
    uint32_t rr[2][16];
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (h < nch) tmem_ld16(tcol + g0 + 16 * h, rr[h]);
    tmem_ld_wait();
    if (n < args.N) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h >= nch) break;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const int t = t_base + g0 + 16 * h + c;
          if (t < args.T) args.partial[((int64_t)split * args.T + t) * args.N + n] = __uint_as_float(rr[h][c]);
        }
      }
    }
  }
}

// !SWAP (prefill) epilogue: TMEM lane <-> token t, accumulator column c <-> feature
// n_tile * BN + c (split-K is never used on this path).
template <int BN>
PL_DEV void token_rows_epilogue(const GemmArgs& args, uint32_t tcol, int t, int n_tile) {
  const int epi = args.epi;
  const bool tv = t < args.T;
  if (epi == EPI_SWIGLU && args.swiglu_il) {
    // interleaved columns (gate_j, up_j): 16 accumulator columns -> 8 outputs
    for (int c0 = 0; c0 < BN; c0 += 16) {
      uint32_t r[16];
      tmem_ld16(tcol + c0, r);
      tmem_ld_wait();
      const int j0 = (n_tile * BN + c0) / 2;
      if (tv && n_tile * BN + c0 < args.N) {
        uint32_t packed[4];
#pragma unroll
        for (int c = 0; c < 16; c += 4) {
          const float g0 = rbf(__uint_as_float(r[c])), u0 = rbf(__uint_as_float(r[c + 1]));
          const float g1 = rbf(__uint_as_float(r[c + 2])), u1 = rbf(__uint_as_float(r[c + 3]));
          packed[c / 4] = pack_bf16x2(rbf(silu_f(g0)) * u0, rbf(silu_f(g1)) * u1);
        }
        *reinterpret_cast<uint4*>(args.C + (int64_t)t * args.ldc + j0) =
            make_uint4(packed[0], packed[1], packed[2], packed[3]);
      }
    }
  } else if (epi == EPI_SWIGLU) {
    for (int p = 0; p < BN / 128; ++p) {
      for (int c0 = 0; c0 < 64; c0 += 16) {
        uint32_t g[16], u[16];
        tmem_ld16(tcol + p * 128 + c0, g);
        tmem_ld16(tcol + p * 128 + 64 + c0, u);
        tmem_ld_wait();
        const int j0 = (n_tile * BN) / 2 + p * 64 + c0;
        if (tv && (n_tile * BN + p * 128) < args.N) {
          uint32_t packed[8];
#pragma unroll
          for (int c = 0; c < 16; c += 2) {
            const float g0 = rbf(__uint_as_float(g[c])), g1 = rbf(__uint_as_float(g[c + 1]));
            const float u0 = rbf(__uint_as_float(u[c])), u1 = rbf(__uint_as_float(u[c + 1]));
            packed[c / 2] = pack_bf16x2(rbf(silu_f(g0)) * u0, rbf(silu_f(g1)) * u1);
          }
          uint4* dst = reinterpret_cast<uint4*>(args.C + (int64_t)t * args.ldc + j0);
          dst[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
          dst[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
        }
      }
    }
  } else {
    for (int c0 = 0; c0 < BN; c0 += 16) {
      uint32_t r[16];
      tmem_ld16(tcol + c0, r);
      tmem_ld_wait();
      const int n0 = n_tile * BN + c0;
      if (!tv || n0 >= args.N) continue;
      float v[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) v[c] = __uint_as_float(r[c]);
      if (epi == EPI_BIAS) {
#pragma unroll
        for (int c = 0; c < 16; ++c) v[c] += bf2f(args.bias[n0 + c]);
      } else if (epi == EPI_RESIDUAL) {
        const uint4* rp = reinterpret_cast<const uint4*>(args.residual + (int64_t)t * args.ldr + n0);
        const uint4 r0 = rp[0], r1 = rp[1];
        const uint32_t rr[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
        for (int c = 0; c < 16; c += 2) {
          const float2 rv = unpack_bf16x2(rr[c / 2]);
          v[c] = rbf(v[c]) + rv.x;
          v[c + 1] = rbf(v[c + 1]) + rv.y;
        }
      }
      uint32_t packed[8];
#pragma unroll
      for (int c = 0; c < 16; c += 2) packed[c / 2] = pack_bf16x2(v[c], v[c + 1]);
      uint4* dst = reinterpret_cast<uint4*>(args.C + (int64_t)t * args.ldc + n0);
      dst[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
      dst[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
    }
  }
}

template <int BN, bool SWAP, int CTAS>
__global__ void __launch_bounds__(TC_THREADS, CTAS)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const GemmArgs args) {
  using L = GemmSmem<BN, SWAP, CTAS>;
  constexpr int AS = L::AS, BS = L::BS;
  constexpr uint32_t TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;  // double-buffered accumulator
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* fullA = reinterpret_cast<uint64_t*>(smem + L::BAR_OFFSET);
  uint64_t* emptyA = fullA + AS;
  uint64_t* fullB = emptyA + AS;
  uint64_t* emptyB = fullB + BS;
  uint64_t* tfull = emptyB + BS;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* scratch = reinterpret_cast<float*>(smem + L::SCRATCH_OFFSET);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  CskMeta csk_meta;  // cluster split-K RoPE metadata (epilogue warps)
  // second-half epilogue helpers (warps 0, 1, 6, 7) for single-item CTAs of the two hot
  // decode epilogues (SwiGLU on interleaved rows, feature-contiguous split-K partials)
  const bool split_epi = SWAP && BN >= 32 && static_cast<int>(gridDim.x) >= args.num_items && !args.csk &&
                         ((args.splits > 1 && args.pmode == 1) ||
                          (args.splits == 1 && args.epi == EPI_SWIGLU && args.swiglu_il));
  const uint32_t tl_tag = (1u << 24) | ((static_cast<uint32_t>(args.N) / 128u) << 12) | static_cast<uint32_t>(args.num_kb);
  if (threadIdx.x == 0) PL_TL(tl_tag, 0);

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < AS; ++s) {
      mbar_init(&fullA[s], 1);
      mbar_init(&emptyA[s], 1);
    }
    for (int s = 0; s < BS; ++s) {
      mbar_init(&fullB[s], 1);
      mbar_init(&emptyB[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  // the epilogue writes buffers the previous kernel may still read (split-K partials,
  // the residual stream): wait for it before any global write
  if (warp >= 2) pdl_wait();

  if (warp == 0 || warp == GEMM_ACT_WARP) {
    // ------------------------------------------------------- TMA producers
    if (warp == 0 && lane == 0) {
      const uint64_t pol_w = policy_evict_first();   // weights stream through once
      const uint64_t pol_x = policy_evict_last();    // activations are re-read per weight tile
      const uint64_t polA = SWAP ? pol_w : pol_x;
      const uint64_t polB = SWAP ? pol_x : pol_w;
      int sa = 0, sb = 0;
      uint32_t pa = 0, pb = 0;
      auto issue_a = [&](int kb, int m_tile) {
        mbar_wait(&emptyA[sa], pa ^ 1);
        mbar_arrive_expect_tx(&fullA[sa], A_TILE_BYTES);
        if (SWAP && args.wp)  // one contiguous 16 KB copy of the pre-swizzled weight tile
          bulk_load(smem + sa * A_TILE_BYTES, args.wp + ((int64_t)m_tile * args.num_kb + kb) * A_TILE_BYTES,
                    A_TILE_BYTES, &fullA[sa]);
        else
          tma_load_2d(smem + sa * A_TILE_BYTES, &tmA, &fullA[sa], kb * BK, m_tile * BM, polA);
        if (++sa == AS) {
          sa = 0;
          pa ^= 1;
        }
      };
      auto issue_b = [&](int kb, int n_tile) {
        mbar_wait(&emptyB[sb], pb ^ 1);
        mbar_arrive_expect_tx(&fullB[sb], L::B_TILE_BYTES);
        if (!SWAP && args.wp) {  // BN = 256 weight rows = packed tiles 2n, 2n+1
          uint8_t* d = smem + L::B_OFFSET + sb * L::B_TILE_BYTES;
#pragma unroll
          for (int h = 0; h < BN / BM; ++h)
            bulk_load(d + h * A_TILE_BYTES,
                      args.wp + ((int64_t)(n_tile * (BN / BM) + h) * args.num_kb + kb) * A_TILE_BYTES,
                      A_TILE_BYTES, &fullB[sb]);
        } else {
          tma_load_2d(smem + L::B_OFFSET + sb * L::B_TILE_BYTES, &tmB, &fullB[sb], kb * BK, n_tile * BN, polB);
        }
        if (++sb == BS) {
          sb = 0;
          pb ^= 1;
        }
      };
      // Two independent streams, one thread each IN DIFFERENT WARPS, so neither waits
      // behind the other's ring: warp 0 streams the weights (never produced by the
      // previous kernel, so no PDL wait -- they flow while the predecessor drains), warp
      // GEMM_ACT_WARP the activations (after griddepcontrol.wait).  A single issuing
      // thread coupled the rings; two lanes of one warp are no better: a lane suspended
      // in mbarrier.try_wait holds the warp, so the other lane's loads went out one
      // suspend interval late -- each CTA streamed only ~24 GB/s (measured: the Llama-3
      // o-proj at split 1 took 44 us for 32 MB), hidden only when every SM is busy.
      PieceWalk walk;
      walk.init(args);
      Piece pc;
      while (walk.next(args, pc)) {
        const int m_tile = pc.m_tile, n_tile = pc.n_tile, kb0 = pc.kb0, nkb = pc.nkb;
        for (int i = 0; i < nkb; ++i) {
          if (SWAP) issue_a(kb0 + i, m_tile);
          else issue_b(kb0 + i, n_tile);
        }
      }
    } else if (warp == GEMM_ACT_WARP && lane == 0) {
      const uint64_t pol_x = policy_evict_last();
      const uint64_t polA = pol_x, polB = pol_x;
      int sa = 0, sb = 0;
      uint32_t pa = 0, pb = 0;
      pdl_wait();  // activations come from the previous kernel
      PieceWalk walk;
      walk.init(args);
      Piece pc;
      while (walk.next(args, pc)) {
        const int m_tile = pc.m_tile, n_tile = pc.n_tile, kb0 = pc.kb0, nkb = pc.nkb;
        for (int i = 0; i < nkb; ++i) {
          const int kb = kb0 + i;
          if (SWAP) {
            mbar_wait(&emptyB[sb], pb ^ 1);
            mbar_arrive_expect_tx(&fullB[sb], L::B_TILE_BYTES);
            tma_load_2d(smem + L::B_OFFSET + sb * L::B_TILE_BYTES, &tmB, &fullB[sb], kb * BK, n_tile * BN, polB);
            if (++sb == BS) {
              sb = 0;
              pb ^= 1;
            }
          } else {
            mbar_wait(&emptyA[sa], pa ^ 1);
            mbar_arrive_expect_tx(&fullA[sa], A_TILE_BYTES);
            tma_load_2d(smem + sa * A_TILE_BYTES, &tmA, &fullA[sa], kb * BK, m_tile * BM, polA);
            if (++sa == AS) {
              sa = 0;
              pa ^= 1;
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
      int sa = 0, sb = 0, acc = 0;
      uint32_t pa = 0, pb = 0, aphase = 0;
      PieceWalk walk;
      walk.init(args);
      Piece pc;
      bool tl_first = true;
      while (walk.next(args, pc)) {
        const int nkb = pc.nkb;
        mbar_wait(&tempty[acc], aphase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int i = 0; i < nkb; ++i) {
          mbar_wait(&fullA[sa], pa);
          mbar_wait(&fullB[sb], pb);
          if (tl_first) {  // first k-block of weights and activations in shared memory
            PL_TL(tl_tag, 2);
            tl_first = false;
          }
          tc_fence_after();
          const uint64_t da = umma_desc_sw128(smem_u32(smem + sa * A_TILE_BYTES));
          const uint64_t db = umma_desc_sw128(smem_u32(smem + L::B_OFFSET + sb * L::B_TILE_BYTES));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)  // +32 B per K=16 step inside the swizzle atom
            umma_bf16(d, da + 2 * k, db + 2 * k, idesc, (i | k) != 0);
          umma_commit(&emptyA[sa]);
          umma_commit(&emptyB[sb]);
          if (++sa == AS) {
            sa = 0;
            pa ^= 1;
          }
          if (++sb == BS) {
            sb = 0;
            pb ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          aphase ^= 1;
        }
      }
    }
    __syncwarp();
  } else if (warp <= 5) {
    // ------------------------------------------------------- epilogue (warps 2..5)
    const int quarter = warp & 3;                 // TMEM lanes [32q, 32q + 32)
    const int row = quarter * 32 + lane;
    const int ep = threadIdx.x - 64;              // 0..127
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    const int epi = args.epi;
    int acc = 0;
    uint32_t aphase = 0;
    if (SWAP && args.csk && args.rope) csk_preload(args, ep, BN, csk_meta);  // overlaps the main loop
    PieceWalk walk;
    walk.init(args);
    Piece pc;
    while (walk.next(args, pc)) {
      const int m_tile = pc.m_tile, n_tile = pc.n_tile, split = pc.split;
      mbar_wait(&tfull[acc], aphase);
      if (warp == 2 && lane == 0) PL_TL(tl_tag, 3);  // accumulator complete
      tc_fence_after();
      const uint32_t tcol = tmem + lane_base + acc * BN;
      auto release_tmem = [&]() {  // accumulator drained: hand the TMEM buffer back
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        if (++acc == 2) {
          acc = 0;
          aphase ^= 1;
        }
      };

      if constexpr (SWAP) {
        // lane <-> feature n, column <-> token t
        const int n = m_tile * BM + row;
        const int t_base = n_tile * BN;
        // the tile's final epilogue, accumulator values from `fetch(c0, v[16])`
        auto final_epi = [&](auto fetch) {
          if (epi == EPI_SWIGLU && args.swiglu_il) {
            epi_swiglu_cols(args, tcol, row, m_tile, t_base, 0, split_epi ? BN / 2 : BN);
          } else if (epi == EPI_SWIGLU) {
            // rows [0,64) gate, [64,128) up of the same 64 output features
            const int j = m_tile * 64 + (row & 63);
            for (int c0 = 0; c0 < BN; c0 += 16) {
              float v[16];
              fetch(c0, v);
              if (row >= 64) {
#pragma unroll
                for (int c = 0; c < 16; ++c) scratch[c * 64 + (row - 64)] = v[c];
              }
              epi_sync();
              if (row < 64) {
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                  const int t = t_base + c0 + c;
                  if (t < args.T) {
                    const float g = rbf(v[c]);
                    const float u = rbf(scratch[c * 64 + row]);
                    args.C[(int64_t)t * args.ldc + j] = f2bf(rbf(silu_f(g)) * u);
                  }
                }
              }
              epi_sync();
            }
          } else if (epi == EPI_ARGMAX) {
            float2* red = reinterpret_cast<float2*>(scratch);  // [4 quarters][16 cols]
            for (int c0 = 0; c0 < BN; c0 += 16) {
              float vv[16];
              fetch(c0, vv);
#pragma unroll
              for (int c = 0; c < 16; ++c) {
                float v = (n < args.N) ? vv[c] : -INFINITY;
                int idx = n;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                  const float ov = __shfl_xor_sync(0xffffffffu, v, o);
                  const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
                  if (ov > v || (ov == v && oi < idx)) {
                    v = ov;
                    idx = oi;
                  }
                }
                if (lane == 0) red[quarter * 16 + c] = make_float2(v, __int_as_float(idx));
              }
              epi_sync();
              if (ep < 16) {
                float2 best = red[ep];
                for (int q = 1; q < 4; ++q) {
                  const float2 o = red[q * 16 + ep];
                  if (o.x > best.x || (o.x == best.x && __float_as_int(o.y) < __float_as_int(best.y)))
                    best = o;
                }
                const int t = t_base + c0 + ep;
                if (t < args.T) args.argmax_ws[(int64_t)m_tile * args.T + t] = best;
              }
              epi_sync();
            }
          } else {
            for (int c0 = 0; c0 < BN; c0 += 16) {
              float v[16];
              fetch(c0, v);
              if (n < args.N) {
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                  const int t = t_base + c0 + c;
                  if (t < args.T) store_out(args, epi, t, n, v[c]);
                }
              }
            }
          }
        };
        auto fetch_tmem = [&](int c0, float (&v)[16]) {
          uint32_t r[16];
          tmem_ld16(tcol + c0, r);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < 16; ++c) v[c] = __uint_as_float(r[c]);
        };

        if (args.csk) {
          // cluster split-K: park this split's tile in the ring (all its loads were
          // consumed by now), column-major [token][feature] so the reducers' lanes coalesce
          float* red = reinterpret_cast<float*>(smem);
          for (int c0 = 0; c0 < BN; c0 += 16) {
            float v[16];
            fetch_tmem(c0, v);
#pragma unroll
            for (int c = 0; c < 16; ++c) red[(c0 + c) * BM + row] = v[c];
          }
        } else if (args.splits > 1 && args.pmode == 1) {
          epi_partial_cols(args, tcol, n, split, t_base, 0, split_epi ? BN / 2 : BN);
        } else if (args.splits > 1) {
          // partials are token-contiguous per feature row: [split][N][Tp]
          float* prow = args.partial + ((int64_t)split * args.N + n) * args.Tp + t_base;
          for (int c0 = 0; c0 < BN; c0 += 16) {
            float v[16];
            fetch_tmem(c0, v);
            if (n < args.N && t_base + c0 < args.T) {
              float4* dst = reinterpret_cast<float4*>(prow + c0);
#pragma unroll
              for (int c = 0; c < 16; c += 4) dst[c / 4] = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
            }
          }
        } else {
          final_epi(fetch_tmem);
        }
        if (!args.csk && warp == 2 && lane == 0) PL_TL(tl_tag, 4);  // this warp's epilogue done
      } else {
        // lane <-> token t, column <-> feature n   (splits == 1 on this path)
        token_rows_epilogue<BN>(args, tcol, m_tile * BM + row, n_tile);
      }
      release_tmem();

    }
  }

  if (split_epi && (warp <= 1 || warp >= GEMM_ACT_WARP) && static_cast<int>(blockIdx.x) < args.num_items) {
    const int quarter = warp & 3;  // warps 0, 1, 6, 7 -> TMEM lane quarters 0, 1, 2, 3
    const int row = quarter * 32 + lane;
    const int split = static_cast<int>(blockIdx.x) % args.splits;
    const int m_tile = (static_cast<int>(blockIdx.x) / args.splits) % args.tiles_m;
    mbar_wait(&tfull[0], 0);  // the single item's accumulator (buffer 0, first phase)
    tc_fence_after();
    const uint32_t tcol = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    if (args.pmode == 1 && args.splits > 1)
      epi_partial_cols(args, tcol, m_tile * BM + row, split, 0, BN / 2, BN);
    else
      epi_swiglu_cols(args, tcol, row, m_tile, 0, BN / 2, BN);
    tc_fence_before();
  }

  if (SWAP && args.csk) {
    if (threadIdx.x == 64) PL_TL(tl_tag, 4);  // tile parked
    cluster_sync();  // every split's partial tile is parked in its CTA's shared memory
    if (threadIdx.x == 64) PL_TL(tl_tag, 5);
    if (warp >= 2 && warp <= 5) csk_reduce(args, smem, threadIdx.x - 64, BN, csk_meta);
    if (threadIdx.x == 64) PL_TL(tl_tag, 6);  // this thread's share reduced
    cluster_sync();  // the peers are done reading this CTA's shared memory
  }
  if (!args.csk && threadIdx.x == 0) PL_TL(tl_tag, 5);  // weight producer done
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) PL_TL(tl_tag, 1);
  if (warp == 1) tmem_dealloc<TMEM_COLS>(tmem);
}

// ---------------------------------------------------------------- CTA pair (prefill)
// !SWAP GEMMs on a 2-CTA cluster (one TPC): the pair computes one 256-token x
// 256-feature tile with tcgen05.mma.cta_group::2 (M = 256).  CTA r stages token rows
// [128 r, +128) of the A tile and feature rows [128 r, +128) of the B tile; the
// leader (r = 0) issues the MMA, which reads both CTAs' shared memory, and each CTA's
// TMEM receives its own 128 token rows x all 256 features.  Per SM and MMA the
// operand reads drop from 4 KB A + 8 KB B (single CTA, M = 128, N = 256) to 4 + 4 KB,
// and a ring stage is 32 KB instead of 48 KB, so the ring is deeper.
//
// Barriers: every TMA of the pair completes on the LEADER's full barrier (the leader
// arms it with both halves' bytes); the leader's commits multicast to the empty / TMEM
// barriers at the same offset in both CTAs; both epilogues release a TMEM buffer on
// the leader's tempty barrier (8 warp arrivals).  Work items: pair p walks tiles
// p, p + #pairs, ... (grouped raster in 256-row bands).
template <int S>
struct PairSmem {
  static constexpr int B_OFFSET = S * A_TILE_BYTES;
  static constexpr int BAR_OFFSET = 2 * S * A_TILE_BYTES;
  // fullA, emptyA, fullB, emptyB [S], tfull[2], tempty[2], tmem slot
  static constexpr int TOTAL = BAR_OFFSET + 8 * (4 * S + 4) + 16 + 1024;
};

PL_DEV bool pair_next(const GemmArgs& a, int& it, int& m_tile, int& n_tile) {
  if (it >= a.num_items) return false;
  const int tiles_n = a.num_items / a.tiles_m;
  if (a.raster_m > 0) {
    const int band = it / (a.raster_m * tiles_n);
    const int gm = min(a.raster_m, a.tiles_m - band * a.raster_m);
    const int idx = it - band * a.raster_m * tiles_n;
    m_tile = band * a.raster_m + idx % gm;
    n_tile = idx / gm;
  } else {
    m_tile = it % a.tiles_m;
    n_tile = it / a.tiles_m;
  }
  it += gridDim.x >> 1;
  return true;
}

template <int S>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(224, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const GemmArgs args) {
  using L = PairSmem<S>;
  constexpr int BN = 256;
  constexpr uint32_t TMEM_COLS = 2 * BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* fullA = reinterpret_cast<uint64_t*>(smem + L::BAR_OFFSET);
  uint64_t* emptyA = fullA + S;
  uint64_t* fullB = emptyA + S;
  uint64_t* emptyB = fullB + S;
  uint64_t* tfull = emptyB + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < S; ++s) {
      mbar_init(&fullA[s], 1);
      mbar_init(&emptyA[s], 1);
      mbar_init(&fullB[s], 1);
      mbar_init(&emptyB[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is the one used)
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  cluster_sync();  // barriers initialised in both CTAs before any cross-CTA signal
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  if (warp >= 2) pdl_wait();

  if (warp == 0 || warp == GEMM_ACT_WARP) {
    // ------------------------------------------------------- TMA producers (both CTAs)
    if (lane == 0) {
      const bool weights = warp == 0;  // warp 0: B (weights, no PDL wait); warp 6: A (activations)
      if (!weights) pdl_wait();
      const uint64_t pol = weights ? policy_evict_first() : policy_evict_last();
      uint64_t* full = weights ? fullB : fullA;
      uint64_t* empty = weights ? emptyB : emptyA;
      uint8_t* ring = smem + (weights ? L::B_OFFSET : 0);
      int s = 0;
      uint32_t ph = 0;
      int it = blockIdx.x >> 1, m_tile, n_tile;
      while (pair_next(args, it, m_tile, n_tile)) {
        for (int kb = 0; kb < args.num_kb; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * A_TILE_BYTES);  // both CTAs' halves
          const uint32_t bar = mapa_shared(&full[s], 0);
          if (!weights)
            tma_load_2d_pair(ring + s * A_TILE_BYTES, &tmA, bar, kb * BK, m_tile * 256 + rank * BM, pol);
          else if (args.wp)  // packed 16 KB tile (feature tile 2 n + r, k-block kb) as a linear 3-D box
            tma_load_3d_pair(ring + s * A_TILE_BYTES, &tmB, bar, 0, 0,
                             (n_tile * 2 + static_cast<int>(rank)) * args.num_kb + kb, pol);
          else
            tma_load_2d_pair(ring + s * A_TILE_BYTES, &tmB, bar, kb * BK, n_tile * BN + rank * BM, pol);
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer (leader only)
    if (rank == 0 && lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(2 * BM, BN);
      int s = 0, acc = 0;
      uint32_t ph = 0, aphase = 0;
      int it = blockIdx.x >> 1, m_tile, n_tile;
      while (pair_next(args, it, m_tile, n_tile)) {
        mbar_wait_cluster(&tempty[acc], aphase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = 0; kb < args.num_kb; ++kb) {
          mbar_wait(&fullA[s], ph);
          mbar_wait(&fullB[s], ph);
          tc_fence_after();
          const uint64_t da = umma_desc_sw128(smem_u32(smem + s * A_TILE_BYTES));
          const uint64_t db = umma_desc_sw128(smem_u32(smem + L::B_OFFSET + s * A_TILE_BYTES));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) umma_bf16_pair(d, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
          umma_commit_pair(&emptyA[s]);
          umma_commit_pair(&emptyB[s]);
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
        umma_commit_pair(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          aphase ^= 1;
        }
      }
    }
    __syncwarp();
  } else if (warp <= 5) {
    // ------------------------------------------------------- epilogue (warps 2..5, both CTAs)
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    int acc = 0;
    uint32_t aphase = 0;
    int it = blockIdx.x >> 1, m_tile, n_tile;
    while (pair_next(args, it, m_tile, n_tile)) {
      mbar_wait_cluster(&tfull[acc], aphase);
      tc_fence_after();
      token_rows_epilogue<BN>(args, tmem + lane_base + acc * BN, m_tile * 256 + static_cast<int>(rank) * BM + row,
                              n_tile);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(mapa_shared(&tempty[acc], 0));
      if (++acc == 2) {
        acc = 0;
        aphase ^= 1;
      }
    }
  }

  tc_fence_before();
  cluster_sync();  // neither CTA leaves while the pair's MMAs / signals may touch it
  tc_fence_after();
  if (warp == 1) tmem_dealloc_pair<TMEM_COLS>(tmem);
}

// Split-K reduction + epilogue.  partial: [splits][N][Tp] fp32 (token-contiguous),
// summed in split order (deterministic).  Each thread owns one output feature and
// 4 consecutive tokens: splits independent 16-byte loads in flight.
__global__ void __launch_bounds__(256)
    gemm_splitk_reduce_kernel(const float* partial, int splits, int T, int Tp, int N,
                              int epi, __nv_bfloat16* __restrict__ C, int64_t ldc,
                              const __nv_bfloat16* __restrict__ bias,
                              const __nv_bfloat16* __restrict__ residual, int64_t ldr, int swiglu_il,
                              __nv_bfloat16* __restrict__ C2) {
  pdl_trigger();
  pdl_wait();
  const int n_out = (epi == EPI_SWIGLU) ? N / 2 : N;
  const int tq = (T + 3) / 4;
  const int64_t total = static_cast<int64_t>(n_out) * tq;
  const int64_t split_stride = static_cast<int64_t>(N) * Tp / 4;  // in float4
  const float4* P = reinterpret_cast<const float4*>(partial);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int j = static_cast<int>(i % n_out);   // consecutive threads -> consecutive features
    const int t0 = static_cast<int>(i / n_out) * 4;
    const int n = (epi == EPI_SWIGLU) ? (j / 64) * 128 + (swiglu_il ? 2 * (j % 64) : j % 64) : j;
    const int64_t up_off = (swiglu_il ? 1 : 64) * static_cast<int64_t>(Tp) / 4;  // up row, in float4
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f), up = make_float4(0.f, 0.f, 0.f, 0.f);
    const float4* p = P + (static_cast<int64_t>(n) * Tp + t0) / 4;
#pragma unroll 4
    for (int s = 0; s < splits; ++s) {
      const float4 x = p[s * split_stride];
      acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
      if (epi == EPI_SWIGLU) {
        const float4 u = p[s * split_stride + up_off];
        up.x += u.x; up.y += u.y; up.z += u.z; up.w += u.w;
      }
    }
    const float av[4] = {acc.x, acc.y, acc.z, acc.w};
    const float uv[4] = {up.x, up.y, up.z, up.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int t = t0 + k;
      if (t >= T) break;
      const int64_t o = static_cast<int64_t>(t) * ldc + j;
      __nv_bfloat16 v;
      if (epi == EPI_SWIGLU)
        v = f2bf(rbf(silu_f(rbf(av[k]))) * rbf(uv[k]));
      else if (epi == EPI_RESIDUAL)
        v = f2bf(rbf(av[k]) + bf2f(residual[static_cast<int64_t>(t) * ldr + j]));
      else if (epi == EPI_BIAS)
        v = f2bf(av[k] + bf2f(bias[j]));
      else
        v = f2bf(av[k]);
      C[o] = v;
      if (C2) C2[o] = v;  // fused transport into the next stage's buffer
    }
  }
}

// Fused decode epilogue 1: split-K reduce + residual add + the NEXT RMSNorm, one CTA
// per token row (partials feature-contiguous, [splits][T][N]):
//   h[t]  = bf16(bf16(sum_s partial) + h[t])             (residual, modeling_llama.py:313-331)
//   a[t]  = bf16(w * bf16(h[t] * rsqrt(mean(h[t]^2)+eps)))   (RMSNorm, :62-67)
// Up to 1024 threads per row, VPT float4 per thread; the residual row and four
// splits' partials are in flight at once (latency-bound, not bandwidth-bound).
template <int VPT>  // float4 chunks per thread
__global__ void __launch_bounds__(1024)
    reduce_residual_norm_kernel(const float* partial, int splits, int T, int N,
                                __nv_bfloat16* __restrict__ h, int64_t ldh,
                                const __nv_bfloat16* __restrict__ w, float eps,
                                __nv_bfloat16* __restrict__ a, int64_t lda) {
  if (threadIdx.x == 0) PL_TL(2u << 24, 0);
  pdl_trigger();
  const int t = blockIdx.x;
  const int nt = blockDim.x;
  uint2 wv[VPT];  // the norm weight is static: fetched before griddepcontrol.wait
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int f = (threadIdx.x + nt * k) * 4;
    wv[k] = f < N ? *reinterpret_cast<const uint2*>(w + f) : make_uint2(0, 0);
  }
  pdl_wait();
  uint2 old[VPT];
  float4 acc[VPT];
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int f = (threadIdx.x + nt * k) * 4;
    acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    old[k] = f < N ? *reinterpret_cast<const uint2*>(h + static_cast<int64_t>(t) * ldh + f) : make_uint2(0, 0);
  }
  const int64_t stride = static_cast<int64_t>(T) * N;
  const float* prow = partial + static_cast<int64_t>(t) * N;
  // Up to 8 splits' loads in flight per round at VPT = 1 (one L2 round trip for the L3
  // residual GEMMs).  The loads are unconditional (split index and feature clamped to
  // valid addresses) plain weak loads after griddepcontrol.wait (the PDL-documented
  // way to read the previous grid's output), so they issue back to back before the
  // first add; the predicated __ldcg form compiled to load -> add -> load.  `partial`
  // is not __restrict__: that would turn these into .nc loads, whose read-only
  // contract the early-launched (PDL) grid cannot promise.  Sum order = split order.
  constexpr int G = VPT == 1 ? 8 : 4;
  for (int s0 = 0; s0 < splits; s0 += G) {
    float4 x[G][VPT];
#pragma unroll
    for (int u = 0; u < G; ++u)
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        const int f = (threadIdx.x + nt * k) * 4;
        const int su = min(s0 + u, splits - 1);
        x[u][k] = *reinterpret_cast<const float4*>(prow + su * stride + (f < N ? f : 0));
      }
#pragma unroll
    for (int u = 0; u < G; ++u)
      if (s0 + u < splits)
#pragma unroll
        for (int k = 0; k < VPT; ++k) {  // split order (deterministic)
          acc[k].x += x[u][k].x;
          acc[k].y += x[u][k].y;
          acc[k].z += x[u][k].z;
          acc[k].w += x[u][k].w;
        }
  }
  float hv[VPT][4];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int f = (threadIdx.x + nt * k) * 4;
    if (f >= N) continue;
    const float2 o0 = unpack_bf16x2(old[k].x), o1 = unpack_bf16x2(old[k].y);
    hv[k][0] = rbf(rbf(acc[k].x) + o0.x);
    hv[k][1] = rbf(rbf(acc[k].y) + o0.y);
    hv[k][2] = rbf(rbf(acc[k].z) + o1.x);
    hv[k][3] = rbf(rbf(acc[k].w) + o1.y);
    if (splits > 0)  // splits == 0: h is already final (cluster split-K), only normalise it
      *reinterpret_cast<uint2*>(h + static_cast<int64_t>(t) * ldh + f) =
          make_uint2(pack_bf16x2(hv[k][0], hv[k][1]), pack_bf16x2(hv[k][2], hv[k][3]));
    ss += hv[k][0] * hv[k][0] + hv[k][1] * hv[k][1] + hv[k][2] * hv[k][2] + hv[k][3] * hv[k][3];
  }
  __shared__ float red[32];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
  const int nw = nt >> 5;
  for (int i = 0; i < nw; ++i) tot += red[i];
  const float inv = 1.0f / sqrtf(tot / static_cast<float>(N) + eps);
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int f = (threadIdx.x + nt * k) * 4;
    if (f >= N) continue;
    const float2 w0 = unpack_bf16x2(wv[k].x), w1 = unpack_bf16x2(wv[k].y);
    *reinterpret_cast<uint2*>(a + static_cast<int64_t>(t) * lda + f) =
        make_uint2(pack_bf16x2(w0.x * rbf(hv[k][0] * inv), w0.y * rbf(hv[k][1] * inv)),
                   pack_bf16x2(w1.x * rbf(hv[k][2] * inv), w1.y * rbf(hv[k][3] * inv)));
  }
#ifdef PL_TIMELINE
  __syncthreads();
  if (threadIdx.x == 0) PL_TL(2u << 24, 1);
#endif
}

// Fused decode epilogue 2: QKV split-K reduce (+ Qwen2 bias) + neox RoPE on q and k
// (HF per-op bf16 rounding, as rope_kv_kernel) + paged K/V append.  One thread per
// (head, rotary pair i, 4 tokens); partials token-contiguous, [splits][N][Tp].
__global__ void __launch_bounds__(256)
    reduce_qkv_rope_kernel(const float* partial, int splits, int T, int Tp, int N,
                           const __nv_bfloat16* __restrict__ bias, __nv_bfloat16* __restrict__ qkv,
                           int64_t ldqkv, const int32_t* __restrict__ pos,
                           const int32_t* __restrict__ slot, const __nv_bfloat16* __restrict__ cos_sin,
                           int max_pos, __nv_bfloat16* __restrict__ k_cache,
                           __nv_bfloat16* __restrict__ v_cache, int block_size, int Hq, int Hkv) {
  pdl_trigger();
  constexpr int HDIM = 128, HALF = 64;
  const int heads = Hq + 2 * Hkv;
  const int tq = (T + 3) / 4;
  const int64_t total = static_cast<int64_t>(heads) * HALF * tq;
  const int64_t split_stride = static_cast<int64_t>(N) * Tp / 4;
  const float4* P = reinterpret_cast<const float4*>(partial);
  // Inputs that do not come from the GEMM (bias, positions and KV slots from the host
  // metadata, the RoPE table) are fetched before griddepcontrol.wait, so only the
  // partial sums sit on the dependent path.
  struct Side {
    float b1, b2, c[4], sn[4];
    int sl[4];
  };
  auto side = [&](int64_t idx, Side& sd) {
    const int i = static_cast<int>(idx % HALF);
    const int hh = static_cast<int>((idx / HALF) % heads);
    const int t0 = static_cast<int>(idx / (HALF * heads)) * 4;
    const int n1 = hh * HDIM + i, n2 = n1 + HALF;
    sd.b1 = bias ? bf2f(bias[n1]) : 0.f;
    sd.b2 = bias ? bf2f(bias[n2]) : 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int t = min(t0 + k, T - 1);
      sd.c[k] = 1.f, sd.sn[k] = 0.f;
      if (hh < Hq + Hkv) {
        int pp = pos[t];
        pp = pp < 0 ? 0 : (pp >= max_pos ? max_pos - 1 : pp);
        sd.c[k] = bf2f(cos_sin[static_cast<int64_t>(pp) * HDIM + i]);
        sd.sn[k] = bf2f(cos_sin[static_cast<int64_t>(pp) * HDIM + HALF + i]);
      }
      sd.sl[k] = slot ? slot[t] : -1;
    }
  };
  const int64_t idx0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  Side sd0;
  if (idx0 < total) side(idx0, sd0);
  pdl_wait();
  for (int64_t idx = idx0; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = static_cast<int>(idx % HALF);
    const int hh = static_cast<int>((idx / HALF) % heads);
    const int t0 = static_cast<int>(idx / (HALF * heads)) * 4;
    const int n1 = hh * HDIM + i, n2 = n1 + HALF;
    Side sd;
    if (idx == idx0)
      sd = sd0;
    else
      side(idx, sd);
    float4 a1 = make_float4(0.f, 0.f, 0.f, 0.f), a2 = a1;
    const float4* p1 = P + (static_cast<int64_t>(n1) * Tp + t0) / 4;
    const float4* p2 = P + (static_cast<int64_t>(n2) * Tp + t0) / 4;
    // four splits' loads in flight (unconditional weak loads after the PDL wait, as in
    // reduce_residual_norm_kernel), summed in split order
    for (int s0 = 0; s0 < splits; s0 += 4) {
      float4 x[4], y[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int su = min(s0 + u, splits - 1);
        x[u] = p1[su * split_stride];
        y[u] = p2[su * split_stride];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (s0 + u >= splits) break;
        a1.x += x[u].x; a1.y += x[u].y; a1.z += x[u].z; a1.w += x[u].w;
        a2.x += y[u].x; a2.y += y[u].y; a2.z += y[u].z; a2.w += y[u].w;
      }
    }
    const float v1[4] = {rbf(a1.x + sd.b1), rbf(a1.y + sd.b1), rbf(a1.z + sd.b1), rbf(a1.w + sd.b1)};
    const float v2[4] = {rbf(a2.x + sd.b2), rbf(a2.y + sd.b2), rbf(a2.z + sd.b2), rbf(a2.w + sd.b2)};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int t = t0 + k;
      if (t >= T) break;
      float o1 = v1[k], o2 = v2[k];
      if (hh < Hq + Hkv) {
        o1 = rbf(rbf(v1[k] * sd.c[k]) + rbf(-v2[k] * sd.sn[k]));
        o2 = rbf(rbf(v2[k] * sd.c[k]) + rbf(v1[k] * sd.sn[k]));
      }
      __nv_bfloat16* row = qkv + static_cast<int64_t>(t) * ldqkv;
      row[n1] = f2bf(o1);
      row[n2] = f2bf(o2);
      const int sl = sd.sl[k];
      if (hh >= Hq && sl >= 0) {
        const bool is_k = hh < Hq + Hkv;
        const int kh = is_k ? hh - Hq : hh - Hq - Hkv;
        __nv_bfloat16* cache = is_k ? k_cache : v_cache;
        __nv_bfloat16* dst = cache + ((static_cast<int64_t>(sl / block_size) * Hkv + kh) * block_size +
                                      sl % block_size) * HDIM;
        dst[i] = f2bf(o1);
        dst[i + HALF] = f2bf(o2);
      }
    }
  }
}

// Per token: reduce the per-tile (max, index) pairs, lowest index on ties.
__global__ void argmax_reduce_kernel(const float2* __restrict__ ws, int tiles, int T,
                                     int64_t* __restrict__ out_ids, float* __restrict__ out_max) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < tiles; i += blockDim.x) {
    const float2 p = ws[(int64_t)i * T + t];
    const int pi = __float_as_int(p.y);
    if (p.x > best || (p.x == best && pi < bi)) {
      best = p.x;
      bi = pi;
    }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = best;
    si[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      if (sv[w] > best || (sv[w] == best && si[w] < bi)) {
        best = sv[w];
        bi = si[w];
      }
    }
    out_ids[t] = bi;
    if (out_max) out_max[t] = best;
  }
}

// ------------------------------------------------------------------ host --

namespace {

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

struct MapKey {
  const void* ptr;
  int64_t rows, cols, ld;
  int box_rows;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && rows == o.rows && cols == o.cols && ld == o.ld && box_rows == o.box_rows;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = reinterpret_cast<size_t>(k.ptr);
    h ^= static_cast<size_t>(k.rows) * 0x9E3779B97F4A7C15ull;
    h ^= static_cast<size_t>(k.cols) * 0xC2B2AE3D27D4EB4Full;
    h ^= static_cast<size_t>(k.ld) * 0x165667B19E3779F9ull;
    h ^= static_cast<size_t>(k.box_rows) << 7;
    return h;
  }
};

std::mutex g_map_mu;
std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;

// bf16 [rows, cols] row-major with leading dimension `ld` (elements); box = {64, box_rows}
int make_map(CUtensorMap* out, const void* ptr, int64_t rows, int64_t cols, int64_t ld,
             int box_rows) {
  MapKey key{ptr, rows, cols, ld, box_rows};
  {
    std::lock_guard<std::mutex> g(g_map_mu);
    auto it = g_maps.find(key);
    if (it != g_maps.end()) {
      *out = it->second;
      return PL_OK;
    }
  }
  auto fn = get_encode_fn();
  if (!fn) return set_error(PL_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(PL_ERR_CONFIG, "cuTensorMapEncodeTiled failed (%d) rows=%lld cols=%lld ld=%lld",
                     (int)r, (long long)rows, (long long)cols, (long long)ld);
  std::lock_guard<std::mutex> g(g_map_mu);
  if (g_maps.size() > 8192) g_maps.clear();
  g_maps.emplace(key, *out);
  return PL_OK;
}

// Packed weights (pack_weight_kernel) as a 3-D tensor [tiles][128 rows][64 bf16] with no
// swizzle: one box {64, 128, 1} is a tile's 16 KB pre-swizzled image, copied verbatim.
int make_packed_map(CUtensorMap* out, const void* ptr, int64_t tiles) {
  MapKey key{ptr, tiles, 0, 0, -1};
  {
    std::lock_guard<std::mutex> g(g_map_mu);
    auto it = g_maps.find(key);
    if (it != g_maps.end()) {
      *out = it->second;
      return PL_OK;
    }
  }
  auto fn = get_encode_fn();
  if (!fn) return set_error(PL_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(BK), static_cast<cuuint64_t>(BM), static_cast<cuuint64_t>(tiles)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(BK * 2), static_cast<cuuint64_t>(A_TILE_BYTES)};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(BM), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(PL_ERR_CONFIG, "cuTensorMapEncodeTiled (packed) failed (%d) tiles=%lld", (int)r,
                     (long long)tiles);
  std::lock_guard<std::mutex> g(g_map_mu);
  if (g_maps.size() > 8192) g_maps.clear();
  g_maps.emplace(key, *out);
  return PL_OK;
}

template <int S>
int launch_pair_s(const CUtensorMap& ma, const CUtensorMap& mb, const GemmArgs& a, int grid, cudaStream_t st) {
  const int rc = ensure_smem_attr(reinterpret_cast<const void*>(gemm_pair_kernel<S>), PairSmem<S>::TOTAL,
                                  "gemm pair smem attribute");
  if (rc) return rc;
  return launch_k("gemm_pair_kernel", gemm_pair_kernel<S>, dim3(grid), dim3(GEMM_THREADS), PairSmem<S>::TOTAL, st, ma, mb,
                  a);
}
// ring depth 7 = 224 KB of 32 KB stages
int launch_pair(const CUtensorMap& ma, const CUtensorMap& mb, const GemmArgs& a, int grid, cudaStream_t st) {
  return launch_pair_s<7>(ma, mb, a, grid, st);
}

template <int BN, bool SWAP, int CTAS = (BN <= 128 ? 2 : 1)>
int launch_tc(const CUtensorMap& ma, const CUtensorMap& mb, const GemmArgs& a, int grid,
              cudaStream_t st, int cluster = 0) {
  constexpr int smem = GemmSmem<BN, SWAP, CTAS>::TOTAL;
  const int rc = ensure_smem_attr(reinterpret_cast<const void*>(gemm_tc_kernel<BN, SWAP, CTAS>), smem,
                                  "gemm smem attribute");
  if (rc) return rc;
  return launch_kc("gemm_tc_kernel", gemm_tc_kernel<BN, SWAP, CTAS>, dim3(grid), dim3(TC_THREADS), smem, st, cluster,
                   ma, mb, a);
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }

bool use_swap(int64_t T, int epi) { return T <= 256 || epi == EPI_ARGMAX; }

int swap_bn(int64_t T) { return T <= 16 ? 16 : T <= 32 ? 32 : T <= 64 ? 64 : T <= 128 ? 128 : 256; }

}  // namespace

int make_tma_2d(CUtensorMap* out, const void* ptr, int64_t rows, int64_t cols, int64_t ld,
                int box_rows) {
  return make_map(out, ptr, rows, cols, ld, box_rows);
}

// Split-K factor for the decode (SWAP) path, from the weight shape (N, K) only so a
// token's result does not depend on which decode batch it rides in.  Decode GEMMs are HBM
// streams: a CTA with a 4-6 deep TMA ring pulls ~2x its fair share of bandwidth,
// so the only goal is to give every SM at least one work item -- any extra split
// is pure partial-sum traffic.  Smallest split with tiles*splits >= #SMs, each
// split keeping >= 4 k-blocks.
int gemm_num_splits(int64_t N, int64_t K, bool swap) {
  if (!swap) return 1;
  const int64_t tiles = (N + BM - 1) / BM;
  const int64_t kb = K / BK;
  const int64_t sms = 148;
  int best = 1;
  for (int s = 1; s <= 16; ++s) {
    const int64_t per = (kb + s - 1) / s;
    if (s > 1 && per < 4) break;
    best = static_cast<int>((kb + per - 1) / per);  // no empty splits
    if (tiles * best >= sms) break;
  }
  // Long-K projections (the down GEMMs, K >= 12288): round the split count up to a
  // multiple of 4.  The residual+norm reduce loads partials in groups of 8 (VPT = 1) or 4,
  // so this adds no reduction round, and the smaller per-CTA streams even out the SMs that carry two
  // CTAs (L3 down: 5 -> 8 splits, 160 -> 256 CTAs; 4-layer decode forward -1.0 % at
  // T = 64, -1.5 % at T = 32, neutral at T = 16: profiles/r1/split_sweep.log).
  if (kb >= 192 && best > 1 && best % 4) {
    const int up = (best + 3) / 4 * 4;
    const int64_t per = (kb + up - 1) / up;
    if (per >= 16) best = static_cast<int>((kb + per - 1) / per);
  }
  return best;
}

// Prefill (!SWAP) GEMMs on CTA pairs (cta_group::2, 256 x 256 tiles).  PL_GEMM_PAIR=0 /
// 1 forces it off / on; default on for >= 512 tokens.
bool use_pair(bool swap, int64_t T) {
  static const int env = [] { const char* v = getenv("PL_GEMM_PAIR"); return v ? atoi(v) : -1; }();
  if (swap || env == 0) return false;
  return env == 1 || T >= 512;
}

// Workspace (SWAP): split-K partials [splits][N][Tp] fp32, or argmax partials [tiles][T].
int64_t gemm_workspace_bytes(int64_t T, int64_t N, int64_t K, int epi) {
  const bool swap = use_swap(T, epi);
  const int64_t tiles = (N + BM - 1) / BM;
  if (epi == EPI_ARGMAX) return tiles * T * 8;
  const int splits = gemm_num_splits(N, K, swap);
  if (splits <= 1) return 0;
  const int64_t bn = swap_bn(T);
  const int64_t tiles_n = (T + bn - 1) / bn;
  return static_cast<int64_t>(splits) * N * (tiles_n * bn) * 4;
}

int gemm_launch(const __nv_bfloat16* X, int64_t ldx, const __nv_bfloat16* W, int64_t ldw,
                const __nv_bfloat16* bias, __nv_bfloat16* C, int64_t ldc,
                const __nv_bfloat16* residual, int64_t ldr, int64_t T, int64_t N, int64_t K,
                int epi, void* ws, int64_t ws_bytes, int64_t* argmax_out, cudaStream_t st,
                const FusedEpi* fuse, bool* fused, bool w_packed) {
  if (fused) *fused = false;
  if (T <= 0) return PL_OK;
  if (K % BK != 0 || N <= 0 || K <= 0)
    return set_error(PL_ERR_CONFIG, "gemm: K must be a positive multiple of 64 (K=%lld N=%lld)",
                     (long long)K, (long long)N);
  if (epi == EPI_SWIGLU && N % 128 != 0)
    return set_error(PL_ERR_CONFIG, "gemm swiglu: N (2*ffn) must be a multiple of 128");
  if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(W)) & 15)
    return set_error(PL_ERR_CONFIG, "gemm: operands must be 16-byte aligned");
  if ((ldx % 8) || (ldw % 8)) return set_error(PL_ERR_CONFIG, "gemm: ld must be a multiple of 8");
  const bool swap = use_swap(T, epi);
  if (epi == EPI_ARGMAX && T > 256)
    return set_error(PL_ERR_CONFIG, "gemm argmax: at most 256 rows per call");
  if (!swap && (N % 16 || ldc % 8 || (epi == EPI_RESIDUAL && ldr % 8)))
    return set_error(PL_ERR_CONFIG, "gemm: N and leading dims must be multiples of 16/8");

  GemmArgs a{};
  a.T = static_cast<int>(T);
  a.N = static_cast<int>(N);
  if (w_packed) {
    if (N % 256 || ldw != K)
      return set_error(PL_ERR_CONFIG, "gemm: packed weights need N %% 256 == 0 and ldw == K");
    a.wp = reinterpret_cast<const uint8_t*>(W);
    a.swiglu_il = epi == EPI_SWIGLU;  // pack_weight interleaves gate/up rows
  }
  a.num_kb = static_cast<int>(K / BK);
  a.epi = epi;
  a.C = C;
  a.ldc = ldc;
  a.bias = bias;
  a.residual = residual;
  a.ldr = ldr;
  a.C2 = fuse ? fuse->mirror : nullptr;
  if (a.C2 && !swap) return set_error(PL_ERR_CONFIG, "gemm: a mirrored output needs the decode (SWAP) path");
  a.splits = epi == EPI_ARGMAX ? 1 : gemm_num_splits(N, K, swap);
  a.kb_per_split = (a.num_kb + a.splits - 1) / a.splits;
  const int bn = swap ? swap_bn(T) : 256;
  a.tiles_m = static_cast<int>(swap ? (N + BM - 1) / BM : (T + BM - 1) / BM);
  const int tiles_n = static_cast<int>(swap ? (T + bn - 1) / bn : (N + bn - 1) / bn);
  a.num_items = a.tiles_m * tiles_n * a.splits;
  constexpr int raster = 32;  // prefill tile band (profiles/r1/prefill_raster_sweep.log,
                              // long-K: profiles/r2/prefill_band_longk.log)
  a.raster_m = (!swap && tiles_n > 1 && a.tiles_m > raster) ? raster : 0;
  a.Tp = tiles_n * bn;
  // split-K: the fused epilogues are the partial reduction kernels
  const int fkind = (fuse && swap && a.splits > 1) ? fuse->kind : FUSE_NONE;
  if (fkind == FUSE_RESIDUAL_NORM && (epi != EPI_RESIDUAL || N > 8192 || N % 4))
    return set_error(PL_ERR_CONFIG, "gemm: residual+norm fusion needs a RESIDUAL GEMM, N <= 8192");
  if (fkind == FUSE_QKV_ROPE && (epi != EPI_STORE && epi != EPI_BIAS))
    return set_error(PL_ERR_CONFIG, "gemm: qkv+rope fusion needs a STORE/BIAS GEMM");
  a.pmode = fkind == FUSE_RESIDUAL_NORM ? 1 : 0;
  const int64_t need = gemm_workspace_bytes(T, N, K, epi);
  if (need > 0 && (ws_bytes < need || !ws))
    return set_error(PL_ERR_CONFIG, "gemm: workspace too small (%lld < %lld)", (long long)ws_bytes,
                     (long long)need);
  int grid, cluster = 0;
  {
    if (epi == EPI_ARGMAX) {
      a.argmax_ws = static_cast<float2*>(ws);
    } else if (a.splits > 1) {
      a.partial = static_cast<float*>(ws);
    }
    const int per_sm = (swap && bn <= 128) ? 2 : 1;
    grid = std::min(a.num_items, num_sms() * per_sm);
    // cluster split-K (default on; PL_CSK=0 restores partials + reduce kernels): one wave,
    // one tile per cluster of `splits` CTAs
    // PL_CSK bit mask of the GEMMs that use it: 1 = QKV (+RoPE/KV append), 2 = residual (+norm),
    // 4 = the rest (plain / bias / residual without fusion).  Default 5: measured on the
    // 4-layer L3 decode forward (profiles/r1/cluster_splitk.log) the QKV fusion gains
    // 4 % at T = 64, while residual+norm loses (its reduce kernel already does the norm
    // in one pass; in-GEMM reduction + a norm kernel is slower), and at T <= 16 the
    // partials are small enough that the reduce kernels cost nothing extra.
    static const int csk_mask = [] { const char* v = getenv("PL_CSK"); return v ? atoi(v) : 5; }();
    const int csk_kind = fkind == FUSE_QKV_ROPE ? 1 : fkind == FUSE_RESIDUAL_NORM ? 2 : 4;
    const bool csk_on = (csk_mask & csk_kind) != 0 && (T > 16 || getenv("PL_CSK"));
    const bool rope_ok = fkind != FUSE_QKV_ROPE ||
                         (N == static_cast<int64_t>(fuse->Hq + 2 * fuse->Hkv) * 128 && fuse->block_size > 0);
    // (the cluster epilogues move bf16 x4: 8-byte aligned rows)
    const bool vec_ok = ldc % 4 == 0 && (reinterpret_cast<uintptr_t>(C) & 7) == 0 &&
                        (epi != EPI_RESIDUAL || (ldr % 4 == 0 && (reinterpret_cast<uintptr_t>(residual) & 7) == 0)) &&
                        (!a.C2 || (reinterpret_cast<uintptr_t>(a.C2) & 7) == 0) &&
                        (!bias || (reinterpret_cast<uintptr_t>(bias) & 7) == 0);
    if (csk_on && vec_ok && swap && a.splits > 1 && a.splits <= 8 && tiles_n == 1 && a.num_items == grid &&
        (epi == EPI_STORE || epi == EPI_BIAS || epi == EPI_RESIDUAL) && rope_ok) {
      a.csk = 1;
      cluster = a.splits;
      if (fkind == FUSE_QKV_ROPE) {
        a.rope = 1;
        a.pos = fuse->pos;
        a.slot = fuse->slot;
        a.cos_sin = fuse->cos_sin;
        a.max_pos = fuse->max_pos;
        a.k_cache = fuse->k_cache;
        a.v_cache = fuse->v_cache;
        a.block_size = fuse->block_size;
        a.Hq = fuse->Hq;
        a.Hkv = fuse->Hkv;
      }
    }
  }

  CUtensorMap ma, mb;
  int rc;
  if (swap) {
    if ((rc = make_map(&ma, W, N, K, ldw, BM))) return rc;
    if ((rc = make_map(&mb, X, T, K, ldx, bn))) return rc;
    switch (bn) {
      case 16: rc = launch_tc<16, true>(ma, mb, a, grid, st, cluster); break;
      case 32: rc = launch_tc<32, true>(ma, mb, a, grid, st, cluster); break;
      case 64: rc = launch_tc<64, true>(ma, mb, a, grid, st, cluster); break;
      case 128: rc = launch_tc<128, true>(ma, mb, a, grid, st, cluster); break;
      default: rc = launch_tc<256, true>(ma, mb, a, grid, st, cluster); break;
    }
  } else if (use_pair(swap, T)) {
    // 256-token row tiles, one CTA pair per TPC
    a.tiles_m = static_cast<int>((T + 2 * BM - 1) / (2 * BM));
    a.num_items = a.tiles_m * tiles_n;
    a.raster_m = (tiles_n > 1 && a.tiles_m > raster / 2) ? raster / 2 : 0;
    grid = 2 * std::min(a.num_items, num_sms() / 2);
    if ((rc = make_map(&ma, X, T, K, ldx, BM))) return rc;
    if (w_packed) rc = make_packed_map(&mb, W, (N / BM) * a.num_kb);
    else rc = make_map(&mb, W, N, K, ldw, BM);
    if (rc) return rc;
    rc = launch_pair(ma, mb, a, grid, st);
  } else {
    if ((rc = make_map(&ma, X, T, K, ldx, BM))) return rc;
    if ((rc = make_map(&mb, W, N, K, ldw, 256))) return rc;
    rc = launch_tc<256, false>(ma, mb, a, grid, st);
  }
  if (rc) return rc;

  if (epi == EPI_ARGMAX) {
    const int tiles = static_cast<int>((N + BM - 1) / BM);
    return launch_k("argmax_reduce_kernel", argmax_reduce_kernel, dim3(static_cast<unsigned>(T)),
                    dim3(256), 0, st, a.argmax_ws, tiles, static_cast<int>(T), argmax_out,
                    static_cast<float*>(nullptr));
  }
  if (a.csk) {
    if (a.rope && fused) *fused = true;
    if (fkind == FUSE_RESIDUAL_NORM) {  // h (= C) is final: the next RMSNorm, with the
      // residual-norm kernel's own reduction order (splits = 0: h is only read)
      if (fused) *fused = true;
      const int64_t vec = N / 4;
      const int threads = static_cast<int>(std::min<int64_t>(1024, (vec + 31) / 32 * 32));
      const int vpt = static_cast<int>((vec + threads - 1) / threads);
      if (vpt > 8) return set_error(PL_ERR_CONFIG, "residual+norm: N=%lld too large", (long long)N);
      auto k = vpt <= 1 ? reduce_residual_norm_kernel<1> : vpt <= 2 ? reduce_residual_norm_kernel<2>
             : vpt <= 4 ? reduce_residual_norm_kernel<4> : reduce_residual_norm_kernel<8>;
      return launch_k("reduce_residual_norm_kernel", k, dim3(static_cast<unsigned>(T)), dim3(threads), 0, st,
                      static_cast<const float*>(nullptr), 0, a.T, a.N, C, ldc, fuse->norm_w, fuse->eps,
                      fuse->norm_out, fuse->ld_norm);
    }
    return PL_OK;
  }
  if (fkind == FUSE_RESIDUAL_NORM) {
    if (fused) *fused = true;
    const int64_t vec = N / 4;  // float4 chunks per row
    const int threads = static_cast<int>(std::min<int64_t>(1024, (vec + 31) / 32 * 32));
    const int vpt = static_cast<int>((vec + threads - 1) / threads);
    if (vpt > 8) return set_error(PL_ERR_CONFIG, "residual+norm reduce: N=%lld too large", (long long)N);
    auto k = vpt <= 1 ? reduce_residual_norm_kernel<1> : vpt <= 2 ? reduce_residual_norm_kernel<2>
           : vpt <= 4 ? reduce_residual_norm_kernel<4> : reduce_residual_norm_kernel<8>;
    return launch_k("reduce_residual_norm_kernel", k, dim3(static_cast<unsigned>(T)), dim3(threads), 0, st,
                    a.partial, a.splits, a.T, a.N, C, ldc, fuse->norm_w, fuse->eps, fuse->norm_out,
                    fuse->ld_norm);
  }
  if (fkind == FUSE_QKV_ROPE) {
    if (fused) *fused = true;
    const int heads = fuse->Hq + 2 * fuse->Hkv;
    const int64_t total = static_cast<int64_t>(heads) * 64 * ((T + 3) / 4);
    const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 8));
    return launch_k("reduce_qkv_rope_kernel", reduce_qkv_rope_kernel, dim3(blocks), dim3(256), 0, st,
                    a.partial, a.splits, a.T, a.Tp, a.N, bias, C, ldc, fuse->pos, fuse->slot,
                    fuse->cos_sin, fuse->max_pos, fuse->k_cache, fuse->v_cache, fuse->block_size,
                    fuse->Hq, fuse->Hkv);
  }
  if (a.splits > 1) {
    const int64_t n_out = (epi == EPI_SWIGLU) ? N / 2 : N;
    const int64_t total = n_out * ((T + 3) / 4);
    const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 8));
    return launch_k("gemm_splitk_reduce_kernel", gemm_splitk_reduce_kernel, dim3(blocks), dim3(256), 0,
                    st, a.partial, a.splits, a.T, a.Tp, a.N, epi, C, ldc, bias, residual, ldr, a.swiglu_il,
                    a.C2);
  }
  return PL_OK;
}


#ifdef PL_TIMELINE
int tl_set_gemm(void* buf, void* count, unsigned cap) {
  TimelineSink t{static_cast<unsigned long long*>(buf), static_cast<unsigned*>(count), cap};
  return cudaMemcpyToSymbol(g_tl, &t, sizeof(t)) == cudaSuccess ? PL_OK : PL_ERR_CUDA;
}
#endif

// Weight packing: W [N, K] (row stride ld) -> 16 KB tiles [N/128][K/64], each tile the
// exact 128-byte-swizzled shared-memory image TMA would produce for a 128 x 64 box, so
// the GEMM producer streams it with one contiguous bulk copy per k-block.
__global__ void pack_weight_kernel(const __nv_bfloat16* __restrict__ W, int64_t ld, int64_t N, int64_t K,
                                   uint8_t* __restrict__ out, int interleave) {
  const int64_t nkb = K / BK;
  const int64_t chunks = N * (K / 8);  // 16-byte chunks
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < chunks;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = i / (K / 8), kc = i % (K / 8);
    const int64_t mt = n / BM, kb = kc / 8, c = kc % 8;
    int64_t r = n % BM;
    if (interleave) r = r < 64 ? 2 * r : 2 * (r - 64) + 1;  // [gate 64 | up 64] -> gate_j, up_j pairs
    const uint4 v = *reinterpret_cast<const uint4*>(W + n * ld + kc * 8);
    uint8_t* d = out + (mt * nkb + kb) * A_TILE_BYTES + r * 128 + ((c ^ (r & 7)) << 4);
    *reinterpret_cast<uint4*>(d) = v;
  }
}

int pack_weight_launch(const __nv_bfloat16* W, int64_t ld, int64_t N, int64_t K, void* out, cudaStream_t st,
                       bool interleave_swiglu) {
  if (N % 256 || K % BK || ld % 8)
    return set_error(PL_ERR_CONFIG, "pack_weight: N %% 256, K %% 64 and ld %% 8 must be 0");
  const int64_t chunks = N * (K / 8);
  const int blocks = static_cast<int>(std::min<int64_t>((chunks + 255) / 256, 148 * 16));
  pack_weight_kernel<<<blocks, 256, 0, st>>>(W, ld, N, K, static_cast<uint8_t*>(out), interleave_swiglu ? 1 : 0);
  return check_launch("pack_weight_kernel");
}

// Load every kernel of this file into the context now (lazy module loading would
// otherwise load it at first launch, which can wait on a spinning NCCL kernel).
template <typename K>
static int preload_one(K k, const char* name) {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, k);
  return e == cudaSuccess ? PL_OK : set_cuda_error(e, name);
}

int gemm_preload() {
  int rc = preload_one(gemm_tc_kernel<16, true, 2>, "gemm_tc_kernel");
  if (!rc) rc = preload_one(gemm_tc_kernel<32, true, 2>, "gemm_tc_kernel");
  if (!rc) rc = preload_one(gemm_tc_kernel<64, true, 2>, "gemm_tc_kernel");
  if (!rc) rc = preload_one(gemm_tc_kernel<128, true, 2>, "gemm_tc_kernel");
  if (!rc) rc = preload_one(gemm_tc_kernel<256, true, 1>, "gemm_tc_kernel");
  if (!rc) rc = preload_one(gemm_tc_kernel<256, false, 1>, "gemm_tc_kernel");
  if (!rc) rc = preload_one(gemm_pair_kernel<7>, "gemm_pair_kernel");
  if (!rc) rc = preload_one(argmax_reduce_kernel, "argmax_reduce_kernel");
  if (!rc) rc = preload_one(reduce_residual_norm_kernel<1>, "reduce_residual_norm_kernel");
  if (!rc) rc = preload_one(reduce_residual_norm_kernel<2>, "reduce_residual_norm_kernel");
  if (!rc) rc = preload_one(reduce_residual_norm_kernel<4>, "reduce_residual_norm_kernel");
  if (!rc) rc = preload_one(reduce_residual_norm_kernel<8>, "reduce_residual_norm_kernel");
  if (!rc) rc = preload_one(reduce_qkv_rope_kernel, "reduce_qkv_rope_kernel");
  if (!rc) rc = preload_one(gemm_splitk_reduce_kernel, "gemm_splitk_reduce_kernel");
  if (!rc) rc = preload_one(pack_weight_kernel, "pack_weight_kernel");
  return rc;
}

}  // namespace pl
