// Persistent decode-layer kernel: one launch streams every dense projection of a
// decoder layer (sm_100a).
//
// A decode micro-batch of T <= 256 tokens is a weight stream: per Llama-3-8B layer
// 436 MB of weights against T x 4096 activations.  Issued as one GEMM kernel per
// projection (plus the split-K reduce / residual-norm kernels), every launch pays a
// fill and a drain on 148 SMs, and the small projections (o: 33.5 MB, qkv: 50 MB)
// never reach HBM rate (r1: o_proj 29 %, qkv 33 % of peak).  Here ONE persistent
// launch per layer walks the chain
//
//     o-proj (+residual) -> RMSNorm -> gate_up (+SwiGLU) -> down (+residual) -> RMSNorm
//     -> next layer's qkv (+bias, RoPE, paged K/V append)
//
// with the weights of every projection flowing through one shared-memory ring
// continuously: a CTA's weight producer never waits for activations, so the next
// projection's weights are already in flight while the previous one drains.  Data
// dependencies are tracked in global memory instead of kernel boundaries:
//
//   gate_up  needs all of RMSNorm(h) -> a global norm step (every CTA normalises a
//            slice once all o tiles are in: per-tile sums of squares, fixed order)
//   down     k-block j needs SwiGLU columns [64 j, +64) = gate_up tile j (per-tile flag)
//   qkv      needs RMSNorm(h) after all down tiles -> the second norm step
//
// Work units are (projection, 128-row weight tile, k-range); the per-CTA unit lists
// are built on the host by list scheduling (chain_plan) from the weight shapes only,
// so a token's result never depends on T or on the batch.  Split-K partials go to a
// global fp32 buffer; the last split to arrive sums all of them in split order.
//
// Roles (224 threads): warp 0 lane 0 weight producer (1-D bulk copies of the packed
// 16 KB tiles), warp 6 lane 0 activation producer (TMA, after the dependency of each
// unit), warp 1 TMEM allocation + MMA issue (tcgen05.mma kind::f16, M = 128 weight
// rows, N = BN tokens, double-buffered fp32 accumulators in TMEM), warps 2-5 epilogue
// (partials, last-arriver reduction, residual / SwiGLU / RoPE + K/V epilogues, norm
// steps).  Rounding points follow HF modeling_llama.py exactly as gemm_tc.cu does.
#include <cstdio>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "pl_internal.h"

namespace pl {

namespace {

constexpr int CH_THREADS = 224;
constexpr int CH_ACT_WARP = 6;
constexpr int CBM = 128;
constexpr int CBK = 64;
constexpr int W_TILE = CBM * CBK * 2;  // 16 KB packed weight tile
constexpr int CH_BUDGET = 196 * 1024;

template <int BN>
struct ChainSmem {
  static constexpr int B_TILE = BN * CBK * 2;
  static constexpr int BS = BN <= 64 ? 4 : (BN == 128 ? 3 : 2);
  static constexpr int AS = (CH_BUDGET - BS * B_TILE) / W_TILE;
  static constexpr int B_OFF = AS * W_TILE;
  static constexpr int XCH_OFF = B_OFF + BS * B_TILE;        // rope exchange [16][128] fp32
  static constexpr int RED_OFF = XCH_OFF + 16 * CBM * 4;     // ss reduce [4][16] fp32
  static constexpr int RR_OFF = RED_OFF + 4 * 16 * 4;        // 1 / rms per token [256]
  static constexpr int BAR_OFF = RR_OFF + 256 * 4;
  static constexpr int TOTAL = BAR_OFF + 8 * (2 * AS + 2 * BS + 4) + 16 + 1024;
  static_assert(AS >= 4, "weight ring too shallow");
};

PL_DEV float ch_silu(float x) { return x / (1.0f + expf(-x)); }
PL_DEV void ch_epi_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
PL_DEV float ldcg_f(const float* p) { return __ldcg(p); }
PL_DEV unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
PL_DEV int ld_acquire_s32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
PL_DEV void st_release_s32(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
PL_DEV int atom_add_acq_rel(int* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
PL_DEV void red_add_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// generic-proxy writes of other CTAs (acquired above) -> this thread's TMA reads
PL_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// bounded spin: a protocol bug surfaces as a trap instead of a hung GPU
template <typename F>
PL_DEV void spin_until(F ready) {
  if (ready()) return;
  const uint64_t t0 = globaltimer_ns();
  while (!ready()) {
    __nanosleep(64);
    if (globaltimer_ns() - t0 > 4000000000ull) __trap();
  }
}

}  // namespace

struct ChainJob {
  const uint8_t* w;    // packed weight tiles [tiles][num_kb] x 16 KB
  float* partial;      // split-K partials [splits][tiles][Tp][128] fp32
  int* arrive;         // per-tile arrival counters, zero between launches
  int kind, dep, tiles, num_kb, splits, kb_per_split, act;
};

struct ChainArgs {
  int T, Tp, njobs, d, ffn;
  ChainJob job[4];
  const int4* units;      // {job, tile, kb0, nkb}
  const int* unit_off;    // CTA c owns units [unit_off[c], unit_off[c + 1])
  __nv_bfloat16* h;       // residual stream [T, d]
  __nv_bfloat16* a;       // normalised activations [T, d]
  __nv_bfloat16* m;       // SwiGLU output [T, ffn]
  __nv_bfloat16* q_out;   // roped q rows [T, ld_q] (the attention's q operand)
  int64_t ld_q;
  float* ss;              // per-tile sums of squares [2][d / 128][Tp]
  const __nv_bfloat16* norm_w[2];
  int has_norm[2];
  float eps;
  const __nv_bfloat16* bias;  // qkv bias (Qwen2) or null
  const int32_t* pos;
  const int32_t* slot;
  const __nv_bfloat16* cos_sin;
  int max_pos;
  __nv_bfloat16* k_cache;
  __nv_bfloat16* v_cache;
  int block_size, Hq, Hkv;
  unsigned long long* ctr;  // monotone: [0] o tiles, [1] norm-A CTAs, [2] down tiles, [3] norm-B CTAs
  unsigned long long tgt[4];  // values the counters reach when this launch's steps are done
  int* gu_flag;             // per gate_up tile: sequence number of the launch that finished it
  int seq;
};

template <int BN>
__global__ void __launch_bounds__(CH_THREADS, 1)
    chain_kernel(const __grid_constant__ CUtensorMap tm0, const __grid_constant__ CUtensorMap tm1,
                 const __grid_constant__ CUtensorMap tm2, const __grid_constant__ ChainArgs args) {
  using L = ChainSmem<BN>;
  constexpr int AS = L::AS, BS = L::BS;
  constexpr uint32_t TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* fullA = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* emptyA = fullA + AS;
  uint64_t* fullB = emptyA + AS;
  uint64_t* emptyB = fullB + BS;
  uint64_t* tfull = emptyB + BS;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* flag = reinterpret_cast<int*>(tmem_slot + 1);
  float* xch = reinterpret_cast<float*>(smem + L::XCH_OFF);
  float* red = reinterpret_cast<float*>(smem + L::RED_OFF);
  float* rr = reinterpret_cast<float*>(smem + L::RR_OFF);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u0 = args.unit_off[blockIdx.x], u1 = args.unit_off[blockIdx.x + 1];

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tm0);
    tma_prefetch_desc(&tm1);
    tma_prefetch_desc(&tm2);
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

  if (warp == 0) {
    // --------------------------------------------------- weight producer: never waits
    // for activations, so the next projection's weights stream while this one drains
    if (lane == 0) {
      int sa = 0;
      uint32_t pa = 0;
      for (int u = u0; u < u1; ++u) {
        const int4 un = args.units[u];
        const ChainJob& J = args.job[un.x];
        const uint8_t* src = J.w + (static_cast<int64_t>(un.y) * J.num_kb + un.z) * W_TILE;
        for (int i = 0; i < un.w; ++i) {
          mbar_wait(&emptyA[sa], pa ^ 1);
          mbar_arrive_expect_tx(&fullA[sa], W_TILE);
          bulk_load(smem + sa * W_TILE, src + static_cast<int64_t>(i) * W_TILE, W_TILE, &fullA[sa]);
          if (++sa == AS) sa = 0, pa ^= 1;
        }
      }
    }
    __syncwarp();
  } else if (warp == CH_ACT_WARP) {
    // --------------------------------------------------- activation producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_last();
      int sb = 0;
      uint32_t pb = 0;
      pdl_wait();  // o_attn / a come from the previous kernels
      for (int u = u0; u < u1; ++u) {
        const int4 un = args.units[u];
        const ChainJob& J = args.job[un.x];
        if (J.dep == 1 || J.dep == 3) {
          const unsigned long long* c = args.ctr + J.dep;
          const unsigned long long tg = args.tgt[J.dep];
          spin_until([&] { return ld_acquire_u64(c) >= tg; });
          fence_proxy_async_global();
        }
        const CUtensorMap* tm = J.act == 0 ? &tm0 : (J.act == 1 ? &tm1 : &tm2);
        for (int i = 0; i < un.w; ++i) {
          const int kb = un.z + i;
          if (J.dep == 2) {  // SwiGLU columns [64 kb, +64) = gate_up tile kb
            const int* f = args.gu_flag + kb;
            const int sq = args.seq;
            if (ld_acquire_s32(f) < sq) spin_until([&] { return ld_acquire_s32(f) >= sq; });
            fence_proxy_async_global();
          }
          mbar_wait(&emptyB[sb], pb ^ 1);
          mbar_arrive_expect_tx(&fullB[sb], L::B_TILE);
          tma_load_2d(smem + L::B_OFF + sb * L::B_TILE, tm, &fullB[sb], kb * CBK, 0, pol);
          if (++sb == BS) sb = 0, pb ^= 1;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // --------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(CBM, BN);
      int sa = 0, sb = 0, acc = 0;
      uint32_t pa = 0, pb = 0, aphase = 0;
      for (int u = u0; u < u1; ++u) {
        const int nkb = args.units[u].w;
        mbar_wait(&tempty[acc], aphase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int i = 0; i < nkb; ++i) {
          mbar_wait(&fullA[sa], pa);
          mbar_wait(&fullB[sb], pb);
          tc_fence_after();
          const uint64_t da = umma_desc_sw128(smem_u32(smem + sa * W_TILE));
          const uint64_t db = umma_desc_sw128(smem_u32(smem + L::B_OFF + sb * L::B_TILE));
#pragma unroll
          for (int k = 0; k < CBK / 16; ++k) umma_bf16(d, da + 2 * k, db + 2 * k, idesc, (i | k) != 0);
          umma_commit(&emptyA[sa]);
          umma_commit(&emptyB[sb]);
          if (++sa == AS) sa = 0, pa ^= 1;
          if (++sb == BS) sb = 0, pb ^= 1;
        }
        umma_commit(&tfull[acc]);
        if (++acc == 2) acc = 0, aphase ^= 1;
      }
    }
    __syncwarp();
  } else {
    // --------------------------------------------------- epilogue (warps 2..5)
    pdl_wait();
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;  // TMEM lane <-> weight row of the tile
    const int ep = threadIdx.x - 64;      // 0..127
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    const int T = args.T, Tp = args.Tp, d = args.d;
    const int dtiles = d / CBM;
    int acc = 0;
    uint32_t aphase = 0;
    bool done_norm[2] = {false, false};

    // Global RMSNorm step w (0: after the o tiles, 1: after the down tiles): once every
    // tile of the producing projection is in, 1/rms per token from the per-tile sums of
    // squares (summed in tile order), then this CTA's slice of a = norm(h) * w.
    auto norm_step = [&](int w) {
      if (ep == 0) {
        const unsigned long long* c = args.ctr + 2 * w;
        const unsigned long long tg = args.tgt[2 * w];
        spin_until([&] { return ld_acquire_u64(c) >= tg; });
      }
      ch_epi_sync();
      const float* ssw = args.ss + static_cast<int64_t>(w) * dtiles * Tp;
      for (int t = ep; t < T; t += 128) {
        float s = 0.f;
        for (int i = 0; i < dtiles; ++i) s += ldcg_f(ssw + static_cast<int64_t>(i) * Tp + t);
        rr[t] = rsqrtf(s / static_cast<float>(d) + args.eps);
      }
      ch_epi_sync();
      const int64_t nvec = static_cast<int64_t>(T) * d / 8;
      const int64_t per = (nvec + gridDim.x - 1) / gridDim.x;
      const int64_t v0 = blockIdx.x * per, v1 = min(nvec, v0 + per);
      const __nv_bfloat16* wn = args.norm_w[w];
      for (int64_t v = v0 + ep; v < v1; v += 128) {
        const int64_t e = v * 8;
        const int t = static_cast<int>(e / d), k = static_cast<int>(e % d);
        const uint4 x = __ldcg(reinterpret_cast<const uint4*>(args.h + e));
        const uint4 g = *reinterpret_cast<const uint4*>(wn + k);
        const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, gs[4] = {g.x, g.y, g.z, g.w};
        uint32_t o[4];
        const float r = rr[t];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 xv = unpack_bf16x2(xs[j]), gv = unpack_bf16x2(gs[j]);
          o[j] = pack_bf16x2(gv.x * rbf(xv.x * r), gv.y * rbf(xv.y * r));
        }
        *reinterpret_cast<uint4*>(args.a + e) = make_uint4(o[0], o[1], o[2], o[3]);
      }
      __threadfence();
      ch_epi_sync();
      if (ep == 0) red_add_release_u64(args.ctr + 2 * w + 1, 1ull);
      done_norm[w] = true;
    };

    for (int u = u0; u < u1; ++u) {
      const int4 un = args.units[u];
      const ChainJob& J = args.job[un.x];
      if (J.dep >= 1 && args.has_norm[0] && !done_norm[0]) norm_step(0);
      if (J.dep >= 3 && args.has_norm[1] && !done_norm[1]) norm_step(1);
      const int tile = un.y;
      const int split = un.z / J.kb_per_split;
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      const uint32_t tcol = tmem + lane_base + acc * BN;
      auto release_tmem = [&]() {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        if (++acc == 2) acc = 0, aphase ^= 1;
      };
      auto fetch_tmem = [&](int c0, float (&v)[16]) {
        uint32_t r[16];
        tmem_ld16(tcol + c0, r);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 16; ++c) v[c] = __uint_as_float(r[c]);
      };

      if (J.kind == 1) {
        // ---- gate_up, whole K in one unit: SwiGLU straight from TMEM.  Packed rows
        // alternate (gate_j, up_j), so lane pairs meet by one shuffle.
        const int j = tile * 64 + (row >> 1);
        for (int c0 = 0; c0 < BN && c0 < T; c0 += 16) {
          float v[16];
          fetch_tmem(c0, v);
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const float other = __shfl_xor_sync(0xffffffffu, v[c], 1);
            const int t = c0 + c;
            if (!(row & 1) && t < T)
              args.m[static_cast<int64_t>(t) * args.ffn + j] = f2bf(rbf(ch_silu(rbf(v[c]))) * rbf(other));
          }
        }
        release_tmem();
        __threadfence();
        ch_epi_sync();
        if (ep == 0) st_release_s32(args.gu_flag + tile, args.seq);
        continue;
      }

      // ---- split-K projections: this split's fp32 partial, then the last arriver
      float* pbase = J.partial + static_cast<int64_t>(tile) * Tp * CBM + row;
      const int64_t split_stride = static_cast<int64_t>(J.tiles) * Tp * CBM;
      if (J.splits > 1) {
        float* p = pbase + split * split_stride;
        for (int c0 = 0; c0 < BN && c0 < T; c0 += 16) {
          float v[16];
          fetch_tmem(c0, v);
#pragma unroll
          for (int c = 0; c < 16; ++c)
            if (c0 + c < T) __stcg(p + static_cast<int64_t>(c0 + c) * CBM, v[c]);
        }
        release_tmem();
        __threadfence();
        ch_epi_sync();
        if (ep == 0) {
          const int old = atom_add_acq_rel(J.arrive + tile, 1);
          const bool last = old == J.splits - 1;
          if (last) J.arrive[tile] = 0;  // stays zero between launches
          *flag = last;
        }
        ch_epi_sync();
        if (!*flag) continue;
      }
      // split-ordered sum of every split's partial (bit-identical whoever arrives last)
      auto fetch_sum = [&](int c0, float (&v)[16]) {
        if (J.splits == 1) {
          fetch_tmem(c0, v);
          return;
        }
#pragma unroll
        for (int c = 0; c < 16; ++c) v[c] = 0.f;
        const int S = J.splits;
        for (int s0 = 0; s0 < S; s0 += 4) {
          float x[4][16];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int s = min(s0 + q, S - 1);
            const float* p = pbase + s * split_stride + static_cast<int64_t>(c0) * CBM;
#pragma unroll
            for (int c = 0; c < 16; ++c) x[q][c] = ldcg_f(p + min(c, T - 1 - c0) * CBM);  // clamped: no predicated loads
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (s0 + q >= S) break;
#pragma unroll
            for (int c = 0; c < 16; ++c) v[c] += x[q][c];
          }
        }
      };

      if (J.kind == 0 || J.kind == 2) {
        // ---- o / down: residual add into h, per-token sum of squares of the new rows
        const int n = tile * CBM + row;
        float* ssw = args.ss + static_cast<int64_t>(J.kind == 2) * dtiles * Tp + static_cast<int64_t>(tile) * Tp;
        for (int c0 = 0; c0 < BN && c0 < T; c0 += 16) {
          float v[16];
          fetch_sum(c0, v);
          float sq[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const int t = c0 + c;
            sq[c] = 0.f;
            if (t < T) {
              __nv_bfloat16* hp = args.h + static_cast<int64_t>(t) * d + n;
              // L2 read: h rows were written by other CTAs earlier in this launch
              const unsigned short hr = __ldcg(reinterpret_cast<const unsigned short*>(hp));
              const __nv_bfloat16 hn = f2bf(rbf(v[c]) + bf2f(__ushort_as_bfloat16(hr)));
              *hp = hn;
              const float f = bf2f(hn);
              sq[c] = f * f;
            }
          }
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const float s = warp_sum(sq[c]);
            if (lane == 0) red[quarter * 16 + c] = s;
          }
          ch_epi_sync();
          if (ep < 16 && c0 + ep < T) ssw[c0 + ep] = ((red[ep] + red[16 + ep]) + red[32 + ep]) + red[48 + ep];
          ch_epi_sync();
        }
        if (J.splits == 1) release_tmem();
        __threadfence();
        ch_epi_sync();
        if (ep == 0) red_add_release_u64(args.ctr + (J.kind == 2 ? 2 : 0), 1ull);
        continue;
      }

      // ---- qkv (kind 3): bias, neox RoPE on q / k heads, paged K/V append; a 128-row
      // tile is one head, rows i and i + 64 rotate together (exchanged in shared memory)
      {
        const int hh = tile;
        const int n = hh * CBM + row;
        const float b = args.bias ? bf2f(args.bias[n]) : 0.f;
        const bool roped = hh < args.Hq + args.Hkv;
        const int i = row & 63;
        for (int c0 = 0; c0 < BN && c0 < T; c0 += 16) {
          float v[16];
          fetch_sum(c0, v);
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            v[c] = rbf(v[c] + b);
            xch[c * CBM + row] = v[c];
          }
          ch_epi_sync();
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const int t = c0 + c;
            if (t >= T) continue;
            float o = v[c];
            if (roped) {
              int pp = args.pos[t];
              pp = pp < 0 ? 0 : (pp >= args.max_pos ? args.max_pos - 1 : pp);
              const float cs = bf2f(args.cos_sin[static_cast<int64_t>(pp) * CBM + i]);
              const float sn = bf2f(args.cos_sin[static_cast<int64_t>(pp) * CBM + 64 + i]);
              const float partner = xch[c * CBM + (row ^ 64)];
              o = row < 64 ? rbf(rbf(v[c] * cs) + rbf(-partner * sn)) : rbf(rbf(v[c] * cs) + rbf(partner * sn));
            }
            if (hh < args.Hq) {
              args.q_out[static_cast<int64_t>(t) * args.ld_q + n] = f2bf(o);
            } else {
              const int sl = args.slot ? args.slot[t] : -1;
              if (sl >= 0) {
                const bool is_k = hh < args.Hq + args.Hkv;
                const int kh = is_k ? hh - args.Hq : hh - args.Hq - args.Hkv;
                __nv_bfloat16* cache = is_k ? args.k_cache : args.v_cache;
                cache[((static_cast<int64_t>(sl / args.block_size) * args.Hkv + kh) * args.block_size +
                       sl % args.block_size) * CBM + row] = f2bf(o);
              }
            }
          }
          ch_epi_sync();
        }
        if (J.splits == 1) release_tmem();
      }
    }
    if (args.has_norm[0] && !done_norm[0]) norm_step(0);
    if (args.has_norm[1] && !done_norm[1]) norm_step(1);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<TMEM_COLS>(tmem);
}

// ------------------------------------------------------------------ host

namespace {

// Unit lists by list scheduling on a fluid model of the weight stream: every CTA
// streams 1 k-block per time unit; a unit finishes at
//   max(cta free + nkb, ready + max(0, nkb - ring))
// (weights prefetch into the ring while its activations are not ready yet).  Units
// go, projection by projection (down units in k order, so early down work needs
// early gate_up tiles), to the CTA that finishes them first.  Depends only on the
// weight shapes and the SM count -- never on T.
struct PlanJob {
  int kind, dep, tiles, num_kb, splits;
};

double simulate(const std::vector<PlanJob>& jobs, int grid, int ring, std::vector<std::vector<int4>>* out) {
  std::vector<double> freet(grid, 0.0);
  if (out) out->assign(grid, {});
  std::vector<double> gu_done;
  double done_prev[4] = {0, 0, 0, 0};  // finish time of each job
  double norm_a = 0, norm_b = 0;
  constexpr double kRed = 0.5, kNorm = 1.5;
  for (int j = 0; j < static_cast<int>(jobs.size()); ++j) {
    const PlanJob& J = jobs[j];
    const int per = (J.num_kb + J.splits - 1) / J.splits;
    struct U {
      int tile, kb0, nkb;
    };
    std::vector<U> units;
    for (int t = 0; t < J.tiles; ++t)
      for (int s = 0; s < J.splits; ++s) {
        const int k0 = s * per, n = std::min(J.num_kb, k0 + per) - k0;
        if (n > 0) units.push_back({t, k0, n});
      }
    if (J.dep == 2)
      std::stable_sort(units.begin(), units.end(), [](const U& a, const U& b) { return a.kb0 < b.kb0; });
    std::vector<double> tile_fin(J.tiles, 0.0);
    for (const U& un : units) {
      double ready = 0;
      if (J.dep == 1) ready = norm_a;
      if (J.dep == 3) ready = norm_b;
      if (J.dep == 2)
        for (int k = un.kb0; k < un.kb0 + un.nkb; ++k) ready = std::max(ready, gu_done[k]);
      int best = 0;
      double bf = 1e300;
      for (int c = 0; c < grid; ++c) {
        const double f = std::max(freet[c] + un.nkb, ready + std::max(0, un.nkb - ring));
        if (f < bf - 1e-9) bf = f, best = c;
      }
      freet[best] = bf;
      tile_fin[un.tile] = std::max(tile_fin[un.tile], bf + (J.splits > 1 ? kRed : 0.0));
      if (out) (*out)[best].push_back(make_int4(j, un.tile, un.kb0, un.nkb));
    }
    double fin = 0;
    for (double f : tile_fin) fin = std::max(fin, f);
    done_prev[j] = fin;
    if (J.kind == 0) norm_a = fin + kNorm;
    if (J.kind == 2) norm_b = fin + kNorm;
    if (J.kind == 1) gu_done = tile_fin;
  }
  double mk = 0;
  for (double f : freet) mk = std::max(mk, f);
  return mk;
}

}  // namespace

// Split factors (from the weight shapes only) and unit lists for a chain of projections.
int chain_plan(const int* kinds, int njobs, const int64_t* N, const int64_t* K, int grid, int ring,
               int* splits_out, std::vector<int4>& units, std::vector<int>& offs) {
  std::vector<PlanJob> jobs(njobs);
  for (int j = 0; j < njobs; ++j) {
    const int dep = kinds[j] == 0 ? 0 : kinds[j] == 1 ? 1 : kinds[j] == 2 ? 2 : (njobs == 1 ? 0 : 3);
    jobs[j] = {kinds[j], dep, static_cast<int>(N[j] / CBM), static_cast<int>(K[j] / CBK), 1};
  }
  // candidate split factors per split-K projection; gate_up never splits (its SwiGLU
  // epilogue reads both halves of a tile from one accumulator)
  auto cands = [](const PlanJob& J) {
    std::vector<int> c;
    if (J.kind == 1) return std::vector<int>{1};
    for (int kb : {32, 16, 8}) {
      const int s = std::max(1, J.num_kb / kb);
      if (std::find(c.begin(), c.end(), s) == c.end()) c.push_back(s);
    }
    return c;
  };
  std::vector<std::vector<int>> cs(njobs);
  for (int j = 0; j < njobs; ++j) cs[j] = cands(jobs[j]);
  std::vector<int> best_s(njobs, 1), cur(njobs, 0);
  double best = 1e300;
  while (true) {
    for (int j = 0; j < njobs; ++j) jobs[j].splits = cs[j][cur[j]];
    const double mk = simulate(jobs, grid, ring, nullptr);
    int parts = 0;
    for (int j = 0; j < njobs; ++j) parts += jobs[j].splits;
    // fewer partials break ties (less L2 traffic on the reduction)
    if (mk < best - 0.25 || (mk < best + 0.25 && parts < [&] {
          int p = 0;
          for (int j = 0; j < njobs; ++j) p += best_s[j];
          return p;
        }())) {
      if (mk < best) best = mk;
      for (int j = 0; j < njobs; ++j) best_s[j] = jobs[j].splits;
    }
    int j = 0;
    while (j < njobs && ++cur[j] == static_cast<int>(cs[j].size())) cur[j++] = 0;
    if (j == njobs) break;
  }
  for (int j = 0; j < njobs; ++j) jobs[j].splits = splits_out[j] = best_s[j];
  std::vector<std::vector<int4>> per;
  simulate(jobs, grid, ring, &per);
  units.clear();
  offs.assign(1, 0);
  for (int c = 0; c < grid; ++c) {
    units.insert(units.end(), per[c].begin(), per[c].end());
    offs.push_back(static_cast<int>(units.size()));
  }
  return PL_OK;
}

int chain_ring_kb(int BN) {
  switch (BN) {
    case 16: return ChainSmem<16>::AS;
    case 32: return ChainSmem<32>::AS;
    case 64: return ChainSmem<64>::AS;
    case 128: return ChainSmem<128>::AS;
    default: return ChainSmem<256>::AS;
  }
}

template <int BN>
static int chain_launch_bn(const CUtensorMap& m0, const CUtensorMap& m1, const CUtensorMap& m2,
                           const ChainArgs& a, int grid, cudaStream_t st) {
  constexpr int smem = ChainSmem<BN>::TOTAL;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(chain_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_cuda_error(e, "chain smem attribute");
    attr = true;
  }
  return launch_k("chain_kernel", chain_kernel<BN>, dim3(grid), dim3(CH_THREADS), smem, st, m0, m1, m2, a);
}

int chain_launch(const ChainLaunch& c, cudaStream_t st) {
  if (c.T <= 0 || c.T > 256) return set_error(PL_ERR_CONFIG, "chain: 1 <= T <= 256 (got %d)", c.T);
  const int BN = c.T <= 16 ? 16 : c.T <= 32 ? 32 : c.T <= 64 ? 64 : c.T <= 128 ? 128 : 256;
  ChainArgs a{};
  a.T = c.T;
  a.Tp = c.Tp;
  a.njobs = c.njobs;
  a.d = c.d;
  a.ffn = c.ffn;
  for (int j = 0; j < c.njobs; ++j) {
    ChainJob& J = a.job[j];
    J.w = static_cast<const uint8_t*>(c.w[j]);
    J.partial = c.partial[j];
    J.arrive = c.arrive[j];
    J.kind = c.kind[j];
    J.dep = c.kind[j] == 0 ? 0 : c.kind[j] == 1 ? 1 : c.kind[j] == 2 ? 2 : (c.has_norm[1] ? 3 : 0);
    J.tiles = static_cast<int>(c.N[j] / CBM);
    J.num_kb = static_cast<int>(c.K[j] / CBK);
    J.splits = c.splits[j];
    J.kb_per_split = (J.num_kb + J.splits - 1) / J.splits;
    J.act = c.kind[j] == 0 ? 0 : c.kind[j] == 2 ? 2 : 1;
  }
  a.units = c.units;
  a.unit_off = c.unit_off;
  a.h = c.h;
  a.a = c.a;
  a.m = c.m;
  a.q_out = c.q_out;
  a.ld_q = c.ld_q;
  a.ss = c.ss;
  a.norm_w[0] = c.norm_w[0];
  a.norm_w[1] = c.norm_w[1];
  a.has_norm[0] = c.has_norm[0];
  a.has_norm[1] = c.has_norm[1];
  a.eps = c.eps;
  a.bias = c.bias;
  a.pos = c.pos;
  a.slot = c.slot;
  a.cos_sin = c.cos_sin;
  a.max_pos = c.max_pos;
  a.k_cache = c.k_cache;
  a.v_cache = c.v_cache;
  a.block_size = c.block_size;
  a.Hq = c.Hq;
  a.Hkv = c.Hkv;
  a.ctr = c.ctr;
  for (int i = 0; i < 4; ++i) a.tgt[i] = c.tgt[i];
  a.gu_flag = c.gu_flag;
  a.seq = c.seq;
  CUtensorMap m0, m1, m2;
  int rc;
  if ((rc = make_tma_2d(&m0, c.o_attn, c.T, c.attn_dim, c.attn_dim, BN))) return rc;
  if ((rc = make_tma_2d(&m1, c.a, c.T, c.d, c.d, BN))) return rc;
  if ((rc = make_tma_2d(&m2, c.m, c.T, c.ffn, c.ffn, BN))) return rc;
  switch (BN) {
    case 16: return chain_launch_bn<16>(m0, m1, m2, a, c.grid, st);
    case 32: return chain_launch_bn<32>(m0, m1, m2, a, c.grid, st);
    case 64: return chain_launch_bn<64>(m0, m1, m2, a, c.grid, st);
    case 128: return chain_launch_bn<128>(m0, m1, m2, a, c.grid, st);
    default: return chain_launch_bn<256>(m0, m1, m2, a, c.grid, st);
  }
}

int chain_preload() {
  cudaFuncAttributes fa;
  const void* ks[5] = {reinterpret_cast<const void*>(chain_kernel<16>), reinterpret_cast<const void*>(chain_kernel<32>),
                       reinterpret_cast<const void*>(chain_kernel<64>), reinterpret_cast<const void*>(chain_kernel<128>),
                       reinterpret_cast<const void*>(chain_kernel<256>)};
  for (const void* k : ks) {
    cudaError_t e = cudaFuncGetAttributes(&fa, k);
    if (e != cudaSuccess) return set_cuda_error(e, "chain_kernel");
  }
  return PL_OK;
}

}  // namespace pl
