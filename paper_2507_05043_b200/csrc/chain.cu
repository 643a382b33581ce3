// Persistent decode-layer kernel: one launch streams every dense projection of a
// decoder layer (sm_100a).
//
// A decode micro-batch of T <= 256 tokens is a weight stream: per Llama-3-8B layer
// 436 MB of weights against T x 4096 activations.  Issued as one GEMM kernel per
// projection (plus split-K reduce / residual-norm kernels), every launch pays a fill
// and a drain on 148 SMs, and the small projections (o: 33.5 MB, qkv: 50 MB) never
// reach HBM rate (r1: o_proj 29 %, qkv 33 % of peak).  Here ONE persistent launch per
// layer walks the chain
//
//     o-proj (+residual) -> RMSNorm -> gate_up (+SwiGLU) -> down (+residual) -> RMSNorm
//     -> next layer's qkv (+bias, RoPE, paged K/V append)
//
// with the weights of every projection flowing through one shared-memory ring: a
// CTA's weight producer never waits for activations, so the next projection's weights
// are in flight while the previous one drains.  Dependencies live in global memory:
//
//   gate_up  needs RMSNorm(h) after o-proj  -> finalisation step A (below)
//   down     k-block j needs SwiGLU columns [64 j, +64) = gate_up tile j (per-tile flag)
//   qkv      needs RMSNorm(h) after down    -> finalisation step B
//
// Work units are (projection, 128-row weight tile, k-range) in one global order
// (projection by projection, down units by k-block so early down work needs early
// gate_up tiles).  CTAs claim units dynamically -- the weight producer takes the next
// unit whenever its ring has room -- so no CTA waits for a specific other CTA to be
// resident: the kernel makes progress with any number of its CTAs on the GPU (NCCL
// kernels of the inter-stage links may hold SMs while a chain runs).
//
// Split-K projections (o, down, qkv) only write fp32 partials per unit (a serial
// split-ordered accumulation in the unit epilogues was measured slower: the splits of
// a tile run concurrently, so the chain of read-modify-writes serialises).  The
// finalisation sums the splits in split order; it is claimed in (token row, 512-feature
// part) pieces by whichever CTAs reach it, every split's load of a piece in flight at
// once -- T x d/512 pieces spread over the GPU instead of one "last arriver" per
// weight tile reading every split of the tile:
//   A / B  h[t] = bf16(bf16(sum of splits, in split order) + h[t]); the piece's sum of
//          squares; the last piece of a row computes 1/rms (parts in order) and writes
//          a[t] = bf16(w * bf16(h[t] / rms))           (modeling_llama.py:62-67, 313-331)
//   Q      q / k / v = bf16(sum + bias); neox RoPE on q and k pairs (i, i + 64) of each
//          head with HF's per-op rounding; q rows for the attention, k / v into the pages
// Split factors come from the weight shapes only (chain_plan), so a decode token's
// result does not depend on T or on the batch.
//
// Roles (224 threads): warp 0 lane 0 weight producer (claims units; 1-D bulk copies of
// the packed 16 KB tiles), warp 6 activation producer (dependency polls, TMA), warp 1
// TMEM allocation + MMA issue (tcgen05.mma kind::f16, M = 128 weight rows, N = BN
// tokens, double-buffered fp32 accumulators in TMEM), warps 2-5 epilogue (partials,
// SwiGLU, finalisation pieces).
#include <cstdio>
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
#ifndef CH_CTAS
#define CH_CTAS 2  // resident chain CTAs per SM (two pipelines per SM stream ~20 % faster)
#endif
#ifndef CH_BUDGET_KB
#define CH_BUDGET_KB (CH_CTAS == 1 ? 200 : 100)
#endif
constexpr int CH_BUDGET = CH_BUDGET_KB * 1024;
constexpr int UQ = 8;  // claimed units in flight between the weight producer and the other roles

template <int BN>
struct ChainSmem {
  static constexpr int B_TILE = BN * CBK * 2;
  // Activation tiles come from L2 with a latency close to HBM's under a full weight
  // stream, so both rings need similar depths in k-blocks (r1: a 3-deep activation
  // ring capped a CTA at ~48 GB/s whatever the weight ring's depth).
#ifndef CH_BS64
#if CH_CTAS == 1
#define CH_BS16 16
#define CH_BS32 12
#define CH_BS64 8
#define CH_BS128 5
#define CH_BS256 3
#else
#define CH_BS16 6
#define CH_BS32 4
#define CH_BS64 3
#define CH_BS128 2
#define CH_BS256 2
#endif
#endif
  static constexpr int BS = BN <= 16 ? CH_BS16 : BN == 32 ? CH_BS32 : BN == 64 ? CH_BS64 : BN == 128 ? CH_BS128 : CH_BS256;
  static constexpr int AS = (CH_BUDGET - BS * B_TILE) / W_TILE;
  static constexpr int B_OFF = AS * W_TILE;
  static constexpr int RED_OFF = B_OFF + BS * B_TILE;  // block reduction [4] + the piece flag
  static constexpr int UQ_OFF = RED_OFF + 64;          // claimed-unit queue [UQ] int4
  static constexpr int BAR_OFF = UQ_OFF + UQ * 16;
  static constexpr int TOTAL = BAR_OFF + 8 * (2 * AS + 2 * BS + 4 + 2 * UQ) + 16 + 1024;
  static_assert(AS >= 2, "weight ring too shallow");
};

PL_DEV float ch_silu(float x) { return x / (1.0f + expf(-x)); }
PL_DEV void ch_epi_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
PL_DEV int ld_acquire_s32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Publishing pattern (as CUTLASS's split-K semaphores): the epilogue threads store,
// bar.sync, then ONE thread performs a .release (or .acq_rel) operation at gpu scope --
// release is cumulative over the stores the barrier ordered before it; readers spin
// with ld.acquire in one thread, then bar.sync, then read through L2 (ld.cg).
PL_DEV void st_release_s32(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
PL_DEV int atom_add_acq_rel(int* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
PL_DEV void red_add_release_s32(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// generic-proxy writes of other CTAs (acquired above) -> this thread's TMA reads
PL_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
PL_DEV float4 ldcg4(const float* p) { return __ldcg(reinterpret_cast<const float4*>(p)); }
PL_DEV uint2 ldcg_u2(const void* p) { return __ldcg(reinterpret_cast<const uint2*>(p)); }

// k-block order inside a unit, rotated by the unit's weight tile: at any moment the
// 148 CTAs then read DIFFERENT activation tiles (a straight k order has every CTA
// request the same 8 KB tile of the shared activation matrix at once, one L2 slice
// serving all of them).  The order depends on the tile only, never on the CTA, so
// every unit's fp32 summation order is fixed.
PL_DEV int rot_kb(const int4& un, int i, int rotate) {
  if (!rotate) return i;
  const int r = (un.y * 37) % un.w;
  const int k = i + r;
  return k >= un.w ? k - un.w : k;
}

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
  float* partial;      // split-K partials [splits][tiles][Tp][128] fp32 (kinds o, down, qkv)
  int kind, dep, tiles, num_kb, splits, kb_per_split, act, n_units;
};

// Per-launch counters (zero at launch; the last CTA to exit clears them again).  Two
// sets alternate by launch parity: the first unit claim happens before
// griddepcontrol.wait, while the previous chain launch may still be draining.
struct ChainCtr {
  int claim;          // next unit index
  int units_done[4];  // per job
  int fin_claim[3];   // finalisation pieces claimed: A (after o), B (after down), Q (qkv)
  int rows_done[2];   // rows of a complete: A, B
  int exited;
  int pad[5];
};
static_assert(sizeof(ChainCtr) == CHAIN_CTR_BYTES, "counter set size");

struct ChainArgs {
  int T, Tp, njobs, d, ffn, n_units;
  ChainJob job[4];
  int fin_job[3];         // job index finalised by step A / B / Q, or -1
  int has_norm[2];        // A / B also write a = RMSNorm(h)
  int pw, pwq;            // feature width of a finalisation piece (residual / qkv)
  int rotate;             // rotated k-block order (rot_kb)
  const int4* units;      // global claim order: {job, tile, kb0, nkb}
  __nv_bfloat16* h;       // residual stream [T, d]
  __nv_bfloat16* a;       // normalised activations [T, d]
  __nv_bfloat16* m;       // SwiGLU output [T, ffn]
  __nv_bfloat16* q_out;   // roped q rows [T, ld_q] (the attention's q operand)
  int64_t ld_q;
  float* part_ss;         // [2][Tp][d / pw] per-piece sums of squares
  int* row_parts;         // [2][Tp] pieces done per row, zero between launches
  const __nv_bfloat16* norm_w[2];
  float eps;
  const __nv_bfloat16* bias;  // qkv bias (Qwen2) or null
  const int32_t* pos;
  const int32_t* slot;
  const __nv_bfloat16* cos_sin;
  int max_pos;
  __nv_bfloat16* k_cache;
  __nv_bfloat16* v_cache;
  int block_size, Hq, Hkv;
  ChainCtr* ctr;          // this launch's counter set
  int* gu_flag;           // per gate_up tile: sequence number of the launch that finished it
  int seq;
  unsigned long long* trace;  // debug (PL_CHAIN_TRACE): per CTA [64 units][4] globaltimer stamps
};

template <int BN>
__global__ void __launch_bounds__(CH_THREADS, CH_CTAS)
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
  uint64_t* uq_full = tempty + 2;
  uint64_t* uq_empty = uq_full + UQ;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(uq_empty + UQ);
  float* red = reinterpret_cast<float*>(smem + L::RED_OFF);
  int* flag = reinterpret_cast<int*>(red + 8);
  int4* uq = reinterpret_cast<int4*>(smem + L::UQ_OFF);
  ChainCtr* ctr = args.ctr;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

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
    for (int q = 0; q < UQ; ++q) {
      mbar_init(&uq_full[q], 1);
      mbar_init(&uq_empty[q], 3);  // activation producer, MMA issuer, epilogue
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
    // --------------------------------------------------- weight producer: claims the
    // next unit whenever its ring has room and never waits for activations, so the
    // next projection's weights stream while this one drains
    if (lane == 0) {
      int sa = 0, q = 0;
      uint32_t pa = 0, qp = 0;
      bool waited = false;
      int nclaimed = 0;
      for (;;) {
        const int idx = atomicAdd(&ctr->claim, 1);
        const int4 un = idx < args.n_units ? args.units[idx] : make_int4(-1, 0, 0, 0);
        mbar_wait(&uq_empty[q], qp ^ 1);
        uq[q] = un;
        const unsigned long long t_claim = args.trace ? globaltimer_ns() : 0ull;
        mbar_arrive(&uq_full[q]);
        if (++q == UQ) q = 0, qp ^= 1;
        if (un.x < 0) break;
        const ChainJob& J = args.job[un.x];
        const uint8_t* src = J.w + (static_cast<int64_t>(un.y) * J.num_kb + un.z) * W_TILE;
#ifndef CH_L2PF
#define CH_L2PF 0
#endif
        // (experiment) warm L2 with the k-blocks the ring cannot hold yet, so more weight
        // bytes are in flight from HBM than shared memory holds
        for (int i = 0; i < un.w && i < AS + CH_L2PF; ++i)
          if (CH_L2PF > 0 && i >= AS)
            bulk_prefetch_l2(src + static_cast<int64_t>(rot_kb(un, i, args.rotate)) * W_TILE, W_TILE);
        for (int i = 0; i < un.w; ++i) {
          if (CH_L2PF > 0 && i + AS + CH_L2PF < un.w)
            bulk_prefetch_l2(src + static_cast<int64_t>(rot_kb(un, i + AS + CH_L2PF, args.rotate)) * W_TILE, W_TILE);
          mbar_wait(&emptyA[sa], pa ^ 1);
          mbar_arrive_expect_tx(&fullA[sa], W_TILE);
          const int kk = rot_kb(un, i, args.rotate);
          bulk_load(smem + sa * W_TILE, src + static_cast<int64_t>(kk) * W_TILE, W_TILE, &fullA[sa]);
          if (++sa == AS) sa = 0, pa ^= 1;
        }
        if (args.trace && nclaimed < 64)
          args.trace[(static_cast<int64_t>(blockIdx.x) * 64 + nclaimed) * 4] =
              (t_claim & ((1ull << 40) - 1)) | (static_cast<unsigned long long>(idx) << 40);
        ++nclaimed;
        if (!waited) {  // the first claim may precede the previous kernel's end; the rest follow it
          pdl_wait();
          waited = true;
        }
      }
    }
    __syncwarp();
  } else if (warp == CH_ACT_WARP) {
    // --------------------------------------------------- activation producer (one warp:
    // lane 0 issues, all lanes poll dependency flags in parallel -- one L2 round trip
    // per 32 flags instead of one per k-block)
    const uint64_t pol = policy_evict_last();
    int sb = 0, q = 0;
    uint32_t pb = 0, qp = 0;
    pdl_wait();  // o_attn / a come from the previous kernels
    for (;;) {
      mbar_wait(&uq_full[q], qp);
      const int4 un = uq[q];
      __syncwarp();
      if (lane == 0) mbar_arrive(&uq_empty[q]);
      if (++q == UQ) q = 0, qp ^= 1;
      if (un.x < 0) break;
      const ChainJob& J = args.job[un.x];
      if (J.dep == 1 || J.dep == 3) {  // the whole normalised activation matrix
        if (lane == 0) {
          const int* c = &ctr->rows_done[J.dep == 3];
          const int T = args.T;
          spin_until([&] { return ld_acquire_s32(c) >= T; });
          fence_proxy_async_global();
        }
      } else if (J.dep == 2) {  // SwiGLU columns [64 kb, +64) = gate_up tile kb
        const int sq = args.seq;
        for (int k0 = 0; k0 < un.w; k0 += 32) {
          const int* f = args.gu_flag + un.z + k0 + lane;
          const bool mine = k0 + lane < un.w;
          bool ok = !mine || ld_acquire_s32(f) >= sq;
          if (!__all_sync(0xffffffffu, ok)) {
            const uint64_t t0 = globaltimer_ns();
            while (!__all_sync(0xffffffffu, ok)) {
              __nanosleep(64);
              ok = !mine || ld_acquire_s32(f) >= sq;
              if (globaltimer_ns() - t0 > 4000000000ull) __trap();
            }
          }
        }
        if (lane == 0) fence_proxy_async_global();
      }
#ifdef CH_EXP_NOB  // experiment: no activation loads (the MMA reads a stale B tile)
      if (false) {
#else
      if (lane == 0) {
#endif
        const CUtensorMap* tm = J.act == 0 ? &tm0 : (J.act == 1 ? &tm1 : &tm2);
        for (int i = 0; i < un.w; ++i) {
          mbar_wait(&emptyB[sb], pb ^ 1);
          mbar_arrive_expect_tx(&fullB[sb], L::B_TILE);
          tma_load_2d(smem + L::B_OFF + sb * L::B_TILE, tm, &fullB[sb], (un.z + rot_kb(un, i, args.rotate)) * CBK, 0,
                      pol);
          if (++sb == BS) sb = 0, pb ^= 1;
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // --------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(CBM, BN);
      int sa = 0, sb = 0, acc = 0, q = 0;
      uint32_t pa = 0, pb = 0, aphase = 0, qp = 0;
      for (;;) {
        mbar_wait(&uq_full[q], qp);
        const int4 un = uq[q];
        mbar_arrive(&uq_empty[q]);
        if (++q == UQ) q = 0, qp ^= 1;
        if (un.x < 0) break;
        const int nkb = un.w;
        mbar_wait(&tempty[acc], aphase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int i = 0; i < nkb; ++i) {
          mbar_wait(&fullA[sa], pa);
#ifndef CH_EXP_NOB
          mbar_wait(&fullB[sb], pb);
#endif
          tc_fence_after();
#ifdef CH_EXP_NOMMA  // experiment: recycle the stages without any MMA (pure load pipeline)
          mbar_arrive(&emptyA[sa]);
          mbar_arrive(&emptyB[sb]);
#else
          const uint64_t da = umma_desc_sw128(smem_u32(smem + sa * W_TILE));
          const uint64_t db = umma_desc_sw128(smem_u32(smem + L::B_OFF + sb * L::B_TILE));
#pragma unroll
          for (int k = 0; k < CBK / 16; ++k) umma_bf16(d, da + 2 * k, db + 2 * k, idesc, (i | k) != 0);
          umma_commit(&emptyA[sa]);
#ifndef CH_EXP_NOB
          umma_commit(&emptyB[sb]);
#endif
#endif
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
    int acc = 0, q = 0;
    uint32_t aphase = 0, qp = 0;
    bool did[3] = {false, false, false};

    // fixed-order sum over the 128 epilogue threads (warp tree, then warps in order)
    auto block_sum = [&](float v) {
      v = warp_sum(v);
      if (lane == 0) red[quarter] = v;
      ch_epi_sync();
      const float s = ((red[0] + red[1]) + red[2]) + red[3];
      ch_epi_sync();
      return s;
    };
    // claim the next piece of finalisation step w (broadcast to all epilogue threads)
    auto claim_piece = [&](int w) {
      if (ep == 0) *flag = atomicAdd(&ctr->fin_claim[w], 1);
      ch_epi_sync();
      const int c = *flag;
      ch_epi_sync();
      return c;
    };

    // ---- finalisation A / B: residual add of the split-summed projection into h, and
    // (has_norm) the next RMSNorm; one piece = (row t, features [p pw, +pw))
    auto fin_residual = [&](int w, int t, int p) {
      const ChainJob& J = args.job[args.fin_job[w]];
      const int S = J.splits, pw = args.pw, P = d / pw;
      const int64_t split_stride = static_cast<int64_t>(J.tiles) * Tp * CBM;
      constexpr int NP = 4;  // float4 positions per thread (pieces of <= 2048 features)
      bool on[NP];
      int n0[NP];
      const float* pp[NP];
      uint2 hr[NP];
      float4 acc4[NP];
#pragma unroll
      for (int u = 0; u < NP; ++u) {
        const int pos = u * 128 + ep;
        on[u] = pos * 4 < pw;
        n0[u] = p * pw + (on[u] ? pos : 0) * 4;
        pp[u] = J.partial + (static_cast<int64_t>(n0[u] / CBM) * Tp + t) * CBM + n0[u] % CBM;
        hr[u] = ldcg_u2(args.h + static_cast<int64_t>(t) * d + n0[u]);
        acc4[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      for (int s0 = 0; s0 < S; s0 += 8) {  // up to 32 float4 loads in flight, summed in split order
        float4 x[NP][8];
#pragma unroll
        for (int u = 0; u < NP; ++u)
#pragma unroll
          for (int k = 0; k < 8; ++k) x[u][k] = ldcg4(pp[u] + min(s0 + k, S - 1) * split_stride);
#pragma unroll
        for (int u = 0; u < NP; ++u)
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (s0 + k < S) {
              acc4[u].x += x[u][k].x;
              acc4[u].y += x[u][k].y;
              acc4[u].z += x[u][k].z;
              acc4[u].w += x[u][k].w;
            }
      }
      float ss = 0.f;
#pragma unroll
      for (int u = 0; u < NP; ++u) {
        const float2 h01 = unpack_bf16x2(hr[u].x), h23 = unpack_bf16x2(hr[u].y);
        const float hv[4] = {rbf(rbf(acc4[u].x) + h01.x), rbf(rbf(acc4[u].y) + h01.y),
                             rbf(rbf(acc4[u].z) + h23.x), rbf(rbf(acc4[u].w) + h23.y)};
        if (on[u]) {
          *reinterpret_cast<uint2*>(args.h + static_cast<int64_t>(t) * d + n0[u]) =
              make_uint2(pack_bf16x2(hv[0], hv[1]), pack_bf16x2(hv[2], hv[3]));
          ss += ((hv[0] * hv[0] + hv[1] * hv[1]) + hv[2] * hv[2]) + hv[3] * hv[3];
        }
      }
      if (!args.has_norm[w]) return;
      ss = block_sum(ss);
      if (ep == 0) {
        args.part_ss[(static_cast<int64_t>(w) * Tp + t) * P + p] = ss;
        const int done = atom_add_acq_rel(args.row_parts + w * Tp + t, 1);
        *flag = done == P - 1;
        if (done == P - 1) args.row_parts[w * Tp + t] = 0;  // zero again for the next launch
      }
      ch_epi_sync();
      const bool last = *flag;
      ch_epi_sync();
      if (!last) return;
      // the row's last piece: 1/rms from the pieces' sums (in piece order), then a[t]
      float tot = 0.f;
      for (int k = 0; k < P; ++k) tot += __ldcg(args.part_ss + (static_cast<int64_t>(w) * Tp + t) * P + k);
      const float r = rsqrtf(tot / static_cast<float>(d) + args.eps);
      const __nv_bfloat16* wn = args.norm_w[w];
      for (int kb = 0; kb < d; kb += 128 * 8 * 8) {  // loads first, then the stores
        uint4 x[8], g[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int k = min(kb + (u * 128 + ep) * 8, d - 8);
          x[u] = __ldcg(reinterpret_cast<const uint4*>(args.h + static_cast<int64_t>(t) * d + k));
          g[u] = *reinterpret_cast<const uint4*>(wn + k);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int k = kb + (u * 128 + ep) * 8;
          if (k >= d) break;
          const uint32_t xs[4] = {x[u].x, x[u].y, x[u].z, x[u].w}, gs[4] = {g[u].x, g[u].y, g[u].z, g[u].w};
          uint32_t o[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 xv = unpack_bf16x2(xs[j]), gv = unpack_bf16x2(gs[j]);
            o[j] = pack_bf16x2(gv.x * rbf(xv.x * r), gv.y * rbf(xv.y * r));
          }
          *reinterpret_cast<uint4*>(args.a + static_cast<int64_t>(t) * d + k) = make_uint4(o[0], o[1], o[2], o[3]);
        }
      }
      ch_epi_sync();
      if (ep == 0) red_add_release_s32(&ctr->rows_done[w], 1);
    };

    // ---- finalisation Q: one piece = (row t, qkv features [p pwq, +pwq)); a thread owns
    // four rotary pairs (i, i + 64) of one head
    auto fin_qkv = [&](int t, int p) {
      const ChainJob& J = args.job[args.fin_job[2]];
      const int S = J.splits, pwq = args.pwq;
      const int64_t split_stride = static_cast<int64_t>(J.tiles) * Tp * CBM;
      int pp = args.pos[t];
      const int sl = args.slot ? args.slot[t] : -1;
      pp = pp < 0 ? 0 : (pp >= args.max_pos ? args.max_pos - 1 : pp);
      constexpr int NP = 2;  // four rotary pairs (i, i + 64) of one head per position
      bool on[NP];
      int n1[NP];
      float4 a1[NP], a2[NP];
      uint2 csr[NP], snr[NP];
#pragma unroll
      for (int u = 0; u < NP; ++u) {
        const int pos = u * 128 + ep;
        on[u] = pos * 8 < pwq;
        const int q = on[u] ? pos : 0;
        const int i0 = (q % 16) * 4;
        n1[u] = p * pwq + (q / 16) * CBM + i0;
        csr[u] = *reinterpret_cast<const uint2*>(args.cos_sin + static_cast<int64_t>(pp) * CBM + i0);
        snr[u] = *reinterpret_cast<const uint2*>(args.cos_sin + static_cast<int64_t>(pp) * CBM + 64 + i0);
        a1[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        a2[u] = a1[u];
      }
      for (int s0 = 0; s0 < S; s0 += 8) {  // eight splits' loads in flight, summed in order
        float4 x1[NP][8], x2[NP][8];
#pragma unroll
        for (int u = 0; u < NP; ++u)
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float* q0 = J.partial + (static_cast<int64_t>(n1[u] / CBM) * Tp + t) * CBM + n1[u] % CBM +
                              min(s0 + k, S - 1) * split_stride;
            x1[u][k] = ldcg4(q0);
            x2[u][k] = ldcg4(q0 + 64);
          }
#pragma unroll
        for (int u = 0; u < NP; ++u)
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (s0 + k < S) {
              a1[u].x += x1[u][k].x, a1[u].y += x1[u][k].y, a1[u].z += x1[u][k].z, a1[u].w += x1[u][k].w;
              a2[u].x += x2[u][k].x, a2[u].y += x2[u][k].y, a2[u].z += x2[u][k].z, a2[u].w += x2[u][k].w;
            }
      }
#pragma unroll
      for (int u = 0; u < NP; ++u) {
        if (!on[u]) continue;
        const int hh = n1[u] / CBM;
        const bool roped = hh < args.Hq + args.Hkv;
        float v1[4] = {a1[u].x, a1[u].y, a1[u].z, a1[u].w}, v2[4] = {a2[u].x, a2[u].y, a2[u].z, a2[u].w};
        const float2 c01 = unpack_bf16x2(csr[u].x), c23 = unpack_bf16x2(csr[u].y);
        const float2 s01 = unpack_bf16x2(snr[u].x), s23 = unpack_bf16x2(snr[u].y);
        const float cs[4] = {c01.x, c01.y, c23.x, c23.y}, sn[4] = {s01.x, s01.y, s23.x, s23.y};
        float o1[4], o2[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float b1 = args.bias ? bf2f(args.bias[n1[u] + j]) : 0.f;
          const float b2 = args.bias ? bf2f(args.bias[n1[u] + 64 + j]) : 0.f;
          v1[j] = rbf(v1[j] + b1);
          v2[j] = rbf(v2[j] + b2);
          o1[j] = roped ? rbf(rbf(v1[j] * cs[j]) + rbf(-v2[j] * sn[j])) : v1[j];
          o2[j] = roped ? rbf(rbf(v2[j] * cs[j]) + rbf(v1[j] * sn[j])) : v2[j];
        }
        const uint2 w1 = make_uint2(pack_bf16x2(o1[0], o1[1]), pack_bf16x2(o1[2], o1[3]));
        const uint2 w2 = make_uint2(pack_bf16x2(o2[0], o2[1]), pack_bf16x2(o2[2], o2[3]));
        if (hh < args.Hq) {
          __nv_bfloat16* qr = args.q_out + static_cast<int64_t>(t) * args.ld_q + n1[u];
          *reinterpret_cast<uint2*>(qr) = w1;
          *reinterpret_cast<uint2*>(qr + 64) = w2;
        } else if (sl >= 0) {
          const bool is_k = hh < args.Hq + args.Hkv;
          const int kh = is_k ? hh - args.Hq : hh - args.Hq - args.Hkv;
          __nv_bfloat16* dst = (is_k ? args.k_cache : args.v_cache) +
                               ((static_cast<int64_t>(sl / args.block_size) * args.Hkv + kh) * args.block_size +
                                sl % args.block_size) * CBM + (n1[u] % CBM);
          *reinterpret_cast<uint2*>(dst) = w1;
          *reinterpret_cast<uint2*>(dst + 64) = w2;
        }
      }
    };

    // finalisation step w (0: A after o, 1: B after down, 2: Q after qkv): wait for every
    // unit of the projection, then claim pieces until none are left
    auto finalise = [&](int w) {
      did[w] = true;
      const int j = args.fin_job[w];
      if (j < 0) return;
      if (ep == 0) {
        const int* c = &ctr->units_done[j];
        const int n = args.job[j].n_units;
        spin_until([&] { return ld_acquire_s32(c) >= n; });
      }
      ch_epi_sync();
      const int P = w == 2 ? args.pwq : args.pw;
      const int pieces = T * ((w == 2 ? args.job[j].tiles * CBM : d) / P);
      for (;;) {
        const int c = claim_piece(w);
        if (c >= pieces) break;
        const int per_row = pieces / T;
        if (w == 2)
          fin_qkv(c / per_row, c % per_row);
        else
          fin_residual(w, c / per_row, c % per_row);
      }
    };

    int nproc = 0;
    for (;;) {
      mbar_wait(&uq_full[q], qp);
      const int4 un = uq[q];
      unsigned long long* trc = (args.trace && ep == 0 && nproc < 64)
                                    ? args.trace + (static_cast<int64_t>(blockIdx.x) * 64 + nproc) * 4 : nullptr;
      ++nproc;
      if (trc) trc[1] = globaltimer_ns();
      ch_epi_sync();  // everyone read the slot
      if (ep == 0) mbar_arrive(&uq_empty[q]);
      if (++q == UQ) q = 0, qp ^= 1;
      if (un.x < 0) break;
      const ChainJob& J = args.job[un.x];
      if (J.dep >= 1 && !did[0]) finalise(0);
      if (J.dep >= 3 && !did[1]) finalise(1);
      const int tile = un.y;
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      if (trc) trc[2] = globaltimer_ns();
      const uint32_t tcol = tmem + lane_base + acc * BN;
      if (J.kind == 1) {
        // ---- gate_up, whole K in one unit: SwiGLU straight from TMEM.  Packed rows
        // alternate (gate_j, up_j), so lane pairs meet by one shuffle.
        const int j = tile * 64 + (row >> 1);
        for (int c0 = 0; c0 < BN && c0 < T; c0 += 16) {
          uint32_t r[16];
          tmem_ld16(tcol + c0, r);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const float v = __uint_as_float(r[c]);
            const float other = __shfl_xor_sync(0xffffffffu, v, 1);
            const int t = c0 + c;
            if (!(row & 1) && t < T)
              args.m[static_cast<int64_t>(t) * args.ffn + j] = f2bf(rbf(ch_silu(rbf(v))) * rbf(other));
          }
        }
      } else {
        // ---- split-K projections: this unit's fp32 partial, token rows of 128 features
        const int split = un.z / J.kb_per_split;
        float* p = J.partial + ((static_cast<int64_t>(split) * J.tiles + tile) * Tp) * CBM + row;
        for (int c0 = 0; c0 < BN && c0 < T; c0 += 16) {
          uint32_t r[16];
          tmem_ld16(tcol + c0, r);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < 16; ++c)
            if (c0 + c < T) __stcg(p + static_cast<int64_t>(c0 + c) * CBM, __uint_as_float(r[c]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) acc = 0, aphase ^= 1;
      ch_epi_sync();
      if (ep == 0) {
        if (J.kind == 1) {
          st_release_s32(args.gu_flag + tile, args.seq);
        } else {
          red_add_release_s32(&ctr->units_done[un.x], 1);
        }
      }
      if (trc) trc[3] = globaltimer_ns();
    }
    if (!did[0]) finalise(0);
    if (!did[1]) finalise(1);
    finalise(2);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<TMEM_COLS>(tmem);
  if (threadIdx.x == 0) {
    // the last CTA out clears this launch's counter set for the launch after next
    __threadfence();
    if (atomicAdd(&ctr->exited, 1) == static_cast<int>(gridDim.x) - 1) {
      __threadfence();
      *ctr = ChainCtr{};
    }
  }
}

// ------------------------------------------------------------------ host

namespace {

// Split factors from a fluid model of the dynamic claiming: every CTA streams 1
// k-block (16 KB) per time unit; units are claimed in the global order (projection by
// projection, split-major) by the CTA that is free first, and a unit finishes at
//   max(cta free + nkb + kUnit, ready + max(0, nkb - ring))
// (its weights prefetch into the ring while its activations are not ready yet; kUnit
// prices a split-K unit's partial write); a finalisation step costs kFin plus
// kFinSplit per split it sums.  Depends only on the weight shapes and the SM count --
// never on T.
struct PlanJob {
  int kind, dep, tiles, num_kb, splits;
};

double simulate(const std::vector<PlanJob>& jobs, int grid, int ring, std::vector<int4>* order) {
  std::vector<double> freet(grid, 0.0);
  if (order) order->clear();
  std::vector<double> gu_done;
  double done_prev[4] = {0, 0, 0, 0};  // finish time of each job
  double norm_a = 0, norm_b = 0;
  constexpr double kUnit = 1.0, kFin = 12.0, kFinSplit = 1.5;
  for (int j = 0; j < static_cast<int>(jobs.size()); ++j) {
    const PlanJob& J = jobs[j];
    const int per = (J.num_kb + J.splits - 1) / J.splits;  // splits are effective: no empty split
    struct U {
      int tile, kb0, nkb;
    };
    std::vector<U> units;  // split-major: split s of a tile follows split s - 1 by a wave
    for (int s = 0; s < J.splits; ++s)
      for (int t = 0; t < J.tiles; ++t) {
        const int k0 = s * per, n = std::min(J.num_kb, k0 + per) - k0;
        if (n > 0) units.push_back({t, k0, n});
      }
    std::vector<double> tile_fin(J.tiles, 0.0);
    const double cu = J.splits > 1 ? kUnit : 0.0;
    for (const U& un : units) {
      double ready = 0;
      if (J.dep == 1) ready = norm_a;
      if (J.dep == 3) ready = norm_b;
      if (J.dep == 2)
        for (int k = un.kb0; k < un.kb0 + un.nkb; ++k) ready = std::max(ready, gu_done[k]);
      int best = 0;
      double bf = 1e300;
      for (int c = 0; c < grid; ++c) {
        const double f = std::max(freet[c] + un.nkb + cu, ready + std::max(0, un.nkb - ring));
        if (f < bf - 1e-9) bf = f, best = c;
      }
      freet[best] = bf;
      tile_fin[un.tile] = std::max(tile_fin[un.tile], bf);
      if (order) order->push_back(make_int4(j, un.tile, un.kb0, un.nkb));
    }
    double fin = 0;
    for (double f : tile_fin) fin = std::max(fin, f);
    done_prev[j] = fin;
    const double fin_cost = kFin + kFinSplit * J.splits;  // reading every split's partial
    done_prev[j] = fin + (J.kind == 1 ? 0.0 : fin_cost);
    if (J.kind == 0) norm_a = done_prev[j];
    if (J.kind == 2) norm_b = done_prev[j];
    if (J.kind == 1) gu_done = tile_fin;
  }
  double mk = 0;
  for (double f : freet) mk = std::max(mk, f);
  for (double f : done_prev) mk = std::max(mk, f);
  return mk;
}

}  // namespace

// Split factors (from the weight shapes only) and the global unit order of a chain.
int chain_plan(const int* kinds, int njobs, const int64_t* N, const int64_t* K, int grid, int ring,
               int* splits_out, std::vector<int4>& units) {
  std::vector<PlanJob> jobs(njobs);
  for (int j = 0; j < njobs; ++j) {
    const int dep = kinds[j] == 0 ? 0 : kinds[j] == 1 ? 1 : kinds[j] == 2 ? 2 : (njobs == 1 ? 0 : 3);
    jobs[j] = {kinds[j], dep, static_cast<int>(N[j] / CBM), static_cast<int>(K[j] / CBK), 1};
  }
  // Split factors by unit size (the fluid model's choices were measured slower: it
  // under-prices partial traffic and the serial tail after the norm barriers): the
  // projections right after a barrier (qkv) get 8-k-block units so the CTAs share the
  // tail finely; the others 16-k-block units; gate_up never splits (its SwiGLU epilogue
  // reads both halves of a tile from one accumulator).
  std::vector<int> best_s(njobs, 1);
  for (int j = 0; j < njobs; ++j) {
    const PlanJob& J = jobs[j];
    if (J.kind == 1) continue;
    const int target = J.kind == 3 ? 8 : 16;
    const int want = std::max(1, J.num_kb / target);
    const int per = (J.num_kb + want - 1) / want;
    best_s[j] = (J.num_kb + per - 1) / per;  // no empty splits
  }
  for (int j = 0; j < njobs; ++j) jobs[j].splits = splits_out[j] = best_s[j];
  simulate(jobs, grid, ring, &units);
  return PL_OK;
}

int chain_ctas_per_sm() { return CH_CTAS; }

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
  const int rc = ensure_smem_attr(reinterpret_cast<const void*>(chain_kernel<BN>), smem, "chain smem attribute");
  if (rc) return rc;
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
    J.kind = c.kind[j];
    J.dep = c.kind[j] == 0 ? 0 : c.kind[j] == 1 ? 1 : c.kind[j] == 2 ? 2 : (c.has_norm[1] ? 3 : 0);
    J.tiles = static_cast<int>(c.N[j] / CBM);
    J.num_kb = static_cast<int>(c.K[j] / CBK);
    J.splits = c.splits[j];
    J.kb_per_split = (J.num_kb + J.splits - 1) / J.splits;
    J.act = c.kind[j] == 0 ? 0 : c.kind[j] == 2 ? 2 : 1;
    J.n_units = 0;
  }
  for (int w = 0; w < 3; ++w) a.fin_job[w] = -1;
  for (int j = 0; j < c.njobs && c.bench; ++j) a.job[j].dep = 0;  // stream only (pl_stage_chain_bench)
  for (int j = 0; j < c.njobs && !c.bench; ++j) {
    if (c.kind[j] == CHAIN_O) a.fin_job[0] = j;
    if (c.kind[j] == CHAIN_DOWN) a.fin_job[1] = j;
    if (c.kind[j] == CHAIN_QKV) a.fin_job[2] = j;
  }
  for (int u = 0; u < c.n_units; ++u) a.job[c.units_host[u].x].n_units++;
  // finalisation piece widths: the largest of 1024 / 512 / 256 (128 for qkv) dividing the row
  a.pw = 256;  // residual pieces: <= 4 float4 per epilogue thread
  for (int w = 2048; w >= 256; w /= 2)
    if (c.d % w == 0) {
      a.pw = w;
      break;
    }
  a.pwq = 128;  // qkv pieces
  if (a.fin_job[2] >= 0)
    for (int w = 2048; w >= 128; w /= 2)
      if (c.N[a.fin_job[2]] % w == 0) {  // <= 2 x 4 rotary pairs per thread
        a.pwq = w;
        break;
      }
  {
    static const int rot = [] { const char* v = getenv("PL_CHAIN_ROT"); return !(v && v[0] == '0'); }();
    a.rotate = rot;
  }
  if (!a.pw || !a.pwq) return set_error(PL_ERR_CONFIG, "chain: d must be a multiple of 256");
  a.units = c.units;
  a.n_units = c.n_units;
  a.h = c.h;
  a.a = c.a;
  a.m = c.m;
  a.q_out = c.q_out;
  a.ld_q = c.ld_q;
  a.part_ss = c.part_ss;
  a.row_parts = c.row_parts;
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
  a.ctr = static_cast<ChainCtr*>(c.ctr);
  a.gu_flag = c.gu_flag;
  a.seq = c.seq;
  a.trace = c.trace;
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
