// GQA attention for the decoder stages (hd = 128).
//
// prefill: causal varlen self-attention over the prompt rows of the fused qkv
//   buffer.  The reference admits a prompt whole into one micro-batch and never
//   splits compute (engine.py:215-223), so a prefill has no prior
//   context: q, k and v come straight from the QKV GEMM output (post-RoPE)
//   instead of the paged cache.  Flash-attention-2 tiling: 64 query rows per
//   CTA (16 per warp), 64-token K/V tiles double-buffered in XOR-swizzled shared
//   memory via cp.async, m16n8k16 bf16 tensor-core MMAs, fp32 online softmax.
//
// decode: one query token per request over its paged KV cache
//   [num_blocks, Hkv, 64, hd].  One CTA per (kv head, request, KV split) serves
//   the whole GQA group, so each KV page is read from HBM exactly once.  Pages
//   arrive by TMA into 128-byte-swizzled shared memory (persistent CTAs, one TMA
//   producer warp, four tensor-core consumer warps); a request's context is cut
//   into ceil(pages/16) even splits, so the reduction order depends on its own
//   context length only, never on the batch.
#include "common.cuh"
#include "pl_internal.h"

namespace pl {

constexpr int HD = 128;
constexpr float LOG2E = 1.4426950408889634f;

// ======================================================= prefill (mma.sync)

PL_DEV void ldmatrix_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
PL_DEV void ldmatrix_x4_trans(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                              uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
PL_DEV void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// 64 x 128 bf16 tile, rows of 256 B = 16 chunks of 16 B, chunk c of row r at c ^ (r & 7).
PL_DEV uint32_t swz(int row, int chunk) { return row * 256 + ((chunk ^ (row & 7)) << 4); }

// One CTA = 128 query rows = the G query heads of one kv head x (128 / G) positions,
// so each K/V tile staged in shared memory serves all G heads of the group (GQA):
// 8 warps of 16 rows, FA2-style online softmax on m16n8k16 tensor cores, K/V
// double-buffered by cp.async.
constexpr int PF_ROWS = 128, PF_THREADS = 256;

PL_DEV void load_kv_tile(uint8_t* smem, const __nv_bfloat16* base, int64_t ld, int rows_valid) {
  // 64 rows x 16 chunks = 1024 chunks, 4 per thread
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = threadIdx.x + i * PF_THREADS;
    const int row = c >> 4, ch = c & 15;
    const bool ok = row < rows_valid;
    const __nv_bfloat16* src = base + (ok ? static_cast<int64_t>(row) * ld : 0) + ch * 8;
    cp_async16_zfill(smem + swz(row, ch), src, ok);
  }
}

__global__ void __launch_bounds__(PF_THREADS, 2)
    attn_prefill_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t ldqkv,
                        const int32_t* __restrict__ cu_seqlens, int Hq, int Hkv, float scale_log2,
                        __nv_bfloat16* __restrict__ out, int64_t ldo) {
  extern __shared__ uint8_t smem_raw[];
  pdl_trigger();
  pdl_wait();
  uint8_t* sQ = smem_raw;                 // 128 rows x 256 B = 32 KB
  uint8_t* sK = smem_raw + 32768;         // 2 x 16 KB
  uint8_t* sV = smem_raw + 32768 * 2;     // 2 x 16 KB

  const int r = blockIdx.z, kh = blockIdx.y;
  const int G = Hq / Hkv;
  const int QT = PF_ROWS / G;             // positions per head in this CTA
  const int seq0 = cu_seqlens[r];
  const int L = cu_seqlens[r + 1] - seq0;
  const int q0 = blockIdx.x * QT;
  if (q0 >= L) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const __nv_bfloat16* kbase = qkv + static_cast<int64_t>(seq0) * ldqkv + (Hq + kh) * HD;
  const __nv_bfloat16* vbase = qkv + static_cast<int64_t>(seq0) * ldqkv + (Hq + Hkv + kh) * HD;

  const int q_hi = min(q0 + QT, L);          // exclusive
  const int n_kv_tiles = (q_hi + 63) / 64;   // causal: keys < q_hi

  // Q: row rho = head (kh G + rho / QT) at position q0 + rho % QT
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int c = threadIdx.x + i * PF_THREADS;
    const int row = c >> 4, ch = c & 15;
    const int pos = q0 + row % QT;
    const bool ok = pos < L;
    const __nv_bfloat16* src =
        qkv + static_cast<int64_t>(seq0 + (ok ? pos : 0)) * ldqkv + (kh * G + row / QT) * HD + ch * 8;
    cp_async16_zfill(sQ + swz(row, ch), src, ok);
  }
  load_kv_tile(sK, kbase, ldqkv, min(64, L));
  load_kv_tile(sV, vbase, ldqkv, min(64, L));
  cp_async_commit();

  // this warp's 16 rows: one head, 16 consecutive positions
  const int head_g = (warp * 16) / QT;
  const int pos0 = q0 + (warp * 16) % QT;
  uint32_t qf[8][4];
  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY};
  float l_r[2] = {0.f, 0.f};

  const uint32_t sQa = smem_u32(sQ), sKa = smem_u32(sK), sVa = smem_u32(sV);
  const int mi = lane >> 3, ri = lane & 7;

  for (int j = 0; j < n_kv_tiles; ++j) {
    const int buf = j & 1;
    if (j + 1 < n_kv_tiles) {
      const int kv0 = (j + 1) * 64;
      load_kv_tile(sK + (buf ^ 1) * 16384, kbase + static_cast<int64_t>(kv0) * ldqkv, ldqkv,
                   min(64, L - kv0));
      load_kv_tile(sV + (buf ^ 1) * 16384, vbase + static_cast<int64_t>(kv0) * ldqkv, ldqkv,
                   min(64, L - kv0));
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (j == 0) {
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const int row = warp * 16 + (mi & 1) * 8 + ri;
        const int ch = ks * 2 + (mi >> 1);
        ldmatrix_x4(qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3], sQa + swz(row, ch));
      }
    }
    const int kv0 = j * 64;
    if (kv0 <= pos0 + 15) {  // tiles wholly above this warp's rows contribute nothing
      // S = Q K^T  (16 rows x 64 keys per warp)
      float s[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
      const uint32_t kt = sKa + buf * 16384;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
        for (int nt = 0; nt < 8; nt += 2) {
          uint32_t b0, b1, b2, b3;
          const int row = nt * 8 + (mi >> 1) * 8 + ri;
          const int ch = ks * 2 + (mi & 1);
          ldmatrix_x4(b0, b1, b2, b3, kt + swz(row, ch));
          mma_bf16_16816(s[nt], qf[ks], b0, b1);
          mma_bf16_16816(s[nt + 1], qf[ks], b2, b3);
        }
      }
      // causal + length mask, online softmax (base 2)
      const int qrow0 = pos0 + (lane >> 2);
      float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int qi = qrow0 + (e >> 1) * 8;
          const int kj = kv0 + nt * 8 + (lane & 3) * 2 + (e & 1);
          float v = s[nt][e] * scale_log2;
          if (kj > qi || kj >= L) v = -INFINITY;
          s[nt][e] = v;
          mx[e >> 1] = fmaxf(mx[e >> 1], v);
        }
      }
      float corr[2];
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        mx[hr] = fmaxf(mx[hr], __shfl_xor_sync(0xffffffffu, mx[hr], 1));
        mx[hr] = fmaxf(mx[hr], __shfl_xor_sync(0xffffffffu, mx[hr], 2));
        const float m_new = fmaxf(m_r[hr], mx[hr]);
        corr[hr] = (m_new == -INFINITY) ? 1.f : exp2f(m_r[hr] - m_new);
        m_r[hr] = m_new;
      }
      float rs[2] = {0.f, 0.f};
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int hr = e >> 1;
          const float p = (m_r[hr] == -INFINITY) ? 0.f : exp2f(s[nt][e] - m_r[hr]);
          s[nt][e] = p;
          rs[hr] += p;
        }
      }
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        rs[hr] += __shfl_xor_sync(0xffffffffu, rs[hr], 1);
        rs[hr] += __shfl_xor_sync(0xffffffffu, rs[hr], 2);
        l_r[hr] = l_r[hr] * corr[hr] + rs[hr];
      }
#pragma unroll
      for (int nt = 0; nt < 16; ++nt) {
        o[nt][0] *= corr[0];
        o[nt][1] *= corr[0];
        o[nt][2] *= corr[1];
        o[nt][3] *= corr[1];
      }
      // O += P V
      const uint32_t vt = sVa + buf * 16384;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {  // 16 keys per k-step
        uint32_t a[4];
        a[0] = pack_bf16x2(s[2 * ks][0], s[2 * ks][1]);
        a[1] = pack_bf16x2(s[2 * ks][2], s[2 * ks][3]);
        a[2] = pack_bf16x2(s[2 * ks + 1][0], s[2 * ks + 1][1]);
        a[3] = pack_bf16x2(s[2 * ks + 1][2], s[2 * ks + 1][3]);
#pragma unroll
        for (int nt = 0; nt < 16; nt += 2) {
          uint32_t b0, b1, b2, b3;
          const int row = ks * 16 + (mi & 1) * 8 + ri;
          const int ch = nt + (mi >> 1);
          ldmatrix_x4_trans(b0, b1, b2, b3, vt + swz(row, ch));
          mma_bf16_16816(o[nt], a, b0, b1);
          mma_bf16_16816(o[nt + 1], a, b2, b3);
        }
      }
    }
    __syncthreads();
  }

  // normalize and store
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
    const int qi = pos0 + (lane >> 2) + hr * 8;
    if (qi >= L) continue;
    const float inv = l_r[hr] > 0.f ? 1.f / l_r[hr] : 0.f;
    __nv_bfloat16* orow = out + static_cast<int64_t>(seq0 + qi) * ldo + (kh * G + head_g) * HD;
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      const int col = nt * 8 + (lane & 3) * 2;
      *reinterpret_cast<uint32_t*>(orow + col) =
          pack_bf16x2(o[nt][hr * 2] * inv, o[nt][hr * 2 + 1] * inv);
    }
  }
}

// Which prefill kernel: 1 = mma.sync (this file), 2 = tcgen05 (attn_tc.cu), 0 = by
// PL_ATTN_TC (default tcgen05; 0 selects mma.sync); tcgen05 needs the qkv row count
// (its TMA maps), so a launch without it takes the mma.sync kernel.
int attn_prefill_impl(int impl, int64_t rows) {
  static const int env = [] { const char* v = getenv("PL_ATTN_TC"); return v ? atoi(v) : -1; }();
  if (impl == 0) impl = env == 0 ? 1 : 2;
  return impl == 2 && rows > 0 ? 2 : 1;
}

int attn_prefill_launch(const __nv_bfloat16* qkv, int64_t ldqkv, const int32_t* cu_seqlens, int R,
                        int max_seqlen, int Hq, int Hkv, int hd, float scale, __nv_bfloat16* out,
                        int64_t ldo, cudaStream_t st, int64_t rows, int impl) {
  if (R <= 0 || max_seqlen <= 0) return PL_OK;
  if (hd != HD) return set_error(PL_ERR_CONFIG, "attention: head_dim must be 128 (got %d)", hd);
  if (Hkv <= 0 || Hq % Hkv) return set_error(PL_ERR_CONFIG, "attention: Hq must be a multiple of Hkv");
  if (attn_prefill_impl(impl, rows) == 2) {
    if (ldqkv % 8 || ldo % 8) return set_error(PL_ERR_CONFIG, "attention: leading dims % 8");
    return attn_prefill_tc_launch(qkv, ldqkv, rows, cu_seqlens, R, max_seqlen, Hq, Hkv, scale * LOG2E, out,
                                  ldo, st);
  }
  const int G = Hq / Hkv;
  if (G > 8 || PF_ROWS % (16 * G))
    return set_error(PL_ERR_CONFIG, "attention prefill: GQA group %d unsupported (1, 2, 4, 8)", G);
  if (ldqkv % 8 || ldo % 8) return set_error(PL_ERR_CONFIG, "attention: leading dims % 8");
  constexpr int smem = 32768 * 3;
  {
    const int rc0 = ensure_smem_attr(reinterpret_cast<const void*>(attn_prefill_kernel), smem, "attn_prefill smem attribute");
    if (rc0) return rc0;
  }
  const int QT = PF_ROWS / G;
  dim3 grid((max_seqlen + QT - 1) / QT, Hkv, R);
  return launch_k("attn_prefill_kernel", attn_prefill_kernel, grid, dim3(PF_THREADS), smem, st, qkv, ldqkv,
                  cu_seqlens, Hq, Hkv, scale * LOG2E, out, ldo);
}

// ======================================================= decode (paged)
//
// Persistent, warp-specialized paged decode attention (one CTA per SM).  A work
// item is (request, kv head, split of <= 8 pages); the CTA walks its items in a
// static round robin.  Warp 0 (one lane) is a TMA producer streaming each 64-token
// K and V page -- four 2-D boxes of 64 dims x 64 tokens, 128-byte swizzle -- through
// a 4-deep shared-memory ring continuously across items; warps 1-4 each own 16
// tokens of every page: S = Q K^T and O += P V on m16n8k16 tensor cores with Q =
// the GQA group padded to 16 rows (fragments loaded straight from global), per-warp
// online softmax, warps merged in shared memory.  A request's context is cut into
// ceil(pages / 16) even splits (its own length only -- batch invariant); the last
// split CTA to finish merges the splits in split order.  PDL: pages that were
// complete before this step are streamed before griddepcontrol.wait; only the page
// holding the newest token waits for the predecessor kernel.

constexpr int PAGE = 64;                 // tokens per KV block
// Pages per split of a request's context (pages spread evenly over ceil(pages / pps)
// splits).  Depends on the request's own length only, so a request's result never
// depends on the batch it rides in.  PL_ATTN_PPS overrides (experiments).
int attn_pages_per_split() {
  static const int v = [] {
    const char* e = getenv("PL_ATTN_PPS");
    const int x = e ? atoi(e) : 16;
    return (x > 0 && x <= 32) ? x : 16;  // <= 32: block-table entries travel one per lane
  }();
  return v;
}
constexpr int HALF_TILE = 64 * 128;      // 64 tokens x 64 dims bf16 (one TMA box)
constexpr int PAGE_BYTES = 4 * HALF_TILE;  // K lo | K hi | V lo | V hi
constexpr int DEC_THREADS = 160;         // producer warp + 4 consumer warps
constexpr int Q_PITCH = HD * 2 + 16;     // padded q row in shared memory (conflict-free)
constexpr int Q_SLOTS = 2;

struct ItemInfo {
  int r, kh, split, p0, np, ctx, pad0, pad1;
};

template <int G>
struct DecodeSmem {
  static constexpr int STAGES = G <= 4 ? 3 : 2;               // 2 CTAs per SM either way
  static constexpr int Q = STAGES * PAGE_BYTES;                // [Q_SLOTS][G][Q_PITCH]
  static constexpr int INFO = Q + Q_SLOTS * G * Q_PITCH;       // [Q_SLOTS] ItemInfo
  static constexpr int RED_O = INFO + Q_SLOTS * 32;            // [4 warps][G][128] fp32
  static constexpr int RED_M = RED_O + 4 * G * HD * 4;         // [4][G]
  static constexpr int RED_L = RED_M + 4 * G * 4;              // [4][G]
  static constexpr int BAR = (RED_L + 4 * G * 4 + 7) & ~7;     // full[S], empty[S], qfull[2], qempty[2]
  static constexpr int FLAG = BAR + 8 * (2 * STAGES + 2 * Q_SLOTS);
  static constexpr int TOTAL = FLAG + 16 + 1024;               // + alignment slack
};

// address of 16-byte chunk `c` (0..15) of token row `row` in a (lo|hi) 128B-swizzled pair
PL_DEV uint32_t kv_addr(uint32_t base, int row, int c) {
  return base + (c >> 3) * HALF_TILE + row * 128 + (((c & 7) ^ (row & 7)) << 4);
}

struct DecodeArgs {
  const __nv_bfloat16* q;
  int64_t ldq;
  const int32_t* block_table;
  int max_blocks;
  const int32_t* ctx_len;
  int R, Hkv, nsplit;
  int pps;  // pages per split
  float scale_log2;
  __nv_bfloat16* out;
  int64_t ldo;
  float* ws_o;
  float2* ws_ml;
  int* counters;
};

// Geometry of item `it` given its request's context length: pages [p0, p0 + np)
// of request r, kv head kh, split `split`; n_pages = the request's page count.
struct ItemGeom {
  int r, kh, split, p0, np, n_pages, ctx;
};
PL_DEV ItemGeom decode_geom(const DecodeArgs& a, int it, int ctx) {
  ItemGeom g;
  g.split = it % a.nsplit;
  g.kh = (it / a.nsplit) % a.Hkv;
  g.r = it / (a.nsplit * a.Hkv);
  g.ctx = ctx;
  g.n_pages = (ctx + PAGE - 1) / PAGE;
  const int ns_r = max(1, (g.n_pages + a.pps - 1) / a.pps);
  const int pps = (g.n_pages + ns_r - 1) / ns_r;
  g.p0 = g.split * pps;
  g.np = max(0, min(g.n_pages, g.p0 + pps) - g.p0);
  return g;
}

PL_DEV int atomic_add_acq_rel_gpu(int* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// Persistent: 2 CTAs per SM walk the (request, kv head, split) items.  Warp 0 is
// the producer, one item ahead: the context lengths of all of the CTA's items
// come in one warp-wide load, the next item's block-table entries (<= 8, one per
// lane) load while the current item's pages stream, and the next item's q (G
// rows, 1-D bulk copies into a 2-slot ring, with the item geometry) is issued
// before the current item's pages.  K/V pages (4 TMA boxes each) go through a
// STAGES-deep ring.  Warps 1-4 never touch global memory until the output:
// S = Q K^T and O += P V on m16n8k16 tensor cores with Q = the GQA group padded
// to 16 rows, per-warp online softmax, warps merged in shared memory.
template <int G>
__global__ void __launch_bounds__(DEC_THREADS, 2)
    attn_decode_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                       const DecodeArgs args) {
  using L = DecodeSmem<G>;
  constexpr int STAGES = L::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  float* red_o = reinterpret_cast<float*>(smem + L::RED_O);
  float* red_m = reinterpret_cast<float*>(smem + L::RED_M);
  float* red_l = reinterpret_cast<float*>(smem + L::RED_L);
  ItemInfo* info = reinterpret_cast<ItemInfo*>(smem + L::INFO);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* empty = full + STAGES;
  uint64_t* qfull = empty + STAGES;
  uint64_t* qempty = qfull + Q_SLOTS;
  int* last_flag = reinterpret_cast<int*>(smem + L::FLAG);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = args.R * args.Hkv * args.nsplit;
  if (threadIdx.x == 0) PL_TL(3u << 24, 0);

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    for (int s = 0; s < Q_SLOTS; ++s) {
      mbar_init(&qfull[s], 1);
      mbar_init(&qempty[s], 4);
    }
    fence_mbar_init();
  }
  __syncthreads();
  pdl_trigger();

  if (warp == 0) {
    // ------------------------------------------------------- producer warp
    if (blockIdx.x >= n_items) {
      if (lane == 0) pdl_wait();
      return;
    }
    const uint64_t pol = policy_evict_first();
    int stage = 0, qs = 0;
    uint32_t phase = 0, qphase = 0;
    // context lengths of this CTA's items k = 0..31: lane k holds item blockIdx.x + k*grid
    int ctx_batch = 0, batch_base = -1;
    auto ctx_of = [&](int k) -> int {  // warp-collective
      if ((k & ~31) != batch_base) {
        batch_base = k & ~31;
        const int itl = blockIdx.x + (batch_base + lane) * gridDim.x;
        ctx_batch = itl < n_items ? __ldg(args.ctx_len + itl / (args.nsplit * args.Hkv)) : 0;
      }
      return __shfl_sync(0xffffffffu, ctx_batch, k & 31);
    };
    auto bt_of = [&](const ItemGeom& g) -> int {  // lane i: page p0 + i (warp-collective)
      return lane < g.np ? __ldg(args.block_table + static_cast<int64_t>(g.r) * args.max_blocks + g.p0 + lane)
                         : 0;
    };
    auto issue_q = [&](const ItemGeom& g) {  // lane 0
      mbar_wait(&qempty[qs], qphase ^ 1);
      info[qs] = ItemInfo{g.r, g.kh, g.split, g.p0, g.np, g.ctx, 0, 0};
      uint8_t* qd = smem + L::Q + qs * G * Q_PITCH;
      const __nv_bfloat16* qsrc = args.q + static_cast<int64_t>(g.r) * args.ldq + g.kh * G * HD;
      mbar_arrive_expect_tx(&qfull[qs], G * HD * 2);
#pragma unroll
      for (int h = 0; h < G; ++h) bulk_load(qd + h * Q_PITCH, qsrc + h * HD, HD * 2, &qfull[qs]);
      if (++qs == Q_SLOTS) {
        qs = 0;
        qphase ^= 1;
      }
    };
    auto issue_page = [&](int page, int kh) {  // lane 0
      mbar_wait(&empty[stage], phase ^ 1);
      const int row0 = (page * args.Hkv + kh) * PAGE;
      uint8_t* dst = smem + stage * PAGE_BYTES;
      mbar_arrive_expect_tx(&full[stage], PAGE_BYTES);
      tma_load_2d(dst, &tmK, &full[stage], 0, row0, pol);
      tma_load_2d(dst + HALF_TILE, &tmK, &full[stage], 64, row0, pol);
      tma_load_2d(dst + 2 * HALF_TILE, &tmV, &full[stage], 0, row0, pol);
      tma_load_2d(dst + 3 * HALF_TILE, &tmV, &full[stage], 64, row0, pol);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
    };

    // first item: pages complete before this step stream ahead of griddepcontrol.wait;
    // the page holding the newest token (the request's last) and q come from the predecessor
    ItemGeom cur = decode_geom(args, blockIdx.x, ctx_of(0));
    int cur_bt = bt_of(cur);
    int pre = 0;
    {
      const int cold = cur.np - (cur.p0 + cur.np == cur.n_pages ? 1 : 0);
      pre = max(0, min(cold, STAGES));
      for (int i = 0; i < pre; ++i) {
        const int pg = __shfl_sync(0xffffffffu, cur_bt, i);
        if (lane == 0) issue_page(pg, cur.kh);
      }
      if (lane == 0) {
        pdl_wait();
        PL_TL(3u << 24, 2);  // predecessor complete
        issue_q(cur);
      }
    }
    for (int k = 0;; ++k) {
      const int it = blockIdx.x + k * gridDim.x;
      const int nx = it + gridDim.x;
      const bool has_next = nx < n_items;
      ItemGeom nxt{};
      int nxt_bt = 0;
      if (has_next) {
        nxt = decode_geom(args, nx, ctx_of(k + 1));
        nxt_bt = bt_of(nxt);  // in flight while this item's pages stream
        if (lane == 0) issue_q(nxt);
      }
      for (int i = pre; i < cur.np; ++i) {
        const int pg = __shfl_sync(0xffffffffu, cur_bt, i);
        if (lane == 0) issue_page(pg, cur.kh);
      }
      pre = 0;
      if (!has_next) break;
      cur = nxt;
      cur_bt = nxt_bt;
    }
    return;
  }

  // --------------------------------------------------------- consumers (warps 1-4)
  // Transposed tiles ("swap AB" for small GQA groups): S^T = K Q^T with M = 16
  // tokens, N = 8 query heads (the group, zero-padded), K = hd; O^T = V^T P^T with
  // M = 16 head dims, N = 8 heads, K = 16 tokens.  Half the MMAs and half the
  // accumulator registers of the Q-rows-as-M form when G <= 8.
  const int cw = warp - 1;  // consumer warp: tokens [16 cw, 16 cw + 16) of every page
  const int ct = threadIdx.x - 32;
  const int mi = lane >> 3, ri = lane & 7;
  const int g8 = lane >> 2, t4 = lane & 3;  // fragment row group / column pair
  int stage = 0, qs = 0;
  uint32_t phase = 0, qphase = 0;
  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    mbar_wait(&qfull[qs], qphase);
    const ItemInfo inf = info[qs];
    const int r = inf.r, kh = inf.kh, split = inf.split, p0 = inf.p0, np = inf.np, ctx = inf.ctx;
    // B fragments of Q^T: head g8 (zero when g8 >= G), dims 16 ks + 2 t4 (+8)
    uint32_t qf[8][2];
    {
      const uint8_t* qb = smem + L::Q + qs * G * Q_PITCH + g8 * Q_PITCH;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const int off = (ks * 16 + t4 * 2) * 2;
        qf[ks][0] = g8 < G ? *reinterpret_cast<const uint32_t*>(qb + off) : 0u;
        qf[ks][1] = g8 < G ? *reinterpret_cast<const uint32_t*>(qb + off + 16) : 0u;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&qempty[qs]);
    if (++qs == Q_SLOTS) {
      qs = 0;
      qphase ^= 1;
    }
    float o[8][4];  // O^T: dims 16 mt + g8 (+8) x heads 2 t4 (+1)
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};  // heads 2 t4, 2 t4 + 1

    for (int i = 0; i < np; ++i) {
      mbar_wait(&full[stage], phase);
#ifdef PL_TIMELINE
      if (ct == 0 && i == np - 1 && it + static_cast<int>(gridDim.x) >= n_items) PL_TL(3u << 24, 3);  // last page in
#endif
      const uint32_t kb = smem_u32(smem + stage * PAGE_BYTES);
      const uint32_t vb = kb + 2 * HALF_TILE;
      float s[4] = {0.f, 0.f, 0.f, 0.f};  // tokens g8, g8+8 x heads 2 t4, 2 t4 + 1
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        uint32_t a[4];
        ldmatrix_x4(a[0], a[1], a[2], a[3], kv_addr(kb, cw * 16 + (mi & 1) * 8 + ri, ks * 2 + (mi >> 1)));
        mma_bf16_16816(s, a, qf[ks][0], qf[ks][1]);
      }
      const int tok0 = (p0 + i) * PAGE + cw * 16;
      if (tok0 + 16 <= ctx) {
#pragma unroll
        for (int e = 0; e < 4; ++e) s[e] *= args.scale_log2;
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) s[e] = (tok0 + g8 + (e >> 1) * 8 < ctx) ? s[e] * args.scale_log2 : -INFINITY;
      }
      float corr[2], rs[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // reduce over the 16 tokens: lanes sharing t4
        float mx = fmaxf(s[h], s[h + 2]);
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
        const float m_new = fmaxf(m_r[h], mx);
        corr[h] = (m_new == -INFINITY) ? 1.f : exp2f(m_r[h] - m_new);
        m_r[h] = m_new;
        const float pa = (m_new == -INFINITY) ? 0.f : exp2f(s[h] - m_new);
        const float pb = (m_new == -INFINITY) ? 0.f : exp2f(s[h + 2] - m_new);
        s[h] = pa;
        s[h + 2] = pb;
        rs[h] = pa + pb;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        rs[h] += __shfl_xor_sync(0xffffffffu, rs[h], 4);
        rs[h] += __shfl_xor_sync(0xffffffffu, rs[h], 8);
        rs[h] += __shfl_xor_sync(0xffffffffu, rs[h], 16);
        l_r[h] = l_r[h] * corr[h] + rs[h];
      }
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        o[mt][0] *= corr[0];
        o[mt][1] *= corr[1];
        o[mt][2] *= corr[0];
        o[mt][3] *= corr[1];
      }
      // P^T as the B operand: transpose the two 8x8 (token x head) blocks in registers
      uint32_t pb0 = pack_bf16x2(s[0], s[1]), pb1 = pack_bf16x2(s[2], s[3]);
      asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %0;" : "+r"(pb0));
      asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %0;" : "+r"(pb1));
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        uint32_t a[4];
        ldmatrix_x4_trans(a[0], a[1], a[2], a[3], kv_addr(vb, cw * 16 + (mi >> 1) * 8 + ri, mt * 2 + (mi & 1)));
        mma_bf16_16816(o[mt], a, pb0, pb1);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);  // this warp is done with the stage
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }

    // merge the four consumer warps (heads >= G are padding)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int head = t4 * 2 + h;
      if (head < G) {
        if (g8 == 0) {
          red_m[cw * G + head] = m_r[h];
          red_l[cw * G + head] = l_r[h];
        }
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          red_o[(cw * G + head) * HD + mt * 16 + g8] = o[mt][h];
          red_o[(cw * G + head) * HD + mt * 16 + g8 + 8] = o[mt][h + 2];
        }
      }
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    const int e = ct;  // head dim owned in the merge
    const int nsplit = args.nsplit;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < 4; ++w) M = fmaxf(M, red_m[w * G + g]);
      float Lsum = 0.f, O = 0.f;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const float mw = red_m[w * G + g];
        if (mw == -INFINITY) continue;
        const float f = exp2f(mw - M);
        Lsum += red_l[w * G + g] * f;
        O += red_o[(w * G + g) * HD + e] * f;
      }
      const int head = kh * G + g;
      if (nsplit == 1) {
        args.out[static_cast<int64_t>(r) * args.ldo + head * HD + e] = f2bf(Lsum > 0.f ? O / Lsum : 0.f);
      } else {
        const int64_t base = (static_cast<int64_t>(r) * args.Hkv * G + head) * nsplit + split;
        args.ws_o[base * HD + e] = O;
        if (e == 0) args.ws_ml[base] = make_float2(M, Lsum);
      }
    }
    if (nsplit > 1) {
      // last split of (request, kv head) to finish merges every split in split order;
      // one acq_rel atomic orders this CTA's partials (published to thread 0 by the
      // barrier) before the arrival, and the merger's loads after it
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (ct == 0)
        *last_flag = atomic_add_acq_rel_gpu(&args.counters[-1 - (r * args.Hkv + kh)], 1) == nsplit - 1;
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (*last_flag) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int head = kh * G + g;
          const int64_t base = (static_cast<int64_t>(r) * args.Hkv * G + head) * nsplit;
          // four splits' loads in flight per round: unconditional weak loads (split
          // index clamped), ordered after the other splits' writes by the acq_rel
          // arrival + barrier; merged in split order as before
          constexpr int MB = 4;
          float M = -INFINITY;
          for (int s0 = 0; s0 < nsplit; s0 += MB) {
            float mx[MB];
#pragma unroll
            for (int u = 0; u < MB; ++u) mx[u] = args.ws_ml[base + min(s0 + u, nsplit - 1)].x;
#pragma unroll
            for (int u = 0; u < MB; ++u) M = fmaxf(M, mx[u]);  // clamped repeats are harmless
          }
          float Lsum = 0.f, O = 0.f;
          for (int s0 = 0; s0 < nsplit; s0 += MB) {
            float2 ml[MB];
            float ov[MB];
#pragma unroll
            for (int u = 0; u < MB; ++u) {
              const int64_t sb = base + min(s0 + u, nsplit - 1);
              ml[u] = args.ws_ml[sb];
              ov[u] = args.ws_o[sb * HD + e];
            }
#pragma unroll
            for (int u = 0; u < MB; ++u) {
              if (s0 + u >= nsplit) break;
              if (ml[u].x == -INFINITY) continue;
              const float w = exp2f(ml[u].x - M);
              Lsum += ml[u].y * w;
              O += ov[u] * w;
            }
          }
          args.out[static_cast<int64_t>(r) * args.ldo + head * HD + e] =
              f2bf(Lsum > 0.f ? O / Lsum : 0.f);
        }
        if (ct == 0) args.counters[-1 - (r * args.Hkv + kh)] = 0;
      }
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");  // red_* reused by the next item
  }
  if (ct == 0) PL_TL(3u << 24, 1);  // after the final consumer barrier
}

// Workspace: [o partials | (m, l) partials | ... free ... | arrival counters].  The
// counters sit at the END of the buffer, slot i at word -(1 + i), so a counter's
// address depends only on (r, kv head) and the buffer size -- never on this launch's R
// or max_ctx.  They must read zero between launches (the merger resets its own); the
// partials of any launch that fits the workspace end below every counter slot of any
// other launch that fits it (the size below reserves R*Hq words for counters), so
// launches of different shapes can share one workspace sized for the largest.
int64_t attn_decode_workspace_bytes(int R, int Hq, int max_ctx, int hd) {
  const int pages = (max_ctx + PAGE - 1) / PAGE;
  const int nsplit = std::max(1, (pages + attn_pages_per_split() - 1) / attn_pages_per_split());
  if (nsplit == 1) return 0;
  const int64_t counters = ((static_cast<int64_t>(R) * Hq * 4 + 255) / 256) * 256;
  return counters + static_cast<int64_t>(R) * Hq * nsplit * (hd * 4 + 8);
}

int attn_decode_launch(const __nv_bfloat16* q, int64_t ldq, const __nv_bfloat16* k_cache,
                       const __nv_bfloat16* v_cache, int64_t num_blocks, int block_size,
                       const int32_t* block_table, int max_blocks, const int32_t* ctx_len, int R,
                       int max_ctx, int Hq, int Hkv, int hd, float scale, __nv_bfloat16* out,
                       int64_t ldo, void* ws, int64_t ws_bytes, cudaStream_t st) {
  if (R <= 0) return PL_OK;
  if (hd != HD) return set_error(PL_ERR_CONFIG, "attention: head_dim must be 128 (got %d)", hd);
  if (block_size != PAGE) return set_error(PL_ERR_CONFIG, "attention: KV block size must be 64");
  if (Hkv <= 0 || Hq % Hkv) return set_error(PL_ERR_CONFIG, "attention: Hq must be a multiple of Hkv");
  if (num_blocks <= 0) return set_error(PL_ERR_CONFIG, "attention: num_blocks must be > 0");
  if (ldq % 8) return set_error(PL_ERR_CONFIG, "attention: ldq % 8");
  const int G = Hq / Hkv;
  const int pages = (max_ctx + PAGE - 1) / PAGE;
  const int nsplit = std::max(1, (pages + attn_pages_per_split() - 1) / attn_pages_per_split());
  const int64_t need = attn_decode_workspace_bytes(R, Hq, max_ctx, hd);
  if (need > 0 && (ws_bytes < need || !ws))
    return set_error(PL_ERR_CONFIG, "attn_decode: workspace too small (%lld < %lld)",
                     (long long)ws_bytes, (long long)need);
  CUtensorMap mk, mv;
  int rc;
  const int64_t rows = num_blocks * Hkv * PAGE;
  if ((rc = make_tma_2d(&mk, k_cache, rows, HD, HD, 64))) return rc;
  if ((rc = make_tma_2d(&mv, v_cache, rows, HD, HD, 64))) return rc;
  int* counters = need > 0 ? reinterpret_cast<int*>(static_cast<uint8_t*>(ws) + (ws_bytes & ~int64_t(3)))
                           : nullptr;  // one past the last word; slot i at counters[-1 - i]
  float* ws_o = need > 0 ? reinterpret_cast<float*>(ws) : nullptr;
  float2* ws_ml = need > 0 ? reinterpret_cast<float2*>(reinterpret_cast<uint8_t*>(ws_o) +
                                                       static_cast<int64_t>(R) * Hq * nsplit * hd * 4)
                           : nullptr;
  DecodeArgs da;
  da.q = q;
  da.ldq = ldq;
  da.block_table = block_table;
  da.max_blocks = max_blocks;
  da.ctx_len = ctx_len;
  da.R = R;
  da.Hkv = Hkv;
  da.nsplit = nsplit;
  da.pps = attn_pages_per_split();
  da.scale_log2 = scale * LOG2E;
  da.out = out;
  da.ldo = ldo;
  da.ws_o = ws_o;
  da.ws_ml = ws_ml;
  da.counters = counters;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int items = R * Hkv * nsplit;
  const dim3 grid(std::min(items, 2 * sms));  // persistent: two CTAs per SM
#define PL_DECODE_CASE(GG)                                                                      \
  case GG: {                                                                                    \
    constexpr int smem = DecodeSmem<GG>::TOTAL;                                                 \
    if ((rc = ensure_smem_attr(reinterpret_cast<const void*>(attn_decode_kernel<GG>), smem,          \
                               "attn_decode smem attribute")))                                  \
      return rc;                                                                                \
    rc = launch_k("attn_decode_kernel", attn_decode_kernel<GG>, grid, dim3(DEC_THREADS), smem,  \
                  st, mk, mv, da);                                                              \
    break;                                                                                      \
  }
  switch (G) {
    PL_DECODE_CASE(1)
    PL_DECODE_CASE(2)
    PL_DECODE_CASE(4)
    PL_DECODE_CASE(8)
    default:
      return set_error(PL_ERR_CONFIG, "attn_decode: GQA group %d unsupported (1,2,4,8)", G);
  }
#undef PL_DECODE_CASE
  return rc;
}


#ifdef PL_TIMELINE
int tl_set_attn(void* buf, void* count, unsigned cap) {
  TimelineSink t{static_cast<unsigned long long*>(buf), static_cast<unsigned*>(count), cap};
  return cudaMemcpyToSymbol(g_tl, &t, sizeof(t)) == cudaSuccess ? PL_OK : PL_ERR_CUDA;
}
#endif

// Load every kernel of this file into the context now (lazy module loading would
// otherwise load it at first launch, which can wait on a spinning NCCL kernel).
template <typename K>
static int preload_one(K k, const char* name) {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, k);
  return e == cudaSuccess ? PL_OK : set_cuda_error(e, name);
}

int attention_preload() {
  int rc = preload_one(attn_prefill_kernel, "attn_prefill_kernel");
  if (!rc) rc = preload_one(attn_decode_kernel<1>, "attn_decode_kernel");
  if (!rc) rc = preload_one(attn_decode_kernel<2>, "attn_decode_kernel");
  if (!rc) rc = preload_one(attn_decode_kernel<4>, "attn_decode_kernel");
  if (!rc) rc = preload_one(attn_decode_kernel<8>, "attn_decode_kernel");
  return rc;
}

}  // namespace pl
