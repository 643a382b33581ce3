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
//   arrive by TMA into 128-byte-swizzled shared memory; QK^T and PV run on
//   m16n8k16 tensor cores; a request's context is cut into ceil(pages/8)
//   even splits, so the reduction order depends on its own context length
//   only, never on the batch.
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

PL_DEV void load_tile_64x128(uint8_t* smem, const __nv_bfloat16* base, int64_t ld, int rows_valid) {
  // 64 rows x 16 chunks = 1024 chunks, 8 per thread
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int c = threadIdx.x + i * 128;
    const int row = c >> 4, ch = c & 15;
    const bool ok = row < rows_valid;
    const __nv_bfloat16* src = base + (ok ? static_cast<int64_t>(row) * ld : 0) + ch * 8;
    cp_async16_zfill(smem + swz(row, ch), src, ok);
  }
}

__global__ void __launch_bounds__(128, 2)
    attn_prefill_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t ldqkv,
                        const int32_t* __restrict__ cu_seqlens, int Hq, int Hkv, float scale_log2,
                        __nv_bfloat16* __restrict__ out, int64_t ldo) {
  extern __shared__ uint8_t smem_raw[];
  pdl_trigger();
  pdl_wait();
  uint8_t* sQ = smem_raw;                 // 16 KB
  uint8_t* sK = smem_raw + 16384;         // 2 x 16 KB
  uint8_t* sV = smem_raw + 16384 * 3;     // 2 x 16 KB

  const int r = blockIdx.z, h = blockIdx.y;
  const int seq0 = cu_seqlens[r];
  const int L = cu_seqlens[r + 1] - seq0;
  const int q0 = blockIdx.x * 64;
  if (q0 >= L) return;
  const int kh = h / (Hq / Hkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const __nv_bfloat16* qbase = qkv + static_cast<int64_t>(seq0 + q0) * ldqkv + h * HD;
  const __nv_bfloat16* kbase = qkv + static_cast<int64_t>(seq0) * ldqkv + (Hq + kh) * HD;
  const __nv_bfloat16* vbase = qkv + static_cast<int64_t>(seq0) * ldqkv + (Hq + Hkv + kh) * HD;

  const int q_hi = min(q0 + 64, L);          // exclusive
  const int n_kv_tiles = (q_hi + 63) / 64;   // causal: keys < q_hi

  load_tile_64x128(sQ, qbase, ldqkv, q_hi - q0);
  load_tile_64x128(sK, kbase, ldqkv, min(64, L));
  load_tile_64x128(sV, vbase, ldqkv, min(64, L));
  cp_async_commit();

  // Q fragments for this warp's 16 rows: 8 k-steps x 4 regs
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
      load_tile_64x128(sK + (buf ^ 1) * 16384, kbase + static_cast<int64_t>(kv0) * ldqkv, ldqkv,
                       min(64, L - kv0));
      load_tile_64x128(sV + (buf ^ 1) * 16384, vbase + static_cast<int64_t>(kv0) * ldqkv, ldqkv,
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
    const int kv0 = j * 64;
    const int qrow0 = q0 + warp * 16 + (lane >> 2);
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
    __syncthreads();
  }

  // normalize and store
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
    const int qi = q0 + warp * 16 + (lane >> 2) + hr * 8;
    if (qi >= L) continue;
    const float inv = l_r[hr] > 0.f ? 1.f / l_r[hr] : 0.f;
    __nv_bfloat16* orow = out + static_cast<int64_t>(seq0 + qi) * ldo + h * HD;
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      const int col = nt * 8 + (lane & 3) * 2;
      *reinterpret_cast<uint32_t*>(orow + col) =
          pack_bf16x2(o[nt][hr * 2] * inv, o[nt][hr * 2 + 1] * inv);
    }
  }
}

int attn_prefill_launch(const __nv_bfloat16* qkv, int64_t ldqkv, const int32_t* cu_seqlens, int R,
                        int max_seqlen, int Hq, int Hkv, int hd, float scale, __nv_bfloat16* out,
                        int64_t ldo, cudaStream_t st) {
  if (R <= 0 || max_seqlen <= 0) return PL_OK;
  if (hd != HD) return set_error(PL_ERR_CONFIG, "attention: head_dim must be 128 (got %d)", hd);
  if (Hkv <= 0 || Hq % Hkv) return set_error(PL_ERR_CONFIG, "attention: Hq must be a multiple of Hkv");
  if (ldqkv % 8 || ldo % 8) return set_error(PL_ERR_CONFIG, "attention: leading dims % 8");
  constexpr int smem = 16384 * 5;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_prefill_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_cuda_error(e, "attn_prefill smem attribute");
    attr = true;
  }
  dim3 grid((max_seqlen + 63) / 64, Hq, R);
  return launch_k("attn_prefill_kernel", attn_prefill_kernel, grid, dim3(128), smem, st, qkv, ldqkv,
                  cu_seqlens, Hq, Hkv, scale * LOG2E, out, ldo);
}

// ======================================================= decode (paged)
//
// One CTA per (kv head, request, split of <= 8 pages).  A single thread streams
// each 64-token K and V page into shared memory with four 2-D TMA boxes
// (64 dims x 64 tokens, 128-byte swizzle) completing on an mbarrier; the four
// warps then each take 16 tokens of the page: S = Q K^T and O += P V on
// m16n8k16 tensor cores with Q = the GQA group padded to 16 rows.  Every warp
// keeps its own online-softmax state; warps are merged in shared memory and
// splits by attn_decode_combine_kernel, both in a fixed order.

constexpr int PAGE = 64;                 // tokens per KV block
constexpr int MAX_PAGES_PER_SPLIT = 8;   // <= 512 tokens per split, pages spread evenly
constexpr int DEC_STAGES = 3;
constexpr int HALF_TILE = 64 * 128;      // 64 tokens x 64 dims bf16 (one TMA box)
constexpr int PAGE_BYTES = 4 * HALF_TILE;  // K lo | K hi | V lo | V hi

struct DecodeSmem {
  static constexpr int Q_OFF = DEC_STAGES * PAGE_BYTES;        // 16 x 128 bf16, 256 B rows
  static constexpr int BAR_OFF = Q_OFF + 16 * 256;
  static constexpr int TOTAL = BAR_OFF + 64 + 1024;            // + alignment slack
};

// address of 16-byte chunk `c` (0..15) of token row `row` in a (lo|hi) 128B-swizzled pair
PL_DEV uint32_t kv_addr(uint32_t base, int row, int c) {
  return base + (c >> 3) * HALF_TILE + row * 128 + (((c & 7) ^ (row & 7)) << 4);
}

template <int G>
__global__ void __launch_bounds__(128)
    attn_decode_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                       const __nv_bfloat16* __restrict__ q, int64_t ldq,
                       const int32_t* __restrict__ block_table, int max_blocks,
                       const int32_t* __restrict__ ctx_len, int Hkv, float scale_log2,
                       __nv_bfloat16* __restrict__ out, int64_t ldo, float* __restrict__ ws_o,
                       float2* __restrict__ ws_ml, int* __restrict__ counters) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem + DecodeSmem::Q_OFF;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + DecodeSmem::BAR_OFF);

  const int kh = blockIdx.x, r = blockIdx.y, split = blockIdx.z, nsplit = gridDim.z;
  const int Hq = Hkv * G;
  const int ctx = ctx_len[r];
  // split layout depends on this request's context only (batch invariance)
  const int n_pages = (ctx + PAGE - 1) / PAGE;
  const int ns_r = max(1, (n_pages + MAX_PAGES_PER_SPLIT - 1) / MAX_PAGES_PER_SPLIT);
  const int pps = (n_pages + ns_r - 1) / ns_r;
  const int p0 = split * pps;
  const int np = max(0, min(n_pages, p0 + pps) - p0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t* bt = block_table + static_cast<int64_t>(r) * max_blocks;

  auto issue = [&](int i) {
    const int st = i % DEC_STAGES;
    const int row0 = (bt[p0 + i] * Hkv + kh) * PAGE;
    uint8_t* dst = smem + st * PAGE_BYTES;
    mbar_arrive_expect_tx(&full[st], PAGE_BYTES);
    const uint64_t pol = policy_evict_first();
    tma_load_2d(dst, &tmK, &full[st], 0, row0, pol);
    tma_load_2d(dst + HALF_TILE, &tmK, &full[st], 64, row0, pol);
    tma_load_2d(dst + 2 * HALF_TILE, &tmV, &full[st], 0, row0, pol);
    tma_load_2d(dst + 3 * HALF_TILE, &tmV, &full[st], 64, row0, pol);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < DEC_STAGES; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    for (int i = 0; i < min(np, DEC_STAGES); ++i) issue(i);
  }
  // Q tile: rows g < G are the group's query heads, rows G..15 zero
  for (int c = threadIdx.x; c < 16 * 16; c += 128) {
    const int row = c >> 4, ch = c & 15;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (row < G) v = *reinterpret_cast<const uint4*>(q + static_cast<int64_t>(r) * ldq + (kh * G + row) * HD + ch * 8);
    *reinterpret_cast<uint4*>(sQ + swz(row, ch)) = v;
  }
  __syncthreads();
  const int mi = lane >> 3, ri = lane & 7;
  uint32_t qf[8][4];
#pragma unroll
  for (int ks = 0; ks < 8; ++ks)
    ldmatrix_x4(qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3],
                smem_u32(sQ) + swz((mi & 1) * 8 + ri, ks * 2 + (mi >> 1)));

  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};

  for (int i = 0; i < np; ++i) {
    const int st = i % DEC_STAGES;
    mbar_wait(&full[st], (i / DEC_STAGES) & 1);
    const uint32_t kb = smem_u32(smem + st * PAGE_BYTES);
    const uint32_t vb = kb + 2 * HALF_TILE;
    float s[2][4];
#pragma unroll
    for (int t = 0; t < 2; ++t) s[t][0] = s[t][1] = s[t][2] = s[t][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      uint32_t b0, b1, b2, b3;
      ldmatrix_x4(b0, b1, b2, b3, kv_addr(kb, warp * 16 + (mi >> 1) * 8 + ri, ks * 2 + (mi & 1)));
      mma_bf16_16816(s[0], qf[ks], b0, b1);
      mma_bf16_16816(s[1], qf[ks], b2, b3);
    }
    const int tok0 = (p0 + i) * PAGE + warp * 16;
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = tok0 + t * 8 + (lane & 3) * 2 + (e & 1);
        const float v = (j < ctx) ? s[t][e] * scale_log2 : -INFINITY;
        s[t][e] = v;
        mx[e >> 1] = fmaxf(mx[e >> 1], v);
      }
    float corr[2], rs[2] = {0.f, 0.f};
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      mx[hr] = fmaxf(mx[hr], __shfl_xor_sync(0xffffffffu, mx[hr], 1));
      mx[hr] = fmaxf(mx[hr], __shfl_xor_sync(0xffffffffu, mx[hr], 2));
      const float m_new = fmaxf(m_r[hr], mx[hr]);
      corr[hr] = (m_new == -INFINITY) ? 1.f : exp2f(m_r[hr] - m_new);
      m_r[hr] = m_new;
    }
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int hr = e >> 1;
        const float p = (m_r[hr] == -INFINITY) ? 0.f : exp2f(s[t][e] - m_r[hr]);
        s[t][e] = p;
        rs[hr] += p;
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
    uint32_t a[4];
    a[0] = pack_bf16x2(s[0][0], s[0][1]);
    a[1] = pack_bf16x2(s[0][2], s[0][3]);
    a[2] = pack_bf16x2(s[1][0], s[1][1]);
    a[3] = pack_bf16x2(s[1][2], s[1][3]);
#pragma unroll
    for (int nt = 0; nt < 16; nt += 2) {
      uint32_t b0, b1, b2, b3;
      ldmatrix_x4_trans(b0, b1, b2, b3, kv_addr(vb, warp * 16 + (mi & 1) * 8 + ri, nt + (mi >> 1)));
      mma_bf16_16816(o[nt], a, b0, b1);
      mma_bf16_16816(o[nt + 1], a, b2, b3);
    }
    __syncthreads();  // every warp is done with stage st
    if (threadIdx.x == 0 && i + DEC_STAGES < np) issue(i + DEC_STAGES);
  }

  // merge the four warps' softmax states (shared memory reused: all loads consumed)
  float* red_o = reinterpret_cast<float*>(smem);               // [4][16][128]
  float* red_m = red_o + 4 * 16 * HD;                           // [4][16]
  float* red_l = red_m + 4 * 16;                                // [4][16]
  __syncthreads();
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
    const int row = (lane >> 2) + hr * 8;
    if ((lane & 3) == 0) {
      red_m[warp * 16 + row] = m_r[hr];
      red_l[warp * 16 + row] = l_r[hr];
    }
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      const int col = nt * 8 + (lane & 3) * 2;
      red_o[(warp * 16 + row) * HD + col] = o[nt][hr * 2];
      red_o[(warp * 16 + row) * HD + col + 1] = o[nt][hr * 2 + 1];
    }
  }
  __syncthreads();
  const int e = threadIdx.x;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) M = fmaxf(M, red_m[w * 16 + g]);
    float L = 0.f, O = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float mw = red_m[w * 16 + g];
      if (mw == -INFINITY) continue;
      const float f = exp2f(mw - M);
      L += red_l[w * 16 + g] * f;
      O += red_o[(w * 16 + g) * HD + e] * f;
    }
    const int head = kh * G + g;
    if (nsplit == 1) {
      out[static_cast<int64_t>(r) * ldo + head * HD + e] = f2bf(L > 0.f ? O / L : 0.f);
    } else {
      const int64_t base = (static_cast<int64_t>(r) * Hq + head) * nsplit + split;
      ws_o[base * HD + e] = O;
      if (e == 0) ws_ml[base] = make_float2(M, L);
    }
  }
  if (nsplit == 1) return;

  // Split merge fused in: the last split CTA of this (request, kv head) to finish
  // combines every split's state in split order (deterministic) and resets the counter.
  __shared__ int last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&counters[r * Hkv + kh], 1) == nsplit - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int head = kh * G + g;
    const int64_t base = (static_cast<int64_t>(r) * Hq + head) * nsplit;
    float M = -INFINITY;
    for (int s = 0; s < nsplit; ++s) M = fmaxf(M, __ldcg(&ws_ml[base + s]).x);
    float Lsum = 0.f, o = 0.f;
    for (int s = 0; s < nsplit; ++s) {
      const float2 ml = __ldcg(&ws_ml[base + s]);
      if (ml.x == -INFINITY) continue;
      const float w = exp2f(ml.x - M);
      Lsum += ml.y * w;
      o += __ldcg(&ws_o[(base + s) * HD + e]) * w;
    }
    out[static_cast<int64_t>(r) * ldo + head * HD + e] = f2bf(Lsum > 0.f ? o / Lsum : 0.f);
  }
  if (threadIdx.x == 0) counters[r * Hkv + kh] = 0;
}

// Workspace: [R*Hkv arrival counters, zero between launches | o partials | (m, l)].
int64_t attn_decode_workspace_bytes(int R, int Hq, int max_ctx, int hd) {
  const int pages = (max_ctx + PAGE - 1) / PAGE;
  const int nsplit = std::max(1, (pages + MAX_PAGES_PER_SPLIT - 1) / MAX_PAGES_PER_SPLIT);
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
  const int nsplit = std::max(1, (pages + MAX_PAGES_PER_SPLIT - 1) / MAX_PAGES_PER_SPLIT);
  const int64_t need = attn_decode_workspace_bytes(R, Hq, max_ctx, hd);
  if (need > 0 && (ws_bytes < need || !ws))
    return set_error(PL_ERR_CONFIG, "attn_decode: workspace too small (%lld < %lld)",
                     (long long)ws_bytes, (long long)need);
  CUtensorMap mk, mv;
  int rc;
  const int64_t rows = num_blocks * Hkv * PAGE;
  if ((rc = make_tma_2d(&mk, k_cache, rows, HD, HD, 64))) return rc;
  if ((rc = make_tma_2d(&mv, v_cache, rows, HD, HD, 64))) return rc;
  // counters are sized for R*Hq (>= R*Hkv) so the layout only depends on (R, Hq, max_ctx)
  const int64_t counter_bytes = ((static_cast<int64_t>(R) * Hq * 4 + 255) / 256) * 256;
  int* counters = need > 0 ? reinterpret_cast<int*>(ws) : nullptr;
  float* ws_o = need > 0 ? reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + counter_bytes)
                         : nullptr;
  float2* ws_ml = need > 0 ? reinterpret_cast<float2*>(reinterpret_cast<uint8_t*>(ws_o) +
                                                       static_cast<int64_t>(R) * Hq * nsplit * hd * 4)
                           : nullptr;
  dim3 grid(Hkv, R, nsplit);
  constexpr int smem = DecodeSmem::TOTAL;
  const float sl2 = scale * LOG2E;
#define PL_DECODE_CASE(GG)                                                                      \
  case GG: {                                                                                    \
    static bool attr = false;                                                                   \
    if (!attr) {                                                                                \
      cudaError_t e = cudaFuncSetAttribute(attn_decode_kernel<GG>,                              \
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem);  \
      if (e != cudaSuccess) return set_cuda_error(e, "attn_decode smem attribute");             \
      attr = true;                                                                              \
    }                                                                                           \
    rc = launch_k("attn_decode_kernel", attn_decode_kernel<GG>, grid, dim3(128), smem, st, mk,  \
                  mv, q, ldq, block_table, max_blocks, ctx_len, Hkv, sl2, out, ldo, ws_o, ws_ml,  \
                  counters);                                                                    \
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

}  // namespace pl
