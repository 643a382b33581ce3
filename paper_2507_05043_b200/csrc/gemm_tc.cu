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
//          W with split-K chosen from (N, K) only -- never from T -- which keeps
//          every token's result independent of the batch it rides in.
//   !SWAP (prefill): tokens are the A operand (M = 128 rows), features are N = 256.
//
// Warp roles (128 threads): warp 0 lane 0 = TMA producer, warp 1 lane 0 = MMA
// issuer, warp 2 = TMEM allocator; afterwards all four warps run the epilogue,
// warp w owning TMEM lanes [32w, 32w+32).
//
// Epilogues (rounding points follow HF modeling_llama.py: every bf16 tensor op
// rounds its fp32 result to bf16):
//   STORE     out = bf16(acc)
//   BIAS      out = bf16(acc + bias[n])                 (Qwen2 qkv bias, modeling_qwen2.py:200-203)
//   RESIDUAL  out = bf16(bf16(acc) + residual[t, n])     (o_proj / down_proj + residual, :313-331)
//   SWIGLU    W rows interleaved in 64-row blocks [gate 64 | up 64]:
//             out[t, j] = bf16(bf16(silu(bf16(g))) * bf16(u))   (LlamaMLP, :182-184)
//   PARTIAL   fp32 partial sums per split (reduced by gemm_splitk_reduce)
//   ARGMAX    per token (max logit, index) over this CTA's 128 vocabulary rows
#include <cudaTypedefs.h>

#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "pl_internal.h"

namespace pl {

constexpr int BK = 64;          // bf16 elements per 128-byte swizzle row
constexpr int BM = 128;         // MMA M (A-operand rows per CTA)
constexpr int A_TILE_BYTES = BM * BK * 2;

struct GemmArgs {
  int T;          // tokens (logical rows of out)
  int N;          // output features of the GEMM (rows of W)
  int num_kb;     // K / 64
  int kb_per_split;
  int epi;
  __nv_bfloat16* C;
  int64_t ldc;
  const __nv_bfloat16* bias;
  const __nv_bfloat16* residual;
  int64_t ldr;
  float* partial;     // [splits][T][N]
  float2* argmax_ws;  // [N/128 tiles][T] (value, index-as-float-bits)
};

template <int BN, int STAGES>
struct GemmSmem {
  static constexpr int B_TILE_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_TILE_BYTES + B_TILE_BYTES;
  static constexpr int BAR_OFFSET = STAGES * STAGE_BYTES;
  // full[S], empty[S], done, tmem slot, + epilogue scratch
  static constexpr int SCRATCH_OFFSET = BAR_OFFSET + 8 * (2 * STAGES + 1) + 16;
  static constexpr int SCRATCH_BYTES = 64 * 16 * 4 * 2;  // swiglu exchange / argmax
  static constexpr int TOTAL = SCRATCH_OFFSET + SCRATCH_BYTES + 1024;  // + alignment slack
};

PL_DEV float silu_f(float x) { return x / (1.0f + expf(-x)); }

template <int BN, bool SWAP, int STAGES>
__global__ void __launch_bounds__(128, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const GemmArgs args) {
  using L = GemmSmem<BN, STAGES>;
  constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFFSET);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  float* scratch = reinterpret_cast<float*>(smem + L::SCRATCH_OFFSET);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int bm = blockIdx.x, bn = blockIdx.y, split = blockIdx.z;
  const int kb0 = split * args.kb_per_split;
  const int kb1 = min(args.num_kb, kb0 + args.kb_per_split);
  const int nkb = kb1 - kb0;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0 && nkb > 0) {
      // weights stream through once; activations are re-read by every weight tile
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      const uint64_t polA = SWAP ? pol_w : pol_x;
      const uint64_t polB = SWAP ? pol_x : pol_w;
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sa = smem + s * L::STAGE_BYTES;
        uint8_t* sb = sa + A_TILE_BYTES;
        mbar_arrive_expect_tx(&full[s], L::STAGE_BYTES);
        const int kc = (kb0 + i) * BK;
        tma_load_2d(sa, &tmA, &full[s], kc, bm * BM, polA);
        tma_load_2d(sb, &tmB, &full[s], kc, bn * BN, polB);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && nkb > 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * L::STAGE_BYTES);
        const uint32_t sb = sa + A_TILE_BYTES;
        const uint64_t da = umma_desc_sw128(sa);
        const uint64_t db = umma_desc_sw128(sb);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          // +32 bytes per K=16 step inside the swizzle atom (encoded >> 4)
          umma_bf16(tmem, da + 2 * k, db + 2 * k, idesc, (i | k) != 0);
        }
        umma_commit(&empty[s]);
      }
      umma_commit(done);
    }
    __syncwarp();
  }

  // ------------------------------------------------------------ epilogue
  if (nkb > 0) {
    mbar_wait(done, 0);
  }
  __syncwarp();
  tc_fence_after();

  const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
  const int row = warp * 32 + lane;  // TMEM lane owned by this thread
  const int epi = args.epi;

  if constexpr (SWAP) {
    // lane <-> feature n, column <-> token t
    const int n = bm * BM + row;
    if (epi == EPI_SWIGLU) {
      // rows [0,64) gate, [64,128) up of the same 64 output features
      const int j = bm * 64 + (row & 63);
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t r[16];
        tmem_ld16(tmem + lane_base + c0, r);
        tmem_ld_wait();
        if (warp >= 2) {
#pragma unroll
          for (int c = 0; c < 16; ++c) scratch[c * 64 + (row - 64)] = __uint_as_float(r[c]);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (warp < 2) {
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const int t = bn * BN + c0 + c;
            if (t < args.T && nkb > 0) {
              const float g = rbf(__uint_as_float(r[c]));
              const float u = rbf(scratch[c * 64 + row]);
              args.C[(int64_t)t * args.ldc + j] = f2bf(rbf(silu_f(g)) * u);
            }
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
    } else if (epi == EPI_ARGMAX) {
      float2* red = reinterpret_cast<float2*>(scratch);  // [4 warps][16 cols]
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t r[16];
        tmem_ld16(tmem + lane_base + c0, r);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          float v = (n < args.N && nkb > 0) ? __uint_as_float(r[c]) : -INFINITY;
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
          if (lane == 0) red[warp * 16 + c] = make_float2(v, __int_as_float(idx));
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x < 16) {
          const int c = threadIdx.x;
          float2 best = red[c];
          for (int w = 1; w < 4; ++w) {
            const float2 o = red[w * 16 + c];
            if (o.x > best.x || (o.x == best.x && __float_as_int(o.y) < __float_as_int(best.y)))
              best = o;
          }
          const int t = bn * BN + c0 + c;
          if (t < args.T) args.argmax_ws[(int64_t)bm * args.T + t] = best;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
    } else {
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t r[16];
        tmem_ld16(tmem + lane_base + c0, r);
        tmem_ld_wait();
        if (n < args.N) {
          const float b = (epi == EPI_BIAS) ? bf2f(args.bias[n]) : 0.f;
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const int t = bn * BN + c0 + c;
            if (t >= args.T) break;
            const float acc = nkb > 0 ? __uint_as_float(r[c]) : 0.f;
            if (epi == EPI_PARTIAL) {
              args.partial[((int64_t)split * args.T + t) * args.N + n] = acc;
            } else if (epi == EPI_RESIDUAL) {
              const float res = bf2f(args.residual[(int64_t)t * args.ldr + n]);
              args.C[(int64_t)t * args.ldc + n] = f2bf(rbf(acc) + res);
            } else {
              args.C[(int64_t)t * args.ldc + n] = f2bf(acc + b);
            }
          }
        }
      }
    }
  } else {
    // lane <-> token t, column <-> feature n
    const int t = bm * BM + row;
    const bool tv = t < args.T;
    if (epi == EPI_SWIGLU) {
      // columns [p*128, p*128+64) gate, [p*128+64, p*128+128) up
      for (int p = 0; p < BN / 128; ++p) {
        for (int c0 = 0; c0 < 64; c0 += 16) {
          uint32_t g[16], u[16];
          tmem_ld16(tmem + lane_base + p * 128 + c0, g);
          tmem_ld16(tmem + lane_base + p * 128 + 64 + c0, u);
          tmem_ld_wait();
          const int j0 = (bn * BN) / 2 + p * 64 + c0;
          if (tv && (bn * BN + p * 128) < args.N) {
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
        tmem_ld16(tmem + lane_base + c0, r);
        tmem_ld_wait();
        const int n0 = bn * BN + c0;
        if (!tv || n0 >= args.N) continue;
        if (epi == EPI_PARTIAL) {
          float4* dst =
              reinterpret_cast<float4*>(args.partial + ((int64_t)split * args.T + t) * args.N + n0);
#pragma unroll
          for (int c = 0; c < 16; c += 4)
            dst[c / 4] = make_float4(__uint_as_float(r[c]), __uint_as_float(r[c + 1]),
                                     __uint_as_float(r[c + 2]), __uint_as_float(r[c + 3]));
          continue;
        }
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

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<TMEM_COLS>(tmem);
}

// Sum split-K partials in split order (deterministic) and apply the epilogue.
__global__ void gemm_splitk_reduce_kernel(const float* __restrict__ partial, int splits, int T,
                                          int N, int epi, __nv_bfloat16* __restrict__ C,
                                          int64_t ldc, const __nv_bfloat16* __restrict__ bias,
                                          const __nv_bfloat16* __restrict__ residual,
                                          int64_t ldr) {
  const int n_out = (epi == EPI_SWIGLU) ? N / 2 : N;
  const int64_t total = (int64_t)T * n_out;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int t = static_cast<int>(i / n_out);
    const int j = static_cast<int>(i % n_out);
    if (epi == EPI_SWIGLU) {
      const int ng = (j / 64) * 128 + (j % 64);
      const int nu = ng + 64;
      float g = 0.f, u = 0.f;
      for (int s = 0; s < splits; ++s) {
        g += partial[((int64_t)s * T + t) * N + ng];
        u += partial[((int64_t)s * T + t) * N + nu];
      }
      C[(int64_t)t * ldc + j] = f2bf(rbf(silu_f(rbf(g))) * rbf(u));
    } else {
      float acc = 0.f;
      for (int s = 0; s < splits; ++s) acc += partial[((int64_t)s * T + t) * N + j];
      if (epi == EPI_RESIDUAL)
        C[(int64_t)t * ldc + j] = f2bf(rbf(acc) + bf2f(residual[(int64_t)t * ldr + j]));
      else if (epi == EPI_BIAS)
        C[(int64_t)t * ldc + j] = f2bf(acc + bf2f(bias[j]));
      else
        C[(int64_t)t * ldc + j] = f2bf(acc);
    }
  }
}

// Per token: reduce the per-tile (max, index) pairs, lowest index on ties.
__global__ void argmax_reduce_kernel(const float2* __restrict__ ws, int tiles, int T,
                                     int64_t* __restrict__ out_ids, float* __restrict__ out_max) {
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

template <int BN, bool SWAP, int STAGES>
int launch_tc(const CUtensorMap& ma, const CUtensorMap& mb, const GemmArgs& a, dim3 grid,
              cudaStream_t st) {
  constexpr int smem = GemmSmem<BN, STAGES>::TOTAL;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel<BN, SWAP, STAGES>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_cuda_error(e, "gemm smem attribute");
    attr_set = true;
  }
  gemm_tc_kernel<BN, SWAP, STAGES><<<grid, 128, smem, st>>>(ma, mb, a);
  return check_launch("gemm_tc_kernel");
}

}  // namespace

int gemm_num_splits(int64_t N, int64_t K, bool swap) {
  // Split-K depends on the weight shape only (batch invariance): aim for
  // ~2 resident CTAs on each of the 148 SMs while keeping >= 8 k-blocks/split.
  if (!swap) return 1;
  const int64_t tiles = (N + BM - 1) / BM;
  const int64_t kb = K / BK;
  int best = 1;
  double best_eff = 0.0;
  for (int s = 1; s <= 16; ++s) {
    if (kb / s < 8 && s > 1) break;
    const int64_t ctas = tiles * s;
    const double waves = static_cast<double>(ctas) / 296.0;
    const double eff = waves / std::ceil(waves) * std::min(1.0, waves);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = s;
    }
  }
  return best;
}

int64_t gemm_workspace_bytes(int64_t T, int64_t N, int64_t K, int epi) {
  const bool swap = T <= 256 || epi == EPI_ARGMAX;
  if (epi == EPI_ARGMAX) return ((N + BM - 1) / BM) * T * 8;
  const int splits = gemm_num_splits(N, K, swap);
  return splits > 1 ? static_cast<int64_t>(splits) * T * N * 4 : 0;
}

int gemm_launch(const __nv_bfloat16* X, int64_t ldx, const __nv_bfloat16* W, int64_t ldw,
                const __nv_bfloat16* bias, __nv_bfloat16* C, int64_t ldc,
                const __nv_bfloat16* residual, int64_t ldr, int64_t T, int64_t N, int64_t K,
                int epi, void* ws, int64_t ws_bytes, int64_t* argmax_out, cudaStream_t st) {
  if (T <= 0) return PL_OK;
  if (K % BK != 0 || N <= 0 || K <= 0)
    return set_error(PL_ERR_CONFIG, "gemm: K must be a positive multiple of 64 (K=%lld N=%lld)",
                     (long long)K, (long long)N);
  if (epi == EPI_SWIGLU && N % 128 != 0)
    return set_error(PL_ERR_CONFIG, "gemm swiglu: N (2*ffn) must be a multiple of 128");
  if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(W)) & 15)
    return set_error(PL_ERR_CONFIG, "gemm: operands must be 16-byte aligned");
  if ((ldx % 8) || (ldw % 8)) return set_error(PL_ERR_CONFIG, "gemm: ld must be a multiple of 8");
  const bool swap = T <= 256 || epi == EPI_ARGMAX;
  if (epi == EPI_ARGMAX && T > 256)
    return set_error(PL_ERR_CONFIG, "gemm argmax: at most 256 rows per call");
  if (!swap && epi != EPI_PARTIAL && (N % 16 || ldc % 8 || (epi == EPI_RESIDUAL && ldr % 8)))
    return set_error(PL_ERR_CONFIG, "gemm: N and leading dims must be multiples of 16/8");

  GemmArgs a{};
  a.T = static_cast<int>(T);
  a.N = static_cast<int>(N);
  a.num_kb = static_cast<int>(K / BK);
  a.epi = epi;
  a.C = C;
  a.ldc = ldc;
  a.bias = bias;
  a.residual = residual;
  a.ldr = ldr;

  const int splits = (epi == EPI_ARGMAX) ? 1 : gemm_num_splits(N, K, swap);
  a.kb_per_split = (a.num_kb + splits - 1) / splits;
  const int final_epi = epi;
  if (epi == EPI_ARGMAX) {
    const int64_t need = ((N + BM - 1) / BM) * T * 8;
    if (ws_bytes < need || !ws) return set_error(PL_ERR_CONFIG, "gemm argmax: workspace too small");
    a.argmax_ws = reinterpret_cast<float2*>(ws);
  } else if (splits > 1) {
    const int64_t need = static_cast<int64_t>(splits) * T * N * 4;
    if (ws_bytes < need || !ws)
      return set_error(PL_ERR_CONFIG, "gemm: split-K workspace too small (%lld < %lld)",
                       (long long)ws_bytes, (long long)need);
    a.partial = reinterpret_cast<float*>(ws);
    a.epi = EPI_PARTIAL;
  }

  CUtensorMap ma, mb;
  int rc;
  if (swap) {
    const int bn = T <= 16 ? 16 : T <= 32 ? 32 : T <= 64 ? 64 : T <= 128 ? 128 : 256;
    if ((rc = make_map(&ma, W, N, K, ldw, BM))) return rc;
    if ((rc = make_map(&mb, X, T, K, ldx, bn))) return rc;
    dim3 grid((N + BM - 1) / BM, (T + bn - 1) / bn, splits);
    switch (bn) {
      case 16: rc = launch_tc<16, true, 6>(ma, mb, a, grid, st); break;
      case 32: rc = launch_tc<32, true, 5>(ma, mb, a, grid, st); break;
      case 64: rc = launch_tc<64, true, 4>(ma, mb, a, grid, st); break;
      case 128: rc = launch_tc<128, true, 4>(ma, mb, a, grid, st); break;
      default: rc = launch_tc<256, true, 4>(ma, mb, a, grid, st); break;
    }
  } else {
    constexpr int BNP = 256;
    if ((rc = make_map(&ma, X, T, K, ldx, BM))) return rc;
    if ((rc = make_map(&mb, W, N, K, ldw, BNP))) return rc;
    dim3 grid((T + BM - 1) / BM, (N + BNP - 1) / BNP, splits);
    rc = launch_tc<BNP, false, 4>(ma, mb, a, grid, st);
  }
  if (rc) return rc;

  if (final_epi == EPI_ARGMAX) {
    const int tiles = static_cast<int>((N + BM - 1) / BM);
    argmax_reduce_kernel<<<static_cast<unsigned>(T), 256, 0, st>>>(
        reinterpret_cast<const float2*>(ws), tiles, static_cast<int>(T), argmax_out, nullptr);
    return check_launch("argmax_reduce_kernel");
  }
  if (splits > 1) {
    const int64_t n_out = (final_epi == EPI_SWIGLU) ? N / 2 : N;
    const int64_t total = T * n_out;
    const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
    gemm_splitk_reduce_kernel<<<blocks, 256, 0, st>>>(a.partial, splits, static_cast<int>(T),
                                                      static_cast<int>(N), final_epi, C, ldc, bias,
                                                      residual, ldr);
    return check_launch("gemm_splitk_reduce_kernel");
  }
  return PL_OK;
}

}  // namespace pl
