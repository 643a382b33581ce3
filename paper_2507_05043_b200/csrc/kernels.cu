// Memory-bound decoder kernels: synthetic init, embedding gather, RMSNorm,
// RoPE + paged-KV append, token feedback scatter.
//
// All are HBM-streaming kernels: 128-bit coalesced loads/stores, fp32 math,
// bf16 rounding at the points HF transformers rounds (modeling_llama.py).
#include "common.cuh"
#include "pl_internal.h"

namespace pl {

// ------------------------------------------------------------ hash init ---
// Counter-based generator shared bit-for-bit with oracle/hashinit.py.

__host__ __device__ inline uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

__global__ void fill_hash_kernel(__nv_bfloat16* __restrict__ dst, int64_t n, uint32_t key,
                                 uint32_t key2, float mult, float offset) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t h = mix32(mix32(static_cast<uint32_t>(i) + key) ^ key2);
    const float v = static_cast<float>(static_cast<int32_t>(h >> 8) - 8388608);
    dst[i] = __float2bfloat16_rn(__fadd_rn(__fmul_rn(v, mult), offset));
  }
}

int fill_hash_launch(__nv_bfloat16* dst, int64_t n, uint32_t seed, uint32_t tensor_id, float scale,
                     float offset, cudaStream_t st) {
  if (n <= 0) return PL_OK;
  if (n > 0xFFFFFFFFll) return set_error(PL_ERR_CONFIG, "fill_hash: tensor too large");
  const uint32_t key = mix32(seed * 0x9E3779B9u + tensor_id * 0x85EBCA6Bu + 0x632BE5ABu);
  const uint32_t key2 = mix32(key ^ 0x5bd1e995u);
  const float mult = scale * (1.0f / 8388608.0f);  // exact: power-of-two scaling
  const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 32));
  fill_hash_kernel<<<blocks, 256, 0, st>>>(dst, n, key, key2, mult, offset);
  return check_launch("fill_hash_kernel");
}

// ---------------------------------------------------------------- embed ---

__global__ void embed_kernel(const int64_t* __restrict__ ids, const int32_t* __restrict__ req_slot,
                             const int64_t* __restrict__ last_token,
                             const __nv_bfloat16* __restrict__ table, int64_t vocab, int d,
                             __nv_bfloat16* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x;
  int64_t id = ids ? ids[t] : last_token[req_slot[t]];
  if (id < 0 || id >= vocab) id = 0;  // defensive: never read outside the table
  const uint4* src = reinterpret_cast<const uint4*>(table + id * d);
  uint4* dst = reinterpret_cast<uint4*>(out + static_cast<int64_t>(t) * d);
  for (int i = threadIdx.x; i < d / 8; i += blockDim.x) dst[i] = ld_nc_v4(src + i);
}

int embed_launch(const int64_t* ids, const int32_t* req_slot, const int64_t* last_token,
                 const __nv_bfloat16* table, int64_t vocab, int64_t T, int d, __nv_bfloat16* out,
                 cudaStream_t st) {
  if (T <= 0) return PL_OK;
  if (d % 8) return set_error(PL_ERR_CONFIG, "embed: d must be a multiple of 8");
  if (!ids && (!req_slot || !last_token))
    return set_error(PL_ERR_CONFIG, "embed: need ids or (req_slot, last_token)");
  return launch_k("embed_kernel", embed_kernel, dim3(static_cast<unsigned>(T)), dim3(128), 0, st,
                  ids, req_slot, last_token, table, vocab, d, out);
}

// -------------------------------------------------------------- rmsnorm ---
// y = bf16( w * bf16( x * rsqrt(mean(x^2) + eps) ) )   (modeling_llama.py:62-67)

template <int VPT>  // 8-element vectors per thread
__global__ void __launch_bounds__(128) rmsnorm_kernel(const __nv_bfloat16* __restrict__ x,
                                                      int64_t ldx,
                                                      const int32_t* __restrict__ row_idx,
                                                      const __nv_bfloat16* __restrict__ w,
                                                      float eps, int d,
                                                      __nv_bfloat16* __restrict__ out,
                                                      int64_t ldo) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const int64_t src_row = row_idx ? row_idx[r] : r;
  const uint4* xs = reinterpret_cast<const uint4*>(x + src_row * ldx);
  const int nvec = d / 8;
  uint4 v[VPT];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int vi = threadIdx.x + i * 128;
    if (vi < nvec) {
      v[i] = xs[vi];
      const uint32_t* p = reinterpret_cast<const uint32_t*>(&v[i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = unpack_bf16x2(p[j]);
        ss += f.x * f.x + f.y * f.y;
      }
    }
  }
  __shared__ float red[4];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  const float tot = red[0] + red[1] + red[2] + red[3];
  const float inv = 1.0f / sqrtf(tot / static_cast<float>(d) + eps);
  const uint4* ws = reinterpret_cast<const uint4*>(w);
  uint4* os = reinterpret_cast<uint4*>(out + static_cast<int64_t>(r) * ldo);
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int vi = threadIdx.x + i * 128;
    if (vi < nvec) {
      const uint4 wv = ws[vi];
      const uint32_t* p = reinterpret_cast<const uint32_t*>(&v[i]);
      const uint32_t* q = reinterpret_cast<const uint32_t*>(&wv);
      uint4 o;
      uint32_t* po = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = unpack_bf16x2(p[j]);
        const float2 g = unpack_bf16x2(q[j]);
        po[j] = pack_bf16x2(g.x * rbf(f.x * inv), g.y * rbf(f.y * inv));
      }
      os[vi] = o;
    }
  }
}

int rmsnorm_launch(const __nv_bfloat16* x, int64_t ldx, const int32_t* row_idx,
                   const __nv_bfloat16* w, float eps, int64_t rows, int d, __nv_bfloat16* out,
                   int64_t ldo, cudaStream_t st) {
  if (rows <= 0) return PL_OK;
  if (d % 8 || ldx % 8 || ldo % 8 || d > 16384)
    return set_error(PL_ERR_CONFIG, "rmsnorm: d and leading dims must be multiples of 8, d<=16384");
  const int vpt = (d / 8 + 127) / 128;
  const dim3 g(static_cast<unsigned>(rows));
  auto k = vpt <= 1 ? rmsnorm_kernel<1> : vpt <= 2 ? rmsnorm_kernel<2> : vpt <= 4 ? rmsnorm_kernel<4>
         : vpt <= 8 ? rmsnorm_kernel<8> : rmsnorm_kernel<16>;
  return launch_k("rmsnorm_kernel", k, g, dim3(128), 0, st, x, ldx, row_idx, w, eps, d, out, ldo);
}

// ------------------------------------------------------ rope + KV append ---
// Neox rotate_half RoPE (modeling_llama.py:138-168) with HF's bf16 rounding:
//   out[i]      = bf16( bf16(x[i] * cos[i]) + bf16(-x[i+h] * sin[i]) )
//   out[i + h]  = bf16( bf16(x[i+h] * cos[i]) + bf16(x[i] * sin[i]) )
// then k (rotated) and v are appended to the paged caches
// [num_blocks, Hkv, block_size, hd] at slot[t].

__global__ void rope_kv_kernel(__nv_bfloat16* __restrict__ qkv, int64_t ldqkv,
                               const int32_t* __restrict__ pos, const int32_t* __restrict__ slot,
                               const __nv_bfloat16* __restrict__ cos_sin, int max_pos,
                               __nv_bfloat16* __restrict__ k_cache,
                               __nv_bfloat16* __restrict__ v_cache, int block_size, int Hq, int Hkv,
                               int hd) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x;
  const int half = hd / 2;
  const int vec_per_head = half / 8;
  int p = pos[t];
  p = p < 0 ? 0 : (p >= max_pos ? max_pos - 1 : p);
  const int s = slot ? slot[t] : -1;
  const int64_t blk = s >= 0 ? s / block_size : 0;
  const int off = s >= 0 ? s % block_size : 0;
  __nv_bfloat16* row = qkv + static_cast<int64_t>(t) * ldqkv;
  const __nv_bfloat16* cs = cos_sin + static_cast<int64_t>(p) * hd;
  const int n_rot = (Hq + Hkv) * vec_per_head;
  for (int i = threadIdx.x; i < n_rot + Hkv * (hd / 8); i += blockDim.x) {
    if (i < n_rot) {
      const int h = i / vec_per_head;
      const int e0 = (i % vec_per_head) * 8;
      uint4* p1 = reinterpret_cast<uint4*>(row + h * hd + e0);
      uint4* p2 = reinterpret_cast<uint4*>(row + h * hd + half + e0);
      const uint4 x1 = *p1, x2 = *p2;
      const uint4 cv = *reinterpret_cast<const uint4*>(cs + e0);
      const uint4 sv = *reinterpret_cast<const uint4*>(cs + half + e0);
      const uint32_t* a = reinterpret_cast<const uint32_t*>(&x1);
      const uint32_t* b = reinterpret_cast<const uint32_t*>(&x2);
      const uint32_t* c = reinterpret_cast<const uint32_t*>(&cv);
      const uint32_t* sn = reinterpret_cast<const uint32_t*>(&sv);
      uint4 o1, o2;
      uint32_t* q1 = reinterpret_cast<uint32_t*>(&o1);
      uint32_t* q2 = reinterpret_cast<uint32_t*>(&o2);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 fa = unpack_bf16x2(a[j]), fb = unpack_bf16x2(b[j]);
        const float2 fc = unpack_bf16x2(c[j]), fs = unpack_bf16x2(sn[j]);
        q1[j] = pack_bf16x2(rbf(fa.x * fc.x) + rbf(-fb.x * fs.x), rbf(fa.y * fc.y) + rbf(-fb.y * fs.y));
        q2[j] = pack_bf16x2(rbf(fb.x * fc.x) + rbf(fa.x * fs.x), rbf(fb.y * fc.y) + rbf(fa.y * fs.y));
      }
      *p1 = o1;
      *p2 = o2;
      if (h >= Hq && s >= 0) {
        const int kh = h - Hq;
        __nv_bfloat16* kc =
            k_cache + ((blk * Hkv + kh) * block_size + off) * static_cast<int64_t>(hd);
        *reinterpret_cast<uint4*>(kc + e0) = o1;
        *reinterpret_cast<uint4*>(kc + half + e0) = o2;
      }
    } else if (s >= 0) {
      const int j = i - n_rot;
      const int kh = j / (hd / 8);
      const int e0 = (j % (hd / 8)) * 8;
      const uint4 v = *reinterpret_cast<const uint4*>(row + (Hq + Hkv + kh) * hd + e0);
      __nv_bfloat16* vc = v_cache + ((blk * Hkv + kh) * block_size + off) * static_cast<int64_t>(hd);
      *reinterpret_cast<uint4*>(vc + e0) = v;
    }
  }
}

int rope_kv_launch(__nv_bfloat16* qkv, int64_t ldqkv, const int32_t* pos, const int32_t* slot,
                   const __nv_bfloat16* cos_sin, int max_pos, __nv_bfloat16* k_cache,
                   __nv_bfloat16* v_cache, int block_size, int64_t T, int Hq, int Hkv, int hd,
                   cudaStream_t st) {
  if (T <= 0) return PL_OK;
  if (hd % 16 || ldqkv % 8) return set_error(PL_ERR_CONFIG, "rope: hd must be a multiple of 16");
  if (slot && (!k_cache || !v_cache || block_size <= 0))
    return set_error(PL_ERR_CONFIG, "rope: caches required when slots are given");
  return launch_k("rope_kv_kernel", rope_kv_kernel, dim3(static_cast<unsigned>(T)), dim3(128), 0, st,
                  qkv, ldqkv, pos, slot, cos_sin, max_pos, k_cache, v_cache, block_size, Hq, Hkv, hd);
}

// -------------------------------------------------------- token scatter ---

__global__ void token_scatter_kernel(const int64_t* __restrict__ ids,
                                     const int32_t* __restrict__ req_slot,
                                     const int32_t* __restrict__ out_pos, int R,
                                     int64_t* __restrict__ last_token,
                                     int64_t* __restrict__ gen_tokens, int gen_stride) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const int64_t id = ids[r];
  const int s = req_slot[r];
  if (last_token) last_token[s] = id;
  if (gen_tokens && out_pos) gen_tokens[static_cast<int64_t>(s) * gen_stride + out_pos[r]] = id;
}

int token_scatter_launch(const int64_t* ids, const int32_t* req_slot, const int32_t* out_pos, int R,
                         int64_t* last_token, int64_t* gen_tokens, int gen_stride,
                         cudaStream_t st) {
  if (R <= 0) return PL_OK;
  return launch_k("token_scatter_kernel", token_scatter_kernel, dim3((R + 127) / 128), dim3(128), 0,
                  st, ids, req_slot, out_pos, R, last_token, gen_tokens, gen_stride);
}


// Load every kernel of this file into the context now (lazy module loading would
// otherwise load it at first launch, which can wait on a spinning NCCL kernel).
template <typename K>
static int preload_one(K k, const char* name) {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, k);
  return e == cudaSuccess ? PL_OK : set_cuda_error(e, name);
}

int kernels_preload() {
  int rc = preload_one(fill_hash_kernel, "fill_hash_kernel");
  if (!rc) rc = preload_one(embed_kernel, "embed_kernel");
  if (!rc) rc = preload_one(rmsnorm_kernel<1>, "rmsnorm_kernel");
  if (!rc) rc = preload_one(rmsnorm_kernel<2>, "rmsnorm_kernel");
  if (!rc) rc = preload_one(rmsnorm_kernel<4>, "rmsnorm_kernel");
  if (!rc) rc = preload_one(rmsnorm_kernel<8>, "rmsnorm_kernel");
  if (!rc) rc = preload_one(rmsnorm_kernel<16>, "rmsnorm_kernel");
  if (!rc) rc = preload_one(rope_kv_kernel, "rope_kv_kernel");
  if (!rc) rc = preload_one(token_scatter_kernel, "token_scatter_kernel");
  return rc;
}

}  // namespace pl
