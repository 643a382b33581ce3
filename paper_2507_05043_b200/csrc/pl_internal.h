// Internal declarations shared by the libb200link translation units.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "../../include/b200link.h"

namespace pl {

enum Epi : int {
  EPI_STORE = PL_EPI_NONE,
  EPI_BIAS = PL_EPI_BIAS,
  EPI_RESIDUAL = PL_EPI_RESIDUAL,
  EPI_SWIGLU = PL_EPI_SWIGLU,
  EPI_ARGMAX = PL_EPI_ARGMAX,
  EPI_PARTIAL = 100,
};

// thread-local error reporting (pl_last_error)
int set_error(int code, const char* fmt, ...);
int set_cuda_error(cudaError_t e, const char* what);
int check_launch(const char* what);

// PDL on/off (env PL_PDL=0 disables programmatic dependent launch)
bool pdl_enabled();

// cudaFuncAttributeMaxDynamicSharedMemorySize for `func` on the CURRENT device, set once
// per (device, function): the attribute is per device, and one process may drive
// stages on several GPUs
int ensure_smem_attr(const void* func, int bytes, const char* what);

// Launch with programmatic stream serialization so the kernel may start while its
// predecessor in the stream drains (see pdl_wait / pdl_trigger in common.cuh).
// cluster_x > 0: launch as clusters of cluster_x consecutive CTAs.
template <typename... KArgs, typename... Args>
int launch_kc(const char* what, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
              cudaStream_t st, int cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (cluster_x > 0) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = static_cast<unsigned>(cluster_x);
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
  if (e != cudaSuccess) return set_cuda_error(e, what);
  return check_launch(what);
}

template <typename... KArgs, typename... Args>
int launch_k(const char* what, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
             cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
  if (e != cudaSuccess) return set_cuda_error(e, what);
  return check_launch(what);
}

// gemm_tc.cu
// cached 2-D bf16 TMA descriptor: [rows, cols] row-major (ld elements), box {64, box_rows}, SW128
int make_tma_2d(CUtensorMap* out, const void* ptr, int64_t rows, int64_t cols, int64_t ld,
                int box_rows);
int gemm_num_splits(int64_t N, int64_t K, bool swap);
int64_t gemm_workspace_bytes(int64_t T, int64_t N, int64_t K, int epi);
// Decode-path epilogue fusions applied by the split-K reduction (stage runtime only).
enum FuseKind : int { FUSE_NONE = 0, FUSE_RESIDUAL_NORM = 1, FUSE_QKV_ROPE = 2 };
struct FusedEpi {
  int kind = FUSE_NONE;
  // fused transport (any kind): every final output row also stored here (ldc), e.g. the
  // next pipeline stage's receive buffer on a peer GPU (decode / SWAP GEMMs only)
  __nv_bfloat16* mirror = nullptr;
  // FUSE_RESIDUAL_NORM: C (= residual) updated in place, then norm_out = rmsnorm(C) * norm_w
  const __nv_bfloat16* norm_w = nullptr;
  float eps = 0.f;
  __nv_bfloat16* norm_out = nullptr;
  int64_t ld_norm = 0;
  // FUSE_QKV_ROPE: RoPE on q,k of C + K/V append to the paged caches
  const int32_t* pos = nullptr;
  const int32_t* slot = nullptr;
  const __nv_bfloat16* cos_sin = nullptr;
  int max_pos = 0;
  __nv_bfloat16* k_cache = nullptr;
  __nv_bfloat16* v_cache = nullptr;
  int block_size = 0, Hq = 0, Hkv = 0;
};

int gemm_launch(const __nv_bfloat16* X, int64_t ldx, const __nv_bfloat16* W, int64_t ldw,
                const __nv_bfloat16* bias, __nv_bfloat16* C, int64_t ldc,
                const __nv_bfloat16* residual, int64_t ldr, int64_t T, int64_t N, int64_t K,
                int epi, void* ws, int64_t ws_bytes, int64_t* argmax_out, cudaStream_t st,
                const FusedEpi* fuse = nullptr, bool* fused = nullptr, bool w_packed = false);
// W [N, K] -> pre-swizzled 16 KB tiles (see gemm_tc.cu); out may not alias W
// interleave_swiglu: [gate 64 | up 64] row blocks become (gate_j, up_j) row pairs (the
// packed SwiGLU epilogue pairs them with one shuffle)
int pack_weight_launch(const __nv_bfloat16* W, int64_t ld, int64_t N, int64_t K, void* out, cudaStream_t st,
                       bool interleave_swiglu = false);

#ifdef PL_TIMELINE
int tl_set_gemm(void* buf, void* count, unsigned cap);
int tl_set_attn(void* buf, void* count, unsigned cap);
#endif

// per-file eager kernel loading (pl_preload_kernels)
int attention_preload();
int kernels_preload();
int gemm_preload();
int transport_preload();

// kernels.cu
int fill_hash_launch(__nv_bfloat16* dst, int64_t n, uint32_t seed, uint32_t tensor_id,
                     float scale, float offset, cudaStream_t st);
int embed_launch(const int64_t* ids, const int32_t* req_slot, const int64_t* last_token,
                 const __nv_bfloat16* table, int64_t vocab, int64_t T, int d, __nv_bfloat16* out,
                 cudaStream_t st);
int rmsnorm_launch(const __nv_bfloat16* x, int64_t ldx, const int32_t* row_idx,
                   const __nv_bfloat16* w, float eps, int64_t rows, int d, __nv_bfloat16* out,
                   int64_t ldo, cudaStream_t st);
int rope_kv_launch(__nv_bfloat16* qkv, int64_t ldqkv, const int32_t* pos, const int32_t* slot,
                   const __nv_bfloat16* cos_sin, int max_pos, __nv_bfloat16* k_cache,
                   __nv_bfloat16* v_cache, int block_size, int64_t T, int Hq, int Hkv, int hd,
                   cudaStream_t st);
int token_scatter_launch(const int64_t* ids, const int32_t* req_slot, const int32_t* out_pos,
                         int R, int64_t* last_token, int64_t* gen_tokens, int gen_stride,
                         cudaStream_t st);

// chain.cu -- persistent decode-layer kernel (o -> norm -> gate_up -> down -> norm -> qkv)
enum ChainKind : int { CHAIN_O = 0, CHAIN_GATE_UP = 1, CHAIN_DOWN = 2, CHAIN_QKV = 3 };
struct ChainLaunch {
  int T = 0, Tp = 0, njobs = 0, d = 0, ffn = 0, attn_dim = 0, grid = 0;
  int kind[4] = {0, 0, 0, 0};
  int64_t N[4] = {0, 0, 0, 0}, K[4] = {0, 0, 0, 0};
  int splits[4] = {1, 1, 1, 1};
  const void* w[4] = {nullptr, nullptr, nullptr, nullptr};  // packed weights (pack_weight_launch)
  float* partial[4] = {nullptr, nullptr, nullptr, nullptr};  // split-K partials [splits][tiles][Tp][128]
  const int4* units = nullptr;  // global claim order {job, tile, kb0, nkb} (device)
  const int4* units_host = nullptr;  // the same list on the host
  int n_units = 0;
  const __nv_bfloat16* o_attn = nullptr;
  __nv_bfloat16 *h = nullptr, *a = nullptr, *m = nullptr, *q_out = nullptr;
  int64_t ld_q = 0;
  float* part_ss = nullptr;  // [2][Tp][d / piece] finalisation sums of squares
  int* row_parts = nullptr;  // [2][Tp] zero between launches
  const __nv_bfloat16* norm_w[2] = {nullptr, nullptr};
  int has_norm[2] = {0, 0};
  float eps = 0.f;
  const __nv_bfloat16* bias = nullptr;
  const int32_t *pos = nullptr, *slot = nullptr;
  const __nv_bfloat16* cos_sin = nullptr;
  int max_pos = 0;
  __nv_bfloat16 *k_cache = nullptr, *v_cache = nullptr;
  int block_size = 0, Hq = 0, Hkv = 0;
  void* ctr = nullptr;  // this launch's counter set (CHAIN_CTR_BYTES, zero; two sets alternate)
  int* gu_flag = nullptr;
  int seq = 0;
  unsigned long long* trace = nullptr;  // debug: [grid][64][4] globaltimer stamps, or null
  int bench = 0;  // pl_stage_chain_bench: no dependencies, no finalisation (weight stream only)
};
constexpr int CHAIN_CTR_BYTES = 64;
int chain_plan(const int* kinds, int njobs, const int64_t* N, const int64_t* K, int grid, int ring,
               int* splits_out, std::vector<int4>& units);
int chain_ring_kb(int BN);
int chain_ctas_per_sm();
int chain_launch(const ChainLaunch& c, cudaStream_t st);
int chain_preload();

// attention.cu
// rows = qkv rows (> 0 enables the tcgen05 kernel, whose TMA maps need the extent);
// impl 0 auto, 1 mma.sync, 2 tcgen05
int attn_prefill_launch(const __nv_bfloat16* qkv, int64_t ldqkv, const int32_t* cu_seqlens, int R,
                        int max_seqlen, int Hq, int Hkv, int hd, float scale, __nv_bfloat16* out,
                        int64_t ldo, cudaStream_t st, int64_t rows = 0, int impl = 0);
// attn_tc.cu
int attn_prefill_tc_launch(const __nv_bfloat16* qkv, int64_t ldqkv, int64_t rows, const int32_t* cu_seqlens,
                           int R, int max_seqlen, int Hq, int Hkv, float scale_log2, __nv_bfloat16* out,
                           int64_t ldo, cudaStream_t st);
int attn_tc_preload();
int64_t attn_decode_workspace_bytes(int R, int Hq, int max_ctx, int hd);
int attn_decode_launch(const __nv_bfloat16* q, int64_t ldq, const __nv_bfloat16* k_cache,
                       const __nv_bfloat16* v_cache, int64_t num_blocks, int block_size,
                       const int32_t* block_table,
                       int max_blocks, const int32_t* ctx_len, int R, int max_ctx, int Hq, int Hkv,
                       int hd, float scale, __nv_bfloat16* out, int64_t ldo, void* ws,
                       int64_t ws_bytes, cudaStream_t st);

}  // namespace pl
