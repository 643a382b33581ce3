// extern "C" entry points of libb200link (declared in include/b200link.h) and
// the thread-local error channel.
#include <atomic>
#include <mutex>
#include <set>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "pl_internal.h"

namespace pl {

namespace {
thread_local char g_err[1024] = "";
std::atomic<int64_t> g_launches{0};
}

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int set_cuda_error(cudaError_t e, const char* what) {
  return set_error(PL_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

int ensure_smem_attr(const void* func, int bytes, const char* what) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  if (done.count({dev, func})) return PL_OK;
  const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return set_cuda_error(e, what);
  done.insert({dev, func});
  return PL_OK;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("PL_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}

int check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, what);
  return PL_OK;
}

}  // namespace pl

using namespace pl;

static cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
static const __nv_bfloat16* B(const void* p) { return static_cast<const __nv_bfloat16*>(p); }
static __nv_bfloat16* BM_(void* p) { return static_cast<__nv_bfloat16*>(p); }

extern "C" {

int32_t pl_abi_version(void) { return PL_ABI_VERSION; }

const char* pl_last_error(void) { return g_err; }

int32_t pl_preload_kernels(void) {
  int rc = gemm_preload();
  if (!rc) rc = attention_preload();
  if (!rc) rc = kernels_preload();
  if (!rc) rc = transport_preload();
  if (!rc) rc = chain_preload();
  if (!rc) rc = attn_tc_preload();
  return rc;
}

int64_t pl_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int32_t pl_device_sm_count(int32_t device) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return n;
}

int32_t pl_fill_hash_bf16(void* dst, int64_t n, uint32_t seed, uint32_t tensor_id, float scale,
                          float offset, void* stream) {
  if (!dst && n > 0) return set_error(PL_ERR_CONFIG, "fill_hash: null dst");
  return fill_hash_launch(BM_(dst), n, seed, tensor_id, scale, offset, S(stream));
}

int32_t pl_embed(const int64_t* ids, const int32_t* req_slot, const int64_t* last_token,
                 const void* table, int64_t vocab, int64_t T, int32_t d, void* out, void* stream) {
  if (!table || !out) return set_error(PL_ERR_CONFIG, "embed: null table/out");
  return embed_launch(ids, req_slot, last_token, B(table), vocab, T, d, BM_(out), S(stream));
}

int32_t pl_rmsnorm(const void* x, int64_t ldx, const int32_t* row_idx, const void* w, float eps,
                   int64_t rows, int32_t d, void* out, int64_t ldo, void* stream) {
  if (!x || !w || !out) return set_error(PL_ERR_CONFIG, "rmsnorm: null argument");
  return rmsnorm_launch(B(x), ldx, row_idx, B(w), eps, rows, d, BM_(out), ldo, S(stream));
}

int64_t pl_gemm_workspace_bytes(int64_t T, int64_t N, int64_t K, int32_t epilogue) {
  return gemm_workspace_bytes(T, N, K, epilogue);
}

int32_t pl_gemm(const void* X, int64_t ldx, const void* W, int64_t ldw, const void* bias, void* C,
                int64_t ldc, const void* residual, int64_t ldr, int64_t T, int64_t N, int64_t K,
                int32_t epilogue, void* workspace, int64_t workspace_bytes, int64_t* argmax_out,
                void* stream) {
  if (!X || !W) return set_error(PL_ERR_CONFIG, "gemm: null operand");
  if (epilogue < PL_EPI_NONE || epilogue > PL_EPI_ARGMAX)
    return set_error(PL_ERR_CONFIG, "gemm: unknown epilogue %d", epilogue);
  if (epilogue == PL_EPI_ARGMAX ? !argmax_out : !C)
    return set_error(PL_ERR_CONFIG, "gemm: null output");
  if (epilogue == PL_EPI_BIAS && !bias) return set_error(PL_ERR_CONFIG, "gemm: bias epilogue needs bias");
  if (epilogue == PL_EPI_RESIDUAL && !residual)
    return set_error(PL_ERR_CONFIG, "gemm: residual epilogue needs residual");
  return gemm_launch(B(X), ldx, B(W), ldw, B(bias), BM_(C), ldc, B(residual), ldr, T, N, K, epilogue,
                     workspace, workspace_bytes, argmax_out, S(stream));
}

int32_t pl_pack_weight(const void* W, int64_t ldw, int64_t N, int64_t K, int32_t interleave, void* out,
                       void* stream) {
  if (!W || !out) return set_error(PL_ERR_CONFIG, "pack_weight: null argument");
  return pack_weight_launch(B(W), ldw, N, K, out, S(stream), interleave != 0);
}

int32_t pl_gemm_packed(const void* X, int64_t ldx, const void* W_packed, const void* bias, void* C,
                       int64_t ldc, const void* residual, int64_t ldr, int64_t T, int64_t N, int64_t K,
                       int32_t epilogue, void* workspace, int64_t workspace_bytes, int64_t* argmax_out,
                       void* stream) {
  if (!X || !W_packed) return set_error(PL_ERR_CONFIG, "gemm: null operand");
  if (epilogue < PL_EPI_NONE || epilogue > PL_EPI_ARGMAX)
    return set_error(PL_ERR_CONFIG, "gemm: unknown epilogue %d", epilogue);
  if (epilogue == PL_EPI_ARGMAX ? !argmax_out : !C)
    return set_error(PL_ERR_CONFIG, "gemm: null output");
  if (epilogue == PL_EPI_BIAS && !bias) return set_error(PL_ERR_CONFIG, "gemm: bias epilogue needs bias");
  if (epilogue == PL_EPI_RESIDUAL && !residual)
    return set_error(PL_ERR_CONFIG, "gemm: residual epilogue needs residual");
  return gemm_launch(B(X), ldx, B(W_packed), K, B(bias), BM_(C), ldc, B(residual), ldr, T, N, K, epilogue,
                     workspace, workspace_bytes, argmax_out, S(stream), nullptr, nullptr, true);
}

int32_t pl_rope_kv_write(void* qkv, int64_t ldqkv, const int32_t* pos, const int32_t* slot,
                         const void* cos_sin, int32_t max_pos, void* k_cache, void* v_cache,
                         int32_t block_size, int64_t T, int32_t Hq, int32_t Hkv, int32_t hd,
                         void* stream) {
  if (!qkv || !pos || !cos_sin) return set_error(PL_ERR_CONFIG, "rope: null argument");
  return rope_kv_launch(BM_(qkv), ldqkv, pos, slot, B(cos_sin), max_pos, BM_(k_cache), BM_(v_cache),
                        block_size, T, Hq, Hkv, hd, S(stream));
}

int32_t pl_attn_prefill(const void* qkv, int64_t ldqkv, const int32_t* cu_seqlens, int32_t R,
                        int32_t max_seqlen, int32_t Hq, int32_t Hkv, int32_t hd, float scale,
                        void* out, int64_t ldo, void* stream) {
  if (!qkv || !cu_seqlens || !out) return set_error(PL_ERR_CONFIG, "attn_prefill: null argument");
  return attn_prefill_launch(B(qkv), ldqkv, cu_seqlens, R, max_seqlen, Hq, Hkv, hd, scale, BM_(out),
                             ldo, S(stream));
}

int32_t pl_attn_prefill_ex(const void* qkv, int64_t ldqkv, int64_t rows, const int32_t* cu_seqlens, int32_t R,
                           int32_t max_seqlen, int32_t Hq, int32_t Hkv, int32_t hd, float scale, void* out,
                           int64_t ldo, int32_t impl, void* stream) {
  if (!qkv || !cu_seqlens || !out) return set_error(PL_ERR_CONFIG, "attn_prefill: null argument");
  if (impl < 0 || impl > 2) return set_error(PL_ERR_CONFIG, "attn_prefill: impl must be 0, 1 or 2");
  return attn_prefill_launch(B(qkv), ldqkv, cu_seqlens, R, max_seqlen, Hq, Hkv, hd, scale, BM_(out),
                             ldo, S(stream), rows, impl);
}

int64_t pl_attn_decode_workspace_bytes(int32_t R, int32_t Hq, int32_t max_ctx, int32_t hd) {
  return attn_decode_workspace_bytes(R, Hq, max_ctx, hd);
}

int32_t pl_attn_decode(const void* q, int64_t ldq, const void* k_cache, const void* v_cache,
                       int64_t num_blocks, int32_t block_size, const int32_t* block_table, int32_t max_blocks,
                       const int32_t* ctx_len, int32_t R, int32_t max_ctx, int32_t Hq, int32_t Hkv,
                       int32_t hd, float scale, void* out, int64_t ldo, void* workspace,
                       int64_t workspace_bytes, void* stream) {
  if (!q || !k_cache || !v_cache || !block_table || !ctx_len || !out)
    return set_error(PL_ERR_CONFIG, "attn_decode: null argument");
  return attn_decode_launch(B(q), ldq, B(k_cache), B(v_cache), num_blocks, block_size, block_table,
                            max_blocks,
                            ctx_len, R, max_ctx, Hq, Hkv, hd, scale, BM_(out), ldo, workspace,
                            workspace_bytes, S(stream));
}

int64_t pl_lmhead_workspace_bytes(int32_t R, int64_t vocab) {
  // d is not an argument: size for the largest stream-K grid (an upper bound for any d)
  return gemm_workspace_bytes(R, vocab, int64_t(64) << 12, EPI_ARGMAX);
}

int32_t pl_lmhead_argmax(const void* h, int64_t ldh, const void* W, int64_t vocab, int32_t d,
                         int32_t R, int64_t* out_ids, void* workspace, int64_t workspace_bytes,
                         void* stream) {
  return pl_gemm(h, ldh, W, d, nullptr, nullptr, 0, nullptr, 0, R, vocab, d, PL_EPI_ARGMAX,
                 workspace, workspace_bytes, out_ids, stream);
}

int32_t pl_token_scatter(const int64_t* ids, const int32_t* req_slot, const int32_t* out_pos,
                         int32_t R, int64_t* last_token, int64_t* gen_tokens, int32_t gen_stride,
                         void* stream) {
  if (!ids || !req_slot) return set_error(PL_ERR_CONFIG, "token_scatter: null argument");
  return token_scatter_launch(ids, req_slot, out_pos, R, last_token, gen_tokens, gen_stride,
                              S(stream));
}

int32_t pl_enable_peer_access(int32_t ndev, const int32_t* devs) {
  if (ndev < 0 || (ndev > 0 && !devs)) return set_error(PL_ERR_CONFIG, "enable_peer_access: bad arguments");
  int prev = 0;
  cudaGetDevice(&prev);
  for (int i = 0; i < ndev; ++i)
    for (int j = 0; j < ndev; ++j) {
      if (devs[i] == devs[j]) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, devs[i], devs[j]);
      if (!can) continue;
      cudaSetDevice(devs[i]);
      const cudaError_t e = cudaDeviceEnablePeerAccess(devs[j], 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
      } else if (e != cudaSuccess) {
        cudaSetDevice(prev);
        return set_cuda_error(e, "cudaDeviceEnablePeerAccess");
      }
    }
  cudaSetDevice(prev);
  return PL_OK;
}

int32_t pl_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  if (bytes <= 0) return PL_OK;
  cudaError_t e = cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDefault, S(stream));
  if (e != cudaSuccess) return set_cuda_error(e, "memcpy_async");
  return PL_OK;
}

#ifdef PL_TIMELINE
// experiment builds only: kernel timeline sink (buf: 2 x u64 per record, count: u32)
PL_API int32_t pl_timeline_set(void* buf, void* count, uint32_t cap) {
  int rc = tl_set_gemm(buf, count, cap);
  if (!rc) rc = tl_set_attn(buf, count, cap);
  return rc;
}
#endif

}  // extern "C"
