/*
 * libb200link -- C ABI of the B200-native pipeline-parallel serving hot path.
 *
 * The reference (`pipelink`, /root/reference/pkg/src/pipelink) has NO FFI: its
 * two hot-path subsystems are virtual.  Each entry point below names the
 * reference call site it replaces:
 *
 *   compute   engine.py:376-388  PipelineEngine._try_start_compute ->
 *             compute_time(stage.profile, phase, mb.batched_tokens) (engine.py:384,
 *             profiles.py:95-121).  The latency-table lookup becomes a real
 *             decoder forward of the stage's layer range: pl_stage_forward, built
 *             from the kernel entry points pl_embed ... pl_lmhead_argmax.
 *   transport engine.py:347-372 / 546-576 (_link_emit_next -> transmission_ns,
 *             transport.py:199-200) and wire.py:124-149 (SocketLinkSender.run
 *             `sendall` of one LinkQueue chunk).  Each LinkQueue chunk becomes
 *             one NCCL send/recv pair: pl_p2p_send / pl_p2p_recv.
 *   throttle  transport.py:199-200 + engine.py:552 (`round(bytes*1e9/bw)` +
 *             latency) reproduced in wall time on the GPU: pl_gate_until_ns.
 *
 * Conventions: plain C types only; every pointer argument is a device pointer
 * unless named *_host; `stream` is a cudaStream_t passed as void*.  Kernel
 * entry points never allocate and never synchronize.  Every function except
 * pl_abi_version / pl_last_error returns a pl_status; on failure
 * pl_last_error() holds a thread-local message.  The Python wrapper maps
 * PL_ERR_CONFIG -> pipelink.errors.ConfigError, PL_ERR_PROTOCOL ->
 * ProtocolError, anything else -> PipelinkError (errors.py:4-39).
 */
#ifndef B200LINK_H_
#define B200LINK_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PL_ABI_VERSION 1

#if defined(__GNUC__)
#define PL_API __attribute__((visibility("default")))
#else
#define PL_API
#endif

typedef enum pl_status {
  PL_OK = 0,
  PL_ERR_CONFIG = 1,   /* bad shape, alignment or argument  -> ConfigError   */
  PL_ERR_PROTOCOL = 2, /* transport / NCCL failure           -> ProtocolError */
  PL_ERR_CUDA = 3,     /* CUDA runtime / launch failure      -> PipelinkError */
} pl_status;

/* Load every kernel of the library into the current device's context now.
 * CUDA loads modules lazily at first launch by default, and a load can wait on
 * a running kernel -- an NCCL receive spinning for its peer would deadlock it.
 * pl_stage_create calls this; call it before any NCCL traffic otherwise. */
PL_API int32_t pl_preload_kernels(void);

/* GEMM epilogues (see pl_gemm). */
typedef enum pl_epilogue {
  PL_EPI_NONE = 0,     /* C = bf16(acc)                                      */
  PL_EPI_BIAS = 1,     /* C = bf16(acc + bias[n])                            */
  PL_EPI_RESIDUAL = 2, /* C = bf16(bf16(acc) + residual[t, n]) (may alias C) */
  PL_EPI_SWIGLU = 3,   /* W rows in 64-row blocks [gate|up]; C[t, N/2]       */
  PL_EPI_ARGMAX = 4,   /* argmax over n of acc, int64 per row                */
} pl_epilogue;

PL_API int32_t pl_abi_version(void);
PL_API const char* pl_last_error(void);
PL_API int32_t pl_device_sm_count(int32_t device);
/* Number of libb200link kernels launched by this process so far (bench.py's gpu_launches). */
PL_API int64_t pl_launch_count(void);

/* ---------------------------------------------------------------- init --- */

/* dst[i] = bf16(float(hash(seed, tensor_id, i) - 2^23) * (scale * 2^-23) + offset):
 * the counter-based synthetic weight init shared bit-for-bit with oracle/hashinit.py. */
PL_API int32_t pl_fill_hash_bf16(void* dst, int64_t n, uint32_t seed, uint32_t tensor_id, float scale,
                          float offset, void* stream);

/* ------------------------------------------------------- decoder kernels - */

/* out[t] = table[ids[t]]                          (ids != NULL: prompt tokens)
 * out[t] = table[last_token[req_slot[t]]]          (ids == NULL: decode feedback) */
PL_API int32_t pl_embed(const int64_t* ids, const int32_t* req_slot, const int64_t* last_token,
                 const void* table, int64_t vocab, int64_t T, int32_t d, void* out, void* stream);

/* out[r] = rmsnorm(x[row_idx ? row_idx[r] : r]) * w, fp32 math, HF rounding points
 * (modeling_llama.py:62-67). */
PL_API int32_t pl_rmsnorm(const void* x, int64_t ldx, const int32_t* row_idx, const void* w, float eps,
                   int64_t rows, int32_t d, void* out, int64_t ldo, void* stream);

/* C[T, N] = epilogue(X[T, K] . W[N, K]^T) on tcgen05 tensor cores.  workspace:
 * pl_gemm_workspace_bytes(T, N, K, epilogue) bytes (split-K or argmax partials). */
PL_API int64_t pl_gemm_workspace_bytes(int64_t T, int64_t N, int64_t K, int32_t epilogue);
PL_API int32_t pl_gemm(const void* X, int64_t ldx, const void* W, int64_t ldw, const void* bias, void* C,
                int64_t ldc, const void* residual, int64_t ldr, int64_t T, int64_t N, int64_t K,
                int32_t epilogue, void* workspace, int64_t workspace_bytes, int64_t* argmax_out,
                void* stream);

/* Pre-swizzle W [N, K] (row stride ldw) into the packed layout the decode GEMMs stream
 * with one 16 KB bulk copy per 128 x 64 tile: [N/128][K/64] tiles, each the 128-byte-
 * swizzled shared-memory image (what pl_stage_pack_weights does to a stage's
 * projections).  interleave = 1 for a gate_up weight (SwiGLU epilogue): rows alternate
 * gate_j / up_j inside each 128-row tile.  out: N*K*2 bytes, not aliasing W;
 * N % 256 == 0, K % 64 == 0. */
PL_API int32_t pl_pack_weight(const void* W, int64_t ldw, int64_t N, int64_t K, int32_t interleave, void* out,
                              void* stream);
/* pl_gemm with W packed by pl_pack_weight (interleave = 1 iff epilogue == SWIGLU). */
PL_API int32_t pl_gemm_packed(const void* X, int64_t ldx, const void* W_packed, const void* bias, void* C,
                              int64_t ldc, const void* residual, int64_t ldr, int64_t T, int64_t N, int64_t K,
                              int32_t epilogue, void* workspace, int64_t workspace_bytes, int64_t* argmax_out,
                              void* stream);

/* Neox RoPE on the q and k heads of qkv[T, (Hq+2Hkv)*hd] in place, then k and v
 * written to the paged caches [num_blocks, Hkv, block_size, hd] at slot[t]
 * (slot < 0 skips the write).  cos_sin: bf16 [max_pos, hd] = [cos | sin]. */
PL_API int32_t pl_rope_kv_write(void* qkv, int64_t ldqkv, const int32_t* pos, const int32_t* slot,
                         const void* cos_sin, int32_t max_pos, void* k_cache, void* v_cache,
                         int32_t block_size, int64_t T, int32_t Hq, int32_t Hkv, int32_t hd,
                         void* stream);

/* Causal varlen GQA attention over the prompt rows of qkv (no prior context;
 * prefill is never split, engine.py:215-223).  out[T, Hq*hd]. */
PL_API int32_t pl_attn_prefill(const void* qkv, int64_t ldqkv, const int32_t* cu_seqlens, int32_t R,
                        int32_t max_seqlen, int32_t Hq, int32_t Hkv, int32_t hd, float scale,
                        void* out, int64_t ldo, void* stream);
/* Same, with the qkv row count (the tcgen05 kernel's TMA maps need it) and the kernel:
 * impl 0 = default (tcgen05; PL_ATTN_TC=0 selects mma.sync), 1 = mma.sync FA2, 2 = tcgen05
 * (FA4-style: S and O in TMEM, TMA-fed K / V ring; GQA groups 1, 2, 4, 8). */
PL_API int32_t pl_attn_prefill_ex(const void* qkv, int64_t ldqkv, int64_t rows, const int32_t* cu_seqlens,
                           int32_t R, int32_t max_seqlen, int32_t Hq, int32_t Hkv, int32_t hd, float scale,
                           void* out, int64_t ldo, int32_t impl, void* stream);

/* One query token per request over its paged KV (ctx_len[r] tokens incl. the
 * current one; caches hold num_blocks blocks).  q rows: [R, Hq*hd], leading dim ldq. */
PL_API int64_t pl_attn_decode_workspace_bytes(int32_t R, int32_t Hq, int32_t max_ctx, int32_t hd);
PL_API int32_t pl_attn_decode(const void* q, int64_t ldq, const void* k_cache, const void* v_cache,
                       int64_t num_blocks, int32_t block_size, const int32_t* block_table, int32_t max_blocks,
                       const int32_t* ctx_len, int32_t R, int32_t max_ctx, int32_t Hq, int32_t Hkv,
                       int32_t hd, float scale, void* out, int64_t ldo, void* workspace,
                       int64_t workspace_bytes, void* stream);

/* Greedy next token: out_ids[r] = argmax_v h[r] . W[v]  (fp32 logits, lowest
 * index on ties).  Replaces the 8-byte token feedback size of engine.py:409. */
PL_API int64_t pl_lmhead_workspace_bytes(int32_t R, int64_t vocab);
PL_API int32_t pl_lmhead_argmax(const void* h, int64_t ldh, const void* W, int64_t vocab, int32_t d,
                         int32_t R, int64_t* out_ids, void* workspace, int64_t workspace_bytes,
                         void* stream);

/* Return hop landing on the head stage: last_token[req_slot[r]] = ids[r] and
 * gen_tokens[req_slot[r] * gen_stride + out_pos[r]] = ids[r]. */
PL_API int32_t pl_token_scatter(const int64_t* ids, const int32_t* req_slot, const int32_t* out_pos,
                         int32_t R, int64_t* last_token, int64_t* gen_tokens, int32_t gen_stride,
                         void* stream);

/* --------------------------------------------------------- stage runtime - */

typedef struct pl_layer_weights {
  const void* attn_norm; /* bf16 [d]                                   */
  const void* w_qkv;     /* bf16 [(Hq+2Hkv)*hd, d]                     */
  const void* b_qkv;     /* bf16 [(Hq+2Hkv)*hd] or NULL (Qwen2 bias)   */
  const void* w_o;       /* bf16 [d, Hq*hd]                            */
  const void* mlp_norm;  /* bf16 [d]                                   */
  const void* w_gate_up; /* bf16 [2*ffn, d], 64-row blocks [gate|up]   */
  const void* w_down;    /* bf16 [d, ffn]                              */
  void* k_cache;         /* bf16 [num_blocks, Hkv, block_size, hd]     */
  void* v_cache;
} pl_layer_weights;

typedef struct pl_stage_config {
  int32_t d, Hq, Hkv, hd, ffn;
  int32_t num_layers;
  int64_t vocab;
  float eps;
  int32_t block_size, max_blocks_per_req, max_pos;
  int64_t num_blocks; /* KV cache blocks per layer */
  int32_t is_first, is_last;
  int32_t max_tokens; /* activation rows the workspace is sized for */
  int32_t max_reqs;   /* requests per micro-batch                   */
  int32_t max_ctx;    /* longest context (tokens)                   */
  const void* embed;      /* bf16 [vocab, d]  (first stage)  */
  const void* final_norm; /* bf16 [d]         (last stage)   */
  const void* lm_head;    /* bf16 [vocab, d]  (last stage)   */
  const void* cos_sin;    /* bf16 [max_pos, hd]              */
} pl_stage_config;

/* Packed int32 micro-batch metadata (one H2D copy per micro-batch):
 *   pos[T] | slot[T] | req_slot[T] | cu_seqlens[R+1] | ctx_len[R] | last_idx[R]
 *   | block_table[R * max_blocks_per_req]                                    */
typedef struct pl_microbatch {
  int32_t T, R;
  int32_t phase;      /* 0 prefill, 1 decode, 2 mixed (allow_mixed_phase, engine.py:184-190):
                         requests [0, n_decode) decode one token each in rows [0, n_decode),
                         the rest are prompts in rows [n_decode, T)                        */
  int32_t max_seqlen; /* prefill: longest prompt in the micro-batch */
  int32_t max_ctx;    /* decode: longest context in the micro-batch */
  const int32_t* meta;
  const int64_t* token_ids;  /* first stage, prefill/mixed: prompt ids [T]    */
  const int64_t* last_token; /* first stage, decode/mixed: feedback table     */
  void* hidden;              /* bf16 [T, d] residual stream: input (non-first),
                                output (non-last), updated in place           */
  int64_t* out_ids;          /* last stage: [R] greedy tokens                 */
  int32_t n_decode;          /* mixed: decode requests leading the batch      */
  void* peer_hidden;         /* decode, non-last stage, or NULL: the last residual
                                epilogue also stores the output rows here -- the
                                next stage's receive buffer, possibly on a peer
                                GPU (fused transport: no link copy)           */
} pl_microbatch;

PL_API int64_t pl_stage_workspace_bytes(const pl_stage_config* cfg);
PL_API int32_t pl_stage_create(const pl_stage_config* cfg, const pl_layer_weights* layers,
                        void* workspace, int64_t workspace_bytes, void** handle);
PL_API int32_t pl_stage_forward(void* handle, const pl_microbatch* mb, void* stream);
/* Repack the stage's projection weights (and lm_head) IN PLACE into pre-swizzled
 * 16 KB tiles [N/128][K/64] -- the shared-memory image of a 128 x 64 TMA box --
 * so every weight k-block streams as one contiguous bulk copy.  Weights whose N
 * is not a multiple of 256 stay row-major.  Synchronizes `stream`; afterwards
 * the weight buffers are only meaningful to this stage. */
PL_API int32_t pl_stage_pack_weights(void* handle, void* stream);
PL_API int32_t pl_stage_destroy(void* handle);

/* Live kernel timing for bench.py: CUDA events around the kernel groups of one
 * layer (a new pass: earlier records cleared; layer < 0 stops recording and keeps
 * them).  pl_stage_probe_read returns, per recorded forward, out_meta[3] = {phase,
 * T, kind} and out_ms[5]: kind 0 (one kernel per projection) = {qkv gemm,
 * rope+attention, o gemm, gate_up gemm, down gemm}; kind 1 (persistent decode
 * chain) = {decode attention, chain kernel, 0, 0, 0}.  Synchronize the stream first. */
PL_API int32_t pl_stage_probe(void* handle, int32_t layer);
/* Debug (PL_CHAIN_TRACE=k in the environment): per-unit globaltimer stamps of the
 * stage's k-th persistent chain launch, [grid][64][4] u64 = {claim time mod 2^40 |
 * claim index << 40, unit popped by the epilogue, accumulator ready, epilogue done}. */
PL_API int32_t pl_stage_chain_trace(void* handle, uint64_t* out_host, int64_t n, int32_t* grid);
/* Benchmark: `iters` launches of a persistent chain holding ONE projection of layer 0
 * (kind 0 o, 1 gate_up, 2 down, 3 qkv) at T tokens, without dependencies or
 * finalisation -- the chain kernel's weight stream alone (results are scratch). */
PL_API int32_t pl_stage_chain_bench(void* handle, int32_t kind, int32_t T, int32_t iters, void* stream);
PL_API int32_t pl_stage_probe_read(void* handle, float* out_ms_host, int32_t* out_meta_host, int32_t cap,
                            int32_t* n_host);

/* ------------------------------------------------------------ transport --- */

/* NCCL 2.28 P2P over NVLink.  One communicator per directed stage hop. */
PL_API int32_t pl_nccl_version(void);
PL_API int32_t pl_nccl_unique_id(uint8_t* id_host, int32_t len); /* len >= 128 */
PL_API int32_t pl_comm_init_rank(const uint8_t* id_host, int32_t nranks, int32_t rank, void** comm);
PL_API int32_t pl_comm_destroy(void* comm);
PL_API int32_t pl_p2p_send(void* comm, const void* buf, int64_t bytes, int32_t peer, void* stream);
PL_API int32_t pl_p2p_recv(void* comm, void* buf, int64_t bytes, int32_t peer, void* stream);

/* Link-throttle gate: block `stream` until %globaltimer >= *t0 + offset_ns. */
PL_API int32_t pl_record_globaltimer(uint64_t* dst, void* stream);
PL_API int32_t pl_gate_until_ns(const uint64_t* t0, uint64_t offset_ns, void* stream);

/* Host<->device plumbing without a Python round trip. */
PL_API int32_t pl_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream);
/* Single-process multi-GPU placement: enable NVLink peer access between every pair of
 * the listed devices, so same-process hops are direct peer copies. */
PL_API int32_t pl_enable_peer_access(int32_t ndev, const int32_t* devs);

/* ------------------------------------------------------------ scheduler --- */

/* Native virtual-clock scheduler: PipelineEngine.run (engine.py:509-600) with
 * choose_n / _round_terms (controller.py:68-186), admit_and_batch
 * (engine.py:155-238), LinkQueue (transport.py:70-160), compute_time
 * (profiles.py:95-121) and transmission_ns / s_to_ns (transport.py:32-33,
 * 199-200) restated bit-exactly.  Host-only; no GPU needed unless a pipeline
 * is attached.  Profiles: per (stage, phase) the sorted points
 * prof_x[prof_off[2s+ph] : prof_off[2s+ph+1]] (tokens) / prof_y (seconds),
 * phase 0 = prefill, 1 = decode; links: S forward hops then the return hop. */
typedef struct pl_sched_config {
  int32_t n_stages, n_links;
  int64_t max_batched_tokens;
  int32_t max_batch_size, n_max; /* n_max: effective (ControllerConfig.effective_n_max) */
  double bubble_epsilon, gain_delta;
  int32_t fixed_compute;         /* BudgetMode.FIXED_COMPUTE */
  int32_t decision_stride;
  int64_t chunk_size;            /* < 0: unchunked (chunk_size None / inf) */
  int32_t fcfs;                  /* SchedulingPolicy.FCFS */
  int32_t allow_mixed;
  int64_t bytes_per_token;       /* hidden_dim * dtype_bytes */
  int64_t feedback_bytes;        /* TOKEN_FEEDBACK_BYTES (placement.py:16) */
  const int64_t* prof_off;       /* [2 * n_stages + 1] */
  const int64_t* prof_x;
  const double* prof_y;
  const double* link_latency_s;  /* [n_links] */
  const double* link_bandwidth;  /* [n_links] bytes/s */
} pl_sched_config;

typedef struct pl_sched_request {
  int64_t id, arrival_ns, input_len, output_len; /* arrival_ns = s_to_ns(arrival_time) */
} pl_sched_request;

PL_API int32_t pl_sched_create(const pl_sched_config* cfg, void** handle);
PL_API int32_t pl_sched_destroy(void* handle);
PL_API int32_t pl_sched_choose_n(void* handle, int64_t queued_tokens, int32_t phase, int32_t* n,
                                 int64_t* budget, double* bubble);
/* Run the trace (trace order) to completion or horizon_ns (< 0: none).  With a
 * pipeline (pl_pipeline_create) every decision also issues its GPU work, and
 * the call returns once the device finished; NULL gives a pure virtual run. */
PL_API int32_t pl_sched_run(void* handle, const pl_sched_request* reqs, int64_t n_reqs,
                            int64_t horizon_ns, void* pipeline);
/* counts[8] = {events, link events, decisions, token emissions, first-compute
 * entries, busy intervals, end_ns, all_finished}. */
PL_API int32_t pl_sched_counts(void* handle, int64_t* counts_host);
/* Logs of the last run (host arrays sized by pl_sched_counts; NULL skips):
 *   events[4n]    time_ns, EventKind, subject, stage
 *   links[7n]     time_ns, link, payload, chunk index, bytes, class (0 prefill,
 *                 1 decode), event (0 enqueue, 1 emit, 2 sent, 3 deliver)
 *   decisions[3n] iteration, n, token budget; bubbles[n]
 *   emissions[2n] time_ns, request id;  first_compute[2n] request id, time_ns
 *   busy[3n]      stage, start_ns, end_ns
 *   req_state[2r] RequestState (0 queued, 1 prefill, 2 decoding, 3 finished),
 *                 tokens emitted; req_times[2r] first token / finish seconds
 *                 (NaN: none), in trace order. */
PL_API int32_t pl_sched_read(void* handle, int64_t* events, int64_t* links, int64_t* decisions,
                             double* bubbles, int64_t* emissions, int64_t* first_compute,
                             int64_t* busy, int64_t* req_state, double* req_times);

/* ------------------------------------------------------------ runtime ----- */

/* The GPU side of a pipeline run on this process (twin of backend.py's
 * GpuBackend): per stage s a pl_stage handle or NULL when the stage lives on
 * another rank, its compute stream and buffers; per link the NCCL
 * communicator when the hop crosses processes (this process is comm-rank 0 on
 * its outgoing hops, 1 on incoming). */
typedef struct pl_pipeline_config {
  int32_t n_stages, n_slots, max_blocks, block_size;
  int64_t num_blocks;
  int32_t max_tokens, max_reqs, d;
  int32_t throttle;      /* gate deliveries at the virtual link timing */
  int32_t record_links;  /* per-chunk device timestamps */
  void* const* stage;    /* [n_stages] */
  void* const* stream;   /* [n_stages] compute streams */
  const int32_t* device; /* [n_stages] CUDA ordinals */
  void* const* meta_dev; /* [n_stages] int32 metadata buffers */
  void* const* ids_dev;  /* [n_stages] int64 prompt-id buffer (head) */
  void* const* hidden;   /* [n_stages * n_slots] bf16 residual-stream payloads */
  void* const* out_ids;  /* [n_stages * n_slots] int64 tokens (last stage) */
  void* const* comm;     /* [n_stages] NCCL communicators or NULL */
  int64_t* const* ids_recv; /* head: [n_slots] return-hop landing buffers */
  int32_t fuse_transport;   /* decode payloads between stages of THIS process: the
                               producer's last residual epilogue stores straight into
                               the next stage's buffer (peer memory over NVLink); the
                               link issues no copy (prefill chunks still copy) */
} pl_pipeline_config;

PL_API int32_t pl_pipeline_create(const pl_pipeline_config* cfg, void** handle);
PL_API int32_t pl_pipeline_destroy(void* handle);
/* The trace of the next run: prompt ids of request i (trace order) are the
 * host array prompt_ids[prompt_off[i] : prompt_off[i+1]] (copied); head
 * outputs last_token [n_requests] and gen_tokens [n_requests, gen_stride]. */
PL_API int32_t pl_pipeline_set_requests(void* handle, int64_t n_requests, const int64_t* prompt_off_host,
                                        const int64_t* prompt_ids_host, int64_t* last_token,
                                        int64_t* gen_tokens, int32_t gen_stride);
/* counts[5] = {stage forwards, token scatters, chunk records, micro-batches,
 * request ids of those micro-batches}. */
PL_API int32_t pl_pipeline_counts(void* handle, int64_t* counts_host);
/* Device-clock results of the last run (seconds since the run's start event on
 * the stage's device; NULL skips):  busy[2n] stage, micro-batch / busy_s[2n]
 * start, end;  fb_mb[n] / fb_s[n] token scatters on the head;  chunks[6n] link,
 * src stage, payload, index, bytes, class / chunk_s[3n] enqueue, emit, sent;
 * mb_log[4n] micro-batch, decode, R, work (context sum or tokens) with
 * request ids mb_req_ids[mb_req_off[i] : mb_req_off[i+1]]. */
PL_API int32_t pl_pipeline_read(void* handle, double* run_time_s, double* decode_start_s,
                                int64_t* busy, double* busy_s, int64_t* fb_mb, double* fb_s,
                                int64_t* chunks, double* chunk_s, int64_t* mb_log,
                                int64_t* mb_req_off, int64_t* mb_req_ids);

#ifdef __cplusplus
}
#endif
#endif /* B200LINK_H_ */
