// Stage runtime: the per-stage decoder forward that replaces the reference's
// simulated compute call `compute_time(stage.profile, phase, mb.batched_tokens)`
// (engine.py:384).  One C call launches every kernel of the stage's layer range
// on the caller's stream, so the Python driver pays one FFI crossing per
// micro-batch per stage instead of ~10 per layer.
//
// Layer (modeling_llama.py:313-331, with the residual add fused into the GEMM
// epilogues so only the single residual stream `hidden` crosses stages):
//   a   = rmsnorm(hidden) * w_attn
//   qkv = a . Wqkv^T (+ b)                      tcgen05 GEMM
//   q,k = rope(q,k); cache[k,v] <- k,v          rope_kv
//   o   = attn(q, k, v)                         prefill (mma.sync FA2) | decode (paged)
//   hidden = hidden + o . Wo^T                  tcgen05 GEMM, RESIDUAL epilogue
//   a   = rmsnorm(hidden) * w_mlp
//   m   = silu(a . Wg^T) * (a . Wu^T)           tcgen05 GEMM, SWIGLU epilogue
//   hidden = hidden + m . Wd^T                  tcgen05 GEMM, RESIDUAL epilogue
// First stage: hidden = embed(ids).  Last stage: final norm of each request's
// last row, lm_head GEMM with fused argmax -> int64 token ids (engine.py:409).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "pl_internal.h"

namespace pl {

namespace {

int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }

struct Layout {
  int64_t a, qkv, o, m, hn, gemm_ws, attn_ws, chain, total;
};

// Decode layers run as persistent chain kernels (chain.cu) when the stage's projection
// weights are packed and T <= 256.  Three chain shapes per stage: the first layer's qkv,
// a middle layer (o, gate_up, down, next qkv) and the last layer (o, gate_up, down).
enum ChainType { CH_QKV_ONLY = 0, CH_FULL = 1, CH_LAST = 2, CH_TYPES = 3 };

struct ChainPlan {
  int njobs = 0;
  int kind[4] = {0, 0, 0, 0};
  int64_t N[4] = {0, 0, 0, 0}, K[4] = {0, 0, 0, 0};
  int splits[4] = {1, 1, 1, 1};
  std::vector<int4> units;  // global claim order
  int64_t units_off = 0;    // byte offset inside the chain region
};

struct ChainLayout {
  ChainPlan plan[CH_TYPES];
  int grid = 0, Tp_max = 0;
  int64_t partial[4] = {0, 0, 0, 0};  // by ChainKind
  int64_t part_ss = 0, row_parts = 0, ctr = 0, gu_flag = 0, bytes = 0;
};

int chain_tp(int T) { return T <= 16 ? 16 : T <= 32 ? 32 : T <= 64 ? 64 : T <= 128 ? 128 : 256; }

ChainLayout chain_layout(const pl_stage_config& c, int grid) {
  ChainLayout C;
  C.grid = grid;
  if (grid <= 0 || c.num_layers <= 0) return C;
  const int64_t d = c.d, qkv_dim = static_cast<int64_t>(c.Hq + 2 * c.Hkv) * c.hd;
  const int64_t attn_dim = static_cast<int64_t>(c.Hq) * c.hd, ffn = c.ffn;
  C.Tp_max = chain_tp(std::min(c.max_reqs, 256));
  const int64_t NN[4] = {d, 2 * ffn, d, qkv_dim}, KK[4] = {attn_dim, d, ffn, d};
  const int kinds[CH_TYPES][4] = {{CHAIN_QKV, 0, 0, 0}, {CHAIN_O, CHAIN_GATE_UP, CHAIN_DOWN, CHAIN_QKV},
                                  {CHAIN_O, CHAIN_GATE_UP, CHAIN_DOWN, 0}};
  const int nj[CH_TYPES] = {1, 4, 3};
  int max_split[4] = {1, 1, 1, 1};
  const int ring = chain_ring_kb(64);  // planning uses one ring depth for every T
  for (int t = 0; t < CH_TYPES; ++t) {
    ChainPlan& P = C.plan[t];
    P.njobs = nj[t];
    for (int j = 0; j < P.njobs; ++j) {
      P.kind[j] = kinds[t][j];
      P.N[j] = NN[P.kind[j]];
      P.K[j] = KK[P.kind[j]];
    }
    chain_plan(P.kind, P.njobs, P.N, P.K, grid, ring, P.splits, P.units);
    for (int j = 0; j < P.njobs; ++j) max_split[P.kind[j]] = std::max(max_split[P.kind[j]], P.splits[j]);
    if (getenv("PL_CHAIN_VERBOSE")) {
      fprintf(stderr, "chain plan %d (grid %d):", t, grid);
      for (int j = 0; j < P.njobs; ++j)
        fprintf(stderr, " kind %d N %lld K %lld splits %d;", P.kind[j], (long long)P.N[j], (long long)P.K[j],
                P.splits[j]);
      fprintf(stderr, " %zu units\n", P.units.size());
    }
  }
  int64_t off = 0;
  for (int k = 0; k < 4; ++k) {
    const int64_t tiles = NN[k] / 128;
    C.partial[k] = off;  // every split-K projection writes partials (also at one split)
    off += align256(k == CHAIN_GATE_UP ? 0 : max_split[k] * tiles * C.Tp_max * 128 * 4);
  }
  C.part_ss = off;
  off += align256(2 * C.Tp_max * (d / 256) * 4);  // pieces of >= 256 features
  C.row_parts = off;
  off += align256(2 * C.Tp_max * 4);
  C.ctr = off;  // two counter sets (launch parity)
  off += align256(2 * CHAIN_CTR_BYTES);
  C.gu_flag = off;
  off += align256(ffn / 64 * 4);
  for (int t = 0; t < CH_TYPES; ++t) {
    C.plan[t].units_off = off;
    off += align256(static_cast<int64_t>(C.plan[t].units.size()) * 16);
  }
  C.bytes = off;
  return C;
}

bool chain_shapes_ok(const pl_stage_config& c) {
  const int64_t qkv_dim = static_cast<int64_t>(c.Hq + 2 * c.Hkv) * c.hd;
  return c.hd == 128 && c.d % 256 == 0 && (2 * static_cast<int64_t>(c.ffn)) % 256 == 0 && c.ffn % 64 == 0 &&
         qkv_dim % 256 == 0 && (static_cast<int64_t>(c.Hq) * c.hd) % 64 == 0 && c.d <= 16384;
}

int device_sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  return n;
}

Layout stage_layout(const pl_stage_config& c) {
  const int64_t T = c.max_tokens, R = c.max_reqs;
  const int64_t qkv_dim = static_cast<int64_t>(c.Hq + 2 * c.Hkv) * c.hd;
  const int64_t attn_dim = static_cast<int64_t>(c.Hq) * c.hd;
  Layout L{};
  int64_t off = 0;
  L.a = off;
  off += align256(T * c.d * 2);
  L.qkv = off;
  off += align256(T * qkv_dim * 2);
  L.o = off;
  off += align256(T * attn_dim * 2);
  L.m = off;
  off += align256(T * static_cast<int64_t>(c.ffn) * 2);
  L.hn = off;
  off += align256(R * c.d * 2);
  // split-K partials are only used on the SWAP (T <= 256) path
  int64_t gws = 0;
  const int64_t Ts[2] = {std::min<int64_t>(T, 256), std::min<int64_t>(R, 256)};
  for (int64_t t : Ts) {
    gws = std::max(gws, gemm_workspace_bytes(t, qkv_dim, c.d, EPI_BIAS));
    gws = std::max(gws, gemm_workspace_bytes(t, c.d, attn_dim, EPI_RESIDUAL));
    gws = std::max(gws, gemm_workspace_bytes(t, 2 * static_cast<int64_t>(c.ffn), c.d, EPI_SWIGLU));
    gws = std::max(gws, gemm_workspace_bytes(t, c.d, c.ffn, EPI_RESIDUAL));
  }
  if (c.is_last) gws = std::max(gws, gemm_workspace_bytes(std::min<int64_t>(R, 256), c.vocab, c.d, EPI_ARGMAX));
  L.gemm_ws = off;
  off += align256(gws);
  L.attn_ws = off;
  off += align256(attn_decode_workspace_bytes(static_cast<int>(R), c.Hq, c.max_ctx, c.hd));
  L.chain = off;
  if (chain_shapes_ok(c)) off += align256(chain_layout(c, device_sms() * chain_ctas_per_sm()).bytes);
  L.total = off;
  return L;
}

}  // namespace

struct ProbeRec {
  cudaEvent_t ev[7];
  int phase, T, kind;  // kind 0: per-projection kernels, 1: attention + chain kernel
};

// Makes the stage's GPU current for the duration of a call (one process may drive
// stages on several GPUs; kernels must launch on the device that owns the stream).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

struct Stage {
  int dev = 0;  // the CUDA device the stage was created on
  pl_stage_config cfg;
  std::vector<pl_layer_weights> layers;
  uint8_t* ws;
  Layout L;
  int probe_layer = -1;
  std::vector<ProbeRec> probes;
  size_t probe_used = 0;
  // weights repacked into pre-swizzled 16 KB tiles (pl_stage_pack_weights)
  bool pk_qkv = false, pk_o = false, pk_gu = false, pk_down = false, pk_lm = false;
  // persistent decode-layer kernels
  bool chain_ok = false;
  ChainLayout CL;
  int ch_seq = 0;  // chain launches so far (gate_up tile flags hold the finishing launch's number)
  // debug: PL_CHAIN_TRACE=k records per-unit globaltimer stamps of the k-th chain launch
  unsigned long long* ch_trace = nullptr;
  int ch_trace_seq = 0;

  int init_chain() {
    chain_ok = false;
    if (!chain_shapes_ok(cfg)) return PL_OK;
    CL = chain_layout(cfg, device_sms() * chain_ctas_per_sm());
    if (CL.bytes == 0) return PL_OK;
    for (int t = 0; t < CH_TYPES; ++t) {
      const ChainPlan& P = CL.plan[t];
      cudaError_t e = cudaMemcpy(ws + L.chain + P.units_off, P.units.data(), P.units.size() * sizeof(int4),
                                 cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return set_cuda_error(e, "chain unit tables");
    }
    return PL_OK;
  }

  // Opt-in (PL_CHAIN=1): measured slower than one kernel per projection on B200 at
  // every decode T (profiles/r2/chain_*.log) -- its software dependency
  // tracking (two global norm barriers, split finalisation, the qkv tail) costs more
  // than the fill/drain it removes between kernels
  bool use_chain(int T) const {
    static const bool on = [] { const char* v = getenv("PL_CHAIN"); return v && v[0] == '1'; }();
    return on && CL.bytes > 0 && pk_qkv && pk_o && pk_gu && pk_down && T <= CL.Tp_max && T <= 256;
  }

  // pl_stage_chain_bench: a chain of ONE projection of layer 0 (kind: 0 o, 1 gate_up, 2
  // down, 3 qkv) with no dependencies and no finalisation -- the weight stream alone
  std::vector<ChainPlan> bench_plans;
  int bench_chain(int kind, int T, cudaStream_t st) {
    if (CL.bytes == 0 || kind < 0 || kind > 3 || T <= 0 || T > CL.Tp_max)
      return set_error(PL_ERR_CONFIG, "chain_bench: unavailable (kind %d, T %d)", kind, T);
    if (bench_plans.empty()) bench_plans.resize(4);
    ChainPlan& P = bench_plans[kind];
    const pl_stage_config& c = cfg;
    const int64_t d = c.d, qkv_dim = static_cast<int64_t>(c.Hq + 2 * c.Hkv) * c.hd;
    const int64_t NN[4] = {d, 2 * static_cast<int64_t>(c.ffn), d, qkv_dim};
    const int64_t KK[4] = {static_cast<int64_t>(c.Hq) * c.hd, d, c.ffn, d};
    if (P.njobs == 0) {
      P.njobs = 1;
      P.kind[0] = kind;
      P.N[0] = NN[kind];
      P.K[0] = KK[kind];
      // the splits the full chain uses for this projection
      const ChainPlan& F = CL.plan[CH_FULL];
      for (int j = 0; j < F.njobs; ++j)
        if (F.kind[j] == kind) P.splits[0] = F.splits[j];
      const int per = static_cast<int>((KK[kind] / 64 + P.splits[0] - 1) / P.splits[0]);
      for (int sp = 0; sp < P.splits[0]; ++sp)
        for (int tl = 0; tl < static_cast<int>(NN[kind] / 128); ++tl) {
          const int k0 = sp * per, n = std::min(static_cast<int>(KK[kind] / 64), k0 + per) - k0;
          if (n > 0) P.units.push_back(make_int4(0, tl, k0, n));
        }
      // unit table in the chain region's tail (the full plan's table is the largest)
      P.units_off = CL.plan[CH_FULL].units_off;
    }
    uint8_t* base = ws + L.chain;
    cudaError_t e = cudaMemcpyAsync(base + P.units_off, P.units.data(), P.units.size() * sizeof(int4),
                                    cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return set_cuda_error(e, "chain_bench units");
    const pl_layer_weights& w = layers[0];
    const void* wts[4] = {w.w_o, w.w_gate_up, w.w_down, w.w_qkv};
    ChainLaunch k;
    k.T = T;
    k.Tp = chain_tp(T);
    k.njobs = 1;
    k.d = c.d;
    k.ffn = c.ffn;
    k.attn_dim = c.Hq * c.hd;
    k.grid = CL.grid;
    k.kind[0] = kind;
    k.N[0] = P.N[0];
    k.K[0] = P.K[0];
    k.splits[0] = P.splits[0];
    k.w[0] = wts[kind];
    k.partial[0] = reinterpret_cast<float*>(base + CL.partial[kind]);
    k.units = reinterpret_cast<const int4*>(base + P.units_off);
    k.units_host = P.units.data();
    k.n_units = static_cast<int>(P.units.size());
    k.o_attn = buf(L.o);
    k.h = buf(L.a);  // scratch: nothing is finalised
    k.a = buf(L.a);
    k.m = buf(L.m);
    k.q_out = buf(L.qkv);
    k.ld_q = qkv_dim;
    k.part_ss = reinterpret_cast<float*>(base + CL.part_ss);
    k.row_parts = reinterpret_cast<int*>(base + CL.row_parts);
    k.eps = c.eps;
    k.seq = ++ch_seq;
    k.ctr = base + CL.ctr + (k.seq & 1) * CHAIN_CTR_BYTES;
    k.gu_flag = reinterpret_cast<int*>(base + CL.gu_flag);
    k.bench = 1;
    return chain_launch(k, st);
  }

  // one chain launch of type `t` for layer l (CH_QKV_ONLY: layer l's qkv; CH_FULL: layer
  // l's o, gate_up, down and layer l+1's qkv; CH_LAST: layer l's o, gate_up, down)
  int launch_chain(int t, int l, int T, const int32_t* pos, const int32_t* slot, __nv_bfloat16* hid,
                   cudaStream_t st) {
    const pl_stage_config& c = cfg;
    const ChainPlan& P = CL.plan[t];
    const pl_layer_weights& w = layers[l];
    const pl_layer_weights& wq = (t == CH_FULL) ? layers[l + 1] : w;
    uint8_t* base = ws + L.chain;
    ChainLaunch k;
    k.T = T;
    k.Tp = chain_tp(T);
    k.njobs = P.njobs;
    k.d = c.d;
    k.ffn = c.ffn;
    k.attn_dim = c.Hq * c.hd;
    k.grid = CL.grid;
    const void* wts[4] = {w.w_o, w.w_gate_up, w.w_down, wq.w_qkv};
    for (int j = 0; j < P.njobs; ++j) {
      const int kd = P.kind[j];
      k.kind[j] = kd;
      k.N[j] = P.N[j];
      k.K[j] = P.K[j];
      k.splits[j] = P.splits[j];
      k.w[j] = wts[kd];
      k.partial[j] = reinterpret_cast<float*>(base + CL.partial[kd]);
    }
    k.units = reinterpret_cast<const int4*>(base + P.units_off);
    k.units_host = P.units.data();
    k.n_units = static_cast<int>(P.units.size());
    k.o_attn = buf(L.o);
    k.h = hid;
    k.a = buf(L.a);
    k.m = buf(L.m);
    k.q_out = buf(L.qkv);
    k.ld_q = static_cast<int64_t>(c.Hq + 2 * c.Hkv) * c.hd;
    k.part_ss = reinterpret_cast<float*>(base + CL.part_ss);
    k.row_parts = reinterpret_cast<int*>(base + CL.row_parts);
    k.has_norm[0] = t != CH_QKV_ONLY;
    k.has_norm[1] = t == CH_FULL;
    k.norm_w[0] = static_cast<const __nv_bfloat16*>(w.mlp_norm);
    k.norm_w[1] = t == CH_FULL ? static_cast<const __nv_bfloat16*>(wq.attn_norm) : nullptr;
    k.eps = c.eps;
    k.bias = static_cast<const __nv_bfloat16*>(wq.b_qkv);
    k.pos = pos;
    k.slot = slot;
    k.cos_sin = static_cast<const __nv_bfloat16*>(c.cos_sin);
    k.max_pos = c.max_pos;
    k.k_cache = static_cast<__nv_bfloat16*>(wq.k_cache);
    k.v_cache = static_cast<__nv_bfloat16*>(wq.v_cache);
    k.block_size = c.block_size;
    k.Hq = c.Hq;
    k.Hkv = c.Hkv;
    k.seq = ++ch_seq;
    k.ctr = base + CL.ctr + (k.seq & 1) * CHAIN_CTR_BYTES;
    if (ch_trace_seq == 0) {
      const char* v = getenv("PL_CHAIN_TRACE");
      ch_trace_seq = v ? atoi(v) : -1;
      if (ch_trace_seq > 0 && cudaMalloc(&ch_trace, static_cast<size_t>(CL.grid) * 64 * 4 * 8) != cudaSuccess)
        ch_trace = nullptr;
      if (ch_trace) cudaMemset(ch_trace, 0, static_cast<size_t>(CL.grid) * 64 * 4 * 8);
    }
    k.trace = (ch_trace && k.seq == ch_trace_seq) ? ch_trace : nullptr;
    k.gu_flag = reinterpret_cast<int*>(base + CL.gu_flag);
    return chain_launch(k, st);
  }

  int pack(cudaStream_t st) {
    const pl_stage_config& c = cfg;
    const int64_t d = c.d, qkv_dim = static_cast<int64_t>(c.Hq + 2 * c.Hkv) * c.hd;
    const int64_t attn_dim = static_cast<int64_t>(c.Hq) * c.hd, ffn = c.ffn;
    struct Job { bool* flag; int64_t N, K; };
    const Job jobs[5] = {{&pk_qkv, qkv_dim, d}, {&pk_o, d, attn_dim}, {&pk_gu, 2 * ffn, d}, {&pk_down, d, ffn},
                         {&pk_lm, c.is_last ? c.vocab : 0, d}};
    int64_t biggest = 0;
    for (const Job& j : jobs)
      if (j.N % 256 == 0 && j.K % 64 == 0 && j.N > 0) biggest = std::max(biggest, j.N * j.K * 2);
    if (biggest == 0) return PL_OK;
    void* tmp = nullptr;
    cudaError_t e = cudaMalloc(&tmp, biggest);
    if (e != cudaSuccess) return set_cuda_error(e, "pack_weights: temp");
    int rc = PL_OK;
    auto pack_one = [&](void* w, int64_t N, int64_t K, bool swiglu) {
      if (rc || !w) return;
      e = cudaMemcpyAsync(tmp, w, N * K * 2, cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) {
        rc = set_cuda_error(e, "pack_weights: copy");
        return;
      }
      rc = pack_weight_launch(static_cast<const __nv_bfloat16*>(tmp), K, N, K, w, st, swiglu);
    };
    for (const Job& j : jobs) {
      if (j.N <= 0 || j.N % 256 || j.K % 64 || *j.flag) continue;
      if (j.flag == &pk_lm) {
        pack_one(const_cast<void*>(c.lm_head), j.N, j.K, false);
      } else {
        for (auto& lw : layers) {
          const void* w = j.flag == &pk_qkv ? lw.w_qkv : j.flag == &pk_o ? lw.w_o : j.flag == &pk_gu ? lw.w_gate_up
                                                                                                 : lw.w_down;
          pack_one(const_cast<void*>(w), j.N, j.K, j.flag == &pk_gu);
        }
      }
      if (rc) break;
      *j.flag = true;
    }
    e = cudaStreamSynchronize(st);
    cudaFree(tmp);
    if (!rc && e != cudaSuccess) rc = set_cuda_error(e, "pack_weights");
    return rc;
  }

  __nv_bfloat16* buf(int64_t off) const { return reinterpret_cast<__nv_bfloat16*>(ws + off); }

  cudaEvent_t* next_probe(int phase, int T, int kind = 0) {
    if (probe_used == probes.size()) {
      if (probes.size() >= 65536) return nullptr;
      ProbeRec r{};
      for (auto& e : r.ev)
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
      probes.push_back(r);
    }
    ProbeRec& r = probes[probe_used++];
    r.phase = phase;
    r.T = T;
    r.kind = kind;
    return r.ev;
  }

  int forward(const pl_microbatch& mb, cudaStream_t st) {
    const pl_stage_config& c = cfg;
    const int T = mb.T, R = mb.R;
    if (T <= 0 || R <= 0) return set_error(PL_ERR_CONFIG, "stage_forward: empty micro-batch");
    if (T > c.max_tokens || R > c.max_reqs)
      return set_error(PL_ERR_CONFIG, "stage_forward: micro-batch (T=%d, R=%d) exceeds capacity (%d, %d)",
                       T, R, c.max_tokens, c.max_reqs);
    const bool decode = mb.phase == 1;
    const bool mixed = mb.phase == 2;
    if (mb.phase < 0 || mb.phase > 2) return set_error(PL_ERR_CONFIG, "stage_forward: bad phase %d", mb.phase);
    if (decode && T != R) return set_error(PL_ERR_CONFIG, "stage_forward: decode needs T == R");
    // decode requests lead the batch: rows [0, Rd); prompts fill rows [Rd, T)
    const int Rd = decode ? R : (mixed ? mb.n_decode : 0);
    const int Rp = R - Rd;
    if (mixed && (Rd <= 0 || Rp <= 0 || T - Rd < Rp))
      return set_error(PL_ERR_CONFIG, "stage_forward: mixed batch needs decode and prompt requests");
    if (!mb.meta || !mb.hidden) return set_error(PL_ERR_CONFIG, "stage_forward: missing buffers");
    const int32_t* pos = mb.meta;
    const int32_t* slot = pos + T;
    const int32_t* req_slot = slot + T;
    const int32_t* cu = req_slot + T;
    const int32_t* ctx = cu + R + 1;
    const int32_t* last_idx = ctx + R;
    const int32_t* bt = last_idx + R;

    const int64_t d = c.d;
    const int64_t qkv_dim = static_cast<int64_t>(c.Hq + 2 * c.Hkv) * c.hd;
    const int64_t attn_dim = static_cast<int64_t>(c.Hq) * c.hd;
    const int64_t ffn = c.ffn;
    __nv_bfloat16* hid = static_cast<__nv_bfloat16*>(mb.hidden);
    __nv_bfloat16* a = buf(L.a);
    __nv_bfloat16* qkv = buf(L.qkv);
    __nv_bfloat16* o = buf(L.o);
    __nv_bfloat16* m = buf(L.m);
    void* gws = ws + L.gemm_ws;
    const int64_t gws_bytes = L.attn_ws - L.gemm_ws;
    const float scale = 1.0f / sqrtf(static_cast<float>(c.hd));
    int rc;

    if (c.is_first) {
      if (Rd > 0) {
        if (!mb.last_token) return set_error(PL_ERR_CONFIG, "stage_forward: decode needs last_token");
        rc = embed_launch(nullptr, req_slot, mb.last_token, static_cast<const __nv_bfloat16*>(c.embed),
                          c.vocab, Rd, c.d, hid, st);
        if (rc) return rc;
      }
      if (Rp > 0) {
        if (!mb.token_ids) return set_error(PL_ERR_CONFIG, "stage_forward: prefill needs token_ids");
        rc = embed_launch(mb.token_ids + Rd, nullptr, nullptr, static_cast<const __nv_bfloat16*>(c.embed),
                          c.vocab, T - Rd, c.d, hid + static_cast<int64_t>(Rd) * c.d, st);
        if (rc) return rc;
      }
    }

    if (decode && use_chain(T) && !mb.peer_hidden) {
      // persistent chain kernels: per layer one attention launch and one chain launch
      for (int l = 0; l < c.num_layers; ++l) {
        const pl_layer_weights& w = layers[l];
        cudaEvent_t* ev = (l == probe_layer) ? next_probe(mb.phase, T, 1) : nullptr;
        if (l == 0) {
          if ((rc = rmsnorm_launch(hid, d, nullptr, static_cast<const __nv_bfloat16*>(w.attn_norm), c.eps, T,
                                   c.d, a, d, st)))
            return rc;
          if ((rc = launch_chain(CH_QKV_ONLY, 0, T, pos, slot, hid, st))) return rc;
        }
        if (ev) cudaEventRecord(ev[0], st);
        rc = attn_decode_launch(qkv, qkv_dim, static_cast<const __nv_bfloat16*>(w.k_cache),
                                static_cast<const __nv_bfloat16*>(w.v_cache), c.num_blocks, c.block_size, bt,
                                c.max_blocks_per_req, ctx, R, mb.max_ctx, c.Hq, c.Hkv, c.hd, scale, o, attn_dim,
                                ws + L.attn_ws, L.chain - L.attn_ws, st);
        if (rc) return rc;
        if (ev) cudaEventRecord(ev[1], st);
        if ((rc = launch_chain(l + 1 < c.num_layers ? CH_FULL : CH_LAST, l, T, pos, slot, hid, st))) return rc;
        if (ev) cudaEventRecord(ev[2], st);
      }
      return finish_last(mb, hid, last_idx, R, gws, gws_bytes, st);
    }

    // Decode-path fusions (split-K reductions double as epilogues): QKV reduce + RoPE +
    // KV append, and residual reduce + the next RMSNorm.  `a_ready` tracks whether the
    // previous fused reduction already produced this layer's normalized input.
    static const bool fuse_on = [] { const char* v = getenv("PL_FUSE"); return !(v && v[0] == '0'); }();
    bool a_ready = false;
    for (int l = 0; l < c.num_layers; ++l) {
      const pl_layer_weights& w = layers[l];
      cudaEvent_t* ev = (l == probe_layer) ? next_probe(mb.phase, T) : nullptr;
      auto mark = [&](int i) {
        if (ev) cudaEventRecord(ev[i], st);
      };
      if (!a_ready &&
          (rc = rmsnorm_launch(hid, d, nullptr, static_cast<const __nv_bfloat16*>(w.attn_norm), c.eps,
                               T, c.d, a, d, st)))
        return rc;
      mark(0);
      FusedEpi qf;
      if (fuse_on) {
        qf.kind = FUSE_QKV_ROPE;
        qf.pos = pos;
        qf.slot = slot;
        qf.cos_sin = static_cast<const __nv_bfloat16*>(c.cos_sin);
        qf.max_pos = c.max_pos;
        qf.k_cache = static_cast<__nv_bfloat16*>(w.k_cache);
        qf.v_cache = static_cast<__nv_bfloat16*>(w.v_cache);
        qf.block_size = c.block_size;
        qf.Hq = c.Hq;
        qf.Hkv = c.Hkv;
      }
      bool roped = false;
      if ((rc = gemm_launch(a, d, static_cast<const __nv_bfloat16*>(w.w_qkv), d,
                            static_cast<const __nv_bfloat16*>(w.b_qkv), qkv, qkv_dim, nullptr, 0, T,
                            qkv_dim, d, w.b_qkv ? EPI_BIAS : EPI_STORE, gws, gws_bytes, nullptr, st,
                            &qf, &roped, pk_qkv)))
        return rc;
      mark(1);
      if (!roped &&
          (rc = rope_kv_launch(qkv, qkv_dim, pos, slot, static_cast<const __nv_bfloat16*>(c.cos_sin),
                               c.max_pos, static_cast<__nv_bfloat16*>(w.k_cache),
                               static_cast<__nv_bfloat16*>(w.v_cache), c.block_size, T, c.Hq, c.Hkv,
                               c.hd, st)))
        return rc;
      if (Rd > 0) {  // one query row per decode request over its paged context
        rc = attn_decode_launch(qkv, qkv_dim, static_cast<const __nv_bfloat16*>(w.k_cache),
                                static_cast<const __nv_bfloat16*>(w.v_cache), c.num_blocks,
                                c.block_size, bt,
                                c.max_blocks_per_req, ctx, Rd, mb.max_ctx, c.Hq, c.Hkv, c.hd, scale, o,
                                attn_dim, ws + L.attn_ws, L.chain - L.attn_ws, st);
        if (rc) return rc;
      }
      if (Rp > 0) {  // causal attention over the prompt rows (cu_seqlens are absolute rows)
        rc = attn_prefill_launch(qkv, qkv_dim, cu + Rd, Rp, mb.max_seqlen, c.Hq, c.Hkv, c.hd, scale, o,
                                 attn_dim, st, T);
        if (rc) return rc;
      }
      mark(2);
      auto norm_fuse = [&](const void* norm_w) {
        FusedEpi f;
        if (fuse_on && norm_w) {
          f.kind = FUSE_RESIDUAL_NORM;
          f.norm_w = static_cast<const __nv_bfloat16*>(norm_w);
          f.eps = c.eps;
          f.norm_out = a;
          f.ld_norm = d;
        }
        return f;
      };
      FusedEpi of = norm_fuse(w.mlp_norm);
      bool normed = false;
      if ((rc = gemm_launch(o, attn_dim, static_cast<const __nv_bfloat16*>(w.w_o), attn_dim, nullptr,
                            hid, d, hid, d, T, d, attn_dim, EPI_RESIDUAL, gws, gws_bytes, nullptr, st,
                            &of, &normed, pk_o)))
        return rc;
      mark(3);
      if (!normed &&
          (rc = rmsnorm_launch(hid, d, nullptr, static_cast<const __nv_bfloat16*>(w.mlp_norm), c.eps, T,
                               c.d, a, d, st)))
        return rc;
      mark(4);
      if ((rc = gemm_launch(a, d, static_cast<const __nv_bfloat16*>(w.w_gate_up), d, nullptr, m, ffn,
                            nullptr, 0, T, 2 * ffn, d, EPI_SWIGLU, gws, gws_bytes, nullptr, st, nullptr,
                            nullptr, pk_gu)))
        return rc;
      mark(5);
      // the next layer's input norm rides on this residual reduction (not across stages);
      // the stage's last residual write also lands in the next stage's buffer (fused
      // transport, pl_microbatch.peer_hidden)
      FusedEpi df = norm_fuse(l + 1 < c.num_layers ? layers[l + 1].attn_norm : nullptr);
      if (l + 1 == c.num_layers && mb.peer_hidden) {
        if (!decode || c.is_last)
          return set_error(PL_ERR_CONFIG, "stage_forward: peer_hidden is for decode micro-batches of non-last stages");
        df.mirror = static_cast<__nv_bfloat16*>(mb.peer_hidden);
      }
      if ((rc = gemm_launch(m, ffn, static_cast<const __nv_bfloat16*>(w.w_down), ffn, nullptr, hid, d,
                            hid, d, T, d, ffn, EPI_RESIDUAL, gws, gws_bytes, nullptr, st, &df,
                            &a_ready, pk_down)))
        return rc;
      mark(6);
    }

    return finish_last(mb, hid, last_idx, R, gws, gws_bytes, st);
  }

  // last stage: final norm of each request's newest row, lm_head + argmax (engine.py:409)
  int finish_last(const pl_microbatch& mb, __nv_bfloat16* hid, const int32_t* last_idx, int R, void* gws,
                  int64_t gws_bytes, cudaStream_t st) {
    const pl_stage_config& c = cfg;
    const int64_t d = c.d;
    int rc;
    if (c.is_last) {
      if (!mb.out_ids) return set_error(PL_ERR_CONFIG, "stage_forward: last stage needs out_ids");
      __nv_bfloat16* hn = buf(L.hn);
      if ((rc = rmsnorm_launch(hid, d, last_idx, static_cast<const __nv_bfloat16*>(c.final_norm), c.eps,
                               R, c.d, hn, d, st)))
        return rc;
      if ((rc = gemm_launch(hn, d, static_cast<const __nv_bfloat16*>(c.lm_head), d, nullptr, nullptr, 0,
                            nullptr, 0, R, c.vocab, d, EPI_ARGMAX, gws, gws_bytes, mb.out_ids, st, nullptr,
                            nullptr, pk_lm)))
        return rc;
    }
    return PL_OK;
  }
};

}  // namespace pl

using namespace pl;

extern "C" {

int64_t pl_stage_workspace_bytes(const pl_stage_config* cfg) {
  if (!cfg) return -1;
  return stage_layout(*cfg).total;
}

int32_t pl_stage_create(const pl_stage_config* cfg, const pl_layer_weights* layers, void* workspace,
                        int64_t workspace_bytes, void** handle) {
  if (!cfg || !handle || (cfg->num_layers > 0 && !layers))
    return set_error(PL_ERR_CONFIG, "stage_create: null argument");
  if (cfg->hd != 128) return set_error(PL_ERR_CONFIG, "stage_create: head_dim must be 128");
  if (cfg->d % 64 || cfg->ffn % 64)
    return set_error(PL_ERR_CONFIG, "stage_create: d and ffn must be multiples of 64");
  if (cfg->block_size != 64) return set_error(PL_ERR_CONFIG, "stage_create: KV block size must be 64");
  if (cfg->is_first && !cfg->embed) return set_error(PL_ERR_CONFIG, "stage_create: first stage needs embed");
  if (cfg->is_last && (!cfg->lm_head || !cfg->final_norm))
    return set_error(PL_ERR_CONFIG, "stage_create: last stage needs lm_head and final_norm");
  const int prc = pl_preload_kernels();  // no lazy module loads once links are live
  if (prc) return prc;
  const Layout L = stage_layout(*cfg);
  if (!workspace || workspace_bytes < L.total)
    return set_error(PL_ERR_CONFIG, "stage_create: workspace %lld < required %lld",
                     (long long)workspace_bytes, (long long)L.total);
  // deterministic initial contents (never read before written)
  cudaError_t e = cudaMemset(workspace, 0, static_cast<size_t>(L.total));
  if (e != cudaSuccess) return set_cuda_error(e, "stage workspace memset");
  Stage* s = new Stage();
  cudaGetDevice(&s->dev);
  s->cfg = *cfg;
  s->layers.assign(layers, layers + cfg->num_layers);
  s->ws = static_cast<uint8_t*>(workspace);
  s->L = L;
  const int rc = s->init_chain();
  if (rc) {
    delete s;
    return rc;
  }
  *handle = s;
  return PL_OK;
}

int32_t pl_stage_forward(void* handle, const pl_microbatch* mb, void* stream) {
  if (!handle || !mb) return set_error(PL_ERR_CONFIG, "stage_forward: null argument");
  Stage* s = static_cast<Stage*>(handle);
  DeviceGuard g(s->dev);
  return s->forward(*mb, static_cast<cudaStream_t>(stream));
}

int32_t pl_stage_pack_weights(void* handle, void* stream) {
  if (!handle) return set_error(PL_ERR_CONFIG, "stage_pack_weights: null handle");
  Stage* s = static_cast<Stage*>(handle);
  DeviceGuard g(s->dev);
  return s->pack(static_cast<cudaStream_t>(stream));
}

// Debug: copy the per-unit stamps of the traced chain launch (PL_CHAIN_TRACE=k) to the
// host: [grid][64][4] u64 = {claim time mod 2^40 | claim index << 40, unit popped by the
// epilogue, accumulator ready, epilogue done}; returns the grid size in *grid.
int32_t pl_stage_chain_trace(void* handle, uint64_t* out_host, int64_t n, int32_t* grid) {
  Stage* s = static_cast<Stage*>(handle);
  if (!s || !out_host || !grid) return set_error(PL_ERR_CONFIG, "chain_trace: null argument");
  *grid = s->CL.grid;
  if (!s->ch_trace) return set_error(PL_ERR_CONFIG, "chain_trace: set PL_CHAIN_TRACE=<launch number>");
  const int64_t total = static_cast<int64_t>(s->CL.grid) * 64 * 4;
  cudaError_t e = cudaMemcpy(out_host, s->ch_trace, std::min(n, total) * 8, cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? PL_OK : set_cuda_error(e, "chain_trace copy");
}

// Benchmark of the persistent chain kernel's weight stream: `iters` launches of a chain
// holding ONE projection of layer 0 (kind 0 o, 1 gate_up, 2 down, 3 qkv) at T tokens,
// without dependencies or finalisation.  Results are scratch.
int32_t pl_stage_chain_bench(void* handle, int32_t kind, int32_t T, int32_t iters, void* stream) {
  Stage* s = static_cast<Stage*>(handle);
  if (!s) return set_error(PL_ERR_CONFIG, "chain_bench: null handle");
  if (!s->pk_qkv || !s->pk_o || !s->pk_gu || !s->pk_down)
    return set_error(PL_ERR_CONFIG, "chain_bench: weights are not packed");
  DeviceGuard g(s->dev);
  for (int i = 0; i < iters; ++i) {
    const int rc = s->bench_chain(kind, T, static_cast<cudaStream_t>(stream));
    if (rc) return rc;
  }
  return PL_OK;
}

int32_t pl_stage_destroy(void* handle) {
  Stage* s = static_cast<Stage*>(handle);
  if (!s) return PL_OK;
  if (s->ch_trace) cudaFree(s->ch_trace);
  for (auto& r : s->probes)
    for (auto& e : r.ev) cudaEventDestroy(e);
  delete s;
  return PL_OK;
}

// Timing probe: CUDA events around each kernel group of one layer, recorded on
// the launch stream (bench.py reads kernel durations live, not under ncu).
// layer >= 0 starts a new pass (records cleared); layer < 0 stops recording.
int32_t pl_stage_probe(void* handle, int32_t layer) {
  Stage* s = static_cast<Stage*>(handle);
  if (!s) return set_error(PL_ERR_CONFIG, "stage_probe: null handle");
  s->probe_layer = layer;
  if (layer >= 0) s->probe_used = 0;  // a new pass; layer < 0 stops and keeps the records
  return PL_OK;
}

// Per recorded forward: out_meta[i*3 + {0,1,2}] = {phase, T, kind}; kind 0 (per-projection
// kernels): out_ms[i*5 + {0..4}] = {qkv gemm, rope+attention, o gemm, gate_up gemm, down gemm};
// kind 1 (persistent chain): out_ms[i*5 + {0,1}] = {decode attention, chain kernel}, rest 0.
// Requires the stream to be synchronized.
int32_t pl_stage_probe_read(void* handle, float* out_ms, int32_t* out_meta, int32_t cap, int32_t* n) {
  Stage* s = static_cast<Stage*>(handle);
  if (!s || !n) return set_error(PL_ERR_CONFIG, "stage_probe_read: null argument");
  const int cnt = static_cast<int>(std::min<size_t>(s->probe_used, static_cast<size_t>(cap)));
  for (int i = 0; i < cnt; ++i) {
    const ProbeRec& r = s->probes[i];
    const int pairs[5][2] = {{0, 1}, {1, 2}, {2, 3}, {4, 5}, {5, 6}};
    const int npairs = r.kind == 1 ? 2 : 5;
    for (int k = 0; k < 5; ++k) {
      float ms = 0.f;
      if (k < npairs) {
        cudaError_t e = cudaEventElapsedTime(&ms, r.ev[pairs[k][0]], r.ev[pairs[k][1]]);
        if (e != cudaSuccess) return set_cuda_error(e, "probe elapsed time");
      }
      out_ms[i * 5 + k] = ms;
    }
    out_meta[i * 3] = r.phase;
    out_meta[i * 3 + 1] = r.T;
    out_meta[i * 3 + 2] = r.kind;
  }
  *n = cnt;
  s->probe_used = 0;
  return PL_OK;
}

}  // extern "C"
