// Native pipeline runtime: the scheduler's hooks issue the real stage forwards
// and link transfers (C++ twin of backend.py's GpuBackend), plus the C ABI of
// the scheduler and the runtime (include/b200link.h, "scheduler" section).
//
// Per local stage: the compute stream (the executor's), a send, a recv and (in
// link-throttle mode) a deliver stream.  Cross-stream ordering uses re-recorded
// CUDA events, never host syncs:
//   compute(s, mb)  waits recv_done(s, slot), the previous occupant's
//                   send_done(s, slot) and, on the head in decode, the latest
//                   token scatter
//   send chunk      waits comp_done(s, slot) (first chunk)
//   recv chunk      waits the previous occupant's send_done(dst, slot)
// The host runs ahead of the GPU by at most RUN_AHEAD forwards per stage.
// Per-micro-batch host data (metadata, prompt ids, scatter indices) lives in a
// pinned ring; an entry is reused only after every copy that read it finished.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <unordered_map>
#include <vector>

#include "../../include/b200link.h"
#include "pl_internal.h"
#include "sched.h"

namespace pl {
namespace {

constexpr int RUN_AHEAD = 24;

inline int64_t align16(int64_t x) { return (x + 15) & ~int64_t(15); }

struct TimingPool {  // timing-enabled events of one device, handed out in order per run
  int dev = 0;
  std::vector<cudaEvent_t> ev;
  size_t used = 0;
  cudaEvent_t take() {
    if (used == ev.size()) {
      cudaEvent_t e;
      cudaSetDevice(dev);
      if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
      ev.push_back(e);
    }
    return ev[used++];
  }
  ~TimingPool() {
    for (auto e : ev) cudaEventDestroy(e);
  }
};

struct StageRt {
  bool local = false;
  void* stage = nullptr;
  int dev = 0;
  cudaStream_t comp = nullptr, send = nullptr, recv = nullptr, deliver = nullptr;
  int32_t* meta_dev = nullptr;
  int64_t* ids_dev = nullptr;
  std::vector<void*> hidden;
  std::vector<int64_t*> out_ids;
  std::vector<cudaEvent_t> ev_comp, ev_send;
  std::vector<cudaEvent_t> recv_ev;  // per slot: the incoming payload's ready event (pool event)
  std::vector<char> has_send;
  cudaEvent_t ahead[RUN_AHEAD];
  int64_t n_fwd = 0;
  cudaEvent_t t0 = nullptr, end = nullptr;
  uint64_t* t0_dev = nullptr;
};

struct RingEntry {
  uint8_t* host = nullptr;
  std::vector<cudaEvent_t> guard;  // per stage (+1: head scatter)
  std::vector<char> armed;
};

struct MbRec {
  int slot, T, R, decode, max_seqlen, max_ctx;  // decode: 0 prefill, 1 decode, 2 mixed
  int n_decode;
  int entry;
  int64_t meta_len;
};

struct BusyRec { int stage; int64_t mb; cudaEvent_t a, b; };
struct FbRec { int64_t mb; cudaEvent_t ev; };
struct ChunkRec { int link, src; int64_t pid; int idx; int64_t size; int cls; cudaEvent_t enq, a, b; };
struct MbLog { int64_t mb; int decode, R; int64_t work; };

}  // namespace

struct Pipeline : sched::Hooks {
  // configuration
  int S = 1, n_slots = 1, max_blocks = 1, block_size = 64, max_tokens = 1, max_reqs = 1, d = 0;
  int64_t num_blocks = 0;
  bool throttle = false, record_links = false, fuse = false;
  std::vector<StageRt> st;
  std::vector<void*> comm;  // per link
  int64_t* last_token = nullptr;
  int64_t* gen_tokens = nullptr;
  int64_t gen_stride = 0;
  std::vector<int64_t*> ids_recv;
  std::vector<int32_t*> scatter_dev;
  std::vector<int64_t> prompt_off, prompt_ids;
  int64_t meta_cap = 0, entry_bytes = 0, ids_off = 0, scat_off = 0;
  std::vector<RingEntry> ring;
  uint8_t* ring_host = nullptr;
  int ring_i = 0;
  std::vector<std::unique_ptr<TimingPool>> pools;  // per device ordinal

  // per-run state
  const sched::Config* cfg = nullptr;
  std::vector<sched::Request>* reqs = nullptr;
  std::vector<int> free_slots;
  std::vector<int32_t> free_blocks;
  std::vector<std::vector<int32_t>> bt;  // per request index (empty: not allocated)
  std::unordered_map<int64_t, MbRec> mbs;
  std::vector<BusyRec> busy;
  std::vector<FbRec> fb;
  std::vector<ChunkRec> chunks;
  std::vector<MbLog> mb_log;
  std::vector<int64_t> mb_req_ids;  // flat request ids of mb_log entries
  std::vector<int64_t> mb_req_off;
  cudaEvent_t first_decode = nullptr;
  cudaEvent_t last_fb = nullptr;
  int err = 0;

  // results
  double run_time_s = 0;

  int error() const override { return err; }

  TimingPool& pool(int dev) {
    if ((int)pools.size() <= dev) pools.resize(dev + 1);
    if (!pools[dev]) {
      pools[dev].reset(new TimingPool());
      pools[dev]->dev = dev;
    }
    return *pools[dev];
  }

  int fail(int code) {
    if (!err) err = code;
    return code;
  }
  bool cu(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return true;
    fail(set_cuda_error(e, what));
    return false;
  }
  bool ok(int rc) {
    if (rc == PL_OK) return true;
    fail(rc);
    return false;
  }

  int meta_len(int T, int R) const { return 3 * T + 3 * R + 1 + R * max_blocks; }

  int init(const pl_pipeline_config& c) {
    S = c.n_stages, n_slots = c.n_slots, max_blocks = c.max_blocks, block_size = c.block_size;
    max_tokens = c.max_tokens, max_reqs = c.max_reqs, d = c.d, num_blocks = c.num_blocks;
    throttle = c.throttle != 0, record_links = c.record_links != 0, fuse = c.fuse_transport != 0;
    if (S < 1 || n_slots < 1 || max_blocks < 1 || block_size < 1 || max_tokens < 1 || max_reqs < 1 || d < 1)
      return set_error(PL_ERR_CONFIG, "pipeline_create: bad sizes");
    st.resize(S);
    for (int s = 0; s < S; ++s) {
      StageRt& r = st[s];
      r.local = c.stage[s] != nullptr;
      if (!r.local) continue;
      r.stage = c.stage[s];
      r.dev = c.device[s];
      r.comp = static_cast<cudaStream_t>(c.stream[s]);
      r.meta_dev = static_cast<int32_t*>(c.meta_dev[s]);
      r.ids_dev = static_cast<int64_t*>(c.ids_dev[s]);
      if (s == 0 && !r.ids_dev) return set_error(PL_ERR_CONFIG, "pipeline_create: head needs ids_dev");
      cudaSetDevice(r.dev);
      cudaError_t e = cudaStreamCreateWithFlags(&r.send, cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&r.recv, cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&r.deliver, cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaMalloc(&r.t0_dev, sizeof(uint64_t));
      if (e != cudaSuccess) return set_cuda_error(e, "pipeline_create: streams");
      r.hidden.resize(n_slots);
      r.out_ids.resize(n_slots, nullptr);
      r.ev_comp.resize(n_slots), r.ev_send.resize(n_slots);
      r.recv_ev.assign(n_slots, nullptr);
      r.has_send.assign(n_slots, 0);
      for (int k = 0; k < n_slots; ++k) {
        r.hidden[k] = c.hidden[s * n_slots + k];
        if (s == S - 1) r.out_ids[k] = static_cast<int64_t*>(c.out_ids[s * n_slots + k]);
        if (!r.hidden[k] || (s == S - 1 && !r.out_ids[k]))
          return set_error(PL_ERR_CONFIG, "pipeline_create: stage %d slot %d buffers missing", s, k);
        for (auto* v : {&r.ev_comp, &r.ev_send}) {
          e = cudaEventCreateWithFlags(&(*v)[k], cudaEventDisableTiming);
          if (e != cudaSuccess) return set_cuda_error(e, "pipeline_create: events");
        }
      }
      for (auto& a : r.ahead) {
        e = cudaEventCreateWithFlags(&a, cudaEventDisableTiming);
        if (e != cudaSuccess) return set_cuda_error(e, "pipeline_create: events");
      }
    }
    const int nl = S >= 2 ? S : 0;
    comm.assign(nl, nullptr);
    for (int l = 0; l < nl; ++l) {
      comm[l] = c.comm ? c.comm[l] : nullptr;
      const int src = l == S - 1 ? S - 1 : l, dst = l == S - 1 ? 0 : l + 1;
      if (st[src].local != st[dst].local && !comm[l])
        return set_error(PL_ERR_CONFIG, "pipeline_create: hop %d crosses processes but has no communicator", l);
    }
    if (st[0].local) {
      ids_recv.resize(n_slots);
      scatter_dev.resize(n_slots);
      cudaSetDevice(st[0].dev);
      for (int k = 0; k < n_slots; ++k) {
        ids_recv[k] = c.ids_recv ? c.ids_recv[k] : nullptr;
        if (S > 1 && !ids_recv[k]) return set_error(PL_ERR_CONFIG, "pipeline_create: ids_recv missing");
        cudaError_t e = cudaMalloc(&scatter_dev[k], sizeof(int32_t) * 2 * max_reqs);
        if (e != cudaSuccess) return set_cuda_error(e, "pipeline_create: scatter buffers");
      }
    }
    prompt_off.assign(1, 0);
    meta_cap = meta_len(max_tokens, max_reqs);
    ids_off = align16(meta_cap * 4);
    scat_off = ids_off + align16(int64_t(max_tokens) * 8);
    entry_bytes = scat_off + align16(int64_t(max_reqs) * 8);
    ring.resize(2 * RUN_AHEAD + n_slots + 8);
    cudaError_t ea = cudaHostAlloc(&ring_host, entry_bytes * (int64_t)ring.size(), cudaHostAllocPortable);
    if (ea != cudaSuccess) return set_cuda_error(ea, "pipeline_create: pinned ring");
    for (size_t i = 0; i < ring.size(); ++i) {
      RingEntry& en = ring[i];
      en.host = ring_host + entry_bytes * (int64_t)i;
      cudaError_t e;
      en.guard.assign(S + 1, nullptr);
      en.armed.assign(S + 1, 0);
      for (int s = 0; s <= S; ++s) {
        const int owner = s < S ? s : 0;
        if (!st[owner].local) continue;
        cudaSetDevice(st[owner].dev);
        e = cudaEventCreateWithFlags(&en.guard[s], cudaEventDisableTiming);
        if (e != cudaSuccess) return set_cuda_error(e, "pipeline_create: ring events");
      }
    }
    return PL_OK;
  }

  ~Pipeline() {
    for (StageRt& r : st) {
      if (!r.local) continue;
      cudaSetDevice(r.dev);
      for (auto* v : {&r.ev_comp, &r.ev_send})
        for (auto e : *v) cudaEventDestroy(e);
      for (auto e : r.ahead) cudaEventDestroy(e);
      for (auto s : {r.send, r.recv, r.deliver})
        if (s) cudaStreamDestroy(s);
      cudaFree(r.t0_dev);
    }
    for (auto p : scatter_dev) cudaFree(p);
    for (RingEntry& en : ring)
      for (auto e : en.guard)
        if (e) cudaEventDestroy(e);
    if (ring_host) cudaFreeHost(ring_host);
  }

  int set_requests(int64_t n, const int64_t* off, const int64_t* ids, int64_t* lt, int64_t* gen, int32_t stride) {
    if (n < 0 || !off || (n > 0 && !ids)) return set_error(PL_ERR_CONFIG, "pipeline_set_requests: bad prompts");
    if (st[0].local && (!lt || !gen || stride < 1))
      return set_error(PL_ERR_CONFIG, "pipeline_set_requests: head buffers missing");
    prompt_off.assign(off, off + n + 1);
    prompt_ids.assign(ids, ids + prompt_off.back());
    last_token = lt, gen_tokens = gen, gen_stride = stride;
    return PL_OK;
  }

  // ------------------------------------------------------------ run setup
  int start(const sched::Config& c, std::vector<sched::Request>& r) {
    cfg = &c, reqs = &r;
    if ((int64_t)r.size() + 1 != (int64_t)prompt_off.size())
      return set_error(PL_ERR_CONFIG, "pipeline: trace has %lld requests, prompts for %lld",
                       (long long)r.size(), (long long)prompt_off.size() - 1);
    for (size_t i = 0; i < r.size(); ++i)
      if (prompt_off[i + 1] - prompt_off[i] != r[i].input_len)
        return set_error(PL_ERR_CONFIG, "pipeline: prompt of request %lld has wrong length", (long long)r[i].id);
    err = 0;
    free_slots.clear();
    for (int k = n_slots - 1; k >= 0; --k) free_slots.push_back(k);
    free_blocks.clear();
    for (int64_t b = num_blocks - 1; b >= 0; --b) free_blocks.push_back((int32_t)b);
    bt.assign(r.size(), {});
    mbs.clear(), busy.clear(), fb.clear(), chunks.clear(), mb_log.clear();
    mb_req_ids.clear(), mb_req_off.assign(1, 0);
    first_decode = last_fb = nullptr;
    for (auto& p : pools)
      if (p) p->used = 0;
    for (StageRt& s : st) {
      if (!s.local) continue;
      std::fill(s.has_send.begin(), s.has_send.end(), 0);
      std::fill(s.recv_ev.begin(), s.recv_ev.end(), nullptr);
      s.n_fwd = 0;
      cudaSetDevice(s.dev);
      s.t0 = pool(s.dev).take();
      if (!cu(cudaEventRecord(s.t0, s.comp), "t0")) return err;
      if (throttle) {
        if (!ok(pl_record_globaltimer(s.t0_dev, s.comp))) return err;
        cudaEvent_t e = pool(s.dev).take();
        cudaEventRecord(e, s.comp);
        cudaStreamWaitEvent(s.deliver, e, 0);
      }
    }
    return PL_OK;
  }

  RingEntry& take_entry(int& idx) {
    idx = ring_i;
    ring_i = (ring_i + 1) % (int)ring.size();
    RingEntry& en = ring[idx];
    for (size_t g = 0; g < en.guard.size(); ++g)
      if (en.armed[g]) {
        cu(cudaEventSynchronize(en.guard[g]), "ring guard");
        en.armed[g] = 0;
      }
    return en;
  }

  // ------------------------------------------------------------ hooks
  void admit(const sched::MicroBatch& mb, int64_t) override {
    if (err) return;
    if (free_slots.empty()) {
      fail(set_error(PL_ERR_PROTOCOL, "no free micro-batch slot"));
      return;
    }
    const int R = (int)mb.reqs.size();
    const bool decode = mb.phase == sched::DECODE;
    const bool mixed = mb.phase == sched::MIXED;
    // mixed batches: admit_and_batch places decoders ahead of prompts (engine.py:184-198)
    int n_dec = 0;
    if (mixed) {
      for (int ri : mb.reqs) {
        if ((*reqs)[ri].state != sched::DECODING) break;
        ++n_dec;
      }
      for (int i = n_dec; i < R; ++i)
        if ((*reqs)[mb.reqs[i]].state == sched::DECODING) {
          fail(set_error(PL_ERR_PROTOCOL, "mixed micro-batch with a decoder after a prompt"));
          return;
        }
    }
    if (R > max_reqs) {
      fail(set_error(PL_ERR_CONFIG, "micro-batch of %d requests exceeds capacity %d", R, max_reqs));
      return;
    }
    for (int ri : mb.reqs) {
      std::vector<int32_t>& row = bt[ri];
      if (!row.empty()) continue;
      const sched::Request& q = (*reqs)[ri];
      const int64_t need = (q.input_len + q.output_len + block_size - 1) / block_size;
      if ((int64_t)free_blocks.size() < need || need > max_blocks) {
        fail(set_error(PL_ERR_CONFIG, "paged KV cache exhausted"));
        return;
      }
      row.assign(max_blocks, 0);
      for (int64_t j = 0; j < need; ++j) {
        row[j] = free_blocks.back();
        free_blocks.pop_back();
      }
    }
    int64_t T = 0;
    if (decode) {
      T = R;
    } else {
      for (int i = 0; i < R; ++i) T += i < n_dec ? 1 : (*reqs)[mb.reqs[i]].input_len;
    }
    if (T > max_tokens) {
      fail(set_error(PL_ERR_CONFIG, "micro-batch of %lld tokens exceeds capacity %d", (long long)T, max_tokens));
      return;
    }
    int entry;
    RingEntry& en = take_entry(entry);
    int32_t* meta = reinterpret_cast<int32_t*>(en.host);
    int32_t* pos = meta;
    int32_t* slot = pos + T;
    int32_t* rslot = slot + T;
    int32_t* cuq = rslot + T;
    int32_t* ctx = cuq + R + 1;
    int32_t* last = ctx + R;
    int32_t* btm = last + R;
    int32_t* scat = reinterpret_cast<int32_t*>(en.host + scat_off);
    int max_seqlen = 1, max_ctx = 0;
    int64_t work = 0;
    cuq[0] = 0;
    int64_t t = 0;
    int64_t* ids = reinterpret_cast<int64_t*>(en.host + ids_off);
    for (int i = 0; i < R; ++i) {
      const int ri = mb.reqs[i];
      const sched::Request& q = (*reqs)[ri];
      const int32_t* row = bt[ri].data();
      std::memcpy(btm + (int64_t)i * max_blocks, row, sizeof(int32_t) * max_blocks);
      scat[i] = ri;
      scat[R + i] = (int32_t)q.tokens;
      if (decode || i < n_dec) {
        const int64_t p = q.input_len + q.tokens - 1;
        pos[t] = (int32_t)p;
        slot[t] = row[p / block_size] * block_size + (int32_t)(p % block_size);
        rslot[t] = ri;
        if (mixed) ids[t] = 0;  // the decode row embeds last_token[req] instead
        ++t;
        cuq[i + 1] = (int32_t)t;
        ctx[i] = (int32_t)(p + 1);
        last[i] = (int32_t)(t - 1);
        max_ctx = std::max<int>(max_ctx, (int)(p + 1));
        work += p + 1;
      } else {
        const int64_t L = q.input_len;
        std::memcpy(ids + t, prompt_ids.data() + prompt_off[ri], sizeof(int64_t) * L);
        for (int64_t p = 0; p < L; ++p, ++t) {
          pos[t] = (int32_t)p;
          slot[t] = row[p / block_size] * block_size + (int32_t)(p % block_size);
          rslot[t] = ri;
        }
        cuq[i + 1] = (int32_t)t;
        ctx[i] = (int32_t)L;
        last[i] = (int32_t)(t - 1);
        max_seqlen = std::max<int>(max_seqlen, (int)L);
        work += L;
      }
    }
    if (!decode && !mixed) max_ctx = max_seqlen;  // unused by the prefill kernel
    const int slot_k = free_slots.back();
    free_slots.pop_back();
    MbRec rec{slot_k, (int)T, R, decode ? 1 : (mixed ? 2 : 0), max_seqlen, max_ctx, n_dec, entry,
              meta_len((int)T, R)};
    mbs.emplace(mb.id, std::move(rec));
    mb_log.push_back(MbLog{mb.id, decode ? 1 : (mixed ? 2 : 0), R, work});
    for (int ri : mb.reqs) mb_req_ids.push_back((*reqs)[ri].id);
    mb_req_off.push_back((int64_t)mb_req_ids.size());
  }

  void compute(int s, const sched::MicroBatch& mb, int64_t) override {
    if (err || !st[s].local) return;
    StageRt& r = st[s];
    MbRec& rec = mbs.at(mb.id);
    const int k = rec.slot;
    cudaSetDevice(r.dev);
    cudaEvent_t ahead = r.ahead[r.n_fwd % RUN_AHEAD];
    if (r.n_fwd >= RUN_AHEAD && !cu(cudaEventSynchronize(ahead), "run-ahead")) return;  // run-ahead cap
    if (r.has_send[k]) cudaStreamWaitEvent(r.comp, r.ev_send[k], 0);
    if (s > 0 && r.recv_ev[k]) cudaStreamWaitEvent(r.comp, r.recv_ev[k], 0);
    // fused transport: a decode payload for a stage of this process is stored by this
    // forward's last residual epilogue straight into the next stage's slot buffer --
    // once that slot's previous occupant has left it
    void* peer = nullptr;
    if (fused_hop(s, rec)) {
      StageRt& rd = st[s + 1];
      if (rd.has_send[k]) cudaStreamWaitEvent(r.comp, rd.ev_send[k], 0);
      peer = rd.hidden[k];
    }
    if (s == 0 && rec.decode != 0 && last_fb) {  // decode rows read the latest token scatter
      cudaStreamWaitEvent(r.comp, last_fb, 0);
      if (!first_decode) {
        first_decode = pool(r.dev).take();
        cudaEventRecord(first_decode, r.comp);
      }
    }
    RingEntry& en = ring[rec.entry];
    if (!cu(cudaMemcpyAsync(r.meta_dev, en.host, sizeof(int32_t) * rec.meta_len, cudaMemcpyHostToDevice, r.comp),
            "meta H2D"))
      return;
    if (s == 0 && rec.decode != 1 &&
        !cu(cudaMemcpyAsync(r.ids_dev, en.host + ids_off, sizeof(int64_t) * rec.T, cudaMemcpyHostToDevice, r.comp),
            "ids H2D"))
      return;
    cudaEventRecord(en.guard[s], r.comp);
    en.armed[s] = 1;
    cudaEvent_t a = pool(r.dev).take(), b = pool(r.dev).take();
    cudaEventRecord(a, r.comp);
    pl_microbatch m{};
    m.T = rec.T, m.R = rec.R, m.phase = rec.decode, m.max_seqlen = rec.max_seqlen, m.max_ctx = rec.max_ctx;
    m.n_decode = rec.n_decode;
    m.meta = r.meta_dev;
    m.token_ids = (s == 0 && rec.decode != 1) ? r.ids_dev : nullptr;
    m.last_token = (s == 0 && rec.decode != 0) ? last_token : nullptr;
    m.hidden = r.hidden[k];
    m.out_ids = s == S - 1 ? r.out_ids[k] : nullptr;
    m.peer_hidden = peer;
    if (!ok(pl_stage_forward(r.stage, &m, r.comp))) return;
    cudaEventRecord(b, r.comp);
    cudaEventRecord(r.ev_comp[k], r.comp);
    busy.push_back(BusyRec{s, mb.id, a, b});
    cudaEventRecord(ahead, r.comp);
    r.n_fwd++;
    if (S == 1) scatter(rec, mb.id, r.out_ids[k], r.comp);
  }

  // decode payloads between two stages of this process travel inside the producer's
  // epilogue (pl_microbatch.peer_hidden) when fused transport is on
  bool fused_hop(int s, const MbRec& rec) const {
    return fuse && rec.decode == 1 && s + 1 < S && st[s].local && st[s + 1].local;
  }

  void emit(int link, const sched::Payload& p, const sched::Chunk& ch, int64_t offset, int64_t now) override {
    if (err) return;
    MbRec& rec = mbs.at(p.mb);
    const int k = rec.slot;
    const bool is_ret = link == S - 1;
    const int src = is_ret ? S - 1 : link, dst = is_ret ? 0 : link + 1;
    StageRt& rs = st[src];
    StageRt& rd = st[dst];
    const bool first = offset == 0, last = ch.last;
    const int64_t size = ch.size;
    uint8_t *sbuf = nullptr, *dbuf = nullptr;
    if (rs.local) {
      cudaSetDevice(rs.dev);
      if (first) cudaStreamWaitEvent(rs.send, rs.ev_comp[k], 0);
      sbuf = static_cast<uint8_t*>(is_ret ? (void*)rs.out_ids[k] : rs.hidden[k]) + offset;
    }
    if (rd.local) dbuf = static_cast<uint8_t*>(is_ret ? (void*)ids_recv[k] : rd.hidden[k]) + offset;
    const int64_t deliver = now + sched::transmission_ns(cfg->links[link], size) +
                            sched::s_to_ns(cfg->links[link].latency_s);
    cudaEvent_t t_emit = nullptr;
    if (rs.local && record_links) {
      t_emit = pool(rs.dev).take();
    }
    if (!is_ret && fused_hop(src, rec)) {
      // the bytes already landed in dst's slot at the end of the producing forward: the
      // chunk is that forward's completion (a zero-length realized chunk); the payload
      // is delivered once, with its last chunk
      if (t_emit) {
        cudaEventRecord(t_emit, rs.send);
        note_chunk(link, src, k, p, ch, t_emit, rs.send);
      }
      if (last) {
        cudaEventRecord(rs.ev_send[k], rs.send);
        rs.has_send[k] = 1;
        cudaEvent_t e = pool(rs.dev).take();
        cudaEventRecord(e, rs.send);
        recv_done(dst, rec, p.mb, e, is_ret, deliver);
      }
      return;
    }
    if (rs.local && rd.local) {
      if (first && rd.has_send[k]) cudaStreamWaitEvent(rs.send, rd.ev_send[k], 0);
      if (t_emit) cudaEventRecord(t_emit, rs.send);
      if (!cu(cudaMemcpyAsync(dbuf, sbuf, size, cudaMemcpyDefault, rs.send), "link copy")) return;
      if (t_emit) note_chunk(link, src, k, p, ch, t_emit, rs.send);
      if (last) {
        cudaEventRecord(rs.ev_send[k], rs.send);
        rs.has_send[k] = 1;
        cudaEvent_t e = pool(rs.dev).take();
        cudaEventRecord(e, rs.send);
        recv_done(dst, rec, p.mb, e, is_ret, deliver);
      }
      return;
    }
    if (rs.local) {
      if (t_emit) cudaEventRecord(t_emit, rs.send);
      if (!ok(pl_p2p_send(comm[link], sbuf, size, 1, rs.send))) return;
      if (t_emit) note_chunk(link, src, k, p, ch, t_emit, rs.send);
      if (last) {
        cudaEventRecord(rs.ev_send[k], rs.send);
        rs.has_send[k] = 1;
      }
    }
    if (rd.local) {
      cudaSetDevice(rd.dev);
      if (first && rd.has_send[k]) cudaStreamWaitEvent(rd.recv, rd.ev_send[k], 0);
      if (!ok(pl_p2p_recv(comm[link], dbuf, size, 0, rd.recv))) return;
      if (last) {
        cudaEvent_t e = pool(rd.dev).take();
        cudaEventRecord(e, rd.recv);
        recv_done(dst, rec, p.mb, e, is_ret, deliver);
      }
    }
  }

  void note_chunk(int link, int src, int k, const sched::Payload& p, const sched::Chunk& ch, cudaEvent_t t_emit,
                  cudaStream_t sst) {
    StageRt& r = st[src];
    cudaEvent_t t_sent = pool(r.dev).take();
    cudaEventRecord(t_sent, sst);
    // enqueue = the producing forward's end (its busy record's end event)
    cudaEvent_t enq = nullptr;
    for (auto it = busy.rbegin(); it != busy.rend(); ++it)
      if (it->stage == src && it->mb == p.mb) {
        enq = it->b;
        break;
      }
    chunks.push_back(ChunkRec{link, src, p.id, ch.index, ch.size, ch.cls, enq, t_emit, t_sent});
    (void)k;
  }

  void recv_done(int dst, MbRec& rec, int64_t mb_id, cudaEvent_t ev, bool is_ret, int64_t deliver_ns) {
    StageRt& r = st[dst];
    cudaSetDevice(r.dev);
    if (throttle) {
      // the payload becomes usable only once the emulated link would have delivered it;
      // gated on a separate stream so the link's own chunk pipeline is not held back
      cudaStreamWaitEvent(r.deliver, ev, 0);
      if (!ok(pl_gate_until_ns(r.t0_dev, (uint64_t)deliver_ns, r.deliver))) return;
      ev = pool(r.dev).take();
      cudaEventRecord(ev, r.deliver);
    }
    if (!is_ret) {
      r.recv_ev[rec.slot] = ev;
      return;
    }
    cudaStreamWaitEvent(r.recv, ev, 0);
    scatter(rec, mb_id, ids_recv[rec.slot], r.recv);
  }

  void scatter(MbRec& rec, int64_t mb_id, int64_t* ids, cudaStream_t stream) {
    StageRt& h = st[0];
    RingEntry& en = ring[rec.entry];
    const int R = rec.R;
    int32_t* dev = scatter_dev[rec.slot];
    if (!cu(cudaMemcpyAsync(dev, en.host + scat_off, sizeof(int32_t) * 2 * R, cudaMemcpyHostToDevice, stream),
            "scatter H2D"))
      return;
    cudaEventRecord(en.guard[S], stream);
    en.armed[S] = 1;
    if (!ok(pl_token_scatter(ids, dev, dev + R, R, last_token, gen_tokens, gen_stride, stream))) return;
    cudaEvent_t e = pool(h.dev).take();
    cudaEventRecord(e, stream);
    fb.push_back(FbRec{mb_id, e});
    last_fb = e;
  }

  void feedback(const sched::MicroBatch& mb, int64_t) override {
    if (err) return;
    auto it = mbs.find(mb.id);
    free_slots.push_back(it->second.slot);
    mbs.erase(it);
    for (int ri : mb.reqs) {
      const sched::Request& q = (*reqs)[ri];
      if (q.state != sched::FINISHED || bt[ri].empty()) continue;
      const int64_t need = (q.input_len + q.output_len + block_size - 1) / block_size;
      for (int64_t j = need - 1; j >= 0; --j) free_blocks.push_back(bt[ri][j]);
      bt[ri].clear();
    }
  }

  // ------------------------------------------------------------ finish
  int finish() {
    run_time_s = 0;
    for (StageRt& r : st) {
      if (!r.local) continue;
      cudaSetDevice(r.dev);
      for (cudaStream_t x : {r.send, r.recv, r.deliver}) {
        cudaEvent_t e = pool(r.dev).take();
        cudaEventRecord(e, x);
        cudaStreamWaitEvent(r.comp, e, 0);
      }
      r.end = pool(r.dev).take();
      cudaEventRecord(r.end, r.comp);
    }
    for (StageRt& r : st) {
      if (!r.local) continue;
      if (!cu(cudaEventSynchronize(r.end), "finish")) return err;
      float ms = 0;
      cudaEventElapsedTime(&ms, r.t0, r.end);
      run_time_s = std::max(run_time_s, ms / 1e3);
    }
    for (RingEntry& en : ring) std::fill(en.armed.begin(), en.armed.end(), 0);
    return cudaGetLastError() == cudaSuccess ? PL_OK : set_error(PL_ERR_CUDA, "pipeline finish");
  }

  double since_t0(int stage, cudaEvent_t e) const {
    float ms = 0;
    if (!e || cudaEventElapsedTime(&ms, st[stage].t0, e) != cudaSuccess) return NAN;
    return ms / 1e3;
  }
};

}  // namespace pl

using namespace pl;

// ------------------------------------------------------------------ scheduler
namespace {

struct SchedHandle {
  sched::Config cfg;
  std::vector<sched::Request> reqs;
  sched::Logs logs;
};

}  // namespace

extern "C" {

int32_t pl_sched_create(const pl_sched_config* c, void** handle) {
  if (!c || !handle) return set_error(PL_ERR_CONFIG, "sched_create: null argument");
  if (c->n_stages < 1 || c->n_stages > 4096) return set_error(PL_ERR_CONFIG, "sched_create: bad stage count");
  const int S = c->n_stages;
  const int nl = S >= 2 ? S : 0;
  if (c->n_links != nl) return set_error(PL_ERR_CONFIG, "sched_create: expected %d links, got %d", nl, c->n_links);
  if (c->max_batched_tokens < 1 || c->max_batch_size < 1 || c->n_max < 1 || c->decision_stride < 1)
    return set_error(PL_ERR_CONFIG, "sched_create: bad controller config");
  std::unique_ptr<SchedHandle> h(new SchedHandle());
  sched::Config& g = h->cfg;
  g.S = S;
  g.max_batched_tokens = c->max_batched_tokens, g.max_batch_size = c->max_batch_size, g.n_max = c->n_max;
  g.bubble_epsilon = c->bubble_epsilon, g.gain_delta = c->gain_delta;
  g.fixed_compute = c->fixed_compute, g.decision_stride = c->decision_stride;
  g.chunk_size = c->chunk_size, g.fcfs = c->fcfs, g.allow_mixed = c->allow_mixed;
  g.bytes_per_token = c->bytes_per_token, g.feedback_bytes = c->feedback_bytes;
  g.profiles.resize(S);
  for (int s = 0; s < S; ++s)
    for (int ph = 0; ph < 2; ++ph) {
      const int64_t a = c->prof_off[2 * s + ph], b = c->prof_off[2 * s + ph + 1];
      if (b - a < 2) return set_error(PL_ERR_CONFIG, "sched_create: stage %d phase %d needs >= 2 points", s, ph);
      g.profiles[s].xs[ph].assign(c->prof_x + a, c->prof_x + b);
      g.profiles[s].ys[ph].assign(c->prof_y + a, c->prof_y + b);
      for (int64_t i = a + 1; i < b; ++i)
        if (c->prof_x[i] <= c->prof_x[i - 1])
          return set_error(PL_ERR_CONFIG, "sched_create: stage %d profile points not increasing", s);
    }
  for (int l = 0; l < nl; ++l) {
    if (!(c->link_bandwidth[l] > 0) || c->link_latency_s[l] < 0)
      return set_error(PL_ERR_CONFIG, "sched_create: bad link %d", l);
    g.links.push_back(sched::Link{c->link_latency_s[l], c->link_bandwidth[l]});
  }
  *handle = h.release();
  return PL_OK;
}

int32_t pl_sched_destroy(void* handle) {
  delete static_cast<SchedHandle*>(handle);
  return PL_OK;
}

int32_t pl_sched_choose_n(void* handle, int64_t queued_tokens, int32_t phase, int32_t* n, int64_t* budget,
                          double* bubble) {
  if (!handle || !n || !budget || !bubble || (phase != 0 && phase != 1))
    return set_error(PL_ERR_CONFIG, "sched_choose_n: bad argument");
  const sched::Decision d = sched::choose_n(static_cast<SchedHandle*>(handle)->cfg, queued_tokens, phase);
  *n = d.n, *budget = d.budget, *bubble = d.bubble;
  return PL_OK;
}

int32_t pl_sched_run(void* handle, const pl_sched_request* reqs, int64_t n_reqs, int64_t horizon_ns,
                     void* pipeline) {
  if (!handle || (n_reqs > 0 && !reqs)) return set_error(PL_ERR_CONFIG, "sched_run: null argument");
  SchedHandle* h = static_cast<SchedHandle*>(handle);
  h->reqs.clear();
  for (int64_t i = 0; i < n_reqs; ++i) {
    sched::Request r;
    r.id = reqs[i].id, r.arrival_ns = reqs[i].arrival_ns;
    r.input_len = reqs[i].input_len, r.output_len = reqs[i].output_len;
    if (r.input_len < 1 || r.output_len < 1) return set_error(PL_ERR_CONFIG, "sched_run: request lengths must be >= 1");
    h->reqs.push_back(r);
  }
  sched::Hooks null_hooks;
  Pipeline* p = static_cast<Pipeline*>(pipeline);
  int cur = 0;
  if (p) cudaGetDevice(&cur);  // a virtual run never touches CUDA
  int rc = p ? p->start(h->cfg, h->reqs) : PL_OK;
  if (rc == PL_OK) {
    rc = sched::run(h->cfg, h->reqs, horizon_ns, p ? static_cast<sched::Hooks&>(*p) : null_hooks, h->logs);
    if (rc == 1)
      rc = set_error(PL_ERR_CONFIG, "duplicate request id in trace");
    else if (rc == 2)
      rc = set_error(PL_ERR_PROTOCOL, "payload enqueued twice on one link");
    else if (rc == 3)
      rc = p ? p->err : PL_ERR_CUDA;
    else if (p)
      rc = p->finish();
  }
  if (p) cudaSetDevice(cur);
  return rc;
}

int32_t pl_sched_counts(void* handle, int64_t* counts) {
  if (!handle || !counts) return set_error(PL_ERR_CONFIG, "sched_counts: null argument");
  const sched::Logs& L = static_cast<SchedHandle*>(handle)->logs;
  int64_t nb = 0;
  for (const auto& v : L.busy) nb += (int64_t)v.size();
  counts[0] = (int64_t)L.events.size();
  counts[1] = (int64_t)L.links.size();
  counts[2] = (int64_t)L.decisions.size();
  counts[3] = (int64_t)L.emissions.size();
  counts[4] = (int64_t)L.first_compute.size();
  counts[5] = nb;
  counts[6] = L.end_ns;
  counts[7] = L.all_finished ? 1 : 0;
  return PL_OK;
}

int32_t pl_sched_read(void* handle, int64_t* events, int64_t* links, int64_t* decisions, double* bubbles,
                      int64_t* emissions, int64_t* first_compute, int64_t* busy, int64_t* req_state,
                      double* req_times) {
  if (!handle) return set_error(PL_ERR_CONFIG, "sched_read: null argument");
  const SchedHandle* h = static_cast<SchedHandle*>(handle);
  const sched::Logs& L = h->logs;
  if (events)
    for (size_t i = 0; i < L.events.size(); ++i) {
      const auto& e = L.events[i];
      int64_t* o = events + 4 * i;
      o[0] = e.t, o[1] = e.kind, o[2] = e.subject, o[3] = e.stage;
    }
  if (links)
    for (size_t i = 0; i < L.links.size(); ++i) {
      const auto& e = L.links[i];
      int64_t* o = links + 7 * i;
      o[0] = e.t, o[1] = e.link, o[2] = e.payload, o[3] = e.index, o[4] = e.size, o[5] = e.cls, o[6] = e.ev;
    }
  if (decisions)
    for (size_t i = 0; i < L.decisions.size(); ++i) {
      int64_t* o = decisions + 3 * i;
      o[0] = L.decisions[i].first, o[1] = L.decisions[i].second.n, o[2] = L.decisions[i].second.budget;
      if (bubbles) bubbles[i] = L.decisions[i].second.bubble;
    }
  if (emissions)
    for (size_t i = 0; i < L.emissions.size(); ++i) {
      emissions[2 * i] = L.emissions[i].first;
      emissions[2 * i + 1] = L.emissions[i].second;
    }
  if (first_compute)
    for (size_t i = 0; i < L.first_compute.size(); ++i) {
      first_compute[2 * i] = L.first_compute[i].first;
      first_compute[2 * i + 1] = L.first_compute[i].second;
    }
  if (busy) {
    int64_t j = 0;
    for (size_t s = 0; s < L.busy.size(); ++s)
      for (const auto& iv : L.busy[s]) {
        busy[3 * j] = (int64_t)s, busy[3 * j + 1] = iv.first, busy[3 * j + 2] = iv.second;
        ++j;
      }
  }
  for (size_t i = 0; i < h->reqs.size(); ++i) {
    const sched::Request& r = h->reqs[i];
    if (req_state) req_state[2 * i] = r.state, req_state[2 * i + 1] = r.tokens;
    if (req_times) {
      req_times[2 * i] = r.has_first ? r.first_token_time : NAN;
      req_times[2 * i + 1] = r.has_finish ? r.finish_time : NAN;
    }
  }
  return PL_OK;
}

// ------------------------------------------------------------------ runtime

int32_t pl_pipeline_create(const pl_pipeline_config* c, void** handle) {
  if (!c || !handle || !c->stage || !c->stream || !c->device || !c->meta_dev || !c->ids_dev || !c->hidden ||
      !c->out_ids)
    return set_error(PL_ERR_CONFIG, "pipeline_create: null argument");
  int cur = 0;
  cudaGetDevice(&cur);
  std::unique_ptr<Pipeline> p(new Pipeline());
  const int rc = p->init(*c);
  cudaSetDevice(cur);
  if (rc) return rc;
  *handle = p.release();
  return PL_OK;
}

int32_t pl_pipeline_destroy(void* handle) {
  delete static_cast<Pipeline*>(handle);
  return PL_OK;
}

int32_t pl_pipeline_set_requests(void* handle, int64_t n_requests, const int64_t* prompt_off,
                                 const int64_t* prompt_ids, int64_t* last_token, int64_t* gen_tokens,
                                 int32_t gen_stride) {
  if (!handle) return set_error(PL_ERR_CONFIG, "pipeline_set_requests: null handle");
  return static_cast<Pipeline*>(handle)->set_requests(n_requests, prompt_off, prompt_ids, last_token, gen_tokens,
                                                      gen_stride);
}

int32_t pl_pipeline_counts(void* handle, int64_t* counts) {
  if (!handle || !counts) return set_error(PL_ERR_CONFIG, "pipeline_counts: null argument");
  const Pipeline* p = static_cast<Pipeline*>(handle);
  counts[0] = (int64_t)p->busy.size();
  counts[1] = (int64_t)p->fb.size();
  counts[2] = (int64_t)p->chunks.size();
  counts[3] = (int64_t)p->mb_log.size();
  counts[4] = (int64_t)p->mb_req_ids.size();
  return PL_OK;
}

int32_t pl_pipeline_read(void* handle, double* run_time_s, double* decode_start_s, int64_t* busy,
                         double* busy_s, int64_t* fb_mb, double* fb_s, int64_t* chunks, double* chunk_s,
                         int64_t* mb_log, int64_t* mb_req_off, int64_t* mb_req_ids) {
  if (!handle) return set_error(PL_ERR_CONFIG, "pipeline_read: null argument");
  const Pipeline* p = static_cast<Pipeline*>(handle);
  if (run_time_s) *run_time_s = p->run_time_s;
  if (decode_start_s) *decode_start_s = p->first_decode ? p->since_t0(0, p->first_decode) : NAN;
  for (size_t i = 0; i < p->busy.size(); ++i) {
    const BusyRec& b = p->busy[i];
    if (busy) busy[2 * i] = b.stage, busy[2 * i + 1] = b.mb;
    if (busy_s) busy_s[2 * i] = p->since_t0(b.stage, b.a), busy_s[2 * i + 1] = p->since_t0(b.stage, b.b);
  }
  for (size_t i = 0; i < p->fb.size(); ++i) {
    if (fb_mb) fb_mb[i] = p->fb[i].mb;
    if (fb_s) fb_s[i] = p->since_t0(0, p->fb[i].ev);
  }
  for (size_t i = 0; i < p->chunks.size(); ++i) {
    const ChunkRec& c = p->chunks[i];
    if (chunks) {
      int64_t* o = chunks + 6 * i;
      o[0] = c.link, o[1] = c.src, o[2] = c.pid, o[3] = c.idx, o[4] = c.size, o[5] = c.cls;
    }
    if (chunk_s) {
      chunk_s[3 * i] = p->since_t0(c.src, c.enq);
      chunk_s[3 * i + 1] = p->since_t0(c.src, c.a);
      chunk_s[3 * i + 2] = p->since_t0(c.src, c.b);
    }
  }
  for (size_t i = 0; i < p->mb_log.size(); ++i) {
    const MbLog& m = p->mb_log[i];
    if (mb_log) {
      int64_t* o = mb_log + 4 * i;
      o[0] = m.mb, o[1] = m.decode, o[2] = m.R, o[3] = m.work;
    }
  }
  if (mb_req_off)
    for (size_t i = 0; i < p->mb_req_off.size(); ++i) mb_req_off[i] = p->mb_req_off[i];
  if (mb_req_ids)
    for (size_t i = 0; i < p->mb_req_ids.size(); ++i) mb_req_ids[i] = p->mb_req_ids[i];
  return PL_OK;
}

}  // extern "C"
