// Native virtual-clock scheduler (see sched.h for the reference map).
//
// Float arithmetic is written to round exactly like the reference's Python:
// int operands are converted to double first (exact below 2^53), products of
// ints stay integer where Python's do (transmission_ns), round() is
// round-half-even (nearbyint under the default rounding mode), and the host
// compiler runs with -ffp-contract=off so no FMA changes a result.
#include <math.h>

#include <algorithm>
#include <map>
#include <queue>
#include <unordered_map>
#include <unordered_set>

#include "sched.h"

namespace pl {
namespace sched {

static const int64_t NS_PER_S = 1000000000LL;

int64_t s_to_ns(double seconds) {  // transport.py:32-33
  return (int64_t)nearbyint(seconds * (double)NS_PER_S);
}

int64_t transmission_ns(const Link& l, int64_t bytes) {  // transport.py:199-200
  return (int64_t)nearbyint((double)(bytes * NS_PER_S) / l.bandwidth);
}

double compute_time(const Profile& p, int phase, int64_t tokens) {  // profiles.py:95-121
  const std::vector<int64_t>& xs = p.xs[phase];
  const std::vector<double>& ys = p.ys[phase];
  const size_t n = xs.size();
  size_t i = (size_t)(std::lower_bound(xs.begin(), xs.end(), tokens) - xs.begin());
  if (i < n && xs[i] == tokens) return ys[i];
  size_t a, b;
  if (i == 0) {
    a = 0, b = 1;
  } else if (i == n) {
    a = n - 2, b = n - 1;
  } else {
    a = i - 1, b = i;
  }
  const double slope = (ys[b] - ys[a]) / (double)(xs[b] - xs[a]);
  const double v = ys[a] + slope * (double)(tokens - xs[a]);
  return v > 1e-12 ? v : 1e-12;
}

static int64_t compute_ns(const Profile& p, int phase, int64_t tokens) {
  const int64_t ns = s_to_ns(compute_time(p, phase, tokens));
  return ns > 1 ? ns : 1;
}

// controller.py:68-112
static void round_terms(const Config& c, int64_t n, int64_t tokens, int phase, int64_t& bottleneck,
                        int64_t& round_ns) {
  int64_t sum = 0, bn = 0;
  for (int s = 0; s < c.S; ++s) {
    const int64_t v = compute_ns(c.profiles[s], phase, tokens);
    sum += v;
    bn = std::max(bn, v);
  }
  int64_t transfers = 0;
  if (c.S >= 2) {
    const int64_t act = tokens * c.bytes_per_token;
    for (int l = 0; l < c.S - 1; ++l) {
      transfers += transmission_ns(c.links[l], act);
      transfers += s_to_ns(c.links[l].latency_s);
    }
    transfers += transmission_ns(c.links[c.S - 1], tokens * c.feedback_bytes);
    transfers += s_to_ns(c.links[c.S - 1].latency_s);
  }
  bottleneck = bn;
  round_ns = std::max(sum + transfers, n * bn);
}

// controller.py:132-186
Decision choose_n(const Config& c, int64_t queued_tokens, int phase) {
  const int64_t pool = std::max<int64_t>(1, std::min(queued_tokens, c.max_batched_tokens));
  auto tokens_for = [&](int64_t n) -> int64_t {
    if (c.fixed_compute) return pool;
    return std::max<int64_t>(1, (int64_t)ceil((double)pool / (double)n));
  };
  auto evaluate = [&](int64_t n, double& bubble, double& util, int64_t& tokens) {
    tokens = tokens_for(n);
    int64_t bn, rnd;
    round_terms(c, n, tokens, phase, bn, rnd);
    util = (double)(n * bn) / (double)rnd;
    bubble = std::min(1.0, std::max(0.0, 1.0 - util));
  };
  int64_t n = 1;
  double bubble, util;
  int64_t tokens;
  evaluate(n, bubble, util, tokens);
  while (true) {
    if (bubble <= c.bubble_epsilon || n >= c.n_max) break;
    double nb, nu;
    int64_t nt;
    evaluate(n + 1, nb, nu, nt);
    if (util > 0 && (nu / util) - 1.0 < c.gain_delta) break;
    n += 1, bubble = nb, util = nu, tokens = nt;
  }
  return Decision{(int)n, tokens, bubble};
}

namespace {

// transport.py:70-160
struct LinkQueue {
  int64_t chunk;  // < 0: unchunked
  bool fcfs;
  std::deque<Payload> dec, pre, all;
  std::unordered_set<int64_t> seen;
  int64_t head_off = 0;
  int head_idx = 0;

  bool enqueue(const Payload& p) {
    if (!seen.insert(p.id).second) return false;
    if (fcfs)
      all.push_back(p);
    else if (p.cls == CLS_DECODE)
      dec.push_back(p);
    else
      pre.push_back(p);
    return true;
  }
  static Chunk whole(std::deque<Payload>& q) {
    Payload p = q.front();
    q.pop_front();
    return Chunk{p.id, 0, p.size, true, p.cls};
  }
  Chunk slice(std::deque<Payload>& q) {
    const Payload& p = q.front();
    const int64_t rem = p.size - head_off;
    const int64_t size = std::min(chunk, rem);
    Chunk c{p.id, head_idx, size, size == rem, p.cls};
    if (c.last) {
      q.pop_front();
      head_off = 0, head_idx = 0;
    } else {
      head_off += size, head_idx += 1;
    }
    return c;
  }
  bool next(Chunk& c) {
    if (fcfs) {
      if (all.empty()) return false;
      c = (all.front().cls == CLS_DECODE || chunk < 0) ? whole(all) : slice(all);
      return true;
    }
    if (!dec.empty()) {
      c = whole(dec);
      return true;
    }
    if (!pre.empty()) {
      c = chunk < 0 ? whole(pre) : slice(pre);
      return true;
    }
    return false;
  }
};

struct Ev {
  int64_t t;
  int kind;
  int64_t subject;
  int64_t seq;
  int a;      // stage (DONE) or link (SENT/DELIVERED)
  Chunk ch;   // SENT/DELIVERED
};
struct EvLater {
  bool operator()(const Ev& x, const Ev& y) const {
    if (x.t != y.t) return x.t > y.t;
    if (x.kind != y.kind) return x.kind > y.kind;
    if (x.subject != y.subject) return x.subject > y.subject;
    return x.seq > y.seq;
  }
};

struct StageRt {
  bool busy = false;
  int64_t cur = -1;  // micro-batch id
  int64_t started = 0;
  std::deque<int64_t> waiting;
};

struct LinkRt {
  LinkQueue q;
  int dst;
  bool ret;
  bool busy = false;
  std::unordered_map<int64_t, Payload> payloads;
  std::unordered_map<int64_t, int64_t> sent;
};

struct Bin {
  int64_t tokens = 0;
  std::vector<int> members;
  int phase = -1;
};

class Engine {
 public:
  Engine(const Config& c, std::vector<Request>& reqs, Hooks& h, Logs& logs)
      : c_(c), reqs_(reqs), hooks_(h), logs_(logs) {}

  int run(int64_t horizon) {
    logs_ = Logs();
    logs_.busy.assign(c_.S, {});
    stages_.assign(c_.S, StageRt());
    links_.clear();
    const int nl = c_.S >= 2 ? c_.S : 0;
    for (int i = 0; i < nl; ++i) {
      LinkRt l{LinkQueue{c_.chunk_size, c_.fcfs != 0}, i == nl - 1 ? 0 : i + 1, i == nl - 1};
      links_.push_back(std::move(l));
    }
    std::unordered_map<int64_t, int> by_id;
    for (size_t i = 0; i < reqs_.size(); ++i) {
      Request& r = reqs_[i];
      if (!by_id.emplace(r.id, (int)i).second) return 1;  // duplicate id: ConfigError
      r.state = QUEUED, r.tokens = 0, r.has_first = r.has_finish = false;
      post(r.arrival_ns, ARRIVAL, r.id, 0, Chunk());
    }
    id_index_ = std::move(by_id);
    int64_t last = 0;
    while (!heap_.empty()) {
      if (hooks_.error()) return 3;
      if (horizon >= 0 && heap_.top().t > horizon) {
        last = horizon;
        break;
      }
      const Ev e = heap_.top();
      heap_.pop();
      if (e.t > last) last = e.t;
      switch (e.kind) {
        case DELIVERED: delivered(e.a, e.ch, e.t); break;
        case DONE: compute_finished(e.a, e.subject, e.t); break;
        case ARRIVAL:
          pending_.push_back(id_index_[e.subject]);
          note(e.t, ARRIVAL, e.subject, -1);
          want_boundary(e.t);
          break;
        case BOUNDARY: boundary(e.t); break;
        default: chunk_sent(e.a, e.ch, e.t); break;
      }
      if (err_) return err_;
    }
    if (hooks_.error()) return 3;
    for (int s = 0; s < c_.S; ++s)
      if (stages_[s].busy) {
        logs_.busy[s].push_back({stages_[s].started, last});
        stages_[s].busy = false;
      }
    std::stable_sort(logs_.links.begin(), logs_.links.end(),
                     [](const LinkRec& a, const LinkRec& b) { return a.t < b.t; });
    logs_.end_ns = last;
    bool all = true;
    for (const Request& r : reqs_) all = all && r.state == FINISHED;
    logs_.all_finished = all;
    return 0;
  }

 private:
  const Config& c_;
  std::vector<Request>& reqs_;
  Hooks& hooks_;
  Logs& logs_;
  std::priority_queue<Ev, std::vector<Ev>, EvLater> heap_;
  int64_t seq_ = 0;
  std::vector<StageRt> stages_;
  std::vector<LinkRt> links_;
  std::unordered_map<int64_t, int> id_index_;
  std::deque<int> pending_, ready_;
  std::map<int64_t, MicroBatch> inflight_;  // by id; also owns the micro-batches
  std::unordered_set<int64_t> boundaries_;
  std::unordered_set<int64_t> first_seen_;
  std::map<std::pair<int64_t, int>, Decision> decisions_;
  std::unordered_map<int64_t, int64_t> cns_[2];
  int64_t iteration_ = 0, next_mb_ = 0, next_payload_ = 0;
  bool have_last_ = false;
  Decision last_{};
  int err_ = 0;

  void post(int64_t t, int kind, int64_t subject, int a, const Chunk& ch) {
    heap_.push(Ev{t, kind, subject, seq_++, a, ch});
  }
  void note(int64_t t, int kind, int64_t subject, int stage) {
    logs_.events.push_back(EventRec{t, kind, subject, stage});
  }
  void note_link(int link, int64_t t, int64_t pid, int idx, int64_t size, int cls, int ev) {
    logs_.links.push_back(LinkRec{t, link, pid, idx, size, cls, ev});
  }
  MicroBatch& mb(int64_t id) { return inflight_.at(id); }

  int64_t cns(int s, int phase, int64_t tokens) {
    auto& m = cns_[phase];
    const int64_t key = tokens * static_cast<int64_t>(c_.profiles.size()) + s;  // unique for any S
    auto it = m.find(key);
    if (it != m.end()) return it->second;
    const int64_t v = compute_ns(c_.profiles[s], phase, tokens);
    m.emplace(key, v);
    return v;
  }

  void launch_compute(int s, int64_t now) {
    StageRt& st = stages_[s];
    if (st.busy || st.waiting.empty()) return;
    const int64_t id = st.waiting.front();
    st.waiting.pop_front();
    st.busy = true, st.cur = id, st.started = now;
    const MicroBatch& m = mb(id);
    const int phase = m.phase == DECODE ? 1 : 0;
    const int64_t dur = cns(s, phase, m.tokens);
    if (s == 0)
      for (int ri : m.reqs)
        if (first_seen_.insert(reqs_[ri].id).second) logs_.first_compute.push_back({reqs_[ri].id, now});
    post(now + dur, DONE, id, s, Chunk());
    hooks_.compute(s, m, now);
  }

  void compute_finished(int s, int64_t id, int64_t now) {
    StageRt& st = stages_[s];
    logs_.busy[s].push_back({st.started, now});
    st.busy = false, st.cur = -1;
    note(now, DONE, id, s);
    const MicroBatch& m = mb(id);
    if (s < c_.S - 1) {
      const int cls = m.phase == DECODE ? CLS_DECODE : CLS_PREFILL;
      enqueue(s, m, std::max<int64_t>(1, m.tokens * c_.bytes_per_token), cls, now);
    } else if (!links_.empty()) {
      enqueue(c_.S - 1, m, std::max<int64_t>(1, c_.feedback_bytes * (int64_t)m.reqs.size()), CLS_DECODE, now);
    } else {
      emit_tokens(id, now);
      want_boundary(now);
    }
    launch_compute(s, now);
    if (s == 0) want_boundary(now);
  }

  void enqueue(int li, const MicroBatch& m, int64_t size, int cls, int64_t now) {
    LinkRt& ln = links_[li];
    Payload p{next_payload_++, cls, size, m.id};
    ln.payloads.emplace(p.id, p);
    ln.sent.emplace(p.id, 0);
    if (!ln.q.enqueue(p)) {
      err_ = 2;
      return;
    }
    note_link(li, now, p.id, -1, size, cls, L_ENQUEUE);
    if (!ln.busy) pump(li, now);
  }

  void pump(int li, int64_t now) {
    LinkRt& ln = links_[li];
    Chunk ch;
    if (!ln.q.next(ch)) {
      ln.busy = false;
      return;
    }
    ln.busy = true;
    note_link(li, now, ch.payload, ch.index, ch.size, ch.cls, L_EMIT);
    post(now + transmission_ns(c_.links[li], ch.size), SENT, ch.payload, li, ch);
    int64_t& off = ln.sent[ch.payload];
    const int64_t o = off;
    off += ch.size;
    hooks_.emit(li, ln.payloads.at(ch.payload), ch, o, now);
  }

  void chunk_sent(int li, const Chunk& ch, int64_t now) {
    note_link(li, now, ch.payload, ch.index, ch.size, ch.cls, L_SENT);
    note(now, SENT, ch.payload, -1);
    post(now + s_to_ns(c_.links[li].latency_s), DELIVERED, ch.payload, li, ch);
    pump(li, now);
  }

  void delivered(int li, const Chunk& ch, int64_t now) {
    LinkRt& ln = links_[li];
    note_link(li, now, ch.payload, ch.index, ch.size, ch.cls, L_DELIVER);
    if (!ch.last) return;
    auto pit = ln.payloads.find(ch.payload);
    const Payload p = pit->second;
    ln.payloads.erase(pit);
    ln.sent.erase(ch.payload);
    note(now, DELIVERED, ch.payload, ln.dst);
    hooks_.delivered(li, p, mb(p.mb), now);
    if (ln.ret) {
      emit_tokens(p.mb, now);
      want_boundary(now);
    } else {
      stages_[ln.dst].waiting.push_back(p.mb);
      launch_compute(ln.dst, now);
    }
  }

  // engine.py:422-442
  void emit_tokens(int64_t id, int64_t now) {
    auto it = inflight_.find(id);
    MicroBatch m = std::move(it->second);
    inflight_.erase(it);
    const double t_s = (double)now / (double)NS_PER_S;
    for (int ri : m.reqs) {
      Request& r = reqs_[ri];
      r.tokens += 1;
      logs_.emissions.push_back({now, r.id});
      if (r.state == RUNNING_PREFILL) {
        r.first_token_time = t_s, r.has_first = true;
        if (r.output_len == 1) {
          r.state = FINISHED, r.finish_time = t_s, r.has_finish = true;
        } else {
          r.state = DECODING;
          ready_.push_back(ri);
        }
      } else if (r.state == DECODING) {
        if (r.tokens >= r.output_len) {
          r.state = FINISHED, r.finish_time = t_s, r.has_finish = true;
        } else {
          ready_.push_back(ri);
        }
      }
    }
    hooks_.feedback(m, now);
  }

  void want_boundary(int64_t now) {
    if (boundaries_.insert(now).second) post(now, BOUNDARY, iteration_ + 1, 0, Chunk());
  }

  Decision decide(int phase) {
    int64_t demand = (int64_t)ready_.size();
    for (const auto& kv : inflight_) demand += kv.second.tokens;
    for (int ri : pending_) demand += reqs_[ri].input_len;
    const auto key = std::make_pair(demand, phase);
    auto it = decisions_.find(key);
    if (it != decisions_.end()) return it->second;
    const Decision d = choose_n(c_, demand, phase);
    decisions_.emplace(key, d);
    return d;
  }

  // engine.py:155-238
  std::vector<MicroBatch> admit_and_batch(const Decision& d, int capacity) {
    std::vector<Bin> bins;
    std::vector<MicroBatch> out;
    if (capacity < 1) return out;
    const int64_t budget = d.budget;
    auto lightest = [&](int phase, int64_t extra) -> int {
      int best = -1;
      for (int i = 0; i < (int)bins.size(); ++i) {
        const Bin& b = bins[i];
        const bool compat = b.phase < 0 || b.phase == phase || c_.allow_mixed;
        if (!compat || b.tokens + extra > budget || (int)b.members.size() >= c_.max_batch_size) continue;
        if (best < 0 || b.tokens < bins[best].tokens) best = i;
      }
      return best;
    };
    auto open = [&]() -> int {
      if ((int)bins.size() >= capacity) return -1;
      bins.emplace_back();
      return (int)bins.size() - 1;
    };
    auto place = [&](int bi, int ri, int64_t tokens, int phase) {
      Bin& b = bins[bi];
      b.members.push_back(ri);
      b.tokens += tokens;
      if (b.phase < 0)
        b.phase = phase;
      else if (b.phase != phase)
        b.phase = MIXED;
    };
    while (!ready_.empty()) {
      int b = lightest(DECODE, 1);
      if (b < 0) b = open();
      if (b < 0) break;
      place(b, ready_.front(), 1, DECODE);
      ready_.pop_front();
    }
    while (!pending_.empty()) {
      const int ri = pending_.front();
      const int64_t in = reqs_[ri].input_len;
      int b = lightest(PREFILL, in);
      if (b < 0) b = open();
      if (b < 0) break;
      place(b, ri, in, PREFILL);
      pending_.pop_front();
    }
    for (Bin& b : bins) {
      if (b.members.empty()) continue;
      MicroBatch m;
      m.id = next_mb_ + (int64_t)out.size();
      m.reqs = std::move(b.members);
      m.phase = b.phase < 0 ? DECODE : b.phase;
      m.tokens = b.tokens;
      out.push_back(std::move(m));
    }
    return out;
  }

  // engine.py:456-505
  void boundary(int64_t now) {
    boundaries_.erase(now);
    StageRt& head = stages_[0];
    if (head.busy || !head.waiting.empty() || (ready_.empty() && pending_.empty())) return;
    const int phase = ready_.empty() ? 0 : 1;  // profile phase: prefill 0, decode 1
    Decision d;
    if (!have_last_ || iteration_ % c_.decision_stride == 0)
      d = decide(phase);
    else
      d = last_;
    const int room = d.n - (int)inflight_.size();
    if (room <= 0) return;
    std::vector<MicroBatch> batches = admit_and_batch(d, room);
    if (batches.empty()) return;
    iteration_ += 1;
    last_ = d, have_last_ = true;
    logs_.decisions.push_back({iteration_, d});
    note(now, BOUNDARY, iteration_, 0);
    next_mb_ += (int64_t)batches.size();
    for (MicroBatch& m : batches) {
      for (int ri : m.reqs)
        if (reqs_[ri].state == QUEUED) reqs_[ri].state = RUNNING_PREFILL;
      const int64_t id = m.id;
      inflight_.emplace(id, std::move(m));
      head.waiting.push_back(id);
      hooks_.admit(inflight_.at(id), now);
    }
    launch_compute(0, now);
  }
};

}  // namespace

int run(const Config& c, std::vector<Request>& reqs, int64_t horizon_ns, Hooks& hooks, Logs& logs) {
  Engine e(c, reqs, hooks, logs);
  return e.run(horizon_ns);
}

}  // namespace sched
}  // namespace pl
