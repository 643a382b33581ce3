// Native virtual-clock scheduler: the reference's pipeline semantics in C++.
//
// Bit-exact restatement (verified against pipelink.PipelineEngine.run by
// tests/test_native_sched.py) of:
//   compute_time            profiles.py:95-121   piecewise-linear table lookup
//   s_to_ns / transmission_ns  transport.py:32-33, 199-200
//   LinkQueue               transport.py:70-160  two-class chunking queue
//   _round_terms / choose_n controller.py:68-186 incremental micro-batch search
//   admit_and_batch         engine.py:155-238    continuous batching
//   PipelineEngine.run      engine.py:264-600    event loop, tie order, logs
// Python's float semantics are reproduced operation for operation (IEEE double,
// round-half-even for round()), so every timestamp and decision matches.
//
// The scheduler calls a Hooks object at the points where the reference
// simulates work; the GPU runtime (runtime.cu) implements them with real
// stage forwards and NCCL chunks, the null hooks give a pure virtual run.
#pragma once

#include <stdint.h>

#include <deque>
#include <set>
#include <vector>

namespace pl {
namespace sched {

enum Kind : int { DELIVERED = 0, DONE = 1, ARRIVAL = 2, BOUNDARY = 3, SENT = 4 };  // engine.py:42-49
enum Phase : int { PREFILL = 0, DECODE = 1, MIXED = 2 };
enum Cls : int { CLS_PREFILL = 0, CLS_DECODE = 1 };
enum ReqState : int { QUEUED = 0, RUNNING_PREFILL = 1, DECODING = 2, FINISHED = 3 };
enum LinkEv : int { L_ENQUEUE = 0, L_EMIT = 1, L_SENT = 2, L_DELIVER = 3 };

struct Profile {
  std::vector<int64_t> xs[2];  // [phase: prefill, decode] sorted token counts
  std::vector<double> ys[2];
};

struct Link {
  double latency_s;
  double bandwidth;  // bytes / s
};

struct Config {
  int S = 1;
  std::vector<Profile> profiles;
  std::vector<Link> links;  // S forward+return hops when S >= 2
  int64_t max_batched_tokens = 1;
  int max_batch_size = 1;
  int n_max = 2;            // effective
  double bubble_epsilon = 0.02;
  double gain_delta = 0.01;
  int fixed_compute = 0;    // BudgetMode.FIXED_COMPUTE
  int decision_stride = 1;
  int64_t chunk_size = -1;  // < 0: unchunked
  int fcfs = 0;             // LinkPolicy.FCFS
  int allow_mixed = 0;
  int64_t bytes_per_token = 1;
  int64_t feedback_bytes = 8;
};

struct Request {
  int64_t id, arrival_ns, input_len, output_len;
  int state = QUEUED;
  int64_t tokens = 0;
  double first_token_time = 0, finish_time = 0;
  bool has_first = false, has_finish = false;
};

struct MicroBatch {
  int64_t id;
  std::vector<int> reqs;  // indices into the request table
  int phase;
  int64_t tokens;
};

struct Payload {
  int64_t id;
  int cls;
  int64_t size;
  int64_t mb;  // micro-batch id
};

struct Chunk {
  int64_t payload;
  int index;
  int64_t size;
  bool last;
  int cls;
};

struct Decision {
  int n;
  int64_t budget;
  double bubble;
};

struct Hooks {
  virtual ~Hooks() = default;
  virtual void admit(const MicroBatch&, int64_t) {}
  virtual void compute(int, const MicroBatch&, int64_t) {}
  virtual void emit(int, const Payload&, const Chunk&, int64_t, int64_t) {}
  virtual void delivered(int, const Payload&, const MicroBatch&, int64_t) {}
  virtual void feedback(const MicroBatch&, int64_t) {}
  virtual int error() const { return 0; }  // non-zero aborts the run
};

struct EventRec { int64_t t; int kind; int64_t subject; int stage; };
struct LinkRec { int64_t t; int link; int64_t payload; int index; int64_t size; int cls; int ev; };

struct Logs {
  std::vector<EventRec> events;
  std::vector<LinkRec> links;
  std::vector<std::pair<int64_t, Decision>> decisions;
  std::vector<std::vector<std::pair<int64_t, int64_t>>> busy;
  std::vector<std::pair<int64_t, int64_t>> emissions;  // (t, request id)
  std::vector<std::pair<int64_t, int64_t>> first_compute;  // (request id, t)
  int64_t end_ns = 0;
  bool all_finished = false;
};

// Reference helpers (exposed for tests)
int64_t s_to_ns(double seconds);
int64_t transmission_ns(const Link& l, int64_t bytes);
double compute_time(const Profile& p, int phase, int64_t tokens);
Decision choose_n(const Config& c, int64_t queued_tokens, int phase);

// Run the trace (requests sorted as given) to completion or horizon (< 0: none).
int run(const Config& c, std::vector<Request>& reqs, int64_t horizon_ns, Hooks& hooks, Logs& logs);

}  // namespace sched
}  // namespace pl
