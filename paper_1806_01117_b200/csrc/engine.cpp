// Executor: runs a reversal schedule of an operator pair on the GPU.
//
// B200-native restatement of the reference runtime (pkg/src/asyncckpt/runtime.py):
//   _ByteLedger            runtime.py:123-159  -> Ledger (identical byte accounting)
//   _Execution.forward     runtime.py:174-180  -> Run::forward (seed at first arrival at n)
//   _Execution.backward    runtime.py:186-190  -> Run::backward
//   wait_transfer          runtime.py:192-199  -> Run::wait_transfer (device-side wait;
//                                                  stall = compute-stream idle time, CUDA events)
//   run_schedule           runtime.py:201-252  -> Run::run_schedule
//   _multistage_forward    runtime.py:269-294  -> Run::multistage_forward
//   _multistage_backward   runtime.py:297-322  -> Run::multistage_backward
//   execute                runtime.py:339-381  -> ackpt_engine_run
//   calibrate              runtime.py:420-466  -> ackpt_engine_calibrate
//
// States live in a pool of HBM buffers.  Save/Load/Tape do not copy: a slot
// or tape entry holds a reference-counted buffer id, the reference's
// "bytes are immutable, keep a reference" semantics (runtime.py:221-233)
// without any device-to-device traffic.  A buffer returns to the free list
// when its last reference drops; all compute runs on one stream, so reuse is
// stream-ordered.  Buffers handed to the copy engines are covered by event
// waits: a store's source is released only after the compute stream waited for
// the store (the reference's own "one store in flight" rule), and a fetch's
// destination is written only after the copy stream waited for the compute
// stream's position at issue time.
//
// The host interpreter never blocks inside the timed window: every wait is a
// cudaStreamWaitEvent.  It runs once "dry" at prepare time to size the pool
// and the timing-event pool exactly; the real run replays identical decisions.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "common.h"
#include "nvtx.h"

namespace ackpt {
// tier.cpp
void tier_reserve_keys(ackpt_tier* t, const std::vector<int64_t>& keys, int64_t bytes);
cudaEvent_t tier_ticket_event(ackpt_tier* t, ackpt_ticket id);
int tier_ticket_status(ackpt_tier* t, ackpt_ticket id, std::string* msg);
int tier_async_status(ackpt_tier* t, ackpt_ticket id, std::string* msg);
void tier_retire(ackpt_tier* t, ackpt_ticket id);
void tier_set_timing(ackpt_tier* t, bool on);
void tier_reset_async(ackpt_tier* t, ackpt_ticket id);
void tier_quiesce(ackpt_tier* t);
bool tier_ticket_times(ackpt_tier* t, ackpt_ticket id, cudaEvent_t* t0, cudaEvent_t* t1);
int64_t tier_slot_bytes(const ackpt_tier* t);
cudaStream_t tier_d2h(const ackpt_tier* t);
double tier_spill_seconds(ackpt_tier* t, int64_t bytes);
int tier_dram_slots(ackpt_tier* t);
}  // namespace ackpt

namespace {

struct SegPlan {
  std::vector<ackpt::Action> actions;
  std::vector<int64_t> last_read;  // slot_read_liveness
};

}  // namespace

struct ackpt_engine {
  ackpt_operator op{};
  int64_t S = 0, n = 0;
  // plan
  bool prepared = false;
  int strategy = -1;
  int64_t slots = 0, interval = 0;
  bool fallback = false;
  ackpt_tier* tier = nullptr;
  SegPlan plain;
  std::vector<int64_t> boundaries;
  std::map<int64_t, SegPlan> seg_by_len;
  // resources
  std::vector<void*> slabs;
  std::vector<void*> bufs;
  void* adj_internal = nullptr;
  std::vector<cudaEvent_t> timing;  // pool of timing events
  cudaEvent_t ev_start = nullptr, ev_end = nullptr, ev_sync = nullptr;
  cudaStream_t compute = nullptr;
  int fuse = 0;
  int prefetch = -1;
  int64_t sample_every = 0;
  int timeline = 0;                               // record a measured event timeline
  std::vector<ackpt_timeline_event> timeline_out;  // of the last run
  // CUDA-graph mode (ackpt_engine_set_graph): a pass captured once and replayed
  struct Graph {
    bool pending = false;  // an eager run with these buffers happened: capture next time
    bool prefetch = true;  // the prefetch order the pass was enqueued with
    const void* init = nullptr;
    const void* seed = nullptr;
    void* out = nullptr;
    cudaGraphExec_t exec = nullptr;
    ackpt_stats st{};  // host-side counters of the captured pass
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> stall_pairs;
    std::vector<ackpt_ticket> issued;
  };
  int graph = 0;
  Graph g;
  void drop_graph() {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    g = Graph{};
  }
};

namespace ackpt {
namespace {

struct Ledger {  // runtime.py:123-159
  int64_t slot_bytes = 0, tape_bytes = 0, transfer_bytes = 0, peak = 0;
  void bump() { peak = std::max(peak, slot_bytes + tape_bytes + transfer_bytes); }
  void set_slots(int64_t b) {
    slot_bytes = b;
    bump();
  }
  void add_tape(int64_t b) {
    tape_bytes += b;
    bump();
  }
  void drop_tape(int64_t b) { tape_bytes -= b; }
  void add_transfer(int64_t b) {
    transfer_bytes += b;
    bump();
  }
  void drop_transfer(int64_t b) { transfer_bytes -= b; }
};

constexpr int kExt = -1;  // the caller's initial state (read-only, never pooled)

void check_op(int rc) {
  if (rc != ACKPT_OK) fail(rc, std::string("operator: ") + ackpt_last_error());
}

bool env_prefetch() {
  const char* v = std::getenv("CKPT_DISABLE_PREFETCH");  // runtime.py:302
  return !(v && std::string(v) == "1");
}

struct Run {
  ackpt_engine* E;
  bool dry;
  cudaStream_t s;
  ackpt_stats st{};
  Ledger ledger;
  // buffer pool
  std::vector<int> refs;
  std::vector<int> free_list;
  // Stream-ordering check (SURVEY §5 race detection, always on, host side):
  // a buffer a store reads or a fetch writes is in flight from begin_store /
  // begin_fetch until its wait_transfer.  Returning it to the pool, handing
  // it out, or enqueueing a kernel that reads a fetch destination or writes
  // an in-flight buffer before that wait is a protocol error (ExecutionError)
  // -- the host-side counterpart of ACKPT_POISON's device-side NaN check.
  enum : int8_t { kIdle = 0, kStoreSrc = 1, kFetchDst = 2 };
  std::vector<int8_t> flight;
  std::map<ackpt_ticket, int> flight_of;
  ackpt_ticket dry_ticket = -2;  // distinct tickets in the dry run too
  void flight_mark(ackpt_ticket t, int id, int8_t kind) {
    if (id < 0) return;  // the caller's input: read-only, never pooled
    if (size_t(id) >= flight.size()) flight.resize(size_t(id) + 1, kIdle);
    if (flight[size_t(id)] != kIdle) order_error(id, "second transfer on a buffer already in flight");
    flight[size_t(id)] = kind;
    flight_of[t] = id;
  }
  void flight_clear(ackpt_ticket t) {
    auto it = flight_of.find(t);
    if (it == flight_of.end()) return;
    flight[size_t(it->second)] = kIdle;
    flight_of.erase(it);
  }
  int8_t flight_state(int id) const {
    return id >= 0 && size_t(id) < flight.size() ? flight[size_t(id)] : int8_t(kIdle);
  }
  [[noreturn]] void order_error(int id, const char* what) const {
    fail(ACKPT_EXECUTION_ERROR, std::string("stream-ordering check: ") + what + " (pool buffer " +
                                    std::to_string(id) + ")");
  }
  int in_use = 0, peak_in_use = 0;
  const void* ext = nullptr;
  // adjoint
  void* adj[2] = {nullptr, nullptr};
  int a = 0;
  bool seeded = false;
  const void* seed_bytes = nullptr;
  // timing events
  size_t next_ev = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> stall_pairs;
  // measured timeline (ackpt_engine_set_timeline): compute launches and
  // stalls bracketed by events on the compute stream, transfers by the
  // tier's marks on its copy streams
  struct Span {
    int32_t kind;
    int64_t from, to;
    cudaEvent_t e0, e1;
  };
  struct Xfer {
    int32_t kind;
    int64_t key;
    ackpt_ticket id;
  };
  std::vector<Span> spans;
  std::vector<Xfer> xfers;

  // Runs `launch` (skipped in the dry run), bracketed by timeline events.
  template <class F>
  void span(int32_t kind, int64_t from, int64_t to, F&& launch) {
    if (!E->timeline) {
      if (!dry) launch();
      return;
    }
    cudaEvent_t e0 = timing_event(), e1 = timing_event();
    if (dry) return;
    ACKPT_CUDA_CHECK(cudaEventRecord(e0, s));
    launch();
    ACKPT_CUDA_CHECK(cudaEventRecord(e1, s));
    spans.push_back({kind, from, to, e0, e1});
  }

  Run(ackpt_engine* e, bool d, cudaStream_t str) : E(e), dry(d), s(str) {
    if (!dry) {
      refs.assign(E->bufs.size(), 0);
      for (int i = int(E->bufs.size()) - 1; i >= 0; --i) free_list.push_back(i);
    }
  }

  // -- buffers --------------------------------------------------------------
  int acquire() {
    if (free_list.empty()) {
      if (!dry) fail(ACKPT_EXECUTION_ERROR, "HBM buffer pool exhausted (plan/dry-run mismatch)");
      refs.push_back(0);
      free_list.push_back(int(refs.size()) - 1);
    }
    int id = free_list.back();
    free_list.pop_back();
    if (flight_state(id) != kIdle) order_error(id, "buffer handed out while a transfer uses it");
    refs[size_t(id)] = 1;
    peak_in_use = std::max(peak_in_use, ++in_use);
    return id;
  }
  void retain(int id) {
    if (id >= 0) ++refs[size_t(id)];
  }
  void release(int id) {
    if (id < 0) return;
    if (--refs[size_t(id)] == 0) {
      if (flight_state(id) != kIdle) order_error(id, "buffer released before its transfer was waited");
      free_list.push_back(id);
      --in_use;
      // ACKPT_POISON=1 (race check): a released buffer is filled
      // with NaN bit patterns on the compute stream.  A copy engine still
      // reading it (a store whose wait is missing) or a kernel reading a
      // fetch destination before its H2D copy landed then sees NaN, which the
      // bit-identity / oracle checks of the test suite turn into failures.
      if (!dry && poison()) {
        ACKPT_CUDA_CHECK(cudaMemsetAsync(E->bufs[size_t(id)], 0xFF, size_t(E->S), s));
        chainable = false;
      }
    }
  }
  // ACKPT_FAULT_ORDER=1 (test only, tests/test_gpu_poison.py): the forward
  // sweep does not hold a boundary state while its store is in flight.
  static bool fault_skip_hold() {
    static const bool on = [] {
      const char* v = std::getenv("ACKPT_FAULT_ORDER");
      return v && v[0] == '1';
    }();
    return on;
  }
  static bool poison() {
    static const bool on = [] {
      const char* v = std::getenv("ACKPT_POISON");
      return v && v[0] == '1';
    }();
    return on;
  }
  // Buffer addresses for enqueued work: kernels may not read a fetch
  // destination, nor write any in-flight buffer, before its wait.
  const void* ptr(int id) const {
    if (flight_state(id) == kFetchDst) order_error(id, "read of a fetch destination before its wait");
    return id == kExt ? ext : E->bufs[size_t(id)];
  }
  void* wptr(int id) const {
    if (flight_state(id) != kIdle) order_error(id, "write to a buffer while a transfer uses it");
    return E->bufs[size_t(id)];
  }

  cudaEvent_t timing_event() {
    if (dry) {
      ++next_ev;
      return nullptr;
    }
    if (next_ev >= E->timing.size()) {  // the dry run sized the pool; grow if a mode changed since
      cudaEvent_t ev;
      ACKPT_CUDA_CHECK(cudaEventCreate(&ev));
      E->timing.push_back(ev);
    }
    return E->timing[next_ev++];
  }

  // -- operator calls (runtime.py:174-190) ------------------------------------
  void do_seed(int state) {
    chainable = false;
    // Seed the adjoint register so that after all n backward steps the result
    // lands in adj[0] (the caller's output buffer).
    a = (E->n % 2 == 0) ? 0 : 1;
    if (!dry) {
      if (seed_bytes) {
        ACKPT_CUDA_CHECK(cudaMemcpyAsync(adj[a], seed_bytes, size_t(E->S), cudaMemcpyDeviceToDevice, s));
      } else {
        if (!E->op.seed) fail(ACKPT_EXECUTION_ERROR, "no adjoint seed: operator has no seed function");
        check_op(E->op.seed(E->op.ctx, ptr(state), adj[a], s));
        ++st.kernel_launches;
      }
    }
    seeded = true;
  }

  // Sampled kernel timing: an event pair around every k-th launch.
  int64_t fwd_calls = 0, bwd_calls = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> fwd_pairs, bwd_pairs;

  template <class F>
  void timed(int64_t& calls, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& pairs, F&& launch) {
    const bool sample = E->sample_every > 0 && (calls++ % E->sample_every) == 0;
    if (!sample) {
      if (!dry) launch();
      return;
    }
    cudaEvent_t e0 = timing_event(), e1 = timing_event();
    if (dry) return;
    ACKPT_CUDA_CHECK(cudaEventRecord(e0, s));
    launch();
    ACKPT_CUDA_CHECK(cudaEventRecord(e1, s));
    pairs.emplace_back(e0, e1);
  }

  int forward(int64_t step, int cur) {
    int out = acquire();
    span(ACKPT_EV_FORWARD, step, step + 1, [&] {
      timed(fwd_calls, fwd_pairs, [&] {
        step_launch([&] { check_op(E->op.forward(E->op.ctx, step, ptr(cur), wptr(out), s)); });
        ++st.kernel_launches;
      });
    });
    release(cur);
    ++st.forward_evals;
    if (step + 1 == E->n && !seeded) do_seed(out);
    return out;
  }

  int advance(int64_t from, int64_t to, int cur) {
    // Advance(from, to): per-step contract by default; one fused launch when
    // the operator provides advance() and fusion is enabled.
    // (length 1 too: a fused execution uses the fused kernel family throughout)
    if (to - from >= 1 && E->fuse && E->op.advance) {
      int out = acquire();
      span(ACKPT_EV_FORWARD, from, to, [&] {
        step_launch([&] { check_op(E->op.advance(E->op.ctx, from, to, ptr(cur), wptr(out), s)); });
        ++st.kernel_launches;
      });
      release(cur);
      st.forward_evals += to - from;
      ++st.fused_advances;
      if (to == E->n && !seeded) do_seed(out);
      return out;
    }
    for (int64_t k = from; k < to; ++k) cur = forward(k, cur);
    return cur;
  }

  void backward(int64_t step, int state) {
    if (!seeded)
      fail(ACKPT_EXECUTION_ERROR, "Reverse " + std::to_string(step) + " before the adjoint was seeded");
    span(ACKPT_EV_BACKWARD, step, step + 1, [&] {
      timed(bwd_calls, bwd_pairs, [&] {
        step_launch([&] { check_op(E->op.backward(E->op.ctx, step, ptr(state), adj[a], adj[1 - a], s)); });
        ++st.kernel_launches;
      });
    });
    a = 1 - a;
    ++st.backward_evals;
  }

  // -- transfers ------------------------------------------------------------
  void wait_transfer(ackpt_ticket t, int64_t at_step) {
    // runtime.py:192-199.  Errors captured by the transfer surface here.
    NvtxRange range("wait");
    flight_clear(t);
    if (dry) {
      next_ev += 2;
      return;
    }
    std::string msg;
    int rc = tier_ticket_status(E->tier, t, &msg);
    if (rc != ACKPT_OK) fail(rc, msg);
    chainable = false;
    cudaEvent_t done = tier_ticket_event(E->tier, t);
    cudaEvent_t before = timing_event(), after = timing_event();
    // under graph capture these are event-record nodes (re-recorded on replay)
    const unsigned rf = capturing ? cudaEventRecordExternal : cudaEventRecordDefault;
    ACKPT_CUDA_CHECK(cudaEventRecordWithFlags(before, s, rf));
    if (done) ACKPT_CUDA_CHECK(cudaStreamWaitEvent(s, done, 0));
    ACKPT_CUDA_CHECK(cudaEventRecordWithFlags(after, s, rf));
    stall_pairs.emplace_back(before, after);
    if (E->timeline) spans.push_back({ACKPT_EV_STALL, at_step, at_step, before, after});
  }

  std::vector<ackpt_ticket> issued;  // checked for file-stage errors after the run
  bool capturing = false;            // enqueued under CUDA-graph stream capture
  // The last operation enqueued on the compute stream was a step launch of
  // the operator (per-step, fused Advance / TapeForward / Reverse run): the
  // next one may be chained to it (g_chain_hint, chain.cuh).  Cleared by
  // every other enqueue (waits, transfers, seeds, poison fills).
  bool chainable = false;
  template <class F>
  void step_launch(F&& launch) {
    struct Hint {  // reset on every exit, exceptions included
      explicit Hint(int on) { g_chain_hint = on; }
      ~Hint() { g_chain_hint = 0; }
    } hint((chainable && !E->timeline && E->sample_every == 0) ? 1 : 0);
    chainable = false;
    launch();
    chainable = true;
  }

  ackpt_ticket begin_store(int64_t key, int state) {
    NvtxRange range("store");
    chainable = false;
    ackpt_ticket t = dry_ticket--;
    if (!dry) {
      check_op(ackpt_tier_begin_store(E->tier, key, key, ptr(state), E->S, s, &t));
      issued.push_back(t);
      if (E->timeline) xfers.push_back({ACKPT_EV_STORE, key, t});
    }
    flight_mark(t, state, kStoreSrc);
    ++st.stores_issued;
    st.link_bytes += E->S;
    return t;
  }

  ackpt_ticket begin_fetch(int64_t key, int dst) {
    NvtxRange range("fetch");
    chainable = false;
    ackpt_ticket t = dry_ticket--;
    if (!dry) {
      int rc = ackpt_tier_begin_fetch(E->tier, key, wptr(dst), E->S, s, &t);
      if (rc != ACKPT_OK) fail(rc, ackpt_last_error());
      issued.push_back(t);
      if (E->timeline) xfers.push_back({ACKPT_EV_FETCH, key, t});
    }
    flight_mark(t, dst, kFetchDst);
    ++st.prefetches_issued;
    st.link_bytes += E->S;
    return t;
  }

  // -- interpreter (runtime.py:201-252) ---------------------------------------
  int run_schedule(const SegPlan& plan, int64_t offset, int state) {
    const int64_t cap = E->slots;
    std::vector<int> slot_buf(size_t(std::max<int64_t>(cap, 0)), -2);
    std::vector<int64_t> slot_step(slot_buf.size(), 0);
    std::vector<int64_t> write_idx(slot_buf.size(), -1);
    int64_t occupied = 0;
    std::vector<std::pair<int64_t, int>> tape;
    int64_t current = 0;
    auto free_slot = [&](int64_t slot) {
      if (slot_buf[size_t(slot)] != -2) {
        release(slot_buf[size_t(slot)]);
        slot_buf[size_t(slot)] = -2;
        --occupied;
      }
    };
    const auto& acts = plan.actions;
    for (size_t idx = 0; idx < acts.size(); ++idx) {
      const Action& act = acts[idx];
      if (act.op == ACKPT_ADVANCE || act.op == ACKPT_TAPE) {
        if (act.a != current)
          fail(ACKPT_EXECUTION_ERROR, "action " + std::to_string(idx) + " starts at " +
                                          std::to_string(act.a) + ", state is at " +
                                          std::to_string(current));
        if (act.op == ACKPT_TAPE && E->fuse && E->op.forward_many) {
          // Temporal fusion: up to 64 taped steps per launch, every output
          // kept (the tape holds the INPUT state of each step).
          for (int64_t rel = act.a; rel < act.b;) {
            const int64_t cnt = std::min<int64_t>(ACKPT_MAX_FUSED, act.b - rel);
            void* outs[ACKPT_MAX_FUSED];
            int ids[ACKPT_MAX_FUSED];
            for (int64_t i = 0; i < cnt; ++i) {
              ids[i] = acquire();
              outs[i] = dry ? nullptr : wptr(ids[i]);
            }
            retain(state);
            tape.emplace_back(rel, state);
            ledger.add_tape(E->S);
            for (int64_t i = 0; i + 1 < cnt; ++i) {  // out[i] is the input of step rel+i+1
              tape.emplace_back(rel + i + 1, ids[i]);
              ledger.add_tape(E->S);
            }
            span(ACKPT_EV_FORWARD, offset + rel, offset + rel + cnt, [&] {
              step_launch([&] { check_op(E->op.forward_many(E->op.ctx, offset + rel, cnt, ptr(state), outs, s)); });
              ++st.kernel_launches;
            });
            release(state);
            state = ids[cnt - 1];
            st.forward_evals += cnt;
            ++st.fused_advances;
            if (offset + rel + cnt == E->n && !seeded) do_seed(state);
            rel += cnt;
          }
        } else if (act.op == ACKPT_TAPE) {
          for (int64_t rel = act.a; rel < act.b; ++rel) {
            retain(state);
            tape.emplace_back(rel, state);  // the INPUT state of step rel
            ledger.add_tape(E->S);
            state = forward(offset + rel, state);
          }
        } else if (act.b > act.a) {
          state = advance(offset + act.a, offset + act.b, state);
        }
        current = act.b;
      } else if (act.op == ACKPT_SAVE) {
        if (act.b < 0 || act.b >= cap)
          fail(ACKPT_SLOT_OUT_OF_RANGE,
               "slot " + std::to_string(act.b) + " outside capacity " + std::to_string(cap));
        free_slot(act.b);
        retain(state);
        slot_buf[size_t(act.b)] = state;
        slot_step[size_t(act.b)] = offset + current;
        ++occupied;
        write_idx[size_t(act.b)] = int64_t(idx);
        ledger.set_slots(occupied * E->S);
      } else if (act.op == ACKPT_LOAD) {
        if (act.a < 0 || act.a >= cap)
          fail(ACKPT_SLOT_OUT_OF_RANGE,
               "slot " + std::to_string(act.a) + " outside capacity " + std::to_string(cap));
        int held = slot_buf[size_t(act.a)];
        if (held == -2) fail(ACKPT_SLOT_UNWRITTEN, "slot " + std::to_string(act.a) + " read before write");
        retain(held);
        release(state);
        state = held;
        current = slot_step[size_t(act.a)] - offset;
        const int64_t w = write_idx[size_t(act.a)];
        if (w >= 0 && plan.last_read[size_t(w)] == int64_t(idx)) {  // final read: free
          free_slot(act.a);
          ledger.set_slots(occupied * E->S);
        }
      } else if (act.op == ACKPT_REVERSE && E->fuse && E->op.backward_many) {
        // Temporal fusion: a run of consecutive Reverse actions over taped
        // states in one launch (the adjoint never leaves the chip).
        size_t run = 1;
        while (idx + run < acts.size() && run < size_t(ACKPT_MAX_FUSED) &&
               acts[idx + run].op == ACKPT_REVERSE && acts[idx + run].a == act.a - int64_t(run))
          ++run;
        if (!seeded)
          fail(ACKPT_EXECUTION_ERROR, "Reverse " + std::to_string(act.a) + " before the adjoint was seeded");
        if (tape.size() < run) fail(ACKPT_EXECUTION_ERROR, "Reverse " + std::to_string(act.a) + " without taped state");
        const void* states[ACKPT_MAX_FUSED];
        int held[ACKPT_MAX_FUSED];
        const int64_t lo = act.a - int64_t(run) + 1;
        for (size_t r = 0; r < run; ++r) {  // pop tops: steps act.a, act.a-1, ...
          const int64_t want = act.a - int64_t(r);
          if (tape.back().first != want)
            fail(ACKPT_EXECUTION_ERROR, "Reverse " + std::to_string(want) + " without taped state");
          held[r] = tape.back().second;
          states[want - lo] = dry ? nullptr : ptr(held[r]);
          tape.pop_back();
          ledger.drop_tape(E->S);
        }
        span(ACKPT_EV_BACKWARD, offset + lo, offset + lo + int64_t(run), [&] {
          step_launch([&] { check_op(E->op.backward_many(E->op.ctx, offset + lo, int64_t(run), states, adj[a], adj[1 - a], s)); });
          ++st.kernel_launches;
        });
        a = 1 - a;
        st.backward_evals += int64_t(run);
        for (size_t r = 0; r < run; ++r) release(held[r]);
        idx += run - 1;
      } else if (act.op == ACKPT_REVERSE) {
        if (tape.empty() || tape.back().first != act.a)
          fail(ACKPT_EXECUTION_ERROR, "Reverse " + std::to_string(act.a) + " without taped state");
        int taped = tape.back().second;
        tape.pop_back();
        ledger.drop_tape(E->S);
        backward(offset + act.a, taped);
        release(taped);
      } else if (act.op == ACKPT_DONE) {
        break;
      } else {
        fail(ACKPT_EXECUTION_ERROR, "unknown action op " + std::to_string(act.op));
      }
    }
    for (int64_t sl = 0; sl < cap; ++sl) free_slot(sl);  // pool.clear()
    for (auto& te : tape) release(te.second);
    ledger.set_slots(0);
    return state;
  }

  // -- multistage (runtime.py:269-322) ----------------------------------------
  int multistage_forward(int state) {
    NvtxRange range("sweep");
    const auto& bs = E->boundaries;
    ackpt_ticket ticket = -1;
    int store_src = -2;
    bool have = false;
    for (size_t idx = 0; idx < bs.size(); ++idx) {
      const int64_t b = bs[idx];
      if (have) {
        wait_transfer(ticket, b);
        ledger.drop_transfer(E->S);
        release(store_src);
      }
      ticket = begin_store(b, state);
      if (!fault_skip_hold()) retain(state);  // (test switch: drop the hold, the ordering check must fire)
      store_src = state;
      have = true;
      ledger.add_transfer(E->S);
      const int64_t end = idx + 1 < bs.size() ? bs[idx + 1] : E->n;
      state = advance(b, end, state);
    }
    if (have) {
      wait_transfer(ticket, E->n);
      ledger.drop_transfer(E->S);
      release(store_src);
    }
    return state;
  }

  void multistage_backward() {
    NvtxRange range("backward");
    const bool pf = E->prefetch < 0 ? env_prefetch() : E->prefetch != 0;
    const auto& bs = E->boundaries;
    const size_t nseg = bs.size();
    std::map<int64_t, std::pair<ackpt_ticket, int>> tickets;
    auto issue = [&](int64_t key) {
      int dst = acquire();
      tickets[key] = {begin_fetch(key, dst), dst};
      ledger.add_transfer(E->S);
    };
    if (pf) issue(bs[nseg - 1]);
    for (size_t jj = nseg; jj-- > 0;) {
      const int64_t start = bs[jj];
      const int64_t end = jj + 1 < nseg ? bs[jj + 1] : E->n;
      if (!pf) issue(start);
      auto it = tickets.find(start);
      auto tk = it->second;
      tickets.erase(it);
      wait_transfer(tk.first, start);
      if (pf && jj > 0) issue(bs[jj - 1]);
      ledger.drop_transfer(E->S);  // fetched bytes go live
      const SegPlan& plan = E->seg_by_len.at(end - start);
      NvtxRange seg(dry ? std::string() : "segment " + std::to_string(start) + "-" + std::to_string(end));
      int last = run_schedule(plan, start, tk.second);
      release(last);
    }
  }

  void finish_stats() {
    st.peak_l1_bytes = ledger.peak;
    st.interval = E->strategy == ACKPT_MULTISTAGE ? E->interval : 0;
    st.fallback = E->fallback ? 1 : 0;
    st.device_buffers = int64_t(E->bufs.size());
  }
};

void alloc_pool(ackpt_engine* E, int64_t need_bufs, size_t need_events) {
  if (int64_t(E->bufs.size()) < need_bufs) {
    const int64_t add = need_bufs - int64_t(E->bufs.size());
    void* slab = nullptr;
    cudaError_t e = cudaMalloc(&slab, size_t(add) * size_t(E->S));
    if (e != cudaSuccess) {
      cudaGetLastError();
      fail(ACKPT_STORAGE_FULL, "HBM buffer pool of " + std::to_string(need_bufs) + " x " +
                                   std::to_string(E->S) + " B: " + cudaGetErrorString(e));
    }
    E->slabs.push_back(slab);
    for (int64_t i = 0; i < add; ++i)
      E->bufs.push_back(static_cast<char*>(slab) + size_t(i) * size_t(E->S));
    if (Run::poison()) {  // never-written = NaN; complete before the (non-blocking) compute stream uses it
      ACKPT_CUDA_CHECK(cudaMemset(slab, 0xFF, size_t(add) * size_t(E->S)));
      ACKPT_CUDA_CHECK(cudaDeviceSynchronize());
    }
  }
  if (!E->adj_internal) ACKPT_CUDA_CHECK(cudaMalloc(&E->adj_internal, size_t(E->S)));
  while (E->timing.size() < need_events) {
    cudaEvent_t ev;
    ACKPT_CUDA_CHECK(cudaEventCreate(&ev));
    E->timing.push_back(ev);
  }
}

SegPlan make_plan(std::vector<Action>&& acts) {
  SegPlan p;
  p.actions = std::move(acts);
  slot_read_liveness(p.actions, p.last_read);
  return p;
}

enum class Mode { kFull, kForwardSweep, kBackwardSweep };

// The stream work of one pass on E->compute (between ev_start and ev_end).
void enqueue_pass(ackpt_engine* E, Run& r, Mode mode, void* final_state) {
  const bool ms = E->strategy == ACKPT_MULTISTAGE && !E->fallback;
  // a captured pass is bracketed outside the graph, around its launch
  if (!r.capturing) ACKPT_CUDA_CHECK(cudaEventRecord(E->ev_start, E->compute));
  if (mode == Mode::kFull) {
    if (ms) {
      int last = r.multistage_forward(kExt);
      r.release(last);
      r.multistage_backward();
    } else {
      int last = r.run_schedule(E->plain, 0, kExt);
      r.release(last);
    }
  } else if (mode == Mode::kForwardSweep) {
    r.seeded = true;  // the caller derives the seed from the final state
    int last = r.multistage_forward(kExt);
    if (final_state)
      ACKPT_CUDA_CHECK(cudaMemcpyAsync(final_state, r.ptr(last), size_t(E->S),
                                       cudaMemcpyDeviceToDevice, E->compute));
    r.release(last);
  } else {
    r.a = (E->n % 2 == 0) ? 0 : 1;
    ACKPT_CUDA_CHECK(cudaMemcpyAsync(r.adj[r.a], r.seed_bytes, size_t(E->S), cudaMemcpyDeviceToDevice,
                                     E->compute));
    r.seeded = true;
    r.multistage_backward();
  }
  // Per-step runs end with the adjoint in adj[0] (seed parity); fused reverse
  // runs swap once per launch, so the result may sit in the internal buffer.
  if (mode != Mode::kForwardSweep && r.a != 0)
    ACKPT_CUDA_CHECK(cudaMemcpyAsync(r.adj[0], r.adj[r.a], size_t(E->S), cudaMemcpyDeviceToDevice,
                                     E->compute));
  if (!r.capturing) ACKPT_CUDA_CHECK(cudaEventRecord(E->ev_end, E->compute));
}

double elapsed_s(cudaEvent_t a, cudaEvent_t b) {
  float msv = 0.f;
  ACKPT_CUDA_CHECK(cudaEventElapsedTime(&msv, a, b));
  return double(msv) * 1e-3;
}

void run_impl(ackpt_engine* E, Mode mode, const void* initial_state, const void* seed,
              void* adjoint_out, void* final_state, ackpt_stats* stats, cudaStream_t caller) {
  if (!E->prepared) fail(ACKPT_VALUE_ERROR, "engine not prepared");
  const bool ms = E->strategy == ACKPT_MULTISTAGE && !E->fallback;
  if (mode != Mode::kFull && !ms)
    fail(ACKPT_VALUE_ERROR, "fallback plans have no Level-2 phase; use execute()");  // runtime.py:395-396
  if (mode == Mode::kFull && !adjoint_out) fail(ACKPT_VALUE_ERROR, "adjoint_out is required");
  if (mode == Mode::kBackwardSweep && !seed) fail(ACKPT_VALUE_ERROR, "seed is required");

  // CUDA-graph mode: replay a captured pass when the buffers match; capture
  // on the second run with the same buffers (the first, eager one performs
  // every first-use allocation, which a capture must not contain).
  const bool graphable = E->graph && mode == Mode::kFull && !E->timeline && E->sample_every == 0;
  auto& G = E->g;
  const bool pf_now = E->prefetch < 0 ? env_prefetch() : E->prefetch != 0;
  const bool same = G.init == initial_state && G.seed == seed && G.out == adjoint_out && G.prefetch == pf_now;
  if (!graphable || !same) E->drop_graph();
  const bool replay = graphable && G.exec;
  const bool capture = graphable && !G.exec && G.pending;

  // Order after the caller's stream, then time on the engine's stream.
  ACKPT_CUDA_CHECK(cudaEventRecord(E->ev_sync, caller));
  ACKPT_CUDA_CHECK(cudaStreamWaitEvent(E->compute, E->ev_sync, 0));

  NvtxRange range(mode == Mode::kFull ? "pass" : mode == Mode::kForwardSweep ? "forward_sweep" : "backward_sweep");
  Run r(E, false, E->compute);
  r.ext = initial_state;
  r.seed_bytes = seed;
  r.adj[0] = adjoint_out;
  r.adj[1] = E->adj_internal;
  if (mode == Mode::kForwardSweep) {
    r.adj[0] = E->adj_internal;  // seed computed at step n is discarded
    r.adj[1] = E->adj_internal;
  }
  auto t0 = std::chrono::steady_clock::now();
  if (replay) {
    NvtxRange gr("graph replay");
    for (ackpt_ticket tk : G.issued) tier_reset_async(E->tier, tk);
    ACKPT_CUDA_CHECK(cudaEventRecord(E->ev_start, E->compute));
    ACKPT_CUDA_CHECK(cudaGraphLaunch(G.exec, E->compute));
    ACKPT_CUDA_CHECK(cudaEventRecord(E->ev_end, E->compute));
  } else if (capture) {
    NvtxRange gc("graph capture");
    r.capturing = true;
    if (E->tier) tier_quiesce(E->tier);
    cudaGraph_t graph = nullptr;
    ACKPT_CUDA_CHECK(cudaStreamBeginCapture(E->compute, cudaStreamCaptureModeRelaxed));
    try {
      enqueue_pass(E, r, mode, final_state);
    } catch (...) {
      cudaStreamEndCapture(E->compute, &graph);
      if (graph) cudaGraphDestroy(graph);
      E->drop_graph();
      throw;
    }
    ACKPT_CUDA_CHECK(cudaStreamEndCapture(E->compute, &graph));
    const cudaError_t ie = cudaGraphInstantiate(&G.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) fail(ACKPT_CUDA_ERROR, std::string("graph instantiate: ") + cudaGetErrorString(ie));
    r.finish_stats();
    G.st = r.st;
    G.stall_pairs = r.stall_pairs;
    G.issued = r.issued;
    t0 = std::chrono::steady_clock::now();
    ACKPT_CUDA_CHECK(cudaEventRecord(E->ev_start, E->compute));
    ACKPT_CUDA_CHECK(cudaGraphLaunch(G.exec, E->compute));
    ACKPT_CUDA_CHECK(cudaEventRecord(E->ev_end, E->compute));
  } else {
    enqueue_pass(E, r, mode, final_state);
    if (graphable) {  // remember the buffers: the next identical run is captured
      G.pending = true;
      G.prefetch = pf_now;
      G.init = initial_state;
      G.seed = seed;
      G.out = adjoint_out;
    }
  }
  const bool graphed = replay || capture;
  const auto t_enq = std::chrono::steady_clock::now();
  ACKPT_CUDA_CHECK(cudaEventSynchronize(E->ev_end));
  const auto t1 = std::chrono::steady_clock::now();
  ACKPT_CUDA_CHECK(cudaStreamWaitEvent(caller, E->ev_end, 0));
  for (ackpt_ticket tk : graphed ? G.issued : r.issued) {  // file-stage I/O errors surface once the run drained
    std::string msg;
    const int rc = tier_async_status(E->tier, tk, &msg);
    if (rc != ACKPT_OK) {
      if (!graphed)
        for (ackpt_ticket x : r.issued) tier_retire(E->tier, x);
      fail(rc, msg);
    }
  }
  if (graphed) {
    if (E->tier) tier_quiesce(E->tier);
    r.st = G.st;
    r.stall_pairs = G.stall_pairs;
  } else {
    if (mode == Mode::kFull && !r.seeded)
      fail(ACKPT_EXECUTION_ERROR, "execution finished without producing an adjoint");  // runtime.py:379-380
    r.finish_stats();
  }
  r.st.wall_seconds = std::chrono::duration<double>(t1 - t0).count();
  r.st.host_enqueue_seconds = std::chrono::duration<double>(t_enq - t0).count();
  r.st.gpu_seconds = elapsed_s(E->ev_start, E->ev_end);
  double stall = 0.0;
  for (auto& pr : r.stall_pairs) stall += std::max(0.0, elapsed_s(pr.first, pr.second));
  r.st.stall_seconds = stall;
  auto sum_pairs = [](const std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& v) {
    double acc = 0.0;
    for (auto& pr : v) acc += elapsed_s(pr.first, pr.second);
    return acc;
  };
  r.st.fwd_sample_seconds = sum_pairs(r.fwd_pairs);
  r.st.fwd_samples = int64_t(r.fwd_pairs.size());
  r.st.bwd_sample_seconds = sum_pairs(r.bwd_pairs);
  r.st.bwd_samples = int64_t(r.bwd_pairs.size());
  E->timeline_out.clear();
  if (E->timeline) {
    auto since = [&](cudaEvent_t ev) { return elapsed_s(E->ev_start, ev); };
    for (const auto& sp : r.spans)
      E->timeline_out.push_back({sp.kind, ACKPT_LANE_COMPUTE, sp.from, sp.to, since(sp.e0), since(sp.e1)});
    for (const auto& x : r.xfers) {
      cudaEvent_t t0e = nullptr, t1e = nullptr;
      if (tier_ticket_times(E->tier, x.id, &t0e, &t1e))
        E->timeline_out.push_back({x.kind, ACKPT_LANE_TRANSFER, x.key, x.key, since(t0e), since(t1e)});
    }
    std::stable_sort(E->timeline_out.begin(), E->timeline_out.end(),
                     [](const ackpt_timeline_event& a, const ackpt_timeline_event& b) { return a.start < b.start; });
  }
  if (!graphed)  // every transfer of the pass completed before ev_end: recycle the tickets
    for (ackpt_ticket x : r.issued) tier_retire(E->tier, x);
  if (stats) *stats = r.st;
}

// A failed run may leave kernels queued that read caller buffers: drain the
// engine's stream before reporting the error.
template <class F>
void run_guarded(ackpt_engine* E, F&& fn) {
  try {
    fn();
  } catch (...) {
    cudaStreamSynchronize(E->compute);
    throw;
  }
}

}  // namespace
}  // namespace ackpt

extern "C" {

ACKPT_API int ackpt_engine_create(const ackpt_operator* op, ackpt_engine** out) {
  return ackpt::guard([&] {
    if (!op || !op->forward || !op->backward) ackpt::fail(ACKPT_VALUE_ERROR, "operator needs forward and backward");
    if (op->n_steps < 1) ackpt::fail(ACKPT_VALUE_ERROR, "n_steps must be >= 1");  // runtime.py:79-80
    if (op->state_bytes <= 0) ackpt::fail(ACKPT_VALUE_ERROR, "state_size must be positive");
    std::unique_ptr<ackpt_engine> e(new ackpt_engine());
    e->op = *op;
    e->S = op->state_bytes;
    e->n = op->n_steps;
    ACKPT_CUDA_CHECK(cudaStreamCreateWithFlags(&e->compute, cudaStreamNonBlocking));
    ACKPT_CUDA_CHECK(cudaEventCreate(&e->ev_start));
    ACKPT_CUDA_CHECK(cudaEventCreate(&e->ev_end));
    ACKPT_CUDA_CHECK(cudaEventCreateWithFlags(&e->ev_sync, cudaEventDisableTiming));
    *out = e.release();
  });
}

ACKPT_API int ackpt_engine_destroy(ackpt_engine* e) {
  return ackpt::guard([&] {
    if (!e) return;
    if (e->compute) cudaStreamSynchronize(e->compute);
    e->drop_graph();
    for (auto s : e->slabs) cudaFree(s);
    if (e->adj_internal) cudaFree(e->adj_internal);
    for (auto ev : e->timing) cudaEventDestroy(ev);
    if (e->ev_start) cudaEventDestroy(e->ev_start);
    if (e->ev_end) cudaEventDestroy(e->ev_end);
    if (e->ev_sync) cudaEventDestroy(e->ev_sync);
    if (e->compute) cudaStreamDestroy(e->compute);
    delete e;
  });
}

ACKPT_API int ackpt_engine_prepare(ackpt_engine* E, int32_t strategy, int64_t slots,
                                   int64_t interval, ackpt_tier* tier) {
  return ackpt::guard([&] {
    using namespace ackpt;
    NvtxRange range("prepare");
    E->prepared = false;
    E->drop_graph();
    E->strategy = strategy;
    E->slots = slots;
    E->interval = 0;
    E->fallback = false;
    E->tier = tier;
    E->boundaries.clear();
    E->seg_by_len.clear();
    E->plain = SegPlan{};
    const int64_t n = E->n;
    std::vector<Action> acts;
    if (strategy == ACKPT_FULL_STORAGE) {
      taped_actions(n, acts);  // runtime.py:364-365
      E->slots = 0;
      E->plain = make_plan(std::move(acts));
    } else if (strategy == ACKPT_REVOLVE) {
      revolve_actions(n, slots, acts);  // runtime.py:366-368
      E->plain = make_plan(std::move(acts));
    } else if (strategy == ACKPT_MULTISTAGE) {
      // plan_multistage (schedule.py:288-329)
      if (!tier) fail(ACKPT_VALUE_ERROR, "Multistage requires a Level-2 backend");
      if (interval < 1) fail(ACKPT_VALUE_ERROR, "interval must be >= 1, got " + std::to_string(interval));
      E->interval = interval;
      if (interval >= n) {
        E->fallback = true;
        revolve_actions(n, slots, acts);
        E->plain = make_plan(std::move(acts));
      } else {
        for (int64_t b = 0; b < n; b += interval) E->boundaries.push_back(b);
        for (int64_t b : E->boundaries) {
          const int64_t len = std::min(b + interval, n) - b;
          if (E->seg_by_len.count(len)) continue;
          std::vector<Action> seg;
          if (len <= slots + 1) taped_actions(len, seg);
          else revolve_actions(len, slots, seg);
          E->seg_by_len[len] = make_plan(std::move(seg));
        }
        tier_reserve_keys(tier, E->boundaries, E->S);
      }
    } else {
      fail(ACKPT_VALUE_ERROR, "unknown strategy " + std::to_string(strategy));
    }
    if (tier) tier_set_timing(tier, E->timeline != 0);
    // Dry run: sizes the HBM pool and the timing-event pool exactly.
    Run r(E, true, nullptr);
    r.adj[0] = r.adj[1] = nullptr;
    if (E->strategy == ACKPT_MULTISTAGE && !E->fallback) {
      int last = r.multistage_forward(kExt);
      r.release(last);
      r.multistage_backward();
      // the backward sweep alone needs the same pool; the forward sweep less
    } else {
      int last = r.run_schedule(E->plain, 0, kExt);
      r.release(last);
    }
    alloc_pool(E, r.peak_in_use + 1, r.next_ev);
    E->prepared = true;
  });
}

ACKPT_API int ackpt_engine_set_fusion(ackpt_engine* e, int32_t fuse_advance) {
  if (e->fuse != fuse_advance) e->drop_graph();
  e->fuse = fuse_advance;
  return ACKPT_OK;
}

ACKPT_API int ackpt_engine_set_kernel_sampling(ackpt_engine* e, int64_t every) {
  e->sample_every = every < 0 ? 0 : every;
  e->prepared = false;  // the timing-event pool is sized by the next prepare
  return ACKPT_OK;
}

ACKPT_API int ackpt_engine_set_graph(ackpt_engine* e, int32_t on) {
  if (!on) e->drop_graph();
  e->graph = on ? 1 : 0;
  return ACKPT_OK;
}

ACKPT_API int ackpt_engine_set_timeline(ackpt_engine* e, int32_t on) {
  e->timeline = on ? 1 : 0;
  e->prepared = false;  // the event pool and the tier's marks are set by the next prepare
  return ACKPT_OK;
}

ACKPT_API int ackpt_engine_timeline(const ackpt_engine* e, ackpt_timeline_event* out, int64_t cap, int64_t* len) {
  return ackpt::guard([&] {
    if (!e || !len) ackpt::fail(ACKPT_VALUE_ERROR, "engine and len are required");
    *len = int64_t(e->timeline_out.size());
    for (int64_t i = 0; i < std::min(cap, *len); ++i) out[i] = e->timeline_out[size_t(i)];
  });
}

ACKPT_API int ackpt_engine_set_prefetch(ackpt_engine* e, int32_t prefetch) {
  if (e->prefetch != prefetch) e->drop_graph();
  e->prefetch = prefetch;
  return ACKPT_OK;
}

ACKPT_API int ackpt_engine_run(ackpt_engine* e, const void* initial_state, const void* seed,
                               void* adjoint_out, ackpt_stats* stats, void* stream) {
  return ackpt::guard([&] {
    ackpt::run_guarded(e, [&] {
      ackpt::run_impl(e, ackpt::Mode::kFull, initial_state, seed, adjoint_out, nullptr, stats,
                      static_cast<cudaStream_t>(stream));
    });
  });
}

ACKPT_API int ackpt_engine_forward_sweep(ackpt_engine* e, const void* initial_state,
                                         void* final_state, ackpt_stats* stats, void* stream) {
  return ackpt::guard([&] {
    ackpt::run_guarded(e, [&] {
      ackpt::run_impl(e, ackpt::Mode::kForwardSweep, initial_state, nullptr, nullptr, final_state,
                      stats, static_cast<cudaStream_t>(stream));
    });
  });
}

ACKPT_API int ackpt_engine_backward_sweep(ackpt_engine* e, const void* seed, void* adjoint_out,
                                          ackpt_stats* stats, void* stream) {
  return ackpt::guard([&] {
    ackpt::run_guarded(e, [&] {
      ackpt::run_impl(e, ackpt::Mode::kBackwardSweep, nullptr, seed, adjoint_out, nullptr, stats,
                      static_cast<cudaStream_t>(stream));
    });
  });
}

ACKPT_API int ackpt_engine_calibrate(ackpt_engine* E, ackpt_tier* tier, int64_t trials,
                                     const void* initial_state, double* t_a, double* t_b,
                                     double* t_t) {
  return ackpt::guard([&] {
    using namespace ackpt;
    NvtxRange range("calibrate");
    if (trials < 3) fail(ACKPT_VALUE_ERROR, "trial_steps must be >= 3, got " + std::to_string(trials));
    if (!tier) fail(ACKPT_VALUE_ERROR, "calibrate requires a Level-2 backend");
    cudaStream_t s = E->compute;
    const size_t S = size_t(E->S);
    // trials + 2 states, 2 adjoints
    std::vector<void*> st(size_t(trials) + 2, nullptr);
    void* adj[2] = {nullptr, nullptr};
    auto cleanup = [&] {
      for (void* p : st)
        if (p) cudaFree(p);
      for (void* p : adj)
        if (p) cudaFree(p);
    };
    std::vector<cudaEvent_t> evs(size_t(6 * trials));
    for (auto& ev : evs) ACKPT_CUDA_CHECK(cudaEventCreate(&ev));
    try {
      for (auto& p : st) ACKPT_CUDA_CHECK(cudaMalloc(&p, S));
      for (auto& p : adj) ACKPT_CUDA_CHECK(cudaMalloc(&p, S));
      ACKPT_CUDA_CHECK(cudaMemcpyAsync(st[0], initial_state, S, cudaMemcpyDeviceToDevice, s));
      // warm-up forward (runtime.py:438)
      check_op(E->op.forward(E->op.ctx, 0, st[0], st[1], s));
      // trial forwards: states[i] is the input of trial i (runtime.py:440-446)
      std::vector<int64_t> steps(static_cast<size_t>(trials));
      for (int64_t i = 0; i < trials; ++i) {
        steps[size_t(i)] = i % E->n;
        ACKPT_CUDA_CHECK(cudaEventRecord(evs[size_t(2 * i)], s));
        check_op(E->op.forward(E->op.ctx, steps[size_t(i)], st[size_t(i) + 1], st[size_t(i) + 2], s));
        ACKPT_CUDA_CHECK(cudaEventRecord(evs[size_t(2 * i + 1)], s));
      }
      // With fused Advance launches the forward sweep runs at the fused
      // per-step cost; calibrate that instead so stores still hide (I grows).
      // One launch of 64 steps, about the length of the sweep's own Advance
      // launches (one per interval): a 16-step launch carried ~8 % of launch
      // ramp and tail at the C2 shape (16.7 vs 15.5 us/step inside the pass),
      // so I came out short and the sweep stalled on its stores.
      double fused_step = -1.0;
      if (E->fuse && E->op.advance && E->n >= 2) {
        const int64_t len = std::min<int64_t>(E->n, std::max<int64_t>(trials, 64));
        cudaEvent_t f0, f1;
        ACKPT_CUDA_CHECK(cudaEventCreate(&f0));
        ACKPT_CUDA_CHECK(cudaEventCreate(&f1));
        check_op(E->op.advance(E->op.ctx, 0, len, st[1], st[0], s));  // warm-up
        ACKPT_CUDA_CHECK(cudaEventRecord(f0, s));
        check_op(E->op.advance(E->op.ctx, 0, len, st[1], st[0], s));
        ACKPT_CUDA_CHECK(cudaEventRecord(f1, s));
        ACKPT_CUDA_CHECK(cudaEventSynchronize(f1));
        float msv = 0.f;
        ACKPT_CUDA_CHECK(cudaEventElapsedTime(&msv, f0, f1));
        fused_step = double(msv) * 1e-3 / double(len);
        cudaEventDestroy(f0);
        cudaEventDestroy(f1);
      }
      // seed from the last state, then trial backwards in reverse (runtime.py:448-453)
      void* fin = st[size_t(trials) + 1];
      if (E->op.seed) check_op(E->op.seed(E->op.ctx, fin, adj[0], s));
      else ACKPT_CUDA_CHECK(cudaMemsetAsync(adj[0], 0, S, s));
      int ai = 0;
      for (int64_t i = trials - 1, k = 0; i >= 0; --i, ++k) {
        ACKPT_CUDA_CHECK(cudaEventRecord(evs[size_t(2 * trials + 2 * k)], s));
        check_op(E->op.backward(E->op.ctx, steps[size_t(i)], st[size_t(i) + 1], adj[ai], adj[1 - ai], s));
        ACKPT_CUDA_CHECK(cudaEventRecord(evs[size_t(2 * trials + 2 * k + 1)], s));
        ai = 1 - ai;
      }
      // store round trips of the final state under keys 0..trials-1 (runtime.py:455-460);
      // host storage for the keys is allocated first so only the copy is timed
      std::vector<int64_t> keys;
      for (int64_t i = 0; i < trials; ++i) keys.push_back(i);
      tier_reserve_keys(tier, keys, E->S);
      ACKPT_CUDA_CHECK(cudaStreamSynchronize(s));
      cudaStream_t d2h = tier_d2h(tier);
      for (int64_t i = 0; i < trials; ++i) {
        ACKPT_CUDA_CHECK(cudaEventRecord(evs[size_t(4 * trials + 2 * i)], d2h));
        ackpt_ticket tk;
        check_op(ackpt_tier_begin_store(tier, i, i, fin, E->S, nullptr, &tk));
        ACKPT_CUDA_CHECK(cudaEventRecord(evs[size_t(4 * trials + 2 * i + 1)], d2h));
        check_op(ackpt_tier_wait(tier, tk, nullptr));
      }
      ACKPT_CUDA_CHECK(cudaStreamSynchronize(d2h));
      ACKPT_CUDA_CHECK(cudaStreamSynchronize(s));
      auto median = [&](int64_t base) {
        std::vector<double> v;
        for (int64_t i = 0; i < trials; ++i) {
          float msv = 0.f;
          ACKPT_CUDA_CHECK(cudaEventElapsedTime(&msv, evs[size_t(base + 2 * i)], evs[size_t(base + 2 * i + 1)]));
          v.push_back(double(msv) * 1e-3);
        }
        std::sort(v.begin(), v.end());
        const size_t m = v.size();
        return m % 2 ? v[m / 2] : 0.5 * (v[m / 2 - 1] + v[m / 2]);  // statistics.median
      };
      // Per-step cost as the pass sees it: the pace of back-to-back launches
      // with no events in between (a single call timed on an idle GPU is
      // dominated by its launch latency, ~8 us against ~2 us per step inside
      // a pass; the reference's per-call Python timing is its own sequential
      // pace, runtime.py:440-453).  The smaller of the two.
      auto chain = [&](bool fwd) {
        cudaEvent_t c0, c1;
        ACKPT_CUDA_CHECK(cudaEventCreate(&c0));
        ACKPT_CUDA_CHECK(cudaEventCreate(&c1));
        ACKPT_CUDA_CHECK(cudaEventRecord(c0, s));
        int ai2 = 0;
        for (int64_t i = 0; i < trials; ++i) {
          if (fwd) {
            check_op(E->op.forward(E->op.ctx, steps[size_t(i)], st[size_t(i) + 1], st[size_t(i) + 2], s));
          } else {
            check_op(E->op.backward(E->op.ctx, steps[size_t(i)], st[size_t(i) + 1], adj[ai2], adj[1 - ai2], s));
            ai2 = 1 - ai2;
          }
        }
        ACKPT_CUDA_CHECK(cudaEventRecord(c1, s));
        ACKPT_CUDA_CHECK(cudaEventSynchronize(c1));
        float msv = 0.f;
        ACKPT_CUDA_CHECK(cudaEventElapsedTime(&msv, c0, c1));
        cudaEventDestroy(c0);
        cudaEventDestroy(c1);
        return double(msv) * 1e-3 / double(trials);
      };
      *t_a = fused_step > 0 ? fused_step : std::min(chain(true), median(0));
      *t_b = std::min(chain(false), median(2 * trials));
      *t_t = median(4 * trials);
      // Cascade tier: once a plan has more boundaries than DRAM slots, every
      // store also costs one spill to the file stage (running beside the next
      // D2H copy), so the sustained per-boundary time is the slower of the two.
      const double spill = tier_spill_seconds(tier, E->S);
      if (spill > 0) {
        const int64_t I0 = interval_length_exact(*t_t, *t_a);
        if ((E->n + I0 - 1) / I0 > int64_t(tier_dram_slots(tier)) - 2) *t_t = std::max(*t_t, spill);
      }
    } catch (...) {
      cleanup();
      for (auto ev : evs) cudaEventDestroy(ev);
      throw;
    }
    cleanup();
    for (auto ev : evs) cudaEventDestroy(ev);
  });
}

ACKPT_API int64_t ackpt_engine_interval(const ackpt_engine* e) { return e ? e->interval : 0; }

}  // extern "C"
