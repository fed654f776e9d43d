/*
 * ackpt.h — C ABI of the B200-native asynchronous multistage checkpointing
 * hot path (arXiv 1806.01117).  Every entry point returns an int status
 * (ACKPT_OK == 0) and never throws across the boundary; the message of the
 * last failure on the calling thread is ackpt_last_error().
 *
 * Reference interfaces replaced (paths relative to the reference package
 * root pkg/src/asyncckpt/):
 *   status codes            errors.py:4-37  (one code per exception class)
 *   ackpt_forward_cost      schedule.py:161-169   forward_cost(n, s)
 *   ackpt_revolve_schedule  schedule.py:188-235   revolve_schedule(ScheduleParams)
 *   ackpt_taped_schedule    schedule.py:279-285   taped_schedule(length)
 *   ackpt_best_split        schedule.py:177-181   _best_split(length, slots, table)
 *   ackpt_interval_length   perfmodel.py:56-64    interval_length(t_t, t_a)
 *   ackpt_lstm_*            lstm.py:110-163       _gates / lstm_forward_step /
 *                                                 lstm_backward_step / loss /
 *                                                 loss_gradient_seed
 *   ackpt_tier_*            storage.py:181-278    TransferTicket + Level2Backend
 *                                                 (begin_store/begin_fetch/wait/poll/contains/close)
 *   ackpt_engine_*          runtime.py:162-381    _Execution / execute / calibrate
 *   ackpt_crc32c            storage.py:49-68      crc32c(data, crc)
 *
 * Memory ownership: device buffers passed in are owned by the caller (torch);
 * the engine owns its checkpoint buffer pool (HBM), the tier owns its pinned
 * host slab.  Streams are plain cudaStream_t handles passed as void*.
 */
#ifndef ACKPT_H_
#define ACKPT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define ACKPT_API __attribute__((visibility("default")))
#else
#define ACKPT_API
#endif

/* ---- status codes: 1..8 mirror errors.py:8-37 in declaration order ---- */
enum {
  ACKPT_OK = 0,
  ACKPT_INFEASIBLE_SCHEDULE = 1, /* errors.py:8  InfeasibleSchedule */
  ACKPT_SIZE_MISMATCH = 2,       /* errors.py:12 SizeMismatch */
  ACKPT_SLOT_OUT_OF_RANGE = 3,   /* errors.py:16 SlotOutOfRange */
  ACKPT_SLOT_UNWRITTEN = 4,      /* errors.py:20 SlotUnwritten */
  ACKPT_MISSING_KEY = 5,         /* errors.py:24 MissingKey */
  ACKPT_CHECKSUM_MISMATCH = 6,   /* errors.py:28 ChecksumMismatch */
  ACKPT_STORAGE_FULL = 7,        /* errors.py:32 StorageFull */
  ACKPT_EXECUTION_ERROR = 8,     /* errors.py:36 ExecutionError */
  ACKPT_VALUE_ERROR = 9,         /* ValueError raised by argument checks */
  ACKPT_CUDA_ERROR = 10,         /* any cudaError_t (reported as ExecutionError) */
  ACKPT_NOT_READY = 11           /* ackpt_tier_poll: transfer still in flight */
};

ACKPT_API const char* ackpt_last_error(void);
ACKPT_API const char* ackpt_version(void);

/* ---- schedule actions (schedule.py:70-114) ---- */
enum {
  ACKPT_ADVANCE = 0, /* a=from_step b=to_step   schedule.py:70  */
  ACKPT_SAVE = 1,    /* a=step      b=slot      schedule.py:78  */
  ACKPT_LOAD = 2,    /* a=slot                  schedule.py:86  */
  ACKPT_TAPE = 3,    /* a=from_step b=to_step   schedule.py:93  */
  ACKPT_REVERSE = 4, /* a=step                  schedule.py:102 */
  ACKPT_DONE = 5     /*                         schedule.py:109 */
};

typedef struct ackpt_action {
  int32_t op;
  int32_t reserved;
  int64_t a;
  int64_t b;
} ackpt_action;

/* Host scheduler.  Tables are built once and cached per process (grow-only,
 * like schedule.py:121-136); values and tie-breaks are bit-exact. */
ACKPT_API int ackpt_forward_cost(int64_t n, int64_t s, int64_t* out);
ACKPT_API int ackpt_best_split(int64_t length, int64_t slots, int64_t* out);
/* Writes up to cap actions (Done included); *len receives the full count, so
 * a call with cap=0 sizes the buffer.  Fails with INFEASIBLE_SCHEDULE/VALUE_ERROR
 * exactly where ScheduleParams.__post_init__ (schedule.py:59-66) raises. */
ACKPT_API int ackpt_revolve_schedule(int64_t n, int64_t s, ackpt_action* out, int64_t cap,
                                     int64_t* len);
ACKPT_API int ackpt_taped_schedule(int64_t length, ackpt_action* out, int64_t cap, int64_t* len);
/* Exact ceil(Fraction(t_t)/Fraction(t_a)), at least 1 (perfmodel.py:56-64). */
ACKPT_API int ackpt_interval_length(double t_t, double t_a, int64_t* out);
/* Threads used by the cost-table build (0 = all hardware threads). */
ACKPT_API int ackpt_set_schedule_threads(int32_t threads);

/* ---- LSTM cell operator on device (lstm.py:39-173, batched) ----
 * State layout in HBM, dtype T (f32 or f64): [h(d, B); c(d, B)] with the batch
 * index fastest, i.e. element (part, j, b) at ((part*d + j)*B + b).  At B=1
 * this is exactly the reference's byte image [h(d), c(d)] (lstm.py:99-107). */
enum { ACKPT_F32 = 0, ACKPT_F64 = 1 };

typedef struct ackpt_lstm ackpt_lstm;

/* Weights are given in float64 exactly as LstmCell holds them
 * (w_*: d x 2d row-major, b_*: d, xs: n x d, target: d) and are rounded to
 * the cell dtype once; the per-step input projection W_x x_k + b is
 * precomputed in float64 and then rounded. */
ACKPT_API int ackpt_lstm_create(int32_t d, int64_t n_steps, int64_t batch, int32_t dtype,
                                const double* w_f, const double* w_i, const double* w_o,
                                const double* w_c, const double* b_f, const double* b_i,
                                const double* b_o, const double* b_c, const double* xs,
                                const double* target, ackpt_lstm** out);
ACKPT_API int ackpt_lstm_destroy(ackpt_lstm* cell);
ACKPT_API int64_t ackpt_lstm_state_bytes(const ackpt_lstm* cell);
/* One forward step k: state_k -> state_{k+1} (lstm.py:123-129). */
ACKPT_API int ackpt_lstm_forward(const ackpt_lstm* cell, int64_t step, const void* state_in,
                                 void* state_out, void* stream);
/* Fused run of steps [from, to): one launch, state kept in registers. */
ACKPT_API int ackpt_lstm_advance(const ackpt_lstm* cell, int64_t from_step, int64_t to_step,
                                 const void* state_in, void* state_out, void* stream);
/* Fused TapeForward: count (<= 64) steps from from_step, every output kept. */
ACKPT_API int ackpt_lstm_forward_many(const ackpt_lstm* cell, int64_t from_step, int64_t count,
                                      const void* state_in, void* const* states_out, void* stream);
/* Fused Reverse run: steps from+count-1 .. from, adjoint in registers. */
ACKPT_API int ackpt_lstm_backward_many(const ackpt_lstm* cell, int64_t from_step, int64_t count,
                                       const void* const* states, const void* adjoint_in,
                                       void* adjoint_out, void* stream);
/* One adjoint step k (lstm.py:132-152). */
ACKPT_API int ackpt_lstm_backward(const ackpt_lstm* cell, int64_t step, const void* state,
                                  const void* adjoint_in, void* adjoint_out, void* stream);
/* seed = [2(h - target), 0] (lstm.py:161-163). */
ACKPT_API int ackpt_lstm_seed(const ackpt_lstm* cell, const void* final_state, void* adjoint_out,
                              void* stream);
/* Per-sequence loss sum_j (h_j - target_j)^2 (lstm.py:155-158), B values of dtype T. */
ACKPT_API int ackpt_lstm_loss(const ackpt_lstm* cell, const void* final_state, void* loss_out,
                              void* stream);

/* ---- generic operator plugin (runtime.py:62-87 OperatorPair) ----
 * The engine calls these on its compute stream; device pointers only. */
typedef int (*ackpt_forward_fn)(void* ctx, int64_t step, const void* state_in, void* state_out,
                                void* stream);
typedef int (*ackpt_backward_fn)(void* ctx, int64_t step, const void* state,
                                 const void* adjoint_in, void* adjoint_out, void* stream);
typedef int (*ackpt_seed_fn)(void* ctx, const void* final_state, void* adjoint_out, void* stream);
/* Optional: fused forward over [from, to); NULL means per-step forward. */
typedef int (*ackpt_advance_fn)(void* ctx, int64_t from_step, int64_t to_step,
                                const void* state_in, void* state_out, void* stream);

/* Optional temporal fusion of a TapeForward run: steps [from, from+count),
 * writing the state after each step to states_out[i] (count <= 64). */
typedef int (*ackpt_forward_many_fn)(void* ctx, int64_t from_step, int64_t count,
                                     const void* state_in, void* const* states_out, void* stream);
/* Optional temporal fusion of a run of Reverse actions: steps
 * from+count-1 down to from, states[i] = state of step from+i, the adjoint
 * kept on chip in between (count <= 64). */
typedef int (*ackpt_backward_many_fn)(void* ctx, int64_t from_step, int64_t count,
                                      const void* const* states, const void* adjoint_in,
                                      void* adjoint_out, void* stream);

typedef struct ackpt_operator {
  void* ctx;
  ackpt_forward_fn forward;
  ackpt_backward_fn backward;
  ackpt_seed_fn seed; /* NULL: the adjoint seed is given to ackpt_engine_run */
  ackpt_advance_fn advance;
  int64_t state_bytes; /* OperatorPair.state_size */
  int64_t n_steps;     /* OperatorPair.n_steps */
  ackpt_forward_many_fn forward_many;   /* NULL: per-step forward */
  ackpt_backward_many_fn backward_many; /* NULL: per-step backward */
} ackpt_operator;

#define ACKPT_MAX_FUSED 64

/* Fills *out with the built-in LSTM operator bound to cell. */
ACKPT_API int ackpt_lstm_operator(ackpt_lstm* cell, ackpt_operator* out);

/* Kernel family of the fused d=8 fp32 launches (advance / forward_many /
 * backward_many): 0 = packed FFMA2, 1 = tcgen05 tensor cores with the
 * 3xTF32 split (default), 2 = mixed (tcgen05 advance / forward_many, FFMA2
 * backward_many), 3 = mma (warp-level mma.sync, register fragments, 3xTF32).  Families differ in rounding (all within the fp32
 * tolerance); switch only between executions.  Env ACKPT_TC=0/1/2 presets. */
ACKPT_API int ackpt_set_fused_family(int32_t family);
ACKPT_API int32_t ackpt_get_fused_family(void);

/* Latency injection (test support, pkg/tests/test_runtime.py:33-52 pad_operators):
 * *out wraps base so each forward / backward call first holds the stream for
 * the given seconds with a device-side delay kernel.  Release with
 * ackpt_pad_operator_destroy(out). */
ACKPT_API int ackpt_pad_operator_create(const ackpt_operator* base, double forward_seconds,
                                        double backward_seconds, ackpt_operator* out);
ACKPT_API int ackpt_pad_operator_destroy(ackpt_operator* op);

/* ---- Level-2 tier: HBM <-> pinned host DRAM (storage.py:181-278) ---- */
typedef struct ackpt_tier ackpt_tier;
typedef int64_t ackpt_ticket;

/* capacity: number of keys the pinned slab can hold; slot_bytes: bytes per key.
 * The slab is allocated here (outside any timed window). */
ACKPT_API int ackpt_tier_create(int64_t capacity, int64_t slot_bytes, ackpt_tier** out);
/* File (NVMe) stage, FileBackend (storage.py:321-340): every key is a file
 * <directory>/ckpt_<key>.bin in the reference's CKPT format (magic, u16
 * version, u64 step, u64 length, payload, u32 CRC32C; tmp + rename), moved
 * HBM <-> pinned staging <-> file on the copy streams.  Corrupt / truncated
 * files -> CHECKSUM_MISMATCH, ENOSPC -> STORAGE_FULL, absent -> MISSING_KEY,
 * reported at wait (or at the end of an engine run).  Files already present
 * in the directory can be fetched (resume). */
ACKPT_API int ackpt_tier_create_file(const char* directory, int64_t slot_bytes, ackpt_tier** out);
/* Three-stage tier (BASELINE config 5): HBM -> pinned
 * host DRAM (dram_slots slots of slot_bytes) -> CKPT files in `directory`
 * (same byte format as ackpt_tier_create_file).  Recent boundaries stay in
 * DRAM; older ones are spilled by an I/O thread (CRC32C, O_DIRECT, atomic
 * publish) and read back (O_DIRECT, verified) ahead of their fetch.  No
 * CUDA-graph capture.  Replaces FileBackend behind a pinned cache
 * (storage.py:321-340) where the host RAM cannot hold every boundary. */
ACKPT_API int ackpt_tier_create_cascade(const char* directory, int64_t slot_bytes, int32_t dram_slots,
                                        ackpt_tier** out);
typedef struct ackpt_cascade_stats {
    int64_t dram_slots;
    int64_t spills, spill_bytes;  /* completed DRAM -> file spills */
    double spill_seconds;         /* host time in the spill thread (CRC + write + publish) */
    int64_t reads, read_bytes;    /* completed file -> DRAM reads */
    double read_seconds;
    int64_t dram_hits;            /* fetches served from a DRAM slot */
    int64_t ring_hits;            /* fetches of spilled keys already read ahead */
    int64_t ring_misses;          /* fetches of spilled keys read on demand */
} ackpt_cascade_stats;
ACKPT_API int ackpt_tier_cascade_stats(ackpt_tier* tier, ackpt_cascade_stats* out);
ACKPT_API int ackpt_tier_destroy(ackpt_tier* tier);
/* Stall injection for contention tests: each transfer holds its copy stream
 * for at least latency_us + bytes / bandwidth (bandwidth <= 0: no limit),
 * like SimulatedBackend.transfer_seconds (storage.py:300-301). */
ACKPT_API int ackpt_tier_set_throttle(ackpt_tier* tier, double latency_s, double bandwidth);
/* Store bytes at device pointer src under key; the copy starts after all work
 * already enqueued on after_stream (may be NULL). */
ACKPT_API int ackpt_tier_begin_store(ackpt_tier* tier, int64_t key, int64_t step,
                                     const void* src, int64_t bytes, void* after_stream,
                                     ackpt_ticket* out);
/* Fetch key into device pointer dst; a missing key is reported at wait
 * (storage.py:310-311 raises inside the worker, surfaced by wait). */
ACKPT_API int ackpt_tier_begin_fetch(ackpt_tier* tier, int64_t key, void* dst, int64_t bytes,
                                     void* after_stream, ackpt_ticket* out);
/* Blocks the host; idempotent.  *step_out (may be NULL) receives the stored
 * step.  A waited ticket's slot is recycled: waiting on it again returns the
 * first wait's status and leaves *step_out unchanged.  The source of a store
 * must not be modified, and the destination of a fetch not read, before the
 * ticket completed (both are read / written by the copy engines). */
ACKPT_API int ackpt_tier_wait(ackpt_tier* tier, ackpt_ticket ticket, int64_t* step_out);
/* The tier's copy streams (cudaStream_t): stores run on *d2h, fetches on
 * *h2d -- for callers that tie buffer lifetimes to them (record_stream). */
ACKPT_API int ackpt_tier_streams(ackpt_tier* tier, void** d2h, void** h2d);
/* Makes stream wait for the ticket on the device (no host block). */
ACKPT_API int ackpt_tier_stream_wait(ackpt_tier* tier, ackpt_ticket ticket, void* stream);
/* ACKPT_OK when complete, ACKPT_NOT_READY while in flight. */
ACKPT_API int ackpt_tier_poll(ackpt_tier* tier, ackpt_ticket ticket);
ACKPT_API int ackpt_tier_contains(ackpt_tier* tier, int64_t key, int32_t* out);
/* Byte length stored under key (MISSING_KEY if absent). */
ACKPT_API int ackpt_tier_key_bytes(ackpt_tier* tier, int64_t key, int64_t* out);
/* Host-visible pointer of a stored key's bytes (pinned), for tests / file stage. */
ACKPT_API int ackpt_tier_host_ptr(ackpt_tier* tier, int64_t key, void** out);
ACKPT_API int ackpt_tier_clear(ackpt_tier* tier);

/* ---- executor (runtime.py:90-381) ---- */
enum { ACKPT_FULL_STORAGE = 0, ACKPT_REVOLVE = 1, ACKPT_MULTISTAGE = 2 };

typedef struct ackpt_stats {
  /* ExecutionStats fields, same meaning (runtime.py:90-98) */
  int64_t forward_evals;
  int64_t backward_evals;
  int64_t stores_issued;
  int64_t prefetches_issued;
  double stall_seconds;
  int64_t peak_l1_bytes;
  double wall_seconds;
  /* B200 extras */
  double gpu_seconds;       /* compute-stream event time, first to last action */
  int64_t kernel_launches;  /* kernels this run enqueued */
  int64_t interval;         /* multistage I actually used (0 otherwise) */
  int64_t fallback;         /* 1 if multistage fell back to plain revolve */
  int64_t device_buffers;   /* HBM state buffers held by the pool */
  int64_t link_bytes;       /* bytes moved over the host link */
  int64_t fused_advances;   /* Advance actions run as one fused launch */
  /* sampled kernel timing (ackpt_engine_set_kernel_sampling): CUDA-event
   * durations of every k-th forward / backward launch inside the run */
  double fwd_sample_seconds;
  int64_t fwd_samples;
  double bwd_sample_seconds;
  int64_t bwd_samples;
  double host_enqueue_seconds; /* host time to enqueue the whole run */
} ackpt_stats;

typedef struct ackpt_engine ackpt_engine;

ACKPT_API int ackpt_engine_create(const ackpt_operator* op, ackpt_engine** out);
ACKPT_API int ackpt_engine_destroy(ackpt_engine* engine);
/* Plans the strategy (and sizes/allocates the HBM buffer pool) outside the
 * timed window, like execute() does before t0 (runtime.py:355-362).
 * MULTISTAGE needs interval >= 1: run ackpt_engine_calibrate + ackpt_interval_length
 * first for the reference's interval=None (runtime.py:325-336). */
ACKPT_API int ackpt_engine_prepare(ackpt_engine* engine, int32_t strategy, int64_t slots,
                                   int64_t interval, ackpt_tier* tier);
/* 0 (default): the reference's per-step operator contract, one launch per
 * forward step.  1: run whole Advance actions as one fused launch when the
 * operator provides advance(); counters are unchanged. */
ACKPT_API int ackpt_engine_set_fusion(ackpt_engine* engine, int32_t fuse_advance);
/* Time every k-th forward and backward launch with a CUDA event pair on the
 * compute stream (0 = off).  Takes effect at the next prepare. */
ACKPT_API int ackpt_engine_set_kernel_sampling(ackpt_engine* engine, int64_t every);
/* CUDA-graph mode (default off): ackpt_engine_run captures a pass into a CUDA
 * graph on the second run with the same buffers (the first runs eagerly and
 * performs every first-use allocation) and replays it with one launch while
 * the plan, fusion, prefetch order and buffers stay the same.  Counters come
 * from the captured pass; times from its event nodes.  Not with the timeline
 * or kernel sampling on.  For launch-bound passes (per-step contract, small
 * states). */
ACKPT_API int ackpt_engine_set_graph(ackpt_engine* engine, int32_t on);
/* Mirrors CKPT_DISABLE_PREFETCH=1 (runtime.py:302): -1 read the env var at run. */
ACKPT_API int ackpt_engine_set_prefetch(ackpt_engine* engine, int32_t prefetch);
/* One forward/backward pass (runtime.py:339-381).  seed may be NULL when the
 * operator has a seed function.  Blocks until the adjoint is ready. */
ACKPT_API int ackpt_engine_run(ackpt_engine* engine, const void* initial_state,
                               const void* seed, void* adjoint_out, ackpt_stats* stats,
                               void* stream);
/* Multistage sweeps over an already prepared, non-fallback plan
 * (runtime.py:384-417).  The forward sweep writes the final state. */
ACKPT_API int ackpt_engine_forward_sweep(ackpt_engine* engine, const void* initial_state,
                                         void* final_state, ackpt_stats* stats, void* stream);
ACKPT_API int ackpt_engine_backward_sweep(ackpt_engine* engine, const void* seed,
                                          void* adjoint_out, ackpt_stats* stats, void* stream);
/* Median per-op times (t_a, t_b, t_t) over trial_steps (runtime.py:420-466);
 * stores overwrite keys 0..trial_steps-1 of the tier. */
ACKPT_API int ackpt_engine_calibrate(ackpt_engine* engine, ackpt_tier* tier, int64_t trial_steps,
                                     const void* initial_state, double* t_a, double* t_b,
                                     double* t_t);
/* Interval the last prepare chose. */
ACKPT_API int64_t ackpt_engine_interval(const ackpt_engine* engine);

/* ---- measured timeline (reporting parity with simulator.py:55-66) ----------
 * With the timeline on, a run records every compute launch (per-step or
 * fused, so one event may span several steps), every stall (compute-stream
 * wait on a transfer, from/to = the step it happened at) and every transfer
 * (copy-stream marks around the copy, plus file I/O for the file stage),
 * in seconds since the run's start event.  Events come sorted by start. */
enum {
  ACKPT_EV_FORWARD = 0, /* "forward_compute" */
  ACKPT_EV_BACKWARD = 1, /* "backward_compute" */
  ACKPT_EV_STORE = 2,
  ACKPT_EV_FETCH = 3,
  ACKPT_EV_STALL = 4
};
enum { ACKPT_LANE_COMPUTE = 0, ACKPT_LANE_TRANSFER = 1 };
typedef struct ackpt_timeline_event {
  int32_t kind;
  int32_t lane;
  int64_t from_step;
  int64_t to_step;
  double start;
  double end;
} ackpt_timeline_event;
/* Takes effect at the next prepare (adds two events per launch: a reporting
 * mode, not for headline timing). */
ACKPT_API int ackpt_engine_set_timeline(ackpt_engine* engine, int32_t on);
/* Events of the last run: *len = count; the first min(cap, count) are copied. */
ACKPT_API int ackpt_engine_timeline(const ackpt_engine* engine, ackpt_timeline_event* out, int64_t cap,
                                    int64_t* len);

/* ---- launch chain of the tensor-core kernels (no reference counterpart) ----
 * Host-only self-test of the chain bookkeeping (which launch may chain to
 * which: same cell, same stream, adjacent, equal tilings, marked); 0 = pass,
 * else ACKPT_EXECUTION_ERROR with the failing case in ackpt_last_error(). */
ACKPT_API int ackpt_chain_selftest(void);

/* ---- CRC32C (storage.py:49-68), hardware crc32 instruction when present ---- */
ACKPT_API uint32_t ackpt_crc32c(const void* data, int64_t len, uint32_t crc);

#ifdef __cplusplus
}
#endif
#endif /* ACKPT_H_ */
