// Internal helpers shared by the native translation units of libackpt.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ackpt.h"

namespace ackpt {

// Typed failure carrying one of the ACKPT_* status codes.  Thrown inside the
// library and converted to a status at every extern "C" boundary.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& msg) : std::runtime_error(msg), code(c) {}
};

void set_last_error(const std::string& msg);

// Set by the executor around a step launch that directly follows another
// step launch of the same operator on the same stream, with nothing else
// enqueued in between (engine.cpp).  The native LSTM operator's callbacks
// pass it on as g_chain_native for the duration of the call, and only then
// may the cell chain the two launches (chain.cuh) -- an operator written in
// Python that calls the cell's public API never chains (its temporaries come
// from an allocator that may hand a buffer a running launch still reads to
// the next one).  0 everywhere else.
extern thread_local int g_chain_hint;
extern thread_local int g_chain_native;

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

// Runs fn and converts any exception into a status code + last-error string.
template <class F>
int guard(F&& fn) {
  try {
    fn();
    return ACKPT_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("out of host memory");
    return ACKPT_STORAGE_FULL;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return ACKPT_EXECUTION_ERROR;
  } catch (...) {
    set_last_error("unknown native failure");
    return ACKPT_EXECUTION_ERROR;
  }
}

// Scheduler internals used by the executor (schedule.cpp).
struct Action {
  int32_t op;
  int64_t a;
  int64_t b;
};

void revolve_actions(int64_t n, int64_t s, std::vector<Action>& out);
void taped_actions(int64_t length, std::vector<Action>& out);
int64_t forward_cost_exact(int64_t n, int64_t s);
int64_t interval_length_exact(double t_t, double t_a);
// slot_read_liveness (schedule.py:347-362): for each action index holding a
// Save, the index of the last Load reading that write, or -1.
void slot_read_liveness(const std::vector<Action>& actions, std::vector<int64_t>& last_read);

// CRC32C helpers (crc32c.cpp).  raw = unconditioned register (no xor in/out).
uint32_t crc32c_raw(const void* data, int64_t len, uint32_t reg);
uint32_t crc32c_shift(uint32_t reg, int64_t len);  // as if len zero bytes followed
uint32_t crc32c_parallel(const void* data, int64_t len, uint32_t crc, int threads);
int io_threads(int64_t len);  // worker threads for a len-byte host I/O job

}  // namespace ackpt

#define ACKPT_CUDA_CHECK(expr)                                                        \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess)                                                            \
      ::ackpt::fail(ACKPT_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)
