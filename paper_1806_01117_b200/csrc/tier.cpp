// Level-2 tier: asynchronous HBM <-> pinned host DRAM checkpoint store.
//
// Replaces the reference's Level2Backend + TransferTicket (storage.py:181-278):
// the FIFO queue and worker thread become two copy-engine streams (one D2H for
// stores, one H2D for fetches) and each TransferTicket becomes a CUDA event.
// The reference's FIFO guarantees ("a fetch enqueued after a store of the same
// key always sees the stored bytes", storage.py:4-6) are kept per key: a
// fetch waits for the key's last store event, and a store into a key waits
// for the key's last fetch event before overwriting the host bytes.
// Worker exceptions surfaced at wait() (storage.py:271-278) map to a ticket
// status returned by ackpt_tier_wait (MissingKey, StorageFull, SizeMismatch).
#include <cuda.h>
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "common.h"
#include "nvtx.h"

namespace ackpt {

// Status written by a host function on a copy stream (file I/O); read after
// the ticket's event completed, which orders it after the host function.
struct AsyncStatus {
  std::atomic<int> err{ACKPT_OK};
  std::string msg;
};

struct TierTicket {
  cudaEvent_t done = nullptr;
  int kind = 0;  // 0 store, 1 fetch
  int64_t key = 0;
  int64_t step = 0;
  int err = ACKPT_OK;
  std::string msg;
  bool complete = false;
  double hold_seconds = 0.0;  // throttle: host-func sleep on the copy stream
  cudaEvent_t t0 = nullptr, t1 = nullptr;  // timeline marks (copy start / done)
  bool waited = false;    // waited / retired by its owner: the slot may be recycled
  bool captured = false;  // enqueued under CUDA-graph capture: a graph node refers to it
  // file stage
  std::shared_ptr<AsyncStatus> async;
  ackpt_tier* tier = nullptr;
  int64_t len = 0;
};

// One file-stage transfer handed to a tier I/O thread (stream-memop path).
struct IoJob {
  TierTicket* tk = nullptr;
  uint32_t seq = 0;   // store / fetch sequence number (1, 2, ...)
  uint32_t need = 0;  // store: fetch seq that must have read the old file; fetch: store seq that wrote it
};

struct KeyEntry {
  int64_t slot = -1;
  unsigned char* big = nullptr;  // dedicated pinned buffer for payloads > slot_bytes
  int64_t big_cap = 0;
  int64_t step = 0;
  int64_t len = 0;
  cudaEvent_t last_store = nullptr;
  cudaEvent_t last_fetch = nullptr;
  bool stored = false, fetched = false;
  uint32_t file_store_seq = 0;  // last I/O-thread store of this key (0: none)
  uint32_t file_fetch_seq = 0;  // last I/O-thread fetch of this key
};

struct Cascade;

}  // namespace ackpt

struct ackpt_tier {
  int64_t capacity = 0;  // max keys (0 = bounded by host memory only)
  int64_t slot_bytes = 0;
  std::vector<unsigned char*> chunks;  // cudaHostAlloc'd
  std::vector<unsigned char*> slot_ptr;
  std::vector<int64_t> free_slots;
  std::unordered_map<int64_t, ackpt::KeyEntry> keys;
  // Tickets by id (ids increase; node-based map, so references stay valid).
  // Waited, uncaptured tickets are erased (compact_tickets), so a long-lived
  // backend holds O(in-flight) tickets; a recycled ticket that failed keeps
  // its error for a repeated wait (recycled_errors).
  std::unordered_map<int64_t, ackpt::TierTicket> tickets;
  int64_t next_ticket = 0;
  std::unordered_map<int64_t, std::pair<int, std::string>> recycled_errors;
  std::vector<cudaEvent_t> event_pool;
  std::vector<cudaEvent_t> all_events;
  bool timing = false;                   // record timeline marks around transfers
  std::vector<cudaEvent_t> timing_pool;  // timing-enabled events (in all_events too)
  cudaStream_t d2h = nullptr, h2d = nullptr;
  cudaEvent_t after = nullptr;
  double latency_s = 0.0, bandwidth = 0.0;
  std::mutex mu;
  // File (NVMe) stage: keys live in CKPT files under `dir`; transfers stage
  // through one pinned buffer per direction (stream FIFO orders their reuse).
  bool file_mode = false;
  std::string dir;
  unsigned char* stage_out = nullptr;
  unsigned char* stage_in = nullptr;
  int64_t stage_cap = 0;
  // File-stage I/O threads.  A store's D2H copy lands in stage_out and the
  // GPU bumps flag kCopied; the store thread then writes the CKPT file and
  // bumps kWritten, which the D2H stream waits on (stream memory operations)
  // before the ticket's event and the next store's copy.  A fetch's file is
  // read into stage_in by the fetch thread as soon as its store is written
  // and the previous fetch's H2D copy consumed stage_in (kConsumed); the H2D
  // stream waits on kStaged before copying.  A host function on the stream
  // would cost ~60-260 us of callback latency per transfer on the box; a
  // stream wait on a host-written flag ~10 us.  Under CUDA-graph capture the
  // host-function path is used (the threads are fed at enqueue time).
  CUresult (*wait_value)(CUstream, CUdeviceptr, cuuint32_t, unsigned) = nullptr;
  CUresult (*write_value)(CUstream, CUdeviceptr, cuuint32_t, unsigned) = nullptr;
  uint32_t* flags = nullptr;  // pinned + mapped, one 64-byte line per flag
  uint32_t store_seq = 0, fetch_seq = 0;  // issued (under mu)
  std::mutex qmu;
  std::condition_variable qcv;
  std::deque<ackpt::IoJob> store_q, fetch_q;
  int busy = 0;  // jobs popped and not finished
  bool stop = false;
  std::atomic<bool> abort{false};  // destroy: stop waiting on flags a failed stream never bumps
  std::thread store_thr, fetch_thr;
  // Three-stage cascade (cascade_impl.h): pinned DRAM slots backed by CKPT
  // files; null for the pinned and file tiers.
  ackpt::Cascade* cascade = nullptr;
  int cascade_slots = 0;
};

namespace ackpt {
// cascade_impl.h (same translation unit)
void cascade_create(ackpt_tier* t, int dram_slots);
void cascade_destroy(ackpt_tier* t);
void cascade_quiesce(ackpt_tier* t);
ackpt_ticket cascade_begin_store(ackpt_tier* t, int64_t key, int64_t step, const void* src, int64_t bytes,
                                 void* after_stream);
ackpt_ticket cascade_begin_fetch(ackpt_tier* t, int64_t key, void* dst, int64_t bytes, void* after_stream);
bool cascade_contains(ackpt_tier* t, int64_t key);
int64_t cascade_key_bytes(ackpt_tier* t, int64_t key);
void* cascade_host_ptr(ackpt_tier* t, int64_t key);
void cascade_clear(ackpt_tier* t);
double cascade_spill_probe(ackpt_tier* t, int64_t bytes);
}  // namespace ackpt

namespace ackpt {
enum Flag { kCopied = 0, kWritten = 16, kConsumed = 32, kStaged = 48 };
}

namespace ackpt {
namespace {

cudaEvent_t new_event(ackpt_tier* t) {
  if (!t->event_pool.empty()) {
    cudaEvent_t e = t->event_pool.back();
    t->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  ACKPT_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  t->all_events.push_back(e);
  return e;
}

// Timeline mark on a copy stream (nullptr unless the engine asked for a timeline).
cudaEvent_t mark(ackpt_tier* t, cudaStream_t s) {
  if (!t->timing) return nullptr;
  cudaEvent_t e;
  if (!t->timing_pool.empty()) {
    e = t->timing_pool.back();
    t->timing_pool.pop_back();
  } else {
    ACKPT_CUDA_CHECK(cudaEventCreate(&e));
    t->all_events.push_back(e);
  }
  ACKPT_CUDA_CHECK(cudaEventRecord(e, s));
  return e;
}

void CUDART_CB hold_stream(void* arg) {
  const double s = *static_cast<const double*>(arg);
  if (s > 0) std::this_thread::sleep_for(std::chrono::duration<double>(s));
}

void reserve_slots(ackpt_tier* t, int64_t count) {
  int64_t have = int64_t(t->slot_ptr.size());
  if (count <= have) return;
  if (t->capacity > 0 && count > t->capacity)
    fail(ACKPT_STORAGE_FULL, "tier capacity " + std::to_string(t->capacity) + " keys exceeded");
  const int64_t add = count - have;
  unsigned char* chunk = nullptr;
  cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&chunk), size_t(add) * size_t(t->slot_bytes),
                                cudaHostAllocDefault);
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(ACKPT_STORAGE_FULL, std::string("pinned host allocation failed: ") + cudaGetErrorString(e));
  }
  t->chunks.push_back(chunk);
  for (int64_t i = 0; i < add; ++i) {
    t->slot_ptr.push_back(chunk + size_t(i) * size_t(t->slot_bytes));
    t->free_slots.push_back(have + i);
  }
}

// Erase waited tickets (their events went back to the pool at retire; no I/O
// job or graph node refers to them any more).
void compact_tickets(ackpt_tier* t) {
  for (auto it = t->tickets.begin(); it != t->tickets.end();) {
    TierTicket& f = it->second;
    if (!f.complete || !f.waited || f.captured) {
      ++it;
      continue;
    }
    int code = f.err;
    std::string msg = f.msg;
    if (code == ACKPT_OK && f.async) {
      code = f.async->err.load(std::memory_order_acquire);
      msg = f.async->msg;
    }
    if (code != ACKPT_OK) t->recycled_errors[it->first] = {code, msg};
    it = t->tickets.erase(it);
  }
}

ackpt_ticket add_ticket(ackpt_tier* t, TierTicket&& tk) {
  static constexpr size_t kCompactAt = 256;
  if (t->tickets.size() >= kCompactAt && t->next_ticket % kCompactAt == 0) compact_tickets(t);
  const int64_t id = t->next_ticket++;
  t->tickets.emplace(id, std::move(tk));
  return ackpt_ticket(id);
}

// nullptr: a recycled ticket (waited before); see recycled_status.
TierTicket* find_ticket(ackpt_tier* t, ackpt_ticket id) {
  if (id < 0 || id >= t->next_ticket) fail(ACKPT_VALUE_ERROR, "unknown transfer ticket");
  auto it = t->tickets.find(id);
  return it == t->tickets.end() ? nullptr : &it->second;
}
int recycled_status(const ackpt_tier* t, ackpt_ticket id, std::string* msg) {
  auto it = t->recycled_errors.find(id);
  if (it == t->recycled_errors.end()) return ACKPT_OK;
  if (msg) *msg = it->second.second;
  return it->second.first;
}

void hold(ackpt_tier* t, cudaStream_t s, TierTicket& tk, int64_t bytes) {
  double secs = t->latency_s + (t->bandwidth > 0 ? double(bytes) / t->bandwidth : 0.0);
  if (secs <= 0) return;
  tk.hold_seconds = secs;
  ACKPT_CUDA_CHECK(cudaLaunchHostFunc(s, hold_stream, &tk.hold_seconds));
}

void retire(ackpt_tier* t, TierTicket& tk) {
  if (tk.complete) return;
  tk.complete = true;
  if (tk.done) {
    t->event_pool.push_back(tk.done);
    tk.done = nullptr;
  }
  for (cudaEvent_t* e : {&tk.t0, &tk.t1})
    if (*e) {
      t->timing_pool.push_back(*e);
      *e = nullptr;
    }
}

// ---- file stage: CKPT format (storage.py:9-18, 83-127) ----------------------
// magic "CKPT" | u16 version=1 | u64 step | u64 length | payload | u32 crc32c(header+payload)
constexpr int kHeader = 22, kTrailer = 4;

std::string ckpt_path(const ackpt_tier* t, int64_t key) {
  return t->dir + "/ckpt_" + std::to_string(key) + ".bin";
}

void put_le(unsigned char* p, uint64_t v, int bytes) {
  for (int i = 0; i < bytes; ++i) p[i] = (unsigned char)(v >> (8 * i));
}
uint64_t get_le(const unsigned char* p, int bytes) {
  uint64_t v = 0;
  for (int i = 0; i < bytes; ++i) v |= uint64_t(p[i]) << (8 * i);
  return v;
}

void set_async(AsyncStatus& st, int code, const std::string& msg) {
  st.msg = msg;
  st.err.store(code, std::memory_order_release);
}

// Payload I/O split over worker threads: slice i of the payload is
// checksummed (raw CRC register from 0) and written / read at file offset
// kHeader + lo by its own thread with pwrite / pread, then the slices' CRCs
// are merged in order (crc32c.cpp).  Returns the raw register after
// `reg` (header CRC) and the payload, or sets `err` to the first errno.
uint32_t payload_io(int fd, unsigned char* buf, int64_t len, uint32_t reg, bool write, int& err) {
  const int threads = io_threads(len);
  const int64_t chunk = ((len + threads - 1) / threads + 4095) & ~int64_t(4095);
  std::vector<uint32_t> part(size_t(threads), 0);
  std::vector<int> errs(size_t(threads), 0);
  auto work = [&](int i) {
    const int64_t lo = int64_t(i) * chunk, hi = std::min(len, lo + chunk);
    if (write) part[size_t(i)] = crc32c_raw(buf + lo, hi - lo, 0);
    for (int64_t off = lo; off < hi;) {
      const ssize_t r = write ? ::pwrite(fd, buf + off, size_t(hi - off), off_t(kHeader + off))
                              : ::pread(fd, buf + off, size_t(hi - off), off_t(kHeader + off));
      if (r < 0 && errno == EINTR) continue;
      if (r <= 0) {
        errs[size_t(i)] = r < 0 ? errno : EIO;
        return;
      }
      off += r;
    }
    if (!write) part[size_t(i)] = crc32c_raw(buf + lo, hi - lo, 0);
  };
  std::vector<std::thread> pool;
  int used = 0;
  for (int i = 0; i < threads && int64_t(i) * chunk < len; ++i, ++used)
    if (i > 0) pool.emplace_back(work, i);
  if (used > 0) work(0);
  for (auto& th : pool) th.join();
  err = 0;
  for (int i = 0; i < used; ++i) {
    if (errs[size_t(i)] && !err) err = errs[size_t(i)];
    const int64_t lo = int64_t(i) * chunk, hi = std::min(len, lo + chunk);
    reg = crc32c_shift(reg, hi - lo) ^ part[size_t(i)];
  }
  return reg;
}

// Write stage_out as the ticket's CKPT file: tmp file + rename
// (write_checkpoint_file, storage.py:109-118).  Errors go to tk->async.  The
// replaced file's second name is returned in `*retired` for the caller to
// unlink off the critical path (null: a detached thread unlinks it).
void write_ckpt(TierTicket* tk, std::string* retired_out = nullptr) {
  NvtxRange range("ckpt write");
  ackpt_tier* t = tk->tier;
  unsigned char header[kHeader];
  std::memcpy(header, "CKPT", 4);
  put_le(header + 4, 1, 2);
  put_le(header + 6, uint64_t(tk->step), 8);
  put_le(header + 14, uint64_t(tk->len), 8);
  const std::string path = ckpt_path(t, tk->key), tmp = path + ".tmp";
  auto failed = [&](int e) {
    std::remove(tmp.c_str());
    set_async(*tk->async, e == ENOSPC ? ACKPT_STORAGE_FULL : ACKPT_EXECUTION_ERROR,
              "writing " + path + ": " + std::strerror(e));
  };
  static const bool trace = std::getenv("ACKPT_FILE_TRACE") != nullptr;
  const auto c0 = std::chrono::steady_clock::now();
  const int fd = ::open(tmp.c_str(), O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
  if (fd < 0) return failed(errno);
  const auto c1 = std::chrono::steady_clock::now();
  int err = 0;
  uint32_t reg = crc32c_raw(header, kHeader, 0xFFFFFFFFu);
  if (::pwrite(fd, header, kHeader, 0) != kHeader) err = errno ? errno : EIO;
  if (!err && tk->len > 0) reg = payload_io(fd, t->stage_out, tk->len, reg, true, err);
  const auto c2 = std::chrono::steady_clock::now();
  unsigned char trailer[kTrailer];
  put_le(trailer, reg ^ 0xFFFFFFFFu, 4);
  if (!err && ::pwrite(fd, trailer, kTrailer, off_t(kHeader + tk->len)) != kTrailer) err = errno ? errno : EIO;
  if (::close(fd) != 0 && !err) err = errno;
  // Publish atomically like the reference's tmp + os.replace
  // (storage.py:109-118), so `path` always holds a complete checkpoint -- but
  // never rename OVER an existing file: ext4 (auto_da_alloc) then forces
  // writeback of the new file's data inside rename(), 15-25 ms per 64 MiB on
  // the box, stalling the compute stream.  renameat2(RENAME_EXCHANGE) swaps
  // the two names in one step instead; the tmp name then holds the previous
  // checkpoint, which is unlinked off the critical path.  Without an existing
  // file a plain rename publishes; on file systems without RENAME_EXCHANGE the
  // old file is moved aside first and moved back if the rename fails.
  std::string retired;
  if (!err) {
    if (::renameat2(AT_FDCWD, tmp.c_str(), AT_FDCWD, path.c_str(), RENAME_EXCHANGE) == 0) {
      // free the tmp name for the next store of this key (a rename onto a new
      // name: no data writeback); the old data is unlinked in the background
      retired = path + ".old." + std::to_string(reinterpret_cast<uintptr_t>(tk));
      if (std::rename(tmp.c_str(), retired.c_str()) != 0) retired = tmp;
    } else if (errno == ENOENT) {  // no previous file
      if (std::rename(tmp.c_str(), path.c_str()) != 0) err = errno;
    } else {
      retired = path + ".old." + std::to_string(reinterpret_cast<uintptr_t>(tk));
      if (std::rename(path.c_str(), retired.c_str()) != 0) retired.clear();
      if (std::rename(tmp.c_str(), path.c_str()) != 0) {
        err = errno;
        if (!retired.empty() && std::rename(retired.c_str(), path.c_str()) == 0) retired.clear();
      }
    }
  }
  if (retired_out) *retired_out = retired;
  else if (!retired.empty()) std::thread([retired] { ::unlink(retired.c_str()); }).detach();
  if (trace) {
    const auto c3 = std::chrono::steady_clock::now();
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "ACKPT_FILE_TRACE store key=%lld open=%.3f io=%.3f close+rename=%.3f ms\n",
                 (long long)tk->key, ms(c0, c1), ms(c1, c2), ms(c2, c3));
  }
  if (err) failed(err);
}

// Host function on the D2H stream (graph-capture path), after the payload
// landed in stage_out.
void CUDART_CB file_store_cb(void* arg) { write_ckpt(static_cast<TierTicket*>(arg)); }

// Read + verify the ticket's CKPT file into stage_in (decode_checkpoint /
// read_checkpoint_file, storage.py:83-127).  Errors go to tk->async.
void read_ckpt(TierTicket* tk) {
  NvtxRange range("ckpt read");
  ackpt_tier* t = tk->tier;
  static const bool trace = std::getenv("ACKPT_FILE_TRACE") != nullptr;
  const auto c0 = std::chrono::steady_clock::now();
  struct Trace {
    bool on;
    int64_t key;
    std::chrono::steady_clock::time_point c0;
    ~Trace() {
      if (on)
        std::fprintf(stderr, "ACKPT_FILE_TRACE fetch key=%lld total=%.3f ms\n", (long long)key,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - c0).count());
    }
  } tr{trace, tk->key, c0};
  const std::string path = ckpt_path(t, tk->key);
  const int fd = ::open(path.c_str(), O_RDONLY | O_CLOEXEC);
  if (fd < 0) {
    set_async(*tk->async, ACKPT_MISSING_KEY, path);
    return;
  }
  struct stat sb;
  const int64_t size = ::fstat(fd, &sb) == 0 ? int64_t(sb.st_size) : -1;
  unsigned char header[kHeader], trailer[kTrailer];
  auto bad = [&](const std::string& why) {
    ::close(fd);
    set_async(*tk->async, ACKPT_CHECKSUM_MISMATCH, path + ": " + why);
  };
  if (size < kHeader + kTrailer) return bad("checkpoint truncated: " + std::to_string(size) + " bytes");
  if (::pread(fd, header, kHeader, 0) != kHeader) return bad("short read");
  if (std::memcmp(header, "CKPT", 4) != 0) return bad("bad magic bytes");
  if (get_le(header + 4, 2) != 1) return bad("unsupported format version");
  const uint64_t step = get_le(header + 6, 8), length = get_le(header + 14, 8);
  if (uint64_t(size) != length + kHeader + kTrailer)
    return bad("length field says " + std::to_string(length) + ", file holds " +
               std::to_string(size - kHeader - kTrailer));
  if (int64_t(length) != tk->len || int64_t(length) > t->stage_cap) return bad("payload size changed");
  int err = 0;
  uint32_t reg = crc32c_raw(header, kHeader, 0xFFFFFFFFu);
  if (length > 0) reg = payload_io(fd, t->stage_in, int64_t(length), reg, false, err);
  if (err) return bad(std::string("short read: ") + std::strerror(err));
  if (::pread(fd, trailer, kTrailer, off_t(kHeader + length)) != kTrailer) return bad("short read");
  ::close(fd);
  if ((reg ^ 0xFFFFFFFFu) != uint32_t(get_le(trailer, 4))) {
    set_async(*tk->async, ACKPT_CHECKSUM_MISMATCH, path + ": crc mismatch");
    return;
  }
  if (int64_t(step) != tk->key)
    set_async(*tk->async, ACKPT_CHECKSUM_MISMATCH,
              path + ": file holds step " + std::to_string(step) + ", expected " + std::to_string(tk->key));
  tk->step = int64_t(step);
}

// Host function on the H2D stream (graph-capture path).
void CUDART_CB file_fetch_cb(void* arg) { read_ckpt(static_cast<TierTicket*>(arg)); }

volatile uint32_t& flag(ackpt_tier* t, Flag f) { return reinterpret_cast<volatile uint32_t*>(t->flags)[f]; }

// Wait until a flag the GPU bumps reaches `seq` (cyclic compare): spin, then
// yield.  False when the tier is being torn down instead.
bool wait_flag(ackpt_tier* t, Flag f, uint32_t seq) {
  for (int i = 0; int32_t(flag(t, f) - seq) < 0; ++i) {
    if (t->abort.load(std::memory_order_relaxed)) return false;
    if (i > 4096) std::this_thread::yield();
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  return true;
}
void set_flag(ackpt_tier* t, Flag f, uint32_t seq) {
  std::atomic_thread_fence(std::memory_order_release);
  flag(t, f) = seq;
}

// Store thread: jobs in issue order; a job's file is written once its copy
// landed and every earlier fetch of the key has read the previous file.
void store_worker(ackpt_tier* t) {
  for (;;) {
    IoJob job;
    {
      std::unique_lock<std::mutex> lk(t->qmu);
      t->qcv.wait(lk, [&] { return t->stop || !t->store_q.empty(); });
      if (t->store_q.empty()) return;
      job = t->store_q.front();
      t->store_q.pop_front();
      ++t->busy;
    }
    bool ok = wait_flag(t, kCopied, job.seq);
    if (ok && job.need) {
      std::unique_lock<std::mutex> lk(t->qmu);
      t->qcv.wait(lk, [&] { return t->abort.load() || int32_t(flag(t, kStaged) - job.need) >= 0; });
      ok = !t->abort.load();
    }
    std::string retired;
    if (ok) write_ckpt(job.tk, &retired);  // (never publish a file whose copy did not land)
    {
      std::lock_guard<std::mutex> lk(t->qmu);
      set_flag(t, kWritten, job.seq);  // always, so the D2H stream never hangs
    }
    t->qcv.notify_all();
    if (!retired.empty()) ::unlink(retired.c_str());
    {
      std::lock_guard<std::mutex> lk(t->qmu);
      --t->busy;
    }
    t->qcv.notify_all();
  }
}

// Fetch thread: reads a job's file into stage_in once the store that wrote
// it is done and the previous fetch's H2D copy has consumed stage_in.
void fetch_worker(ackpt_tier* t) {
  for (;;) {
    IoJob job;
    {
      std::unique_lock<std::mutex> lk(t->qmu);
      t->qcv.wait(lk, [&] { return t->stop || !t->fetch_q.empty(); });
      if (t->fetch_q.empty()) return;
      job = t->fetch_q.front();
      t->fetch_q.pop_front();
      ++t->busy;
    }
    bool ok = true;
    if (job.need) {
      std::unique_lock<std::mutex> lk(t->qmu);
      t->qcv.wait(lk, [&] { return t->abort.load() || int32_t(flag(t, kWritten) - job.need) >= 0; });
      ok = !t->abort.load();
    }
    if (ok) ok = wait_flag(t, kConsumed, job.seq - 1);
    if (ok) read_ckpt(job.tk);
    {
      std::lock_guard<std::mutex> lk(t->qmu);
      set_flag(t, kStaged, job.seq);  // always, so the H2D stream never hangs
      --t->busy;
    }
    t->qcv.notify_all();
  }
}

// Stream-memop path available (driver entry points resolved, flags mapped)?
bool io_threads_on(ackpt_tier* t) {
  if (t->flags) return true;
  static const bool env_off = [] {
    const char* e = std::getenv("ACKPT_FILE_HOSTFN");
    return e && e[0] == '1';
  }();
  if (env_off) return false;
  void* w = nullptr;
  void* v = nullptr;
  cudaDriverEntryPointQueryResult q1, q2;
  if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &w, cudaEnableDefault, &q1) != cudaSuccess ||
      cudaGetDriverEntryPoint("cuStreamWriteValue32", &v, cudaEnableDefault, &q2) != cudaSuccess ||
      q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess || !w || !v) {
    cudaGetLastError();
    return false;
  }
  uint32_t* f = nullptr;
  if (cudaHostAlloc(reinterpret_cast<void**>(&f), 256, cudaHostAllocMapped) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  std::memset(f, 0, 256);
  t->wait_value = reinterpret_cast<CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned)>(w);
  t->write_value = reinterpret_cast<CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned)>(v);
  t->flags = f;
  t->store_thr = std::thread(store_worker, t);
  t->fetch_thr = std::thread(fetch_worker, t);
  return true;
}

CUdeviceptr flag_dev(ackpt_tier* t, Flag f) {
  void* d = nullptr;
  ACKPT_CUDA_CHECK(cudaHostGetDevicePointer(&d, t->flags + f, 0));
  return CUdeviceptr(reinterpret_cast<uintptr_t>(d));
}
void stream_wait(ackpt_tier* t, cudaStream_t s, Flag f, uint32_t seq) {
  if (t->wait_value(reinterpret_cast<CUstream>(s), flag_dev(t, f), seq, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
    fail(ACKPT_CUDA_ERROR, "cuStreamWaitValue32 failed");
}
void stream_write(ackpt_tier* t, cudaStream_t s, Flag f, uint32_t seq) {
  if (t->write_value(reinterpret_cast<CUstream>(s), flag_dev(t, f), seq, CU_STREAM_WRITE_VALUE_DEFAULT) !=
      CUDA_SUCCESS)
    fail(ACKPT_CUDA_ERROR, "cuStreamWriteValue32 failed");
}
void enqueue_job(ackpt_tier* t, bool store, const IoJob& job) {
  {
    std::lock_guard<std::mutex> lk(t->qmu);
    (store ? t->store_q : t->fetch_q).push_back(job);
  }
  t->qcv.notify_all();
}
// Block until the I/O threads have no queued or running job.
void io_drain(ackpt_tier* t) {
  if (!t->flags) return;
  std::unique_lock<std::mutex> lk(t->qmu);
  t->qcv.wait(lk, [&] { return t->store_q.empty() && t->fetch_q.empty() && t->busy == 0; });
}
void io_stop(ackpt_tier* t) {
  if (!t->flags) return;
  {
    std::lock_guard<std::mutex> lk(t->qmu);
    t->stop = true;
    t->abort.store(true);  // the streams were drained: only a failed stream leaves a flag behind
  }
  t->qcv.notify_all();
  if (t->store_thr.joinable()) t->store_thr.join();
  if (t->fetch_thr.joinable()) t->fetch_thr.join();
}

bool capturing(void* after_stream) {
  if (!after_stream) return false;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(static_cast<cudaStream_t>(after_stream), &cs) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return cs != cudaStreamCaptureStatusNone;
}

// File-stage transfers go through the I/O threads unless the enqueue is being
// captured into a CUDA graph (or a throttle needs the host-function hold).
bool use_io_threads(ackpt_tier* t, void* after_stream) {
  if (t->latency_s > 0 || t->bandwidth > 0) return false;
  if (after_stream) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(static_cast<cudaStream_t>(after_stream), &cs) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    if (cs != cudaStreamCaptureStatusNone) return false;
  }
  return io_threads_on(t);
}

// Payload length of an existing CKPT file: -1 when absent, -2 when the header
// is not a valid CKPT header for the file's size (bad magic / version, or
// length + header + trailer != file size; `why` says which).  Allocations are
// never sized from an unvalidated header; the fetch of such a file fails with
// ChecksumMismatch at wait, like decode_checkpoint (storage.py:83-106).
int64_t file_payload_len(const ackpt_tier* t, int64_t key, std::string* why = nullptr) {
  const int fd = ::open(ckpt_path(t, key).c_str(), O_RDONLY | O_CLOEXEC);
  if (fd < 0) return -1;
  struct stat sb;
  unsigned char header[kHeader];
  const bool got = ::fstat(fd, &sb) == 0 && ::pread(fd, header, kHeader, 0) == kHeader;
  ::close(fd);
  auto bad = [&](const std::string& w) {
    if (why) *why = ckpt_path(t, key) + ": " + w;
    return int64_t(-2);
  };
  if (!got) return bad("checkpoint truncated");
  if (std::memcmp(header, "CKPT", 4) != 0) return bad("bad magic bytes");
  if (get_le(header + 4, 2) != 1) return bad("unsupported format version");
  const uint64_t length = get_le(header + 14, 8);
  if (length > uint64_t(sb.st_size) || uint64_t(sb.st_size) != length + kHeader + kTrailer)
    return bad("length field says " + std::to_string(length) + ", file holds " +
               std::to_string(int64_t(sb.st_size) - kHeader - kTrailer));
  return int64_t(length);
}

void ensure_stage(ackpt_tier* t, int64_t bytes) {
  if (bytes <= t->stage_cap) return;
  ACKPT_CUDA_CHECK(cudaStreamSynchronize(t->d2h));
  ACKPT_CUDA_CHECK(cudaStreamSynchronize(t->h2d));
  io_drain(t);
  if (t->stage_out) cudaFreeHost(t->stage_out);
  if (t->stage_in) cudaFreeHost(t->stage_in);
  t->stage_out = t->stage_in = nullptr;
  t->stage_cap = 0;
  if (cudaHostAlloc(reinterpret_cast<void**>(&t->stage_out), size_t(bytes), cudaHostAllocDefault) != cudaSuccess ||
      cudaHostAlloc(reinterpret_cast<void**>(&t->stage_in), size_t(bytes), cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    fail(ACKPT_STORAGE_FULL, "pinned staging allocation failed");
  }
  t->stage_cap = bytes;
}

unsigned char* key_ptr(const ackpt_tier* t, const KeyEntry& ke) {
  return ke.big ? ke.big : t->slot_ptr[size_t(ke.slot)];
}

// Gives `key` host storage for `bytes`: a slab slot when it fits slot_bytes,
// else a dedicated pinned buffer (grown on demand; pending copies on the key
// are drained before a buffer is replaced).  Throws StorageFull.
KeyEntry& ensure_storage(ackpt_tier* t, int64_t key, int64_t bytes) {
  KeyEntry& ke = t->keys[key];
  if (bytes <= t->slot_bytes) {
    if (ke.big || ke.slot >= 0) return ke;
    if (t->free_slots.empty()) reserve_slots(t, int64_t(t->slot_ptr.size()) + 1);
    ke.slot = t->free_slots.back();
    t->free_slots.pop_back();
    return ke;
  }
  if (ke.big_cap < bytes) {
    if (ke.stored) ACKPT_CUDA_CHECK(cudaEventSynchronize(ke.last_store));
    if (ke.fetched) ACKPT_CUDA_CHECK(cudaEventSynchronize(ke.last_fetch));
    if (ke.big) cudaFreeHost(ke.big);
    ke.big = nullptr;
    ke.big_cap = 0;
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&ke.big), size_t(bytes), cudaHostAllocDefault);
    if (e != cudaSuccess) {
      cudaGetLastError();
      ke.big = nullptr;
      fail(ACKPT_STORAGE_FULL, std::string("pinned host allocation failed: ") + cudaGetErrorString(e));
    }
    ke.big_cap = bytes;
  }
  if (ke.slot >= 0) {
    t->free_slots.push_back(ke.slot);
    ke.slot = -1;
  }
  return ke;
}

}  // namespace

// Engine-side helpers (engine.cpp): host storage for every key of a plan is
// allocated at prepare time, outside the timed window.
void tier_reserve_keys(ackpt_tier* t, const std::vector<int64_t>& keys, int64_t bytes) {
  std::lock_guard<std::mutex> lk(t->mu);
  if (t->cascade) return;  // its DRAM slots and read buffers exist since creation
  if (bytes <= t->slot_bytes) {
    int64_t absent = 0;
    for (int64_t k : keys) {
      auto it = t->keys.find(k);
      if (it == t->keys.end() || (it->second.slot < 0 && !it->second.big)) ++absent;
    }
    const int64_t used = int64_t(t->slot_ptr.size() - t->free_slots.size());
    reserve_slots(t, used + absent);
  }
  for (int64_t k : keys) ensure_storage(t, k, bytes);
}
cudaEvent_t tier_ticket_event(ackpt_tier* t, ackpt_ticket id) {
  std::lock_guard<std::mutex> lk(t->mu);
  TierTicket* tk = find_ticket(t, id);
  return (!tk || tk->complete) ? nullptr : tk->done;
}
// Asynchronous (file-stage) status of a ticket whose event has completed.
int tier_async_status(ackpt_tier* t, ackpt_ticket id, std::string* msg) {
  std::lock_guard<std::mutex> lk(t->mu);
  TierTicket* tk = find_ticket(t, id);
  if (!tk) return recycled_status(t, id, msg);
  if (!tk->async) return ACKPT_OK;
  const int e = tk->async->err.load(std::memory_order_acquire);
  if (e != ACKPT_OK && msg) *msg = tk->async->msg;
  return e;
}
int tier_ticket_status(ackpt_tier* t, ackpt_ticket id, std::string* msg) {
  std::lock_guard<std::mutex> lk(t->mu);
  TierTicket* tk = find_ticket(t, id);
  if (!tk) return recycled_status(t, id, msg);
  if (msg) *msg = tk->msg;
  return tk->err;
}
// Clear a file-stage ticket's asynchronous status before a CUDA-graph replay
// re-runs its host functions.
void tier_reset_async(ackpt_tier* t, ackpt_ticket id) {
  std::lock_guard<std::mutex> lk(t->mu);
  TierTicket* tk = find_ticket(t, id);  // graph tickets are never recycled
  if (tk && tk->async) tk->async->err.store(ACKPT_OK, std::memory_order_release);
}
// Drain the copy streams and forget the per-key copy-ordering events, so no
// stream wait crosses a CUDA-graph capture boundary (before a capture, after
// a graphed run): the events last recorded inside a capture are graph nodes.
// The per-key events are then re-recorded on the idle copy streams (outside
// any capture), so a later eager transfer or ensure_storage can wait on them.
void tier_quiesce(ackpt_tier* t) {
  if (t->cascade) return cascade_quiesce(t);  // (its workers take t->mu: drain without it)
  std::lock_guard<std::mutex> lk(t->mu);
  ACKPT_CUDA_CHECK(cudaStreamSynchronize(t->d2h));
  ACKPT_CUDA_CHECK(cudaStreamSynchronize(t->h2d));
  io_drain(t);
  for (auto& kv : t->keys) {
    KeyEntry& ke = kv.second;
    if (ke.last_store) ACKPT_CUDA_CHECK(cudaEventRecord(ke.last_store, t->d2h));
    if (ke.last_fetch) ACKPT_CUDA_CHECK(cudaEventRecord(ke.last_fetch, t->h2d));
    ke.fetched = false;
  }
}
void tier_set_timing(ackpt_tier* t, bool on) {
  std::lock_guard<std::mutex> lk(t->mu);
  t->timing = on;
}
// Cascade tiers: seconds one boundary store takes on the spill stage (CRC +
// O_DIRECT write of a `bytes` payload) and the number of DRAM slots; -1 / 0
// for the other tiers (engine calibrate, runtime.py:420-466).
double tier_spill_seconds(ackpt_tier* t, int64_t bytes) {
  if (!t->cascade) return -1.0;
  const double s = cascade_spill_probe(t, bytes);  // drains the workers: no t->mu here
  return s;
}
int tier_dram_slots(ackpt_tier* t) { return t->cascade ? t->cascade_slots : 0; }
bool tier_ticket_times(ackpt_tier* t, ackpt_ticket id, cudaEvent_t* t0, cudaEvent_t* t1) {
  std::lock_guard<std::mutex> lk(t->mu);
  TierTicket* tk = find_ticket(t, id);
  if (!tk) return false;
  *t0 = tk->t0;
  *t1 = tk->t1;
  return tk->t0 && tk->t1;
}

// The engine's tickets once its run drained (every transfer of a pass has
// completed by then): events back to the pool, the slot recyclable.
void tier_retire(ackpt_tier* t, ackpt_ticket id) {
  std::lock_guard<std::mutex> lk(t->mu);
  TierTicket* tk = find_ticket(t, id);
  if (!tk) return;
  retire(t, *tk);
  tk->waited = true;
}
int64_t tier_slot_bytes(const ackpt_tier* t) { return t->slot_bytes; }
cudaStream_t tier_d2h(const ackpt_tier* t) { return t->d2h; }
double tier_throttle_seconds(const ackpt_tier* t, int64_t bytes) {
  return t->latency_s + (t->bandwidth > 0 ? double(bytes) / t->bandwidth : 0.0);
}

}  // namespace ackpt

extern "C" {

ACKPT_API int ackpt_tier_create(int64_t capacity, int64_t slot_bytes, ackpt_tier** out) {
  return ackpt::guard([&] {
    if (slot_bytes <= 0) ackpt::fail(ACKPT_VALUE_ERROR, "slot_bytes must be positive");
    if (capacity < 0) ackpt::fail(ACKPT_VALUE_ERROR, "capacity must be >= 0");
    std::unique_ptr<ackpt_tier> t(new ackpt_tier());
    t->capacity = capacity;
    t->slot_bytes = slot_bytes;
    int lo = 0, hi = 0;
    ACKPT_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    ACKPT_CUDA_CHECK(cudaStreamCreateWithPriority(&t->d2h, cudaStreamNonBlocking, hi));
    ACKPT_CUDA_CHECK(cudaStreamCreateWithPriority(&t->h2d, cudaStreamNonBlocking, hi));
    ACKPT_CUDA_CHECK(cudaEventCreateWithFlags(&t->after, cudaEventDisableTiming));
    if (capacity > 0) ackpt::reserve_slots(t.get(), capacity);
    *out = t.release();
  });
}

ACKPT_API int ackpt_tier_create_file(const char* directory, int64_t slot_bytes, ackpt_tier** out) {
  int rc = ackpt_tier_create(0, slot_bytes > 0 ? slot_bytes : 1, out);
  if (rc != ACKPT_OK) return rc;
  return ackpt::guard([&] {
    ackpt_tier* t = *out;
    t->file_mode = true;
    t->dir = directory ? directory : ".";
    ackpt::ensure_stage(t, slot_bytes > 0 ? slot_bytes : 1);
  });
}

ACKPT_API int ackpt_tier_destroy(ackpt_tier* t) {
  return ackpt::guard([&] {
    if (!t) return;
    if (t->d2h) cudaStreamSynchronize(t->d2h);
    if (t->h2d) cudaStreamSynchronize(t->h2d);
    ackpt::io_stop(t);
    ackpt::cascade_destroy(t);
    if (t->flags) cudaFreeHost(t->flags);
    for (auto e : t->all_events) cudaEventDestroy(e);
    for (auto& kv : t->keys) {
      if (kv.second.last_store) cudaEventDestroy(kv.second.last_store);
      if (kv.second.last_fetch) cudaEventDestroy(kv.second.last_fetch);
      if (kv.second.big) cudaFreeHost(kv.second.big);
    }
    if (t->after) cudaEventDestroy(t->after);
    for (auto c : t->chunks) cudaFreeHost(c);
    if (t->stage_out) cudaFreeHost(t->stage_out);
    if (t->stage_in) cudaFreeHost(t->stage_in);
    if (t->d2h) cudaStreamDestroy(t->d2h);
    if (t->h2d) cudaStreamDestroy(t->h2d);
    delete t;
  });
}

ACKPT_API int ackpt_tier_set_throttle(ackpt_tier* t, double latency_s, double bandwidth) {
  return ackpt::guard([&] {
    if (latency_s < 0) ackpt::fail(ACKPT_VALUE_ERROR, "latency must be >= 0");
    t->latency_s = latency_s;
    t->bandwidth = bandwidth;
  });
}

ACKPT_API int ackpt_tier_begin_store(ackpt_tier* t, int64_t key, int64_t step, const void* src,
                                     int64_t bytes, void* after_stream, ackpt_ticket* out) {
  return ackpt::guard([&] {
    std::lock_guard<std::mutex> lk(t->mu);
    if (t->cascade) {
      if (step < 0) ackpt::fail(ACKPT_VALUE_ERROR, "step must be >= 0");
      if (bytes < 0) ackpt::fail(ACKPT_VALUE_ERROR, "bytes must be >= 0");
      *out = ackpt::cascade_begin_store(t, key, step, src, bytes, after_stream);
      return;
    }
    if (step < 0) ackpt::fail(ACKPT_VALUE_ERROR, "step must be >= 0");
    ackpt::TierTicket tk;
    tk.kind = 0;
    tk.key = key;
    tk.step = step;
    if (bytes < 0) ackpt::fail(ACKPT_VALUE_ERROR, "bytes must be >= 0");
    if (t->file_mode) {
      // D2H into the staging buffer, then write the CKPT file from a host
      // function on the same stream (stores serialise on the D2H stream).
      ackpt::ensure_stage(t, bytes);
      ackpt::KeyEntry& ke = t->keys[key];
      const bool threads = ackpt::use_io_threads(t, after_stream);
      if (after_stream) {
        ACKPT_CUDA_CHECK(cudaEventRecord(t->after, static_cast<cudaStream_t>(after_stream)));
        ACKPT_CUDA_CHECK(cudaStreamWaitEvent(t->d2h, t->after, 0));
      }
      if (ke.fetched) ACKPT_CUDA_CHECK(cudaStreamWaitEvent(t->d2h, ke.last_fetch, 0));
      uint32_t seq = 0;
      if (threads) {  // stage_out is free once the previous store's file is written
        seq = ++t->store_seq;
        ackpt::stream_wait(t, t->d2h, ackpt::kWritten, seq - 1);
      }
      cudaEvent_t m0 = ackpt::mark(t, t->d2h);
      if (bytes > 0)
        ACKPT_CUDA_CHECK(cudaMemcpyAsync(t->stage_out, src, size_t(bytes), cudaMemcpyDeviceToHost, t->d2h));
      ke.step = step;
      ke.len = bytes;
      ackpt_ticket id = ackpt::add_ticket(t, std::move(tk));
      ackpt::TierTicket& ref = *ackpt::find_ticket(t, id);
      ref.captured = ackpt::capturing(after_stream);
      ref.tier = t;
      ref.len = bytes;
      ref.async = std::make_shared<ackpt::AsyncStatus>();
      if (threads) {
        ackpt::stream_write(t, t->d2h, ackpt::kCopied, seq);
        ackpt::enqueue_job(t, true, {&ref, seq, ke.file_fetch_seq});
        ackpt::stream_wait(t, t->d2h, ackpt::kWritten, seq);
        ke.file_store_seq = seq;
      } else {
        ACKPT_CUDA_CHECK(cudaLaunchHostFunc(t->d2h, ackpt::file_store_cb, &ref));
        ke.file_store_seq = 0;
      }
      ackpt::hold(t, t->d2h, ref, bytes);
      ref.done = ackpt::new_event(t);
      ACKPT_CUDA_CHECK(cudaEventRecord(ref.done, t->d2h));
      ref.t0 = m0;
      ref.t1 = ackpt::mark(t, t->d2h);
      if (!ke.last_store) ACKPT_CUDA_CHECK(cudaEventCreateWithFlags(&ke.last_store, cudaEventDisableTiming));
      ACKPT_CUDA_CHECK(cudaEventRecord(ke.last_store, t->d2h));
      ke.stored = true;
      *out = id;
      return;
    }
    ackpt::KeyEntry* kp = nullptr;
    try {
      kp = &ackpt::ensure_storage(t, key, bytes);
    } catch (const ackpt::Error& e) {  // surfaced at wait (storage.py:271-278)
      tk.err = e.code;
      tk.msg = e.what();
      tk.complete = true;
      *out = ackpt::add_ticket(t, std::move(tk));
      return;
    }
    ackpt::KeyEntry& ke = *kp;
    if (after_stream) {
      ACKPT_CUDA_CHECK(cudaEventRecord(t->after, static_cast<cudaStream_t>(after_stream)));
      ACKPT_CUDA_CHECK(cudaStreamWaitEvent(t->d2h, t->after, 0));
    }
    if (ke.fetched) ACKPT_CUDA_CHECK(cudaStreamWaitEvent(t->d2h, ke.last_fetch, 0));
    cudaEvent_t m0 = ackpt::mark(t, t->d2h);
    if (bytes > 0)
      ACKPT_CUDA_CHECK(cudaMemcpyAsync(ackpt::key_ptr(t, ke), src, size_t(bytes),
                                       cudaMemcpyDeviceToHost, t->d2h));
    ke.step = step;
    ke.len = bytes;
    ackpt_ticket id = ackpt::add_ticket(t, std::move(tk));
    ackpt::TierTicket& ref = *ackpt::find_ticket(t, id);
      ref.captured = ackpt::capturing(after_stream);
    ackpt::hold(t, t->d2h, ref, bytes);
    ref.done = ackpt::new_event(t);
    ACKPT_CUDA_CHECK(cudaEventRecord(ref.done, t->d2h));
    ref.t0 = m0;
    ref.t1 = ackpt::mark(t, t->d2h);
    if (!ke.last_store) ACKPT_CUDA_CHECK(cudaEventCreateWithFlags(&ke.last_store, cudaEventDisableTiming));
    ACKPT_CUDA_CHECK(cudaEventRecord(ke.last_store, t->d2h));
    ke.stored = true;
    *out = id;
  });
}

ACKPT_API int ackpt_tier_begin_fetch(ackpt_tier* t, int64_t key, void* dst, int64_t bytes,
                                     void* after_stream, ackpt_ticket* out) {
  return ackpt::guard([&] {
    std::lock_guard<std::mutex> lk(t->mu);
    if (t->cascade) {
      *out = ackpt::cascade_begin_fetch(t, key, dst, bytes, after_stream);
      return;
    }
    ackpt::TierTicket tk;
    tk.kind = 1;
    tk.key = key;
    auto it = t->keys.find(key);
    if (t->file_mode) {
      // Keys stored earlier in this tier, or CKPT files already on disk (resume).
      int64_t len = -1;
      std::string why;
      if (it != t->keys.end() && it->second.stored) len = it->second.len;
      else len = ackpt::file_payload_len(t, key, &why);
      if (len < 0) {
        tk.err = len == -1 ? ACKPT_MISSING_KEY : ACKPT_CHECKSUM_MISMATCH;
        tk.msg = len == -1 ? ackpt::ckpt_path(t, key) : why;
        tk.complete = true;
        *out = ackpt::add_ticket(t, std::move(tk));
        return;
      }
      if (bytes >= 0 && bytes < len) {
        tk.err = ACKPT_SIZE_MISMATCH;
        tk.msg = "destination holds " + std::to_string(bytes) + " bytes, key " + std::to_string(key) +
                 " holds " + std::to_string(len);
        tk.complete = true;
        *out = ackpt::add_ticket(t, std::move(tk));
        return;
      }
      ackpt::ensure_stage(t, len);
      ackpt::KeyEntry& ke = t->keys[key];
      tk.step = ke.stored ? ke.step : key;
      const bool threads = ackpt::use_io_threads(t, after_stream);
      if (after_stream) {
        ACKPT_CUDA_CHECK(cudaEventRecord(t->after, static_cast<cudaStream_t>(after_stream)));
        ACKPT_CUDA_CHECK(cudaStreamWaitEvent(t->h2d, t->after, 0));
      }
      // (I/O-thread path: the fetch thread orders itself after the key's store)
      if (ke.stored && !threads) ACKPT_CUDA_CHECK(cudaStreamWaitEvent(t->h2d, ke.last_store, 0));
      cudaEvent_t m0 = ackpt::mark(t, t->h2d);
      ackpt_ticket id = ackpt::add_ticket(t, std::move(tk));
      ackpt::TierTicket& ref = *ackpt::find_ticket(t, id);
      ref.captured = ackpt::capturing(after_stream);
      ref.tier = t;
      ref.len = len;
      ref.async = std::make_shared<ackpt::AsyncStatus>();
      if (threads) {
        const uint32_t seq = ++t->fetch_seq;
        ackpt::enqueue_job(t, false, {&ref, seq, ke.file_store_seq});
        ke.file_fetch_seq = seq;
        ackpt::stream_wait(t, t->h2d, ackpt::kStaged, seq);
        if (len > 0)
          ACKPT_CUDA_CHECK(cudaMemcpyAsync(dst, t->stage_in, size_t(len), cudaMemcpyHostToDevice, t->h2d));
        ackpt::stream_write(t, t->h2d, ackpt::kConsumed, seq);
      } else {
        ACKPT_CUDA_CHECK(cudaLaunchHostFunc(t->h2d, ackpt::file_fetch_cb, &ref));
        if (len > 0)
          ACKPT_CUDA_CHECK(cudaMemcpyAsync(dst, t->stage_in, size_t(len), cudaMemcpyHostToDevice, t->h2d));
      }
      ackpt::hold(t, t->h2d, ref, len);
      ref.done = ackpt::new_event(t);
      ACKPT_CUDA_CHECK(cudaEventRecord(ref.done, t->h2d));
      ref.t0 = m0;
      ref.t1 = ackpt::mark(t, t->h2d);
      if (!ke.last_fetch) ACKPT_CUDA_CHECK(cudaEventCreateWithFlags(&ke.last_fetch, cudaEventDisableTiming));
      ACKPT_CUDA_CHECK(cudaEventRecord(ke.last_fetch, t->h2d));
      ke.fetched = true;
      *out = id;
      return;
    }
    if (it == t->keys.end() || !it->second.stored) {
      tk.err = ACKPT_MISSING_KEY;  // storage.py:310-311
      tk.msg = "key " + std::to_string(key) + " never stored";
      tk.complete = true;
      *out = ackpt::add_ticket(t, std::move(tk));
      return;
    }
    ackpt::KeyEntry& ke = it->second;
    if (bytes >= 0 && bytes < ke.len) {
      tk.err = ACKPT_SIZE_MISMATCH;
      tk.msg = "destination holds " + std::to_string(bytes) + " bytes, key " +
               std::to_string(key) + " holds " + std::to_string(ke.len);
      tk.complete = true;
      *out = ackpt::add_ticket(t, std::move(tk));
      return;
    }
    tk.step = ke.step;
    if (after_stream) {
      ACKPT_CUDA_CHECK(cudaEventRecord(t->after, static_cast<cudaStream_t>(after_stream)));
      ACKPT_CUDA_CHECK(cudaStreamWaitEvent(t->h2d, t->after, 0));
    }
    ACKPT_CUDA_CHECK(cudaStreamWaitEvent(t->h2d, ke.last_store, 0));
    cudaEvent_t m0 = ackpt::mark(t, t->h2d);
    if (ke.len > 0)
      ACKPT_CUDA_CHECK(cudaMemcpyAsync(dst, ackpt::key_ptr(t, ke), size_t(ke.len),
                                       cudaMemcpyHostToDevice, t->h2d));
    ackpt_ticket id = ackpt::add_ticket(t, std::move(tk));
    ackpt::TierTicket& ref = *ackpt::find_ticket(t, id);
      ref.captured = ackpt::capturing(after_stream);
    ackpt::hold(t, t->h2d, ref, ke.len);
    ref.done = ackpt::new_event(t);
    ACKPT_CUDA_CHECK(cudaEventRecord(ref.done, t->h2d));
    ref.t0 = m0;
    ref.t1 = ackpt::mark(t, t->h2d);
    if (!ke.last_fetch) ACKPT_CUDA_CHECK(cudaEventCreateWithFlags(&ke.last_fetch, cudaEventDisableTiming));
    ACKPT_CUDA_CHECK(cudaEventRecord(ke.last_fetch, t->h2d));
    ke.fetched = true;
    *out = id;
  });
}

ACKPT_API int ackpt_tier_wait(ackpt_tier* t, ackpt_ticket ticket, int64_t* step_out) {
  cudaEvent_t ev = nullptr;
  bool recycled = false;
  int rc = ackpt::guard([&] {
    std::lock_guard<std::mutex> lk(t->mu);
    ackpt::TierTicket* tk = ackpt::find_ticket(t, ticket);
    if (!tk) {  // waited before and recycled: idempotent, the first wait's status
      recycled = true;
      std::string msg;
      const int e = ackpt::recycled_status(t, ticket, &msg);
      if (e != ACKPT_OK) ackpt::fail(e, msg);
      return;
    }
    if (step_out) *step_out = tk->step;
    if (tk->err != ACKPT_OK) {
      tk->waited = true;
      ackpt::fail(tk->err, tk->msg);
    }
    ev = tk->complete ? nullptr : tk->done;
  });
  if (rc != ACKPT_OK || recycled) return rc;
  // Block without holding the lock (other threads may issue transfers).
  return ackpt::guard([&] {
    if (ev) ACKPT_CUDA_CHECK(cudaEventSynchronize(ev));
    std::lock_guard<std::mutex> lk(t->mu);
    ackpt::TierTicket& tk = *ackpt::find_ticket(t, ticket);  // not recyclable before waited
    ackpt::retire(t, tk);
    tk.waited = true;
    if (step_out) *step_out = tk.step;
    if (tk.async) {  // file-stage errors, raised by the worker side (storage.py:271-278)
      const int e = tk.async->err.load(std::memory_order_acquire);
      if (e != ACKPT_OK) ackpt::fail(e, tk.async->msg);
    }
  });
}

ACKPT_API int ackpt_tier_stream_wait(ackpt_tier* t, ackpt_ticket ticket, void* stream) {
  return ackpt::guard([&] {
    std::lock_guard<std::mutex> lk(t->mu);
    ackpt::TierTicket* tk = ackpt::find_ticket(t, ticket);
    if (!tk) {
      std::string msg;
      const int e = ackpt::recycled_status(t, ticket, &msg);
      if (e != ACKPT_OK) ackpt::fail(e, msg);
      return;
    }
    if (tk->err != ACKPT_OK) ackpt::fail(tk->err, tk->msg);
    if (!tk->complete && tk->done)
      ACKPT_CUDA_CHECK(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), tk->done, 0));
  });
}

ACKPT_API int ackpt_tier_poll(ackpt_tier* t, ackpt_ticket ticket) {
  int ready = ACKPT_OK;
  int rc = ackpt::guard([&] {
    std::lock_guard<std::mutex> lk(t->mu);
    ackpt::TierTicket* tk = ackpt::find_ticket(t, ticket);
    if (!tk || tk->complete) return;
    cudaError_t e = cudaEventQuery(tk->done);
    if (e == cudaErrorNotReady) {
      ready = ACKPT_NOT_READY;
      return;
    }
    ACKPT_CUDA_CHECK(e);
    ackpt::retire(t, *tk);
  });
  return rc != ACKPT_OK ? rc : ready;
}

ACKPT_API int ackpt_tier_contains(ackpt_tier* t, int64_t key, int32_t* out) {
  return ackpt::guard([&] {
    std::lock_guard<std::mutex> lk(t->mu);
    if (t->cascade) {
      *out = ackpt::cascade_contains(t, key) ? 1 : 0;
      return;
    }
    auto it = t->keys.find(key);
    *out = (it != t->keys.end() && it->second.stored) ? 1 : 0;
    if (!*out && t->file_mode) *out = ackpt::file_payload_len(t, key) != -1 ? 1 : 0;  // the file exists
  });
}

ACKPT_API int ackpt_tier_key_bytes(ackpt_tier* t, int64_t key, int64_t* out) {
  return ackpt::guard([&] {
    std::lock_guard<std::mutex> lk(t->mu);
    if (t->cascade) {
      *out = ackpt::cascade_key_bytes(t, key);
      return;
    }
    auto it = t->keys.find(key);
    if (t->file_mode && (it == t->keys.end() || !it->second.stored)) {
      std::string why;
      const int64_t len = ackpt::file_payload_len(t, key, &why);
      if (len == -1) ackpt::fail(ACKPT_MISSING_KEY, ackpt::ckpt_path(t, key));
      if (len < 0) ackpt::fail(ACKPT_CHECKSUM_MISMATCH, why);
      *out = len;
      return;
    }
    if (it == t->keys.end() || !it->second.stored)
      ackpt::fail(ACKPT_MISSING_KEY, "key " + std::to_string(key) + " never stored");
    *out = it->second.len;
  });
}

ACKPT_API int ackpt_tier_host_ptr(ackpt_tier* t, int64_t key, void** out) {
  return ackpt::guard([&] {
    std::lock_guard<std::mutex> lk(t->mu);
    if (t->cascade) {
      *out = ackpt::cascade_host_ptr(t, key);
      return;
    }
    if (t->file_mode) ackpt::fail(ACKPT_VALUE_ERROR, "file-stage keys live on disk, not in pinned memory");
    auto it = t->keys.find(key);
    if (it == t->keys.end() || !it->second.stored)
      ackpt::fail(ACKPT_MISSING_KEY, "key " + std::to_string(key) + " never stored");
    *out = ackpt::key_ptr(t, it->second);
  });
}

ACKPT_API int ackpt_tier_clear(ackpt_tier* t) {
  return ackpt::guard([&] {
    ACKPT_CUDA_CHECK(cudaStreamSynchronize(t->d2h));
    ACKPT_CUDA_CHECK(cudaStreamSynchronize(t->h2d));
    ackpt::io_drain(t);
    if (t->cascade) ackpt::cascade_quiesce(t);
    std::lock_guard<std::mutex> lk(t->mu);
    if (t->cascade) ackpt::cascade_clear(t);
    for (auto& kv : t->keys) {
      if (kv.second.slot >= 0) t->free_slots.push_back(kv.second.slot);
      if (kv.second.big) cudaFreeHost(kv.second.big);
      if (kv.second.last_store) cudaEventDestroy(kv.second.last_store);
      if (kv.second.last_fetch) cudaEventDestroy(kv.second.last_fetch);
    }
    t->keys.clear();
    for (auto& kv : t->tickets) {
      ackpt::retire(t, kv.second);
      kv.second.waited = true;
    }
    ackpt::compact_tickets(t);
  });
}

}  // extern "C"

extern "C" ACKPT_API int ackpt_tier_streams(ackpt_tier* t, void** d2h, void** h2d) {
  return ackpt::guard([&] {
    if (d2h) *d2h = t->d2h;
    if (h2d) *h2d = t->h2d;
  });
}

#include "cascade_impl.h"
