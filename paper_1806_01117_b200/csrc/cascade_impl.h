// Three-stage Level-2 tier: HBM -> pinned host DRAM -> CKPT files (NVMe).
// Part of tier.cpp's translation unit (included at its end; it uses the
// tier's tickets, events, copy streams and CKPT helpers).
//
// SURVEY §8(f) row 1 / BASELINE config 5: the pinned tier of tier.cpp with a
// bounded number of DRAM slots (the host-RAM budget), backed by the
// reference's file format (storage.py:9-18, 83-127, 321-340).
//
// * A store copies HBM -> a DRAM slot on the D2H stream (the slot's memory is
//   the CKPT file image: header | payload | crc | pad, payload at +22).
//   Once more than `dram_slots - kSpillMargin` resident keys have no file
//   copy, the oldest is spilled by the spill thread: header, CRC32C, O_DIRECT
//   write of the 4 KiB-padded image, ftruncate to the exact CKPT length,
//   atomic publish (renameat2 exchange).  A store that needs a slot evicts
//   the least recently stored key whose spill was issued; its D2H copy waits
//   (cuStreamWaitValue32) for that spill and for any H2D copy still reading
//   the slot.
// * A fetch of a resident key is one H2D copy from its slot.  A fetch of a
//   spilled key is served from a ring of kRing pinned read buffers: the read
//   thread reads and verifies the file (O_DIRECT, CRC32C) and bumps a flag
//   the H2D stream waits on.  Every fetch also starts reading the next two
//   lower spilled keys (the multistage backward fetches boundaries in
//   descending order, runtime.py:297-322): NVMe -> DRAM two intervals ahead,
//   DRAM -> HBM one ahead (the executor's own prefetch).
// * Errors (ENOSPC -> StorageFull, bad CRC / header -> ChecksumMismatch,
//   absent -> MissingKey) surface at wait / the end of an engine run; every
//   flag is still bumped, so no stream waits forever.
// Not supported: CUDA-graph capture (the threads are fed at enqueue time) and
// the throttle.
#pragma once

namespace ackpt {

constexpr int kRing = 3;         // file read buffers
constexpr int kSpillMargin = 2;  // resident keys kept spillable ahead of demand
constexpr int64_t kDirectAlign = 4096;

struct CascadeKey {
  int64_t step = 0, len = 0;
  uint32_t version = 0;  // bumped by every store of the key
  int slot = -1;         // resident DRAM slot, -1 if not resident
  uint64_t order = 0;    // store order: eviction takes the oldest
  uint32_t spill_gen = 0;   // spill of the resident copy issued with this slot flag value (0: none)
  int spill_slot = -1;      // slot the last spill reads (the file is complete once spilled >= spill_gen)
  bool on_file = false;     // a CKPT file of `version` is complete
  bool stored = false;      // stored through this tier (else: a file found on disk, resume)
  int err = ACKPT_OK;       // sticky spill error of this version
  std::string msg;
};

struct RingEntry {
  int64_t key = -1;
  uint32_t version = 0;
  uint32_t gen = 0;        // read flag value of this occupancy (0: never used)
  bool fetched = false;    // an H2D copy of this occupancy was enqueued (it bumps consumed)
  std::shared_ptr<AsyncStatus> status;
};

struct SpillJob {
  int64_t key = 0, step = 0, len = 0;
  int slot = 0;
  uint32_t copied = 0, gen = 0, version = 0;
};

struct ReadJob {
  int64_t key = 0, len = 0;
  int buf = 0;
  uint32_t gen = 0, need_consumed = 0;
  int spill_slot = -1;
  uint32_t spill_gen = 0;
  std::shared_ptr<AsyncStatus> status;
};

struct CascadeStats {
  int64_t spills = 0, spill_bytes = 0, reads = 0, read_bytes = 0, dram_hits = 0, ring_hits = 0, ring_misses = 0;
  double spill_seconds = 0.0, read_seconds = 0.0;
};

struct Cascade {
  int dram_slots = 0;
  int64_t image_bytes = 0;  // CKPT image of one slot, padded to kDirectAlign
  std::vector<unsigned char*> slot_mem, ring_mem;
  std::vector<int64_t> slot_key;  // key resident in each slot (-1 free)
  std::vector<uint32_t> copy_gen, spill_gen_issued, read_gen;
  std::vector<cudaEvent_t> slot_store_ev, slot_fetch_ev;
  std::vector<bool> slot_fetched;
  std::unordered_map<int64_t, CascadeKey> keys;
  RingEntry ring[kRing];
  int ring_next = 0;
  uint64_t order = 0;
  uint32_t* flags = nullptr;  // mapped pinned: copied[K] spilled[K] read[R] consumed[R], 16 B apart
  std::mutex qmu;
  std::condition_variable qcv;
  std::deque<SpillJob> spill_q;
  std::deque<ReadJob> read_q;
  int busy = 0;
  bool stop = false;
  std::atomic<bool> abort{false};
  std::thread spill_thr, read_thr;
  CascadeStats stats;
};

namespace {

enum CFlag { kCopiedF = 0, kSpilledF = 1, kReadF = 2, kConsumedF = 3 };

uint32_t* cflag_ptr(Cascade* c, CFlag f, int i) {
  const int K = c->dram_slots;
  const int base = f == kCopiedF ? 0 : f == kSpilledF ? K : f == kReadF ? 2 * K : 2 * K + kRing;
  return c->flags + 4 * (base + i);
}
volatile uint32_t& cflag(Cascade* c, CFlag f, int i) { return *reinterpret_cast<volatile uint32_t*>(cflag_ptr(c, f, i)); }

bool cwait(Cascade* c, CFlag f, int i, uint32_t v) {
  for (int n = 0; int32_t(cflag(c, f, i) - v) < 0; ++n) {
    if (c->abort.load(std::memory_order_relaxed)) return false;
    if (n > 4096) std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  return true;
}
void cset(Cascade* c, CFlag f, int i, uint32_t v) {
  std::atomic_thread_fence(std::memory_order_release);
  cflag(c, f, i) = v;
}

CUdeviceptr cflag_dev(Cascade* c, CFlag f, int i) {
  void* d = nullptr;
  ACKPT_CUDA_CHECK(cudaHostGetDevicePointer(&d, cflag_ptr(c, f, i), 0));
  return CUdeviceptr(reinterpret_cast<uintptr_t>(d));
}
void c_stream_wait(ackpt_tier* t, cudaStream_t s, CFlag f, int i, uint32_t v) {
  if (t->wait_value(reinterpret_cast<CUstream>(s), cflag_dev(t->cascade, f, i), v, CU_STREAM_WAIT_VALUE_GEQ) !=
      CUDA_SUCCESS)
    fail(ACKPT_CUDA_ERROR, "cuStreamWaitValue32 failed");
}
void c_stream_write(ackpt_tier* t, cudaStream_t s, CFlag f, int i, uint32_t v) {
  if (t->write_value(reinterpret_cast<CUstream>(s), cflag_dev(t->cascade, f, i), v, CU_STREAM_WRITE_VALUE_DEFAULT) !=
      CUDA_SUCCESS)
    fail(ACKPT_CUDA_ERROR, "cuStreamWriteValue32 failed");
}

// O_DIRECT I/O of a kDirectAlign-padded image, split over worker threads;
// returns 0 or the first errno.
int direct_io(int fd, unsigned char* buf, int64_t bytes, bool write) {
  const int threads = std::max(1, io_threads(bytes));
  const int64_t chunk = ((bytes + threads - 1) / threads + kDirectAlign - 1) / kDirectAlign * kDirectAlign;
  std::vector<int> errs(size_t(threads), 0);
  auto work = [&](int i) {
    const int64_t lo = int64_t(i) * chunk, hi = std::min(bytes, lo + chunk);
    for (int64_t off = lo; off < hi;) {
      const ssize_t r = write ? ::pwrite(fd, buf + off, size_t(hi - off), off_t(off))
                              : ::pread(fd, buf + off, size_t(hi - off), off_t(off));
      if (r < 0 && errno == EINTR) continue;
      if (r < 0) {
        errs[size_t(i)] = errno;
        return;
      }
      if (r == 0) return;  // read: end of file (the image's padding)
      off += r;
    }
  };
  std::vector<std::thread> pool;
  for (int i = 1; i < threads && int64_t(i) * chunk < bytes; ++i) pool.emplace_back(work, i);
  work(0);
  for (auto& th : pool) th.join();
  for (int e : errs)
    if (e) return e;
  return 0;
}

uint32_t parallel_crc_raw(const unsigned char* p, int64_t len, uint32_t reg) {
  const int threads = std::max(1, io_threads(len));
  if (threads == 1 || len < (int64_t(4) << 20)) return crc32c_raw(p, len, reg);
  const int64_t chunk = (len + threads - 1) / threads;
  std::vector<uint32_t> part(size_t(threads), 0);
  std::vector<std::thread> pool;
  auto work = [&](int i) {
    const int64_t lo = int64_t(i) * chunk, hi = std::min(len, lo + chunk);
    if (lo < hi) part[size_t(i)] = crc32c_raw(p + lo, hi - lo, 0);
  };
  for (int i = 1; i < threads; ++i) pool.emplace_back(work, i);
  work(0);
  for (auto& th : pool) th.join();
  for (int i = 0; i < threads; ++i) {
    const int64_t lo = int64_t(i) * chunk, hi = std::min(len, lo + chunk);
    if (lo < hi) reg = crc32c_shift(reg, hi - lo) ^ part[size_t(i)];
  }
  return reg;
}

// Writes the slot's image as <dir>/ckpt_<key>.bin; 0 or errno.
int spill_write(ackpt_tier* t, const SpillJob& j, double* seconds) {
  Cascade* c = t->cascade;
  unsigned char* img = c->slot_mem[size_t(j.slot)];
  std::memcpy(img, "CKPT", 4);
  put_le(img + 4, 1, 2);
  put_le(img + 6, uint64_t(j.step), 8);
  put_le(img + 14, uint64_t(j.len), 8);
  const auto t0 = std::chrono::steady_clock::now();
  const uint32_t reg = parallel_crc_raw(img, kHeader + j.len, 0xFFFFFFFFu);
  put_le(img + kHeader + j.len, reg ^ 0xFFFFFFFFu, 4);
  const int64_t exact = kHeader + j.len + kTrailer;
  const int64_t padded = (exact + kDirectAlign - 1) / kDirectAlign * kDirectAlign;
  std::memset(img + exact, 0, size_t(padded - exact));
  const std::string path = ckpt_path(t, j.key), tmp = path + ".tmp";
  int fd = ::open(tmp.c_str(), O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC | O_DIRECT, 0644);
  if (fd < 0 && errno == EINVAL) fd = ::open(tmp.c_str(), O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
  if (fd < 0) return errno;
  int err = direct_io(fd, img, padded, true);
  if (!err && ::ftruncate(fd, off_t(exact)) != 0) err = errno;
  if (::close(fd) != 0 && !err) err = errno;
  if (err) {
    ::unlink(tmp.c_str());
    return err;
  }
  if (::renameat2(AT_FDCWD, tmp.c_str(), AT_FDCWD, path.c_str(), RENAME_EXCHANGE) == 0) {
    ::unlink(tmp.c_str());  // the previous version (same name exchange: O_DIRECT data, no writeback)
  } else if (std::rename(tmp.c_str(), path.c_str()) != 0) {
    err = errno;
    ::unlink(tmp.c_str());
  }
  *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return err;
}

void spill_worker(ackpt_tier* t) {
  Cascade* c = t->cascade;
  for (;;) {
    SpillJob j;
    {
      std::unique_lock<std::mutex> lk(c->qmu);
      c->qcv.wait(lk, [&] { return c->stop || !c->spill_q.empty(); });
      if (c->spill_q.empty()) return;
      j = c->spill_q.front();
      c->spill_q.pop_front();
      ++c->busy;
    }
    double secs = 0.0;
    int err = 0;
    if (cwait(c, kCopiedF, j.slot, j.copied)) err = spill_write(t, j, &secs);
    else err = ECANCELED;
    {
      std::lock_guard<std::mutex> lk(t->mu);
      auto it = c->keys.find(j.key);
      if (it != c->keys.end() && it->second.version == j.version) {
        if (err) {
          it->second.err = err == ENOSPC ? ACKPT_STORAGE_FULL : ACKPT_EXECUTION_ERROR;
          it->second.msg = "spilling " + ckpt_path(t, j.key) + ": " + std::strerror(err);
        } else {
          it->second.on_file = true;
        }
      }
      if (!err) {
        ++c->stats.spills;
        c->stats.spill_bytes += j.len;
        c->stats.spill_seconds += secs;
      }
    }
    {
      std::lock_guard<std::mutex> lk(c->qmu);
      cset(c, kSpilledF, j.slot, j.gen);  // always: a D2H copy may wait on it
      --c->busy;
    }
    c->qcv.notify_all();
  }
}

// Read + verify <dir>/ckpt_<key>.bin into ring buffer j.buf (read_ckpt's
// checks: size, magic, version, length, CRC32C, step).
void read_job(ackpt_tier* t, const ReadJob& j) {
  Cascade* c = t->cascade;
  const std::string path = ckpt_path(t, j.key);
  unsigned char* img = c->ring_mem[size_t(j.buf)];
  const auto t0 = std::chrono::steady_clock::now();
  int fd = ::open(path.c_str(), O_RDONLY | O_CLOEXEC | O_DIRECT);
  if (fd < 0 && errno == EINVAL) fd = ::open(path.c_str(), O_RDONLY | O_CLOEXEC);
  if (fd < 0) {
    set_async(*j.status, ACKPT_MISSING_KEY, path);
    return;
  }
  struct stat sb;
  const int64_t size = ::fstat(fd, &sb) == 0 ? int64_t(sb.st_size) : -1;
  auto bad = [&](const std::string& why) {
    ::close(fd);
    set_async(*j.status, ACKPT_CHECKSUM_MISMATCH, path + ": " + why);
  };
  if (size < kHeader + kTrailer) return bad("checkpoint truncated: " + std::to_string(size) + " bytes");
  if (size > c->image_bytes) return bad("payload size changed");
  const int64_t padded = (size + kDirectAlign - 1) / kDirectAlign * kDirectAlign;
  const int err = direct_io(fd, img, padded, false);
  ::close(fd);
  if (err) {
    set_async(*j.status, ACKPT_CHECKSUM_MISMATCH, path + ": short read: " + std::strerror(err));
    return;
  }
  if (std::memcmp(img, "CKPT", 4) != 0) return set_async(*j.status, ACKPT_CHECKSUM_MISMATCH, path + ": bad magic bytes");
  if (get_le(img + 4, 2) != 1) return set_async(*j.status, ACKPT_CHECKSUM_MISMATCH, path + ": unsupported format version");
  const int64_t length = int64_t(get_le(img + 14, 8));
  if (length + kHeader + kTrailer != size || length != j.len)
    return set_async(*j.status, ACKPT_CHECKSUM_MISMATCH, path + ": length field says " + std::to_string(length));
  const uint32_t reg = parallel_crc_raw(img, kHeader + length, 0xFFFFFFFFu);
  if ((reg ^ 0xFFFFFFFFu) != uint32_t(get_le(img + kHeader + length, 4)))
    return set_async(*j.status, ACKPT_CHECKSUM_MISMATCH, path + ": crc mismatch");
  if (int64_t(get_le(img + 6, 8)) != j.key)
    return set_async(*j.status, ACKPT_CHECKSUM_MISMATCH, path + ": file holds another step");
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::lock_guard<std::mutex> lk(t->mu);
  ++c->stats.reads;
  c->stats.read_bytes += length;
  c->stats.read_seconds += secs;
}

void read_worker(ackpt_tier* t) {
  Cascade* c = t->cascade;
  for (;;) {
    ReadJob j;
    {
      std::unique_lock<std::mutex> lk(c->qmu);
      c->qcv.wait(lk, [&] { return c->stop || !c->read_q.empty(); });
      if (c->read_q.empty()) return;
      j = c->read_q.front();
      c->read_q.pop_front();
      ++c->busy;
    }
    bool ok = cwait(c, kConsumedF, j.buf, j.need_consumed);  // the previous occupant was copied out
    if (ok && j.spill_slot >= 0) ok = cwait(c, kSpilledF, j.spill_slot, j.spill_gen);  // its file is complete
    if (ok) read_job(t, j);
    else set_async(*j.status, ACKPT_EXECUTION_ERROR, "cascade tier shut down");
    {
      std::lock_guard<std::mutex> lk(c->qmu);
      cset(c, kReadF, j.buf, j.gen);  // always: the H2D copy waits on it
      --c->busy;
    }
    c->qcv.notify_all();
  }
}

void cascade_drain(ackpt_tier* t) {
  Cascade* c = t->cascade;
  std::unique_lock<std::mutex> lk(c->qmu);
  c->qcv.wait(lk, [&] { return c->spill_q.empty() && c->read_q.empty() && c->busy == 0; });
}

void enqueue_spill(ackpt_tier* t, int64_t key, CascadeKey& k) {
  Cascade* c = t->cascade;
  const int s = k.slot;
  const uint32_t gen = ++c->spill_gen_issued[size_t(s)];
  k.spill_gen = gen;
  k.spill_slot = s;
  {
    std::lock_guard<std::mutex> lk(c->qmu);
    c->spill_q.push_back({key, k.step, k.len, s, c->copy_gen[size_t(s)], gen, k.version});
  }
  c->qcv.notify_all();
}

// Keep up to dram_slots - kSpillMargin resident keys without a spill issued.
void spill_ahead(ackpt_tier* t) {
  Cascade* c = t->cascade;
  for (;;) {
    int dirty = 0;
    CascadeKey* oldest = nullptr;
    int64_t oldest_key = 0;
    for (int s = 0; s < c->dram_slots; ++s) {
      const int64_t key = c->slot_key[size_t(s)];
      if (key < 0) continue;
      CascadeKey& k = c->keys[key];
      if (k.spill_gen != 0 && k.spill_slot == s) continue;
      ++dirty;
      if (!oldest || k.order < oldest->order) {
        oldest = &k;
        oldest_key = key;
      }
    }
    if (dirty <= c->dram_slots - kSpillMargin || !oldest) return;
    enqueue_spill(t, oldest_key, *oldest);
  }
}

// A DRAM slot for a new copy; the returned slot's previous occupant (if any)
// is evicted, and *wait_spill / *wait_fetch say what its D2H copy must wait for.
int acquire_slot(ackpt_tier* t, int64_t key, uint32_t* wait_spill) {
  Cascade* c = t->cascade;
  *wait_spill = 0;
  CascadeKey& self = c->keys[key];
  if (self.slot >= 0) {  // re-store of a resident key: same slot, after its spill (if any) read it
    const int s = self.slot;
    if (self.spill_gen != 0 && self.spill_slot == s) *wait_spill = self.spill_gen;
    return s;
  }
  for (int s = 0; s < c->dram_slots; ++s)
    if (c->slot_key[size_t(s)] < 0) return s;
  // evict the oldest resident key; it must be spilled first
  int victim = -1;
  for (int s = 0; s < c->dram_slots; ++s) {
    const CascadeKey& k = c->keys[c->slot_key[size_t(s)]];
    if (victim < 0 || k.order < c->keys[c->slot_key[size_t(victim)]].order) victim = s;
  }
  const int64_t vkey = c->slot_key[size_t(victim)];
  CascadeKey& v = c->keys[vkey];
  if (!(v.spill_gen != 0 && v.spill_slot == victim)) enqueue_spill(t, vkey, v);
  *wait_spill = v.spill_gen;
  v.slot = -1;
  c->slot_key[size_t(victim)] = -1;
  return victim;
}

}  // namespace

void cascade_create(ackpt_tier* t, int dram_slots) {
  if (dram_slots < kSpillMargin + 2) fail(ACKPT_VALUE_ERROR, "cascade tier needs at least 4 DRAM slots");
  std::unique_ptr<Cascade> c(new Cascade());
  c->dram_slots = dram_slots;
  c->image_bytes = (kHeader + t->slot_bytes + kTrailer + kDirectAlign - 1) / kDirectAlign * kDirectAlign;
  void* w = nullptr;
  void* v = nullptr;
  cudaDriverEntryPointQueryResult q1, q2;
  if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &w, cudaEnableDefault, &q1) != cudaSuccess ||
      cudaGetDriverEntryPoint("cuStreamWriteValue32", &v, cudaEnableDefault, &q2) != cudaSuccess ||
      q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess || !w || !v) {
    cudaGetLastError();
    fail(ACKPT_CUDA_ERROR, "cascade tier needs cuStreamWaitValue32 / cuStreamWriteValue32");
  }
  t->wait_value = reinterpret_cast<CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned)>(w);
  t->write_value = reinterpret_cast<CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned)>(v);
  const size_t nflags = size_t(2 * dram_slots + 2 * kRing) * 16;
  ACKPT_CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&c->flags), nflags, cudaHostAllocMapped));
  std::memset(c->flags, 0, nflags);
  auto alloc = [&](std::vector<unsigned char*>& v2, int count) {
    for (int i = 0; i < count; ++i) {
      unsigned char* p = nullptr;
      if (cudaHostAlloc(reinterpret_cast<void**>(&p), size_t(c->image_bytes), cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        fail(ACKPT_STORAGE_FULL, "pinned host allocation of the cascade tier failed");
      }
      v2.push_back(p);  // page aligned: O_DIRECT-able
    }
  };
  t->cascade = c.get();  // visible to cleanup on failure below
  try {
    alloc(c->slot_mem, dram_slots);
    alloc(c->ring_mem, kRing);
    c->slot_key.assign(size_t(dram_slots), -1);
    c->copy_gen.assign(size_t(dram_slots), 0);
    c->spill_gen_issued.assign(size_t(dram_slots), 0);
    c->read_gen.assign(size_t(kRing), 0);
    c->slot_store_ev.assign(size_t(dram_slots), nullptr);
    c->slot_fetch_ev.assign(size_t(dram_slots), nullptr);
    c->slot_fetched.assign(size_t(dram_slots), false);
    for (int s = 0; s < dram_slots; ++s) {
      ACKPT_CUDA_CHECK(cudaEventCreateWithFlags(&c->slot_store_ev[size_t(s)], cudaEventDisableTiming));
      ACKPT_CUDA_CHECK(cudaEventCreateWithFlags(&c->slot_fetch_ev[size_t(s)], cudaEventDisableTiming));
    }
  } catch (...) {
    for (auto p : c->slot_mem) cudaFreeHost(p);
    for (auto p : c->ring_mem) cudaFreeHost(p);
    for (auto e : c->slot_store_ev) if (e) cudaEventDestroy(e);
    for (auto e : c->slot_fetch_ev) if (e) cudaEventDestroy(e);
    cudaFreeHost(c->flags);
    t->cascade = nullptr;
    throw;
  }
  c->spill_thr = std::thread(spill_worker, t);
  c->read_thr = std::thread(read_worker, t);
  t->cascade_slots = dram_slots;
  c.release();
}

void cascade_destroy(ackpt_tier* t) {
  Cascade* c = t->cascade;
  if (!c) return;
  cascade_drain(t);  // queued spills complete, like the reference worker before its sentinel (storage.py:258-263)
  {
    std::lock_guard<std::mutex> lk(c->qmu);
    c->stop = true;
  }
  c->qcv.notify_all();
  c->abort.store(true);  // the streams were drained: only a failed stream leaves a flag behind
  if (c->spill_thr.joinable()) c->spill_thr.join();
  if (c->read_thr.joinable()) c->read_thr.join();
  for (auto p : c->slot_mem) cudaFreeHost(p);
  for (auto p : c->ring_mem) cudaFreeHost(p);
  for (auto e : c->slot_store_ev) cudaEventDestroy(e);
  for (auto e : c->slot_fetch_ev) cudaEventDestroy(e);
  cudaFreeHost(c->flags);
  delete c;
  t->cascade = nullptr;
}

void cascade_quiesce(ackpt_tier* t) {
  ACKPT_CUDA_CHECK(cudaStreamSynchronize(t->d2h));
  ACKPT_CUDA_CHECK(cudaStreamSynchronize(t->h2d));
  cascade_drain(t);
}

ackpt_ticket cascade_begin_store(ackpt_tier* t, int64_t key, int64_t step, const void* src, int64_t bytes,
                                 void* after_stream) {
  Cascade* c = t->cascade;
  if (capturing(after_stream)) fail(ACKPT_VALUE_ERROR, "the cascade tier cannot be captured into a CUDA graph");
  TierTicket tk;
  tk.kind = 0;
  tk.key = key;
  tk.step = step;
  if (bytes > t->slot_bytes) {
    tk.err = ACKPT_SIZE_MISMATCH;
    tk.msg = "payload of " + std::to_string(bytes) + " bytes exceeds the cascade slot (" +
             std::to_string(t->slot_bytes) + ")";
    tk.complete = true;
    return add_ticket(t, std::move(tk));
  }
  uint32_t wait_spill = 0;
  const int s = acquire_slot(t, key, &wait_spill);
  CascadeKey& k = c->keys[key];
  if (after_stream) {
    ACKPT_CUDA_CHECK(cudaEventRecord(t->after, static_cast<cudaStream_t>(after_stream)));
    ACKPT_CUDA_CHECK(cudaStreamWaitEvent(t->d2h, t->after, 0));
  }
  if (wait_spill) c_stream_wait(t, t->d2h, kSpilledF, s, wait_spill);  // the old image is on file
  if (c->slot_fetched[size_t(s)]) ACKPT_CUDA_CHECK(cudaStreamWaitEvent(t->d2h, c->slot_fetch_ev[size_t(s)], 0));
  cudaEvent_t m0 = mark(t, t->d2h);
  if (bytes > 0)
    ACKPT_CUDA_CHECK(cudaMemcpyAsync(c->slot_mem[size_t(s)] + kHeader, src, size_t(bytes), cudaMemcpyDeviceToHost,
                                     t->d2h));
  c_stream_write(t, t->d2h, kCopiedF, s, ++c->copy_gen[size_t(s)]);
  ACKPT_CUDA_CHECK(cudaEventRecord(c->slot_store_ev[size_t(s)], t->d2h));
  c->slot_key[size_t(s)] = key;
  c->slot_fetched[size_t(s)] = false;
  k.slot = s;
  k.step = step;
  k.len = bytes;
  ++k.version;
  k.order = ++c->order;
  k.spill_gen = 0;
  k.spill_slot = -1;
  k.on_file = false;
  k.stored = true;
  k.err = ACKPT_OK;
  k.msg.clear();
  for (auto& r : c->ring)  // a read-ahead of the old version is stale
    if (r.key == key) r.key = -1;
  ackpt_ticket id = add_ticket(t, std::move(tk));
  TierTicket& ref = *find_ticket(t, id);
  ref.done = new_event(t);
  ACKPT_CUDA_CHECK(cudaEventRecord(ref.done, t->d2h));
  ref.t0 = m0;
  ref.t1 = mark(t, t->d2h);
  spill_ahead(t);
  return id;
}

namespace {

// Ring buffer holding (or about to hold) `key`'s current version; issues the
// read if needed.  Returns the buffer index.
int ring_load(ackpt_tier* t, int64_t key, const CascadeKey* k, int64_t len) {
  Cascade* c = t->cascade;
  const uint32_t version = k ? k->version : 0;
  for (int b = 0; b < kRing; ++b)
    if (c->ring[b].key == key && c->ring[b].version == version && c->ring[b].gen) return b;
  // the least recently issued occupancy
  const int b = c->ring_next;
  c->ring_next = (c->ring_next + 1) % kRing;
  RingEntry& e = c->ring[b];
  const uint32_t prev = c->read_gen[size_t(b)];
  if (prev && !e.fetched) cset(c, kConsumedF, b, prev);  // an unused read-ahead: nothing will copy it out
  e.key = key;
  e.version = version;
  e.gen = ++c->read_gen[size_t(b)];
  e.fetched = false;
  e.status = std::make_shared<AsyncStatus>();
  ReadJob j;
  j.key = key;
  j.len = len;
  j.buf = b;
  j.gen = e.gen;
  j.need_consumed = prev;
  j.spill_slot = k ? k->spill_slot : -1;
  j.spill_gen = k ? k->spill_gen : 0;
  j.status = e.status;
  {
    std::lock_guard<std::mutex> lk(c->qmu);
    c->read_q.push_back(j);
  }
  c->qcv.notify_all();
  return b;
}

// Up to two spilled keys below `key`, nearest first: NVMe -> DRAM ahead of their fetch.
void read_ahead(ackpt_tier* t, int64_t key) {
  Cascade* c = t->cascade;
  std::vector<int64_t> below;
  for (auto& kv : c->keys)
    if (kv.first < key && kv.second.stored && kv.second.slot < 0 && kv.second.spill_gen && kv.second.err == ACKPT_OK)
      below.push_back(kv.first);
  std::sort(below.begin(), below.end(), std::greater<int64_t>());
  for (size_t i = 0; i < below.size() && i < size_t(kRing - 1); ++i) {
    const CascadeKey& k = c->keys[below[i]];
    ring_load(t, below[i], &k, k.len);
  }
}

}  // namespace

ackpt_ticket cascade_begin_fetch(ackpt_tier* t, int64_t key, void* dst, int64_t bytes, void* after_stream) {
  Cascade* c = t->cascade;
  if (capturing(after_stream)) fail(ACKPT_VALUE_ERROR, "the cascade tier cannot be captured into a CUDA graph");
  TierTicket tk;
  tk.kind = 1;
  tk.key = key;
  auto it = c->keys.find(key);
  const CascadeKey* k = (it != c->keys.end() && it->second.stored) ? &it->second : nullptr;
  int64_t len = -1;
  std::string why;
  if (k) len = k->len;
  else len = file_payload_len(t, key, &why);  // resume from a file of an earlier run
  auto done_with = [&](int code, const std::string& msg) {
    tk.err = code;
    tk.msg = msg;
    tk.complete = true;
    return add_ticket(t, std::move(tk));
  };
  if (len == -1) return done_with(ACKPT_MISSING_KEY, ckpt_path(t, key));
  if (len < 0) return done_with(ACKPT_CHECKSUM_MISMATCH, why);
  if (len > t->slot_bytes) return done_with(ACKPT_SIZE_MISMATCH, "key " + std::to_string(key) + " exceeds the slot");
  if (bytes >= 0 && bytes < len)
    return done_with(ACKPT_SIZE_MISMATCH, "destination holds " + std::to_string(bytes) + " bytes, key " +
                                              std::to_string(key) + " holds " + std::to_string(len));
  if (k && k->err != ACKPT_OK) return done_with(k->err, k->msg);
  tk.step = k ? k->step : key;
  if (after_stream) {
    ACKPT_CUDA_CHECK(cudaEventRecord(t->after, static_cast<cudaStream_t>(after_stream)));
    ACKPT_CUDA_CHECK(cudaStreamWaitEvent(t->h2d, t->after, 0));
  }
  std::shared_ptr<AsyncStatus> status;
  cudaEvent_t m0 = nullptr;
  if (k && k->slot >= 0) {  // resident: one H2D copy from the slot
    const int s = k->slot;
    ACKPT_CUDA_CHECK(cudaStreamWaitEvent(t->h2d, c->slot_store_ev[size_t(s)], 0));
    m0 = mark(t, t->h2d);
    if (len > 0)
      ACKPT_CUDA_CHECK(
          cudaMemcpyAsync(dst, c->slot_mem[size_t(s)] + kHeader, size_t(len), cudaMemcpyHostToDevice, t->h2d));
    ACKPT_CUDA_CHECK(cudaEventRecord(c->slot_fetch_ev[size_t(s)], t->h2d));
    c->slot_fetched[size_t(s)] = true;
    ++c->stats.dram_hits;
  } else {  // from the file, through a ring buffer (often read ahead already)
    bool hit = false;
    for (auto& r : c->ring)
      hit = hit || (r.key == key && r.version == (k ? k->version : 0) && r.gen);
    ++(hit ? c->stats.ring_hits : c->stats.ring_misses);
    const int b = ring_load(t, key, k, len);
    RingEntry& e = c->ring[b];
    c_stream_wait(t, t->h2d, kReadF, b, e.gen);
    m0 = mark(t, t->h2d);
    if (len > 0)
      ACKPT_CUDA_CHECK(cudaMemcpyAsync(dst, c->ring_mem[size_t(b)] + kHeader, size_t(len), cudaMemcpyHostToDevice,
                                       t->h2d));
    c_stream_write(t, t->h2d, kConsumedF, b, e.gen);
    e.fetched = true;
    status = e.status;
    e.key = -1;  // consumed: the buffer may be refilled after the copy
  }
  ackpt_ticket id = add_ticket(t, std::move(tk));
  TierTicket& ref = *find_ticket(t, id);
  ref.async = status;
  ref.done = new_event(t);
  ACKPT_CUDA_CHECK(cudaEventRecord(ref.done, t->h2d));
  ref.t0 = m0;
  ref.t1 = mark(t, t->h2d);
  if (k) read_ahead(t, key);
  return id;
}

bool cascade_contains(ackpt_tier* t, int64_t key) {
  auto it = t->cascade->keys.find(key);
  if (it != t->cascade->keys.end() && it->second.stored) return true;
  return file_payload_len(t, key) != -1;
}

int64_t cascade_key_bytes(ackpt_tier* t, int64_t key) {
  auto it = t->cascade->keys.find(key);
  if (it != t->cascade->keys.end() && it->second.stored) return it->second.len;
  std::string why;
  const int64_t len = file_payload_len(t, key, &why);
  if (len == -1) fail(ACKPT_MISSING_KEY, ckpt_path(t, key));
  if (len < 0) fail(ACKPT_CHECKSUM_MISMATCH, why);
  return len;
}

void* cascade_host_ptr(ackpt_tier* t, int64_t key) {
  auto it = t->cascade->keys.find(key);
  if (it == t->cascade->keys.end() || !it->second.stored) fail(ACKPT_MISSING_KEY, "key " + std::to_string(key) + " never stored");
  if (it->second.slot < 0) fail(ACKPT_VALUE_ERROR, "key " + std::to_string(key) + " was spilled to " + ckpt_path(t, key));
  return t->cascade->slot_mem[size_t(it->second.slot)] + kHeader;
}

void cascade_clear(ackpt_tier* t) {
  Cascade* c = t->cascade;
  for (int b = 0; b < kRing; ++b) {
    if (c->read_gen[size_t(b)]) cset(c, kConsumedF, b, c->read_gen[size_t(b)]);
    c->ring[b] = RingEntry{};
  }
  std::fill(c->slot_key.begin(), c->slot_key.end(), -1);
  std::fill(c->slot_fetched.begin(), c->slot_fetched.end(), false);
  c->keys.clear();
}

// Seconds to spill (CRC + O_DIRECT write + publish) one payload of `bytes`
// from a free ring buffer; the probe file is removed again.
double cascade_spill_probe(ackpt_tier* t, int64_t bytes) {
  Cascade* c = t->cascade;
  cascade_drain(t);
  ACKPT_CUDA_CHECK(cudaStreamSynchronize(t->h2d));
  const int b = 0;
  if (c->read_gen[size_t(b)]) cset(c, kConsumedF, b, c->read_gen[size_t(b)]);
  c->ring[b] = RingEntry{};
  unsigned char* img = c->ring_mem[size_t(b)];
  std::memset(img + kHeader, 0x5A, size_t(bytes));
  const std::string path = t->dir + "/ckpt_probe.tmp";
  const auto t0 = std::chrono::steady_clock::now();
  put_le(img + 14, uint64_t(bytes), 8);
  const uint32_t reg = parallel_crc_raw(img, kHeader + bytes, 0xFFFFFFFFu);
  put_le(img + kHeader + bytes, reg, 4);
  const int64_t padded = (kHeader + bytes + kTrailer + kDirectAlign - 1) / kDirectAlign * kDirectAlign;
  int fd = ::open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC | O_DIRECT, 0644);
  if (fd < 0 && errno == EINVAL) fd = ::open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
  if (fd < 0) fail(ACKPT_EXECUTION_ERROR, "cascade probe: " + std::string(std::strerror(errno)));
  const int err = direct_io(fd, img, padded, true);
  ::close(fd);
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  ::unlink(path.c_str());
  if (err) fail(err == ENOSPC ? ACKPT_STORAGE_FULL : ACKPT_EXECUTION_ERROR, "cascade probe: " + std::string(std::strerror(err)));
  return secs;
}

}  // namespace ackpt

extern "C" {

ACKPT_API int ackpt_tier_create_cascade(const char* directory, int64_t slot_bytes, int32_t dram_slots,
                                        ackpt_tier** out) {
  int rc = ackpt_tier_create(0, slot_bytes > 0 ? slot_bytes : 1, out);
  if (rc != ACKPT_OK) return rc;
  rc = ackpt::guard([&] {
    ackpt_tier* t = *out;
    t->dir = directory ? directory : ".";
    ackpt::cascade_create(t, dram_slots);
  });
  if (rc != ACKPT_OK) {
    ackpt_tier_destroy(*out);
    *out = nullptr;
  }
  return rc;
}

ACKPT_API int ackpt_tier_cascade_stats(ackpt_tier* t, ackpt_cascade_stats* out) {
  return ackpt::guard([&] {
    if (!t->cascade) ackpt::fail(ACKPT_VALUE_ERROR, "not a cascade tier");
    std::lock_guard<std::mutex> lk(t->mu);
    const ackpt::CascadeStats& s = t->cascade->stats;
    out->dram_slots = t->cascade->dram_slots;
    out->spills = s.spills;
    out->spill_bytes = s.spill_bytes;
    out->spill_seconds = s.spill_seconds;
    out->reads = s.reads;
    out->read_bytes = s.read_bytes;
    out->read_seconds = s.read_seconds;
    out->dram_hits = s.dram_hits;
    out->ring_hits = s.ring_hits;
    out->ring_misses = s.ring_misses;
  });
}

}  // extern "C"
