// CRC32C (Castagnoli), bit-compatible with the reference's table-driven
// crc32c(data, crc) (storage.py:49-68): reflected polynomial 0x82F63B78,
// initial and final xor 0xFFFFFFFF, chaining through the crc argument.
//
// Speed (the file stage checksums every stored / fetched state):
// * the SSE4.2 crc32 instruction has 3-cycle latency and 1/cycle throughput,
//   so long buffers run three independent chains over adjacent thirds and
//   merge them;
// * merging uses linearity of the raw (unconditioned) CRC register:
//     raw(A || B, r) = shift(raw(A, r), |B|) xor raw(B, 0),
//   shift(r, n) = r * x^(8n) mod P in the reflected GF(2) representation,
//   with x^(2^k) mod P tabulated (the standard combine construction);
//   Attribution: mulmod / the x^(2^k) table / the shift below follow zlib's
//   multmodp / x2nmodp / crc32_combine (Mark Adler, zlib license), adapted
//   to the Castagnoli polynomial;
// * crc32c_parallel splits a buffer over worker threads the same way.
// Without SSE4.2 a slicing-by-8 table is used.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "common.h"

#if defined(__x86_64__)
#include <cpuid.h>
#include <nmmintrin.h>
#endif

namespace {

constexpr uint32_t kPoly = 0x82F63B78u;

struct Tables {
  uint32_t t[8][256];
  uint32_t x2n[64];  // x^(2^k) mod P
  Tables() {
    for (uint32_t b = 0; b < 256; ++b) {
      uint32_t c = b;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ kPoly : c >> 1;
      t[0][b] = c;
    }
    for (uint32_t b = 0; b < 256; ++b)
      for (int s = 1; s < 8; ++s) t[s][b] = (t[s - 1][b] >> 8) ^ t[0][t[s - 1][b] & 0xFF];
    x2n[0] = 1u << 30;  // x^1 (bit 31 is x^0 in the reflected form)
    for (int k = 1; k < 64; ++k) x2n[k] = mulmod(x2n[k - 1], x2n[k - 1]);
  }
  // a * b mod P, reflected: bit 31 is the x^0 coefficient.
  static uint32_t mulmod(uint32_t a, uint32_t b) {
    uint32_t m = 1u << 31, p = 0;
    for (;;) {
      if (a & m) {
        p ^= b;
        if ((a & (m - 1)) == 0) break;
      }
      m >>= 1;
      b = (b & 1) ? (b >> 1) ^ kPoly : b >> 1;
    }
    return p;
  }
};

const Tables& tables() {
  static Tables tb;
  return tb;
}

// x^(8 n) mod P
uint32_t x8n(int64_t n) {
  const auto& T = tables();
  uint32_t p = 1u << 31;
  for (int k = 3; n > 0; n >>= 1, ++k)
    if (n & 1) p = Tables::mulmod(T.x2n[k & 63], p);
  return p;
}

uint32_t crc_sw(const unsigned char* p, int64_t n, uint32_t c) {
  const auto& T = tables().t;
  while (n >= 8) {
    uint64_t v;
    std::memcpy(&v, p, 8);
    v ^= c;
    c = T[7][v & 0xFF] ^ T[6][(v >> 8) & 0xFF] ^ T[5][(v >> 16) & 0xFF] ^ T[4][(v >> 24) & 0xFF] ^
        T[3][(v >> 32) & 0xFF] ^ T[2][(v >> 40) & 0xFF] ^ T[1][(v >> 48) & 0xFF] ^ T[0][v >> 56];
    p += 8;
    n -= 8;
  }
  while (n-- > 0) c = (c >> 8) ^ T[0][(c ^ *p++) & 0xFF];
  return c;
}

#if defined(__x86_64__)
__attribute__((target("sse4.2"))) uint32_t crc_hw1(const unsigned char* p, int64_t n, uint32_t c) {
  uint64_t c64 = c;
  while (n >= 8) {
    uint64_t v;
    std::memcpy(&v, p, 8);
    c64 = _mm_crc32_u64(c64, v);
    p += 8;
    n -= 8;
  }
  uint32_t c32 = uint32_t(c64);
  while (n-- > 0) c32 = _mm_crc32_u8(c32, *p++);
  return c32;
}

// Three chains over adjacent thirds (multiples of 8 bytes), merged.
__attribute__((target("sse4.2"))) uint32_t crc_hw(const unsigned char* p, int64_t n, uint32_t c) {
  if (n < 3 * 4096) return crc_hw1(p, n, c);
  const int64_t m = (n / 3) & ~int64_t(7);
  const unsigned char *a = p, *b = p + m, *d = p + 2 * m;
  uint64_t ca = c, cb = 0, cd = 0;
  for (int64_t i = 0; i < m; i += 8) {
    uint64_t va, vb, vd;
    std::memcpy(&va, a + i, 8);
    std::memcpy(&vb, b + i, 8);
    std::memcpy(&vd, d + i, 8);
    ca = _mm_crc32_u64(ca, va);
    cb = _mm_crc32_u64(cb, vb);
    cd = _mm_crc32_u64(cd, vd);
  }
  const uint32_t sh = x8n(m);
  uint32_t r = Tables::mulmod(sh, uint32_t(ca)) ^ uint32_t(cb);
  r = Tables::mulmod(sh, r) ^ uint32_t(cd);
  return crc_hw1(p + 3 * m, n - 3 * m, r);
}

bool have_sse42() {
  unsigned a, b, c, d;
  if (!__get_cpuid(1, &a, &b, &c, &d)) return false;
  return (c & bit_SSE4_2) != 0;
}
#endif

}  // namespace

namespace ackpt {

uint32_t crc32c_raw(const void* data, int64_t len, uint32_t reg) {
  const auto* p = static_cast<const unsigned char*>(data);
#if defined(__x86_64__)
  static const bool hw = have_sse42();
  return hw ? crc_hw(p, len, reg) : crc_sw(p, len, reg);
#else
  return crc_sw(p, len, reg);
#endif
}

int io_threads(int64_t len) {
  static const int hw = int(std::thread::hardware_concurrency());
  static const int cap = [] {  // ACKPT_IO_THREADS: probe override of the worker cap
    const char* e = std::getenv("ACKPT_IO_THREADS");
    return e ? std::max(1, std::atoi(e)) : 8;
  }();
  const int64_t by_size = len / (int64_t(4) << 20);  // >= 4 MiB per worker
  return int(std::max<int64_t>(1, std::min<int64_t>({by_size, int64_t(cap), hw > 0 ? hw : 1})));
}

uint32_t crc32c_shift(uint32_t reg, int64_t len) { return len > 0 ? Tables::mulmod(x8n(len), reg) : reg; }

uint32_t crc32c_parallel(const void* data, int64_t len, uint32_t crc, int threads) {
  const auto* p = static_cast<const unsigned char*>(data);
  uint32_t reg = crc ^ 0xFFFFFFFFu;
  if (threads <= 1 || len < (int64_t(4) << 20)) return crc32c_raw(p, len, reg) ^ 0xFFFFFFFFu;
  const int64_t chunk = ((len + threads - 1) / threads + 7) & ~int64_t(7);
  std::vector<uint32_t> part(size_t(threads), 0);
  std::vector<std::thread> pool;
  for (int i = 0; i < threads; ++i) {
    const int64_t lo = int64_t(i) * chunk, hi = std::min(len, lo + chunk);
    if (lo >= hi) break;
    pool.emplace_back([&, i, lo, hi] { part[size_t(i)] = crc32c_raw(p + lo, hi - lo, 0); });
  }
  for (size_t i = 0; i < pool.size(); ++i) {
    pool[i].join();
    const int64_t lo = int64_t(i) * chunk, hi = std::min(len, lo + chunk);
    reg = crc32c_shift(reg, hi - lo) ^ part[i];
  }
  return reg ^ 0xFFFFFFFFu;
}

}  // namespace ackpt

extern "C" ACKPT_API uint32_t ackpt_crc32c(const void* data, int64_t len, uint32_t crc) {
  if (len >= (int64_t(16) << 20)) return ackpt::crc32c_parallel(data, len, crc, ackpt::io_threads(len));
  return ackpt::crc32c_raw(data, len, crc ^ 0xFFFFFFFFu) ^ 0xFFFFFFFFu;
}
