// CRC32C (Castagnoli), bit-compatible with the reference's table-driven
// crc32c(data, crc) (storage.py:49-68): reflected polynomial 0x82F63B78,
// initial and final xor 0xFFFFFFFF, chaining through the crc argument.
// Uses the SSE4.2 crc32 instruction (8 bytes per instruction) when the host
// CPU has it, else a slicing-by-8 table.
#include <cstring>

#include "common.h"

#if defined(__x86_64__)
#include <cpuid.h>
#include <nmmintrin.h>
#endif

namespace {

struct Tables {
  uint32_t t[8][256];
  Tables() {
    for (uint32_t b = 0; b < 256; ++b) {
      uint32_t c = b;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ 0x82F63B78u : c >> 1;
      t[0][b] = c;
    }
    for (uint32_t b = 0; b < 256; ++b)
      for (int s = 1; s < 8; ++s) t[s][b] = (t[s - 1][b] >> 8) ^ t[0][t[s - 1][b] & 0xFF];
  }
};

const Tables& tables() {
  static Tables tb;
  return tb;
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
__attribute__((target("sse4.2"))) uint32_t crc_hw(const unsigned char* p, int64_t n, uint32_t c) {
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

bool have_sse42() {
  unsigned a, b, c, d;
  if (!__get_cpuid(1, &a, &b, &c, &d)) return false;
  return (c & bit_SSE4_2) != 0;
}
#endif

}  // namespace

extern "C" ACKPT_API uint32_t ackpt_crc32c(const void* data, int64_t len, uint32_t crc) {
  const auto* p = static_cast<const unsigned char*>(data);
  uint32_t c = crc ^ 0xFFFFFFFFu;
#if defined(__x86_64__)
  static const bool hw = have_sse42();
  c = hw ? crc_hw(p, len, c) : crc_sw(p, len, c);
#else
  c = crc_sw(p, len, c);
#endif
  return c ^ 0xFFFFFFFFu;
}
