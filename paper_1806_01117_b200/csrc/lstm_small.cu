// CTA-per-sequence LSTM kernels (any B, any d <= 128, f32 or f64; the path
// for every fp32 batch <= 2048 and every shape outside the batch-tiled fp32
// kernels): the reference's own workload is a single sequence (B = 1,
// float64 byte image, lstm.py:99-107), where one thread per sequence would
// run all 4 d^2 products serially.  Here a CTA owns one sequence (or, for
// short launches at large B, loops over sequences) and its 4d threads own
// the gate rows:
//   phase 1  thread n = gate row (g, j): a[n] = act_g(xb_k[n] + sum_k W[n][k] h[k])
//            (the gate activation is applied by the row's own thread)
//   phase 2  thread j < d: c' and h' (forward), or the gate adjoints
//            da[g][j] and dc (reverse, lstm.py:141-151)
//   phase 3  (reverse) all 4d threads: dh[m] = sum_{g,j} W[g][j][m] da[g][j],
//            one gate each, then a fixed-order sum
// with __syncthreads between phases and the state in shared memory across
// steps, so a fused Advance / TapeForward / Reverse run is one launch.  The
// shared copy of W has row stride d+1 so both the row-per-thread gate product
// and the column-per-thread transposed product are bank-conflict free, and the
// next step's bias (and, in reverse, state) is loaded during the current step
// so no global-load latency sits on the step's dependency chain.  Launches
// are programmatic dependent launches: a kernel lets the next one start at
// once, and the next stages W and its first bias (constants) before
// `griddepcontrol.wait`, overlapping its prologue with this one's steps --
// the per-step contract is a chain of such launches.  Same
// formulas and math-library calls as the generic kernels (lstm_generic.cu),
// so float64 results stay within 1e-12 of the reference.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <unordered_map>
#include <utility>

#include "lstm_cell.h"

namespace ackpt {
namespace sb {

__device__ __forceinline__ float sigmoid(float z) { return 1.0f / (1.0f + expf(-z)); }
__device__ __forceinline__ double sigmoid(double z) { return 1.0 / (1.0 + exp(-z)); }
__device__ __forceinline__ float tanh_(float z) { return tanhf(z); }
__device__ __forceinline__ double tanh_(double z) { return tanh(z); }

// gates f, i, o: sigmoid; candidate g: tanh (lstm.py:120-126)
template <typename T>
__device__ __forceinline__ T act(T z, bool cand) { return cand ? tanh_(z) : sigmoid(z); }

__device__ __forceinline__ void pdl_launch_next() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void pdl_wait_prev() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

struct Ptrs {
  const void* p[ACKPT_MAX_FUSED];
};

// Where a CTA reads W from: W[n][k] = g[n * grs + k * gcs] for the gate rows
// and W[r][m] = p[r * prs + m] for the transposed product.  Shared copy with
// row stride d+1 when it fits (both products conflict-free); else global
// memory, the gate rows from the transposed copy (coalesced across n) and the
// product from the row-major one (coalesced across m).
template <typename T>
struct WView {
  const T* g;
  int grs, gcs;
  const T* p;
  int prs;
};

// a[n] = xb + W[n] . h for this thread's gate row n (n < 4d): two
// interleaved accumulators (even / odd k) halve the dependent FMA chain
template <typename T>
__device__ __forceinline__ T gate_row(const WView<T>& w, T xb, const T* h, int d, int n) {
  const T* row = w.g + int64_t(n) * w.grs;
  T acc0 = xb, acc1 = T(0);
  int k = 0;
#pragma unroll 4
  for (; k + 1 < d; k += 2) {
    acc0 = fma(row[int64_t(k) * w.gcs], h[k], acc0);
    acc1 = fma(row[int64_t(k + 1) * w.gcs], h[k + 1], acc1);
  }
  if (k < d) acc0 = fma(row[int64_t(k) * w.gcs], h[k], acc0);
  return acc0 + acc1;
}

// (W's location is a template parameter so the products compile to LDS /
// LDG rather than generic loads)
template <bool kSmemW, typename T>
__device__ __forceinline__ WView<T> stage_w(T* ws, const T* __restrict__ wh, const T* __restrict__ wht, int d) {
  if (!kSmemW) return {wht, 1, 4 * d, wh, d};
  // blockDim = 4d: thread n copies column n % d of rows n / d + 4 t (coalesced reads)
  const int r0 = int(threadIdx.x) / d, k = int(threadIdx.x) - r0 * d;
#pragma unroll 8
  for (int t = 0; t < d; ++t) ws[(r0 + 4 * t) * (d + 1) + k] = __ldg(wh + threadIdx.x + size_t(4 * d) * t);
  __syncthreads();
  return {ws, d + 1, 1, ws, d + 1};
}

// Forward over `count` steps from `from` for sequence b.  tape: store every
// step's state to outs.p[i]; otherwise the final state to `out`.
template <typename T>
__device__ __forceinline__ void fwd_seq(const T* __restrict__ in, T* __restrict__ out, int64_t B, int d,
                                        const WView<T>& w, const T* __restrict__ xb_all, int64_t from, int count,
                                        bool tape, const Ptrs& outs, T* h, T* c, T* a, T xb, int64_t b) {
  const int n = threadIdx.x;
  if (n < d) {
    h[n] = in[int64_t(n) * B + b];
    c[n] = in[int64_t(d + n) * B + b];
  }
  __syncthreads();
  for (int i = 0; i < count; ++i) {
    const T xb_next = i + 1 < count ? __ldg(xb_all + (from + i + 1) * 4 * d + n) : T(0);
    a[n] = act(gate_row(w, xb, h, d, n), n >= 3 * d);
    xb = xb_next;
    __syncthreads();
    if (n < d) {
      const T f = a[n], ig = a[d + n], o = a[2 * d + n], g = a[3 * d + n];
      const T cn = f * c[n] + ig * g;  // lstm.py:127
      c[n] = cn;
      h[n] = o * tanh_(cn);            // lstm.py:128
      if (tape) {
        T* dst = static_cast<T*>(const_cast<void*>(outs.p[i]));
        dst[int64_t(n) * B + b] = h[n];
        dst[int64_t(d + n) * B + b] = cn;
      }
    }
    __syncthreads();
  }
  if (!tape && n < d) {
    out[int64_t(n) * B + b] = h[n];
    out[int64_t(d + n) * B + b] = c[n];
  }
}

// kPersist: CTAs loop over sequences (W staged once per CTA); else one
// sequence per CTA.
template <typename T, bool kSmemW, bool kPersist>
__global__ void fwd(const T* __restrict__ in, T* __restrict__ out, int64_t B, int d, const T* __restrict__ wh,
                    const T* __restrict__ wht, const T* __restrict__ xb_all, int64_t from, int count, bool tape,
                    const __grid_constant__ Ptrs outs) {
  extern __shared__ __align__(16) unsigned char raw[];
  T* h = reinterpret_cast<T*>(raw);
  T* c = h + d;
  T* a = c + d;  // 4d
  pdl_launch_next();
  const WView<T> w = stage_w<kSmemW>(a + 4 * d, wh, wht, d);
  const T xb = __ldg(xb_all + from * 4 * d + threadIdx.x);
  pdl_wait_prev();  // the input state is the previous launch's output
  if (kPersist) {
    for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
      fwd_seq(in, out, B, d, w, xb_all, from, count, tape, outs, h, c, a, xb, b);
      __syncthreads();
    }
  } else {
    fwd_seq(in, out, B, d, w, xb_all, from, count, tape, outs, h, c, a, xb, int64_t(blockIdx.x));
  }
}

// Reverse over steps from+count-1 .. from for sequence b; states.p[i] is the
// state of step from+i.  Software-pipelined across steps: the transposed
// product of step i (needs step i's gate adjoints) and the gate rows of step
// i-1 (need only step i-1's state) are independent, so each thread runs them
// as interleaved chains in one phase -- two barriers per step.
template <typename T, bool kSmemW>
__device__ __forceinline__ void rev_seq(const T* __restrict__ adj_in, T* __restrict__ adj_out, int64_t B, int d,
                                        const WView<T>& w, const T* __restrict__ xb_all, int64_t from, int count,
                                        const Ptrs& states, T* hb, T* cb, T* dc, T* a, T* da, T* part, T xb_top,
                                        T xbn_first, int64_t b) {
  T xbn = xbn_first;
  const int n = threadIdx.x;
  const int g = n / d, m = n - g * d;
  T dhn = T(0), hs = T(0), cs = T(0);  // threads n < d: dh[n]; state of the step after next
  if (n < d) {
    dhn = adj_in[int64_t(n) * B + b];
    dc[n] = adj_in[int64_t(d + n) * B + b];
    const T* st = static_cast<const T*>(states.p[count - 1]);
    hb[n] = st[int64_t(n) * B + b];
    cb[n] = st[int64_t(d + n) * B + b];
    if (count > 1) {
      st = static_cast<const T*>(states.p[count - 2]);
      hs = st[int64_t(n) * B + b];
      cs = st[int64_t(d + n) * B + b];
    }
  }
  __syncthreads();
  a[n] = act(gate_row(w, xb_top, hb, d, n), n >= 3 * d);
  __syncthreads();
  int cur = 0;
  for (int i = count - 1; i >= 0; --i) {
    const int nxt = cur ^ 1;
    if (n < d) {
      const T* cc = cb + cur * d;
      const T f = a[n], ig = a[d + n], o = a[2 * d + n], gg = a[3 * d + n];
      const T cn = f * cc[n] + ig * gg;
      const T t = tanh_(cn);
      const T dco = dc[n] + dhn * o * (T(1) - t * t);  // lstm.py:143
      da[n] = dco * cc[n] * f * (T(1) - f);           // lstm.py:144
      da[d + n] = dco * gg * ig * (T(1) - ig);        // lstm.py:145
      da[2 * d + n] = dhn * t * o * (T(1) - o);       // lstm.py:142,146
      da[3 * d + n] = dco * ig * (T(1) - gg * gg);    // lstm.py:147
      dc[n] = dco * f;                                // lstm.py:151
      if (i > 0) {
        hb[nxt * d + n] = hs;
        cb[nxt * d + n] = cs;
        if (i > 1) {
          const T* st = static_cast<const T*>(states.p[i - 2]);
          hs = st[int64_t(n) * B + b];
          cs = st[int64_t(d + n) * B + b];
        }
      }
    }
    __syncthreads();
    {
      // lstm.py:149-150: dh = sum_g W_g^T da_g; thread (g, m) sums gate g
      // (then a fixed-order reduction); interleaved with step i-1's gate row
      // (computed unconditionally so the two chains share one basic block;
      // unused when i == 0)
      const T* wg = w.p + int64_t(g) * d * w.prs + m;
      const T* dg = da + g * d;
      T acc = T(0);
#pragma unroll 4
      for (int j = 0; j < d; ++j) acc = fma(wg[int64_t(j) * w.prs], dg[j], acc);
      // (with W in global memory -- d = 96, 128 -- the unused i == 0 row
      // would cost a full pass over W, so it is skipped there)
      if (kSmemW || i > 0) {
        const T an = act(gate_row(w, xbn, hb + nxt * d, d, n), n >= 3 * d);
        a[n] = an;
      }
      part[n] = acc;
      if (i > 1) xbn = __ldg(xb_all + (from + i - 2) * 4 * d + n);
    }
    __syncthreads();
    if (n < d) dhn = (part[n] + part[d + n]) + (part[2 * d + n] + part[3 * d + n]);
    cur = nxt;
  }
  if (n < d) {
    adj_out[int64_t(n) * B + b] = dhn;
    adj_out[int64_t(d + n) * B + b] = dc[n];
  }
}

template <typename T, bool kSmemW, bool kPersist>
__global__ void rev(const T* __restrict__ adj_in, T* __restrict__ adj_out, int64_t B, int d, const T* __restrict__ wh,
                    const T* __restrict__ wht, const T* __restrict__ xb_all, int64_t from, int count,
                    const __grid_constant__ Ptrs states) {
  extern __shared__ __align__(16) unsigned char raw[];
  T* hb = reinterpret_cast<T*>(raw);  // [2][d] h of the step being reversed / the next one
  T* cb = hb + 2 * d;                 // [2][d] c, same
  T* dc = cb + 2 * d;                 // d
  T* a = dc + d;                      // 4d activated gates of the step being reversed
  T* da = a + 4 * d;                  // 4d gate adjoints
  T* part = da + 4 * d;               // 4d per-gate partial dh
  pdl_launch_next();
  const WView<T> w = stage_w<kSmemW>(part + 4 * d, wh, wht, d);
  const int n = threadIdx.x;
  const T xb_top = __ldg(xb_all + (from + count - 1) * 4 * d + n);
  const T xbn_first = count > 1 ? __ldg(xb_all + (from + count - 2) * 4 * d + n) : T(0);
  pdl_wait_prev();
  if (kPersist) {  // as in fwd
    for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
      rev_seq<T, kSmemW>(adj_in, adj_out, B, d, w, xb_all, from, count, states, hb, cb, dc, a, da, part, xb_top,
                         xbn_first, b);
      __syncthreads();  // the next sequence reuses the shared state
    }
  } else {
    rev_seq<T, kSmemW>(adj_in, adj_out, B, d, w, xb_all, from, count, states, hb, cb, dc, a, da, part, xb_top,
                       xbn_first, int64_t(blockIdx.x));
  }
}

// grid = one CTA per sequence, 4d threads; programmatic stream serialisation
// unless ACKPT_PDL=0
// Grid: one CTA per sequence up to what the SMs hold at once; beyond that the
// CTAs loop over sequences (W staged once per CTA, not once per sequence).
template <class K>
unsigned seq_grid(K kernel, int threads, size_t smem, int64_t B) {
  static std::mutex mu;
  static std::unordered_map<const void*, std::pair<size_t, unsigned>> cache;
  unsigned cap = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(reinterpret_cast<const void*>(kernel));
    if (it != cache.end() && it->second.first == smem) cap = it->second.second;
  }
  if (!cap) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) != cudaSuccess) {
      cudaGetLastError();
      per_sm = 1;
    }
    cap = unsigned(std::max(1, per_sm) * std::max(1, sms));
    std::lock_guard<std::mutex> lk(mu);
    cache[reinterpret_cast<const void*>(kernel)] = {smem, cap};
  }
  return unsigned(std::min<int64_t>(B, cap));
}

struct Launch {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  Launch(const ackpt_lstm* c, size_t smem, cudaStream_t s, unsigned grid) {
    static const bool pdl = [] {
      const char* e = std::getenv("ACKPT_PDL");
      return !(e && e[0] == '0');
    }();
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(unsigned(4 * c->d));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
  }
};

}  // namespace sb

bool sb_ok(const ackpt_lstm* c) {
  static const int64_t max_b = [] {  // ACKPT_SB_MAX: probe override of the batch cap
    const char* e = std::getenv("ACKPT_SB_MAX");
    return e ? std::atoll(e) : int64_t(kSmallBatch);
  }();
  return c->B <= max_b && c->d <= kMaxD;
}

// Batches small enough that a CTA per sequence beats the batch-tiled fp32
// kernels (whose 128/256-sequence tiles would run mostly empty): measured
// crossover, overridable with ACKPT_SB_FIRST=<max batch>.
bool sb_first(const ackpt_lstm* c) {
  static const int64_t max_b = [] {
    const char* e = std::getenv("ACKPT_SB_FIRST");
    return e ? std::atoll(e) : int64_t(kSbFirstBatch);
  }();
  return c->B <= max_b && sb_ok(c);
}

// shared-memory budget of the small-batch kernels (W copied in when it fits)
constexpr size_t kSmallWBytes = 160 * 1024;

template <typename T>
void sb_forward(const ackpt_lstm* c, int64_t from, int count, const void* in, void* out, void* const* outs,
                cudaStream_t s) {
  sb::Ptrs o{};
  if (outs)
    for (int i = 0; i < count; ++i) o.p[i] = outs[i];
  const size_t base = size_t(6) * c->d * sizeof(T), wbytes = size_t(4) * c->d * (c->d + 1) * sizeof(T);
  // staged even for one step: the row-per-thread product straight from global
  // memory touches one cache line per thread per load (uncoalesced)
  const bool w_smem = base + wbytes <= kSmallWBytes;
  const size_t smem = base + (w_smem ? wbytes : 0);
  // one CTA per sequence while the SMs hold them all (or W is read from
  // global memory: nothing to amortise); beyond that persistent CTAs
  auto one = w_smem ? sb::fwd<T, true, false> : sb::fwd<T, false, false>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(one, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  unsigned grid = unsigned(c->B);
  auto kern = one;
  if (w_smem) {
    // short launches (per-step operators) are bound by staging W once per
    // sequence; long fused runs amortise it and run faster one sequence per CTA
    const unsigned cap = count < 8 ? sb::seq_grid(one, 4 * c->d, smem, c->B) : grid;
    if (cap < grid) {
      kern = sb::fwd<T, true, true>;
      if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      grid = sb::seq_grid(kern, 4 * c->d, smem, c->B);
    }
  }
  sb::Launch L(c, smem, s, grid);
  ACKPT_CUDA_CHECK(cudaLaunchKernelEx(&L.cfg, kern, static_cast<const T*>(in), static_cast<T*>(out), c->B, c->d,
                                      static_cast<const T*>(c->d_wh), static_cast<const T*>(c->d_wht),
                                      static_cast<const T*>(c->d_xb), from, count, outs != nullptr, o));
}

template <typename T>
void sb_reverse(const ackpt_lstm* c, int64_t from, int count, const void* const* states, const void* adj_in,
                void* adj_out, cudaStream_t s) {
  sb::Ptrs p{};
  for (int i = 0; i < count; ++i) p.p[i] = states[i];
  const size_t base = size_t(17) * c->d * sizeof(T), wbytes = size_t(4) * c->d * (c->d + 1) * sizeof(T);
  // staged even for one step: the row-per-thread product straight from global
  // memory touches one cache line per thread per load (uncoalesced)
  const bool w_smem = base + wbytes <= kSmallWBytes;
  const size_t smem = base + (w_smem ? wbytes : 0);
  auto one = w_smem ? sb::rev<T, true, false> : sb::rev<T, false, false>;  // as in sb_forward
  if (smem > 48 * 1024) cudaFuncSetAttribute(one, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  unsigned grid = unsigned(c->B);
  auto kern = one;
  if (w_smem) {
    const unsigned cap = count < 8 ? sb::seq_grid(one, 4 * c->d, smem, c->B) : grid;  // as in sb_forward
    if (cap < grid) {
      kern = sb::rev<T, true, true>;
      if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      grid = sb::seq_grid(kern, 4 * c->d, smem, c->B);
    }
  }
  sb::Launch L(c, smem, s, grid);
  ACKPT_CUDA_CHECK(cudaLaunchKernelEx(&L.cfg, kern, static_cast<const T*>(adj_in), static_cast<T*>(adj_out), c->B,
                                      c->d, static_cast<const T*>(c->d_wh), static_cast<const T*>(c->d_wht),
                                      static_cast<const T*>(c->d_xb), from, count, p));
}

template void sb_forward<float>(const ackpt_lstm*, int64_t, int, const void*, void*, void* const*, cudaStream_t);
template void sb_forward<double>(const ackpt_lstm*, int64_t, int, const void*, void*, void* const*, cudaStream_t);
template void sb_reverse<float>(const ackpt_lstm*, int64_t, int, const void* const*, const void*, void*,
                                cudaStream_t);
template void sb_reverse<double>(const ackpt_lstm*, int64_t, int, const void* const*, const void*, void*,
                                 cudaStream_t);

}  // namespace ackpt
