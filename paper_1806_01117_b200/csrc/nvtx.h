// NVTX ranges of the executor and the tier (domain "ackpt"): the pass, its
// forward sweep / backward phase, every backward segment, transfer issue and
// wait, calibration, graph capture / replay, and the file stage's disk I/O.
// Header-only NVTX v3: without a tool attached (nsys, ncu --nvtx) a range is
// one predictable branch; with one, e.g.
//   ncu --nvtx --nvtx-include "ackpt@backward/" python bench.py ...
// profiles only the kernels the backward phase launches.
#pragma once

#include <nvtx3/nvToolsExt.h>

#include <string>

namespace ackpt {

inline nvtxDomainHandle_t nvtx_domain() {
  static const nvtxDomainHandle_t d = nvtxDomainCreateA("ackpt");
  return d;
}

struct NvtxRange {
  explicit NvtxRange(const char* msg) { push(msg); }
  explicit NvtxRange(const std::string& msg) { push(msg.c_str()); }
  ~NvtxRange() { nvtxDomainRangePop(nvtx_domain()); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;

 private:
  static void push(const char* msg) {
    nvtxEventAttributes_t a{};
    a.version = NVTX_VERSION;
    a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
    a.messageType = NVTX_MESSAGE_TYPE_ASCII;
    a.message.ascii = msg;
    nvtxDomainRangePushEx(nvtx_domain(), &a);
  }
};

}  // namespace ackpt
