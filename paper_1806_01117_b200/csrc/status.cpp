// Thread-local last-error string and library version (C ABI).
#include <string>

#include "common.h"

namespace ackpt {
namespace {
thread_local std::string tl_last_error;
}
void set_last_error(const std::string& msg) { tl_last_error = msg; }
}  // namespace ackpt

extern "C" {
ACKPT_API const char* ackpt_last_error(void) { return ackpt::tl_last_error.c_str(); }
ACKPT_API const char* ackpt_version(void) { return "ackpt 0.1.0 sm_100a"; }
}
