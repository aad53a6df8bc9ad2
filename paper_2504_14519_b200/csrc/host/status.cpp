// Status strings and version of the libslimpipe C-ABI (include/slimpipe.h).
#include "slimpipe.h"

#include <string>

#include "errors.hpp"

namespace sp {
std::string& last_error() {
  thread_local std::string msg;
  return msg;
}
}  // namespace sp

extern "C" {

const char* sp_status_string(int code) {
  switch (code) {
    case SP_OK: return "ok";
    case SP_ERR_INVALID: return "invalid argument";
    case SP_ERR_RUNTIME: return "runtime error";
    case SP_ERR_CUDA: return "CUDA error";
    case SP_ERR_NCCL: return "NCCL error";
    case SP_ERR_UNSUPPORTED: return "unsupported shape";
    case SP_ERR_NO_DEVICE: return "no CUDA device";
    default: return "unknown status";
  }
}

int sp_version(void) { return 1; }

const char* sp_last_error(void) { return sp::last_error().c_str(); }

}  // extern "C"
