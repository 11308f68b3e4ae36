// Thread-local last-error slot behind eplab_last_error (no exceptions cross the ABI).
#include <cstring>
#include <string>

#include "eplab_b200.h"
#include "host/errors.hpp"

namespace eplab_host {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
const std::string& last_error() { return g_last_error; }
}  // namespace eplab_host

extern "C" {
const char* eplab_version(void) { return "0.1.0-b200"; }

size_t eplab_last_error(char* buf, size_t len) {
  const std::string& s = eplab_host::last_error();
  if (buf && len) {
    size_t n = s.size() < len - 1 ? s.size() : len - 1;
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return s.size();
}
}
