// status.cpp — storage for the thread-local last-error message.
#include "status.h"

#include <cstring>

namespace ftb {
namespace {
thread_local std::string g_msg;
thread_local std::string g_field;
}  // namespace

void set_last_error(ftb_status, const std::string& msg, const std::string& field) {
  g_msg = msg;
  g_field = field;
}
void clear_last_error() {
  g_msg.clear();
  g_field.clear();
}

static size_t copy_out(const std::string& s, char* buf, size_t n) {
  if (buf && n) {
    size_t k = s.size() < n - 1 ? s.size() : n - 1;
    std::memcpy(buf, s.data(), k);
    buf[k] = '\0';
  }
  return s.size();
}

}  // namespace ftb

extern "C" size_t ftb_last_error(char* buf, size_t n) { return ftb::copy_out(ftb::g_msg, buf, n); }
extern "C" size_t ftb_last_error_field(char* buf, size_t n) {
  return ftb::copy_out(ftb::g_field, buf, n);
}
