// status.h — thread-local error reporting behind ftb_last_error(), and the
// C++ exception types the planner throws internally. Each maps to one
// mktune.errors class (errors.py:10-47); the C ABI converts them to codes.
#pragma once
#include <stdexcept>
#include <string>

#include "../../include/ftb.h"

namespace ftb {

struct FtbError : std::runtime_error {
  ftb_status code;
  std::string field;
  FtbError(ftb_status c, const std::string& msg, const std::string& f = "")
      : std::runtime_error(msg), code(c), field(f) {}
};

inline FtbError input_error(const std::string& msg, const std::string& field = "") {
  return FtbError(FTB_INPUT_ERROR, msg, field);
}
inline FtbError capacity_error(const std::string& msg) { return FtbError(FTB_CAPACITY_ERROR, msg); }
inline FtbError empty_error(const std::string& msg, const std::string& constraint = "") {
  return FtbError(FTB_EMPTY_RESULT, msg, constraint);
}
inline FtbError internal_error(const std::string& msg) { return FtbError(FTB_INTERNAL_ERROR, msg); }
inline FtbError cuda_error(const std::string& msg) { return FtbError(FTB_CUDA_ERROR, msg); }

void set_last_error(ftb_status code, const std::string& msg, const std::string& field = "");
void clear_last_error();

// Run `fn` and translate any exception into a status code + last-error text.
template <class F>
ftb_status guarded(F&& fn) {
  try {
    clear_last_error();
    fn();
    return FTB_OK;
  } catch (const FtbError& e) {
    set_last_error(e.code, e.what(), e.field);
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error(FTB_INTERNAL_ERROR, "out of host memory");
    return FTB_INTERNAL_ERROR;
  } catch (const std::exception& e) {
    set_last_error(FTB_INTERNAL_ERROR, e.what());
    return FTB_INTERNAL_ERROR;
  }
}

}  // namespace ftb
