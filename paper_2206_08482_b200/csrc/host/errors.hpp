// Error plumbing shared by the C-ABI layer: C++ exceptions inside the library,
// integer codes + a thread-local message at the extern "C" boundary.
#pragma once

#include <stdexcept>
#include <string>

#include "gmi.h"

namespace gmi {

// Carries one of the GMI_ERR_* codes from include/gmi.h.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& msg) : std::runtime_error(msg), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }
[[noreturn]] inline void invalid(const std::string& msg) { fail(GMI_ERR_INVALID, msg); }

void set_last_error(const std::string& msg);

// Runs `fn`, translating exceptions into a return code and the thread-local message.
template <class Fn>
int guarded(Fn&& fn) noexcept {
  try {
    fn();
    set_last_error("");
    return GMI_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return GMI_ERR_INVALID;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return GMI_ERR_DOMAIN;
  } catch (...) {
    set_last_error("unknown exception");
    return GMI_ERR_DOMAIN;
  }
}

}  // namespace gmi

#define GMI_CUDA_CHECK(expr)                                                                  \
  do {                                                                                        \
    cudaError_t _e = (expr);                                                                  \
    if (_e != cudaSuccess)                                                                    \
      ::gmi::fail(GMI_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e) + " at " + \
                                    __FILE__ + ":" + std::to_string(__LINE__));               \
  } while (0)
