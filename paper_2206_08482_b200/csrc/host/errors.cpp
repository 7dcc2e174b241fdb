#include "errors.hpp"

namespace gmi {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

}  // namespace gmi

extern "C" const char* gmi_last_error(void) { return gmi::g_last_error.c_str(); }

extern "C" int gmi_exit_code(int err) {
  if (err == GMI_OK) return 0;
  if (err == GMI_ERR_INVALID || err == GMI_ERR_CONFIG) return 2;
  return 1;
}

extern "C" int gmi_version(void) { return 1; }
