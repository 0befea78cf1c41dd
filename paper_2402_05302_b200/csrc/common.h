// Internal helpers shared by the library's translation units (error reporting).
#pragma once
#include <cstdarg>
#include <cstdio>
#include <string>

#include "cannikin.h"

namespace cannikin {

// Thread-local last-error text (cannikin_last_error).
void set_error_text(const char* fmt, ...);
void clear_error();

inline cannikin_status fail(cannikin_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  set_error_text("%s", buf);
  return st;
}

}  // namespace cannikin
