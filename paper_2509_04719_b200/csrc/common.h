// Shared host-side helpers of libstadi: status plumbing and error messages.
#pragma once

#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/stadi.h"

namespace stadi {

// Thread-local message of the last context-less error (stadi_last_error(NULL)).
std::string &tls_error();

inline stadi_status fail(std::string *sink, stadi_status st, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (sink) *sink = buf;
  tls_error() = buf;
  return st;
}

}  // namespace stadi
