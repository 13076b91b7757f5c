// common.h -- shared host helpers of libgts (error state).
#pragma once
#include <cstdint>

namespace gts {
// Sets the thread-local error message and returns `code` (gts_last_error).
int set_error(int code, const char *fmt, ...);
}  // namespace gts
