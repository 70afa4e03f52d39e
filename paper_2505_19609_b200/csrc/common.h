// Internal helpers shared by the host planner and the device entry points of libskrull.so.
#pragma once
#include <cstdarg>
#include <cstdio>

#include "skrull.h"

namespace skr {

skr_status fail(skr_status s, const char* fmt, ...);
void clear_error();

}  // namespace skr

#define SKR_EXPORT extern "C" __attribute__((visibility("default")))

#define SKR_REQUIRE(cond, ...)                      \
  do {                                              \
    if (!(cond)) return ::skr::fail(SKR_E_ARG, __VA_ARGS__); \
  } while (0)
