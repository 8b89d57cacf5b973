// Shared host-side helpers: status/last-error plumbing, dtype sizes.
#pragma once

#include <cstdint>
#include <cstdio>
#include <string>

#include "cm.h"

namespace cm {

void set_error(const std::string& msg);
int fail(int status, const std::string& msg);

inline size_t dtype_size(int dtype) {
  switch (dtype) {
    case CM_FLOAT32: return 4;
    case CM_FLOAT64: return 8;
    case CM_BFLOAT16: return 2;
    case CM_INT32: return 4;
    case CM_INT64: return 8;
    default: return 0;
  }
}

inline const char* dtype_name(int dtype) {
  switch (dtype) {
    case CM_FLOAT32: return "float32";
    case CM_FLOAT64: return "float64";
    case CM_BFLOAT16: return "bfloat16";
    case CM_INT32: return "int32";
    case CM_INT64: return "int64";
    default: return "?";
  }
}

// Reference-schedule helpers (hostlogic.cpp)
void chunk_partition(int64_t n, int p, int64_t* off, int64_t* len);
void rhd_layout(int64_t n, int p, int64_t* off, int64_t* len);
void segments_of(int64_t n, int p, int layout, int piece, int npieces, int64_t* off, int64_t* len);
int rhd_vrank(int rank, int p);  // -1 for folded odd ranks

}  // namespace cm

#define CM_CHECK_ARG(cond, msg) \
  do {                          \
    if (!(cond)) return ::cm::fail(CM_ERR_VALUE, (msg)); \
  } while (0)
