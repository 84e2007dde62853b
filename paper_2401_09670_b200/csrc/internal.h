// internal.h — error plumbing shared by the C-ABI translation units.
#pragma once
#include "../../include/ds.h"

namespace ds {
// Record `msg` as this thread's last error and return `st`.
ds_status fail(ds_status st, const char *fmt, ...);
}  // namespace ds
