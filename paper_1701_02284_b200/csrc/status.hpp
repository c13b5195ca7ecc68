// Thread-local error text behind tc_last_error() (tc_abi.h).  No exception
// crosses the C ABI: every entry point converts failures into a tc_status.
#pragma once

#include <string>

#include "tc_abi.h"

namespace tcb {
void set_error(const std::string& msg);
tc_status fail(tc_status st, const std::string& msg);
}  // namespace tcb
