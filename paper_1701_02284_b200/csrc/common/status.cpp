#include "status.hpp"

namespace tcb {
namespace {
thread_local std::string t_last_error;
}
void set_error(const std::string& msg) { t_last_error = msg; }
tc_status fail(tc_status st, const std::string& msg) {
    t_last_error = msg;
    return st;
}
}  // namespace tcb

extern "C" const char* tc_last_error(void) { return tcb::t_last_error.c_str(); }
