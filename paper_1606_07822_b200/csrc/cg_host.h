// cg_host.h -- host-side helpers shared by the translation units of libcachegram_b200.
#pragma once

#include <string>

namespace cgint {
// Sets the thread-local message returned by cg_last_error().
void set_last_error(const std::string& msg);
}  // namespace cgint
