#pragma once
#include <string>

namespace eplab_host {
void set_last_error(const std::string& msg);
const std::string& last_error();
}  // namespace eplab_host
