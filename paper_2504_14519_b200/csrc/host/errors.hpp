// Per-thread last-error text behind sp_last_error() (include/slimpipe.h).
#pragma once
#include <string>

namespace sp {
std::string& last_error();
}
