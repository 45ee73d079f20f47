// Thread-local error reporting for the C-ABI (tpipe_last_error()).
#pragma once
namespace tpipe {
// Formats the message, stores it thread-locally, returns `code` (negative).
int set_error(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
}  // namespace tpipe
