#include "runtime/errors.h"

#include <cstdarg>
#include <cstdio>

#include "tpipe.h"

namespace tpipe {
static thread_local char g_err[512] = "";

int set_error(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}
}  // namespace tpipe

extern "C" __attribute__((visibility("default"))) const char* tpipe_last_error(void) {
    return tpipe::g_err;
}
