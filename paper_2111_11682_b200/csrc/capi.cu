// C-ABI bookkeeping: error string and version.
#include <cstdio>

#include "common.cuh"

static thread_local char g_err[512] = "";

void culsh_set_error(const char *msg, const char *file, int line) {
    const char *base = file;
    for (const char *p = file; *p; ++p)
        if (*p == '/') base = p + 1;
    snprintf(g_err, sizeof(g_err), "%s (%s:%d)", msg, base, line);
}

extern "C" const char *culsh_last_error(void) { return g_err; }

extern "C" const char *culsh_version(void) { return "culsh 0.1.0 sm_100a"; }
