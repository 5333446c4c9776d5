// pald_internal.h -- shared by the translation units of libpald_gpu.so.
#pragma once

// Records the thread-local message returned by pald_gpu_last_error() and
// returns `code`.
int pald_gpu_set_error(int code, const char* message);
