/*
 * ptdr_debug.h -- developer-only entry points of libptdr.so (not part of the product API).
 */
#ifndef PTDR_DEBUG_H_
#define PTDR_DEBUG_H_

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* With PTDR_TRACE=1 in the environment, the dense pipeline kernel records clock64()
 * stamps for the first 512 tiles handled by CTA 0: 16 unsigned long long per tile,
 * fields 0-3 producer (before/after empty wait, dependency satisfied, loads issued),
 * 4-7 consumer (wait start, data ready, stage released, tile done), 8 = phase.
 * Synchronizes the device and copies min(bytes, 64 KiB) to `host`.  Returns the
 * number of bytes copied, or a negative value if tracing is off or a copy failed. */
int ptdr_debug_trace_copy(void* host, size_t bytes);

#ifdef __cplusplus
}
#endif

#endif /* PTDR_DEBUG_H_ */
