/* sas_debug.h — test-only entry points of libsas.so (not part of the drop-in
 * boundary): the kernel-row exponential used by K3, on host and device. */
#ifndef SAS_DEBUG_H_
#define SAS_DEBUG_H_
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
double sas_debug_exp64_host(double x);
int sas_debug_exp64(const double* x_dev, double* y_dev, int64_t n, void* stream);
#ifdef __cplusplus
}
#endif
#endif
