/* pg_network.h — network- and optimizer-level C-ABI: the B200 drop-in for
 * partgan's build_network / forward / infer / backward (one network, host
 * tensors) and adam_step (host vectors).
 *
 * Reference interfaces replaced (file:line under /root/reference/proj):
 *   build_network   include/partgan/network.hpp:58-59,   src/network.cpp:308-343
 *   forward         include/partgan/network.hpp:80,      src/network.cpp:402-419
 *   infer           include/partgan/network.hpp:83,      src/network.cpp:421-427
 *   backward        include/partgan/network.hpp:91,      src/network.cpp:429-480
 *   Network::params / buffers  include/partgan/network.hpp:33-38
 *   adam_step       include/partgan/optim.hpp:29,        src/optim.cpp:20-34
 * Host tensors are the reference's row-major f64 layout ([B][C][H][W] or
 * [B][F]); the device computes in fp32 (math mode PG_MATH_*), parameters stay
 * device-resident between calls.  Errors carry the reference's message text
 * (pg_last_error()): "trace already consumed by a previous backward call",
 * "trace does not belong to this network", "output gradient shape ... does
 * not match network output ...", "adam_step: length mismatch (...)",
 * "adam_step: non-finite gradient rejected" (PG_ENONFINITE, state untouched).
 * The C++ mirror of the reference API built on these calls is
 * include/partgan_b200.hpp.
 */
#ifndef PG_NETWORK_H
#define PG_NETWORK_H

#include <stdint.h>

#include "pg_kernels.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pg_net pg_net;
typedef struct pg_trace pg_trace;

/* build_network: layer list text (pg_trainer.h grammar), per-sample input
 * shape (rank 1 [F] or rank 3 [C,H,W]), init stream seed, init std.  The
 * first batch a forward call sees sizes the device buffers; larger batches
 * regrow them (parameters and buffers are kept). */
int pg_net_create(const char* spec, const long* in_shape, int in_rank, uint64_t seed, double init_std, int math,
                  int device, pg_net** out);
void pg_net_destroy(pg_net* net);
/* counts in the reference flat layouts; out_shape[4] / *out_rank: per-sample output shape */
long pg_net_param_count(const pg_net* net);
long pg_net_buffer_count(const pg_net* net);
int pg_net_out_shape(const pg_net* net, long* out_shape, int* out_rank);
/* Network::params() / buffers() in the reference order (f64) */
int pg_net_get_params(pg_net* net, double* out);
int pg_net_set_params(pg_net* net, const double* in);
int pg_net_get_buffers(pg_net* net, double* out);
int pg_net_set_buffers(pg_net* net, const double* in);
/* forward: x [B][in] -> y [B][out]; train != 0: batch statistics + running
 * update (Mode::train), else running statistics (Mode::eval).  trace != NULL
 * receives a single-use trace for pg_net_backward (free it with
 * pg_trace_destroy); trace == NULL is infer() (no state touched in eval). */
int pg_net_forward(pg_net* net, const double* x, int B, int train, double* y, pg_trace** trace);
/* backward: gy [B][out] -> fresh parameter gradients (reference layout) and
 * the input gradient gx [B][in] (either output may be NULL) */
int pg_net_backward(pg_net* net, pg_trace* trace, const double* gy, int B, double* gparams, double* gx);
void pg_trace_destroy(pg_trace* trace);

/* adam_step on host vectors of length n (m, v, params in/out; *t advanced):
 * the step runs on `device` in fp32 (f64 bias corrections, as the group
 * optimizer).  Non-finite gradients: PG_ENONFINITE, nothing modified. */
int pg_adam_step_host(long n, double* params, const double* grads, double* m, double* v, long* t, double lr,
                      double beta1, double beta2, double eps, int device);

#ifdef __cplusplus
}
#endif

#endif /* PG_NETWORK_H */
