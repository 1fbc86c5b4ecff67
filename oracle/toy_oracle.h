/* TEST INFRASTRUCTURE ONLY -- CPU restatement (plain C, fp64) of the reference's
 * ToyModel oracle, used as the numerical checker for the sm_100a ToyModel path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 *
 * Restates, function by function (file:line in /root/reference/proj):
 *   toy_make_model       <- src/oracle.cpp:94-111   (mt19937_64 + libstdc++ U(a,b))
 *   toy_make_batch       <- src/oracle.cpp:113-123
 *   toy_list_schedule    <- src/listsched.hpp:52-163 (incl. relaxed mode, kEps ties)
 *   toy_run_iteration    <- src/oracle.cpp:162-300,304-351 (Engine + replay order)
 *   toy_sequential_sgd   <- src/oracle.cpp:125-151
 *   toy_max_relative_diff<- src/oracle.cpp:412-425
 * Synchronous schemes only (GPipe/DAPPLE/GEMS/Chimera); the PipeDream per-micro-batch
 * update (oracle.cpp:205-214,339-341) is out of scope.
 *
 * Parity pinning: tests/test_oracle_pin.py checks every function here against the
 * reference library built in place (oracle/_ref) and against tests/golden fixtures
 * (SURVEY.md Appendix D.3 known answers).
 *
 * Layouts: a task is 6 int32 {kind, pipeline_id, micro_batch, stage, worker,
 * replica_group} (kind 0 = Forward, 1 = Backward, others ignored), workers'
 * lists concatenated; ToyModel parameters are one flat array, per stage
 * [W_s (out x in row-major), b_s (out)].
 */
#ifndef TOY_ORACLE_H
#define TOY_ORACLE_H
#include <stdint.h>

int toy_make_model(const int* dims, int n_dims, uint64_t seed, double* params);
int toy_make_batch(const int* dims, int n_dims, int size, uint64_t seed, double* inputs,
                   double* targets);
int toy_list_schedule(int workers, const int* counts, const int* tasks, double f_dur,
                      double b_dur, double p2p_fwd, double p2p_bwd, int relaxed,
                      double* starts, double* ends, double* makespan);
int toy_run_iteration(int D, int W, int N, int B, int halved_backward, int workers,
                      const int* counts, const int* tasks, const int* dims, int n_dims,
                      const double* params, const double* inputs, const double* targets,
                      int batch, double lr, double* params_out, int* peak_stash);
int toy_sequential_sgd(const int* dims, int n_dims, const double* params,
                       const double* inputs, const double* targets, int batch, double lr,
                       double* params_out);
double toy_max_relative_diff(const int* dims, int n_dims, const double* a, const double* b);
#endif
