/* loadflow/sched_rule.h -- MinatoLoader's adaptive worker rule (Eq. 1-2;
 * reference proj/src/scheduler.cpp:16-24), header-only C so the host C++ API
 * (scheduler_loop) and the CUDA shard runner (csrc/shard.cpp, where "workers" are
 * in-flight launch groups on the stream pool) apply the identical arithmetic.
 *
 *   delta   = clip(round_half_away(alpha * (1 - q / q_max) + beta * (c - theta_c)),
 *                  -clip, +clip)
 *   workers = min(max_workers, max(1, current + delta))
 */
#ifndef LOADFLOW_SCHED_RULE_H
#define LOADFLOW_SCHED_RULE_H

#include <math.h>

static inline int lf_round_half_away(double x) {
    return (int)(x >= 0 ? floor(x + 0.5) : ceil(x - 0.5));
}

static inline int lf_sched_delta(double q_size_avg, double c_usage, double alpha, double beta,
                                 double theta_c, double q_max, int clip) {
    const int d = lf_round_half_away(alpha * (1.0 - q_size_avg / q_max) + beta * (c_usage - theta_c));
    return d < -clip ? -clip : (d > clip ? clip : d);
}

static inline int lf_sched_update(int current, int delta, int max_workers) {
    const int w = current + delta;
    return w < 1 ? 1 : (w > max_workers ? max_workers : w);
}

#endif
