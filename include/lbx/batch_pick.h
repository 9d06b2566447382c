/*
 * lbx/batch_pick.h -- the batch-size rule behind lbx_batch_pick (include/lbx/batcher.h), header-only
 * so the config-5 simulator (tools/lb_sim.cpp, built standalone against the reference) applies the
 * same rule as the live batcher.  It is the batching decision the reference's FIFO service never
 * makes: Engine::on_job_ready (proj/src/sim.cpp:409-429) serves one job per GPU at a constant
 * decode_ms (proj/include/latentbox/sim.hpp:19).
 */
#ifndef LBX_BATCH_PICK_H
#define LBX_BATCH_PICK_H

#include <stdint.h>

/* cost_ms[b-1] = GPU time of a batch of b (b = 1..n_cost, linear past n_cost).  Returns the batch
 * size b in [1, min(queued, max_batch)]:
 *  - queued < max_batch / 2: the b that minimises the mean completion time of the `queued` requests
 *    if they were all served FIFO in batches of b (the last one partial) -- a batch holds its first
 *    requests back until it finishes, so with a short queue only a large per-request gain pays;
 *  - a backlog of max_batch / 2 or more (a burst: requests keep arriving, which the mean over the
 *    queue alone does not see): the lowest GPU time per request, a larger batch winning by 2%.
 * The config-5 simulation with the measured B200 curve chose the max_batch / 2 switch over 8 and
 * 32.  No curve: min(queued, max_batch). */
static inline double lbx_batch_cost_at(const double* cost_ms, uint32_t n_cost, uint32_t b) {
  return b <= n_cost ? cost_ms[b - 1] : cost_ms[n_cost - 1] * b / n_cost;
}
static inline uint32_t lbx_batch_pick_rule(const double* cost_ms, uint32_t n_cost, uint32_t queued,
                                           uint32_t max_batch) {
  const uint32_t lim = queued < max_batch ? queued : max_batch;
  if (lim == 0) return 0;
  if (!cost_ms || n_cost == 0) return lim;
  uint32_t best = 1;
  if (2 * queued >= max_batch) {  /* backlog: throughput */
    double per = cost_ms[0];
    for (uint32_t b = 2; b <= lim; ++b) {
      const double c = lbx_batch_cost_at(cost_ms, n_cost, b) / b;
      if (c < per * 0.98) {
        best = b;
        per = c;
      }
    }
    return best;
  }
  double best_mean = 0.0;
  for (uint32_t b = 1; b <= lim; ++b) {
    const double mb = lbx_batch_cost_at(cost_ms, n_cost, b);
    const uint32_t k = queued / b, r = queued - k * b;  /* k full batches, then one of r */
    /* sum of completion times: b requests finish at i * mb for i = 1..k, r at k * mb + m(r) */
    double sum = (double)b * mb * (double)k * (double)(k + 1) / 2.0;
    if (r) sum += (double)r * ((double)k * mb + lbx_batch_cost_at(cost_ms, n_cost, r));
    const double mean = sum / (double)queued;
    if (b == 1 || mean < best_mean * (1.0 - 1e-9)) {
      best = b;
      best_mean = mean;
    }
  }
  return best;
}

#endif /* LBX_BATCH_PICK_H */
