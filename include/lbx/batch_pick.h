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
 * size in [1, min(queued, max_batch)] with the lowest time per request; a larger batch must beat
 * the best smaller one by 2%.  No curve: min(queued, max_batch). */
static inline uint32_t lbx_batch_pick_rule(const double* cost_ms, uint32_t n_cost, uint32_t queued,
                                           uint32_t max_batch) {
  const uint32_t lim = queued < max_batch ? queued : max_batch;
  if (lim == 0) return 0;
  if (!cost_ms || n_cost == 0) return lim;
  uint32_t best = 1;
  double per = cost_ms[0];
  for (uint32_t b = 2; b <= lim; ++b) {
    const double c = (b <= n_cost ? cost_ms[b - 1] : cost_ms[n_cost - 1] * b / n_cost) / b;
    if (c < per * 0.98) {
      best = b;
      per = c;
    }
  }
  return best;
}

#endif /* LBX_BATCH_PICK_H */
