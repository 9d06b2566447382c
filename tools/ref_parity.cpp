// Test-only comparator (built by tests/test_c5_replay_cpu.py): the config-5 harness restatement
// (tools/lb_sim.*) against the reference simulator compiled from its own sources
// (oracle/_ref/libref_sim.a, recipe oracle/ref.mk).  Checks, on the same seeds:
//   1. generate_trace (proj/src/synth.cpp:103-172) == lbsim::synth: every record and object size;
//   2. DualCache (proj/src/dual_cache.cpp) == lbsim::Cache: outcome, promotion and tail-hit flags of
//      every lookup, window counters and final resident order, with alpha moved every 997 lookups;
//   3. gradient_ms / step_alpha (proj/src/tuner.cpp:35-46) on the windows of that replay.
// Prints "OK ..." and exits 0, or the first mismatch and exits 1.
#include <cstdio>
#include <cstdlib>

#include "latentbox/dual_cache.hpp"
#include "latentbox/synth.hpp"
#include "latentbox/tuner.hpp"
#include "lb_sim.hpp"

static int fail(const char* what, size_t i) {
  std::printf("MISMATCH %s at %zu\n", what, i);
  return 1;
}

int main(int argc, char** argv) {
  const uint64_t seed = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 7;
  const bool lognormal = argc > 2 && argv[2][0] == 'l';
  lbx::SynthConfig rc;
  rc.n_objects_initial = 3000;
  rc.arrival_rate = 150;
  rc.duration_days = 6;
  rc.requests_per_day = 40000;
  rc.seed = seed;
  if (lognormal) rc.size_model.kind = lbx::SizeModel::Kind::Lognormal;
  lbsim::SynthCfg mc;
  mc.n_objects_initial = rc.n_objects_initial;
  mc.arrival_rate = rc.arrival_rate;
  mc.days = rc.duration_days;
  mc.requests_per_day = rc.requests_per_day;
  mc.seed = seed;
  mc.lognormal = lognormal;

  const lbx::SynthResult ref = lbx::generate_trace(rc);
  const lbsim::Workload mine = lbsim::synth(mc);
  if (ref.trace.size() != mine.trace.size()) return fail("trace length", 0);
  for (size_t i = 0; i < ref.trace.size(); ++i)
    if (ref.trace[i].ts_ms != mine.trace[i].ts_ms || ref.trace[i].object_id != mine.trace[i].object_id)
      return fail("trace record", i);
  if (ref.objects_total != mine.objects_total) return fail("objects_total", 0);
  for (uint64_t id = 1; id <= ref.objects_total; ++id) {
    const auto& a = ref.catalog.at(id);
    const auto& b = mine.meta[id - 1];
    if (a.image_bytes != b.image_bytes || a.latent_bytes != b.latent_bytes) return fail("catalog", id);
  }

  uint64_t img_total = 0;
  for (const auto& m : mine.meta) img_total += m.image_bytes;
  lbx::DualCacheConfig dc;
  dc.capacity_bytes = img_total / 50;
  dc.alpha = 0.5;
  dc.tail_fraction = 0.1;
  dc.promotion_threshold = 3;
  lbx::DualCache rcache(dc);
  lbsim::Cache mcache(dc.capacity_bytes, 0.5, 0.1, 3);
  size_t promotions = 0, windows = 0;
  double alpha = 0.5;
  lbx::TunerConfig tc;
  for (size_t i = 0; i < mine.trace.size(); ++i) {
    const uint64_t id = mine.trace[i].object_id;
    const lbx::ObjectMeta rm = ref.catalog.at(id);
    const lbx::LookupResult a = rcache.lookup(id, rm);
    bool promoted = false, tail = false;
    const lbsim::Outcome b = mcache.lookup(id, mine.meta[id - 1], &promoted, &tail);
    if ((int)a.outcome != (int)b || a.promoted != promoted || a.tail_hit != tail) return fail("lookup", i);
    promotions += promoted;
    if (b == lbsim::Outcome::FullMiss) {
      rcache.admit_latent(id, rm);
      mcache.admit_latent(id, mine.meta[id - 1]);
    }
    if (i % 997 == 996) {  // a tuning window: compare counters and the gradient, then move alpha
      const lbx::WindowCounters rcnt = rcache.snapshot_and_reset_counters();
      const lbsim::Counters mcnt = mcache.take_counters();
      if (rcnt.total_requests != mcnt.total || rcnt.image_misses != mcnt.image_misses ||
          rcnt.full_misses != mcnt.full_misses || rcnt.image_tail_hits != mcnt.image_tail_hits ||
          rcnt.latent_tail_hits != mcnt.latent_tail_hits)
        return fail("window counters", i);
      const double gr = lbx::gradient_ms(lbx::rates_from_counters(rcnt), 40.0, 140.0);
      const double gm = lbsim::gradient_ms(mcnt, 40.0, 140.0);
      if (gr != gm) return fail("gradient", i);
      const double ar = lbx::step_alpha(tc, alpha, gr);
      const double am = lbsim::step_alpha(alpha, gm, tc.step, tc.alpha_lo, tc.alpha_hi);
      if (ar != am) return fail("step_alpha", i);
      // exaggerated moves exercise budget shrinkage and eviction cascades
      alpha = (windows % 4 < 2) ? std::min(1.0, alpha + 0.07) : std::max(0.0, alpha - 0.11);
      rcache.set_alpha(alpha);
      mcache.set_alpha(alpha);
      ++windows;
    }
  }
  const auto ra = rcache.resident_ids();
  const auto mb = mcache.resident();
  if (ra != mb) return fail("resident set", 0);
  std::printf("OK requests=%zu objects=%llu promotions=%zu windows=%zu resident=%zu\n", mine.trace.size(),
              (unsigned long long)mine.objects_total, promotions, windows, mb.size());
  return 0;
}
