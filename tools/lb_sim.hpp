// Config-5 harness: a minimal restatement of the reference's workload generator, dual-format
// cache, split tuner and request coalescing, for replaying decode-on-miss against real GPU decodes.
//
// Restated (not copied) from the reference, behaviour pinned by tests/test_c5_replay_cpu.py against
// the reference compiled from its own sources (oracle/ref.mk):
//   synth()  <- lbx::generate_trace   proj/src/synth.cpp:103-172 (Vose alias :21-62, draw_meta :64-83)
//   Cache    <- lbx::DualCache        proj/src/dual_cache.cpp:75-206 (budgets :59-73, enforce :75-92,
//                                      lookup :132-196, set_alpha :198-206)
//   tuner    <- rates/gradient/step   proj/src/tuner.cpp:17-59, fire_window proj/src/sim.cpp:271-299
//   coalescing (single flight)       proj/src/router.cpp:117-130, sim.cpp:333-336
//   percentiles (nearest rank)       proj/src/sim.cpp:136-151
#pragma once
#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

namespace lbsim {

struct Meta {
  uint64_t image_bytes = 0, latent_bytes = 0;
};
struct Rec {
  uint64_t ts_ms = 0, object_id = 0;
};

struct SynthCfg {
  uint64_t n_objects_initial = 10000;
  double arrival_rate = 0.0;
  double zipf = 1.11, decay = 1.3;
  uint32_t days = 30;
  uint64_t requests_per_day = 100000;
  uint64_t seed = 1;
  double image_mb = 1.5, latent_mb = 0.29, sigma = 0.35;
  bool lognormal = false;
};

struct Workload {
  std::vector<Rec> trace;
  std::vector<Meta> meta;  // meta[id - 1]
  uint64_t objects_total = 0;
};

Workload synth(const SynthCfg& cfg);

enum class Outcome : uint8_t { ImageHit = 0, LatentHit = 1, FullMiss = 2 };

struct Counters {
  uint64_t total = 0, image_misses = 0, full_misses = 0, image_tail_hits = 0, latent_tail_hits = 0;
};

// Two byte-budgeted segmented-LRU tiers (image, latent), split by alpha, each with a tail of
// fraction tau; promotion to the image tier after h latent hits.
class Cache {
 public:
  Cache(uint64_t capacity, double alpha, double tau, uint32_t h);
  Outcome lookup(uint64_t id, const Meta& m, bool* promoted = nullptr, bool* tail_hit = nullptr);
  void admit_latent(uint64_t id, const Meta& m) { admit(1, id, m.latent_bytes); }
  void admit_image(uint64_t id, const Meta& m) { admit(0, id, m.image_bytes); }
  void set_alpha(double a);
  double alpha() const { return alpha_; }
  Counters take_counters() {
    Counters c = ctr_;
    ctr_ = Counters{};
    return c;
  }
  uint64_t used(int t) const { return t_[t].main_used + t_[t].tail_used; }
  std::vector<uint64_t> resident() const;  // MRU->LRU per tier, image tier first

 private:
  struct Node {
    uint64_t id, bytes;
    uint32_t hits;
    int prev, next;
    uint8_t tier, tail;
  };
  struct List {
    int head = -1, tail = -1;
  };
  struct Tier {
    List main, tl;
    uint64_t main_used = 0, tail_used = 0, budget = 0, main_budget = 0;
  };
  void budgets();
  void enforce(int t);
  void unlink(int n);
  void push_front(int t, bool tail_seg, int n);
  void admit(int t, uint64_t id, uint64_t bytes);
  int alloc(uint64_t id, uint64_t bytes);
  void release(int n);

  uint64_t cap_;
  double alpha_, tau_;
  uint32_t h_;
  Tier t_[2];
  std::vector<Node> nodes_;
  std::vector<int> free_;
  std::unordered_map<uint64_t, int> where_;
  Counters ctr_;
};

// Split-tuner arithmetic (Eq. 1/2 of the paper, proj/src/tuner.cpp:17-46).
double gradient_ms(const Counters& c, double t_decode, double t_fetch);
double step_alpha(double alpha, double gradient, double step, double lo, double hi);

// Nearest-rank percentile, v sorted ascending (proj/src/sim.cpp:143-149).
double pct(const std::vector<double>& v, double q);

// ---------------------------------------------------------------- replay
struct ReplayCfg {
  double time_scale = 10.0;         // replay speed-up on trace timestamps
  double cache_frac = 0.01;         // cache capacity as a fraction of the unique-object footprint
  double tau = 0.10;
  uint32_t h = 8;
  double alpha0 = 0.5;
  bool adaptive = true;             // LbAdaptive
  uint64_t window = 0;              // 0: max(10000, N/60) as the reference auto-scales
  double step = 0.005, ewma = 0.1;
  double fetch_ms = 140.0, net_ms = 10.0, nominal_decode_ms = 40.0;
  double warmup_fraction = 0.20;
  // batched decode service
  int gpus = 8;
  int max_batch = 32;
  double max_wait_ms = 0.0;        // 0 = work-conserving: an idle GPU takes whatever is queued
  std::vector<double> service_ms;   // service_ms[b-1] = GPU time of a batch of b (measured)
  bool cost_policy = false;         // batch size by lbx_batch_pick over service_ms (else greedy)
};

// A decode job: the leader request of an in-flight object (LatentHit or FullMiss).
struct Job {
  uint64_t leader, object_id;
  double t_arrive, t_ready;         // ready = arrival (+ fetch for full misses)
  double t_start = 0, t_end = 0;    // filled by the service model or the live batcher
  int gpu = -1;
  uint32_t batch = 0;
};

struct ReplayOut {
  std::vector<Job> jobs;
  std::vector<uint8_t> outcome;                 // per request
  std::vector<int64_t> job_of;                  // per request: job index it waited on, -1 image hit
  uint64_t image_hits = 0, latent_hits = 0, full_misses = 0, coalesced = 0, windows = 0;
  double final_alpha = 0;
};

// Cache/tuner/coalescing pass over the trace plus the batched FIFO GPU service model in virtual
// time (least-loaded idle GPU takes up to max_batch ready jobs once the oldest waited max_wait).
ReplayOut replay(const Workload& w, const ReplayCfg& cfg);

struct LatencyReport {
  double decode_p50, decode_p99, decode_mean;   // t_end - t_ready over decode jobs (post warm-up)
  double e2e_p50, e2e_p99, e2e_mean;            // completion - arrival over all requests
  uint64_t n_decodes, n_requests;
  double mean_batch;
};
LatencyReport report(const ReplayOut& r, const ReplayCfg& cfg, const Workload& w);

}  // namespace lbsim
