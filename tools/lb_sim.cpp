// Config-5 harness: restated workload / cache / tuner / coalescing and the virtual-time batched
// decode service model.  See lb_sim.hpp for the reference mapping (file:line).
#include "../include/lbx/batch_pick.h"  // the live batcher's rule
#include "lb_sim.hpp"

#include <algorithm>
#include <cmath>
#include <deque>
#include <numeric>
#include <queue>
#include <random>
#include <stdexcept>

namespace lbsim {

// ================================================================ workload
namespace {
inline double u01(std::mt19937_64& r) { return double(r() >> 11) * 0x1.0p-53; }

struct Alias {
  std::vector<double> prob;
  std::vector<uint32_t> alias;
  explicit Alias(const std::vector<double>& w) {
    const size_t n = w.size();
    prob.assign(n, 0.0);
    alias.assign(n, 0);
    double total = 0.0;
    for (double x : w) total += x;
    std::vector<double> sc(n);
    for (size_t i = 0; i < n; ++i) sc[i] = w[i] * double(n) / total;
    std::vector<uint32_t> lo, hi;
    lo.reserve(n);
    hi.reserve(n);
    for (size_t i = 0; i < n; ++i) (sc[i] < 1.0 ? lo : hi).push_back(uint32_t(i));
    while (!lo.empty() && !hi.empty()) {
      const uint32_t s = lo.back(), l = hi.back();
      lo.pop_back();
      hi.pop_back();
      prob[s] = sc[s];
      alias[s] = l;
      sc[l] -= 1.0 - sc[s];
      (sc[l] < 1.0 ? lo : hi).push_back(l);
    }
    for (uint32_t i : hi) prob[i] = 1.0;
    for (uint32_t i : lo) prob[i] = 1.0;
  }
  uint32_t draw(std::mt19937_64& r) const {
    const size_t n = prob.size();
    const double u = u01(r) * double(n);
    uint32_t i = uint32_t(u);
    if (i >= n) i = uint32_t(n - 1);
    return (u - double(i)) < prob[i] ? i : alias[i];
  }
};

Meta size_draw(const SynthCfg& c, std::mt19937_64& r) {
  const double mb = 1024.0 * 1024.0;
  Meta m;
  if (!c.lognormal) {
    m.image_bytes = uint64_t(std::llround(c.image_mb * mb));
    m.latent_bytes = uint64_t(std::llround(c.latent_mb * mb));
    return m;
  }
  const double mu = std::log(c.image_mb * mb) - 0.5 * c.sigma * c.sigma;
  const double a = u01(r), b = u01(r);
  const double z = std::sqrt(-2.0 * std::log(1.0 - a)) * std::cos(2.0 * M_PI * b);
  const double img = std::exp(mu + c.sigma * z);
  m.image_bytes = std::max<uint64_t>(2, uint64_t(std::llround(img)));
  m.latent_bytes =
      std::min(m.image_bytes - 1, std::max<uint64_t>(1, uint64_t(std::llround(img * (c.latent_mb / c.image_mb)))));
  return m;
}
}  // namespace

Workload synth(const SynthCfg& c) {
  std::mt19937_64 r(c.seed);
  const uint64_t arrivals = uint64_t(std::floor(c.arrival_rate * double(c.days)));
  const uint64_t n = c.n_objects_initial + arrivals;
  std::vector<uint32_t> born(n, 0);
  for (uint64_t k = 0; k < arrivals; ++k)
    born[c.n_objects_initial + k] = std::min<uint32_t>(uint32_t(std::floor(double(k + 1) / c.arrival_rate)), c.days - 1);
  std::vector<uint32_t> rank(n);
  std::iota(rank.begin(), rank.end(), 0u);
  for (size_t i = n - 1; i > 0; --i) {
    const size_t j = size_t(u01(r) * double(i + 1));
    std::swap(rank[i], rank[std::min(j, i)]);
  }
  std::vector<double> zw(n);
  for (uint64_t i = 0; i < n; ++i) zw[i] = std::pow(double(rank[i]) + 1.0, -c.zipf);
  Workload w;
  w.objects_total = n;
  w.meta.reserve(n);
  for (uint64_t i = 0; i < n; ++i) w.meta.push_back(size_draw(c, r));
  w.trace.reserve(c.requests_per_day * c.days);
  const uint64_t day_ms = 86'400'000ull;
  std::vector<double> wt(n);
  std::vector<std::pair<uint64_t, uint32_t>> buf;
  buf.reserve(c.requests_per_day);
  for (uint32_t d = 0; d < c.days; ++d) {
    for (uint64_t i = 0; i < n; ++i)
      wt[i] = born[i] > d ? 0.0 : zw[i] * std::pow(double(d - born[i]) + 1.0, -c.decay);
    Alias tab(wt);
    buf.clear();
    for (uint64_t q = 0; q < c.requests_per_day; ++q) {
      uint32_t o = tab.draw(r);
      while (wt[o] == 0.0) o = tab.draw(r);
      const uint64_t ts = uint64_t(d) * day_ms + uint64_t(u01(r) * double(day_ms));
      buf.emplace_back(ts, o);
    }
    std::stable_sort(buf.begin(), buf.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    for (const auto& [ts, o] : buf) w.trace.push_back(Rec{ts, uint64_t(o) + 1});
  }
  return w;
}

// ================================================================ cache
namespace {
uint64_t scaled(double frac, uint64_t total) {  // floor with ulp-wobble guard (dual_cache.cpp:59-66)
  const double x = frac * double(total);
  const double rr = std::round(x);
  if (std::abs(x - rr) < std::max(1e-9, 4e-15 * x)) return uint64_t(rr);
  return uint64_t(std::floor(x));
}
}  // namespace

Cache::Cache(uint64_t capacity, double alpha, double tau, uint32_t h) : cap_(capacity), alpha_(alpha), tau_(tau), h_(h) {
  budgets();
}

void Cache::budgets() {
  t_[0].budget = scaled(alpha_, cap_);
  t_[1].budget = scaled(1.0 - alpha_, cap_);
  for (auto& t : t_) t.main_budget = scaled(1.0 - tau_, t.budget);
}

int Cache::alloc(uint64_t id, uint64_t bytes) {
  int n;
  if (!free_.empty()) {
    n = free_.back();
    free_.pop_back();
  } else {
    n = (int)nodes_.size();
    nodes_.push_back({});
  }
  nodes_[n] = Node{id, bytes, 0, -1, -1, 0, 0};
  return n;
}
void Cache::release(int n) { free_.push_back(n); }

void Cache::unlink(int n) {
  Node& x = nodes_[n];
  List& l = x.tail ? t_[x.tier].tl : t_[x.tier].main;
  if (x.prev >= 0) nodes_[x.prev].next = x.next; else l.head = x.next;
  if (x.next >= 0) nodes_[x.next].prev = x.prev; else l.tail = x.prev;
  x.prev = x.next = -1;
}

void Cache::push_front(int t, bool tail_seg, int n) {
  Node& x = nodes_[n];
  x.tier = (uint8_t)t;
  x.tail = tail_seg;
  List& l = tail_seg ? t_[t].tl : t_[t].main;
  x.prev = -1;
  x.next = l.head;
  if (l.head >= 0) nodes_[l.head].prev = n; else l.tail = n;
  l.head = n;
}

void Cache::enforce(int t) {
  Tier& T = t_[t];
  while (T.main_used > T.main_budget) {  // demote main LRU to tail MRU
    const int n = T.main.tail;
    unlink(n);
    T.main_used -= nodes_[n].bytes;
    T.tail_used += nodes_[n].bytes;
    push_front(t, true, n);
  }
  while (T.tail_used > T.budget - T.main_budget) {  // evict tail LRU
    const int n = T.tl.tail;
    unlink(n);
    T.tail_used -= nodes_[n].bytes;
    where_.erase(nodes_[n].id);
    release(n);
  }
}

void Cache::admit(int t, uint64_t id, uint64_t bytes) {
  if (where_.count(id)) throw std::logic_error("admit: already cached");
  if (bytes > t_[t].budget) return;  // bypass
  const int n = alloc(id, bytes);
  push_front(t, false, n);
  t_[t].main_used += bytes;
  where_[id] = n;
  enforce(t);
}

Outcome Cache::lookup(uint64_t id, const Meta& m, bool* promoted, bool* tail_hit) {
  if (promoted) *promoted = false;
  ctr_.total++;
  auto f = where_.find(id);
  if (f == where_.end()) {
    ctr_.image_misses++;
    ctr_.full_misses++;
    if (tail_hit) *tail_hit = false;
    return Outcome::FullMiss;
  }
  const int n = f->second;
  const int t = nodes_[n].tier;
  const bool was_tail = nodes_[n].tail;
  if (tail_hit) *tail_hit = was_tail;
  // move to the MRU end of the tier's main segment
  unlink(n);
  if (was_tail) {
    t_[t].tail_used -= nodes_[n].bytes;
    t_[t].main_used += nodes_[n].bytes;
  }
  push_front(t, false, n);
  if (t == 0) {
    if (was_tail) ctr_.image_tail_hits++;
    enforce(0);
    return Outcome::ImageHit;
  }
  ctr_.image_misses++;
  if (was_tail) ctr_.latent_tail_hits++;
  enforce(1);
  auto g = where_.find(id);
  if (g == where_.end()) return Outcome::LatentHit;  // evicted by its own move (budgets shrank)
  const int c = g->second;
  if (nodes_[c].hits + 1 >= h_) {
    if (m.image_bytes <= t_[0].main_budget) {
      unlink(c);
      if (nodes_[c].tail) t_[1].tail_used -= nodes_[c].bytes; else t_[1].main_used -= nodes_[c].bytes;
      nodes_[c].bytes = m.image_bytes;
      nodes_[c].hits = 0;
      push_front(0, false, c);
      t_[0].main_used += m.image_bytes;
      enforce(0);
      if (promoted) *promoted = true;
    } else {
      nodes_[c].hits = h_ - 1;
    }
  } else {
    nodes_[c].hits++;
  }
  return Outcome::LatentHit;
}

void Cache::set_alpha(double a) {
  alpha_ = a;
  budgets();
  enforce(0);
  enforce(1);
}

std::vector<uint64_t> Cache::resident() const {
  std::vector<uint64_t> out;
  for (int t = 0; t < 2; ++t)
    for (const List* l : {&t_[t].main, &t_[t].tl})
      for (int n = l->head; n >= 0; n = nodes_[n].next) out.push_back(nodes_[n].id);
  return out;
}

// ================================================================ tuner
double gradient_ms(const Counters& c, double td, double tf) {
  if (c.total == 0) return 0.0;
  const double tot = double(c.total);
  const double mr_img = double(c.image_misses) / tot, d_img = double(c.image_tail_hits) / tot;
  double mr_lat = 0.0, d_lat = 0.0;
  if (c.image_misses) {
    mr_lat = double(c.full_misses) / double(c.image_misses);
    d_lat = double(c.latent_tail_hits) / double(c.image_misses);
  }
  return -d_img * (td + tf * mr_lat) + tf * mr_img * d_lat;
}

double step_alpha(double a, double g, double step, double lo, double hi) {
  if (g < 0.0) a += step;
  else if (g > 0.0) a -= step;
  return std::clamp(a, lo, hi);
}

double pct(const std::vector<double>& v, double q) {
  if (v.empty()) return 0.0;
  const size_t idx = size_t(std::ceil(q * double(v.size())));
  return v[std::min(v.size() - 1, idx == 0 ? 0 : idx - 1)];
}

// ================================================================ replay (virtual time)
ReplayOut replay(const Workload& w, const ReplayCfg& cfg) {
  const size_t N = w.trace.size();
  ReplayOut out;
  out.outcome.assign(N, 0);
  out.job_of.assign(N, -1);
  const uint64_t footprint = w.objects_total * w.meta[0].image_bytes;
  Cache cache(uint64_t(double(footprint) * cfg.cache_frac), cfg.alpha0, cfg.tau, cfg.h);
  const uint64_t W = cfg.window ? cfg.window : std::max<uint64_t>(10'000, N / 60);
  uint64_t win_lookups = 0;
  double t_decode = 0.0;
  bool seen_decode = false;

  auto service = [&](uint32_t b) {
    const auto& s = cfg.service_ms;
    if (s.empty()) return cfg.nominal_decode_ms;
    return s[std::min<size_t>(b, s.size()) - 1] * (b > s.size() ? double(b) / double(s.size()) : 1.0);
  };

  // events: ready jobs wait in a FIFO; GPUs become free at gpu_free[g]
  std::vector<double> gpu_free(cfg.gpus, 0.0);
  std::deque<int> ready;               // job indices in ready order
  std::unordered_map<uint64_t, int> inflight;  // object -> job (coalescing)
  // pending completions (t_done, job) to release coalescing and observe latency in time order
  using Done = std::pair<double, int>;
  std::priority_queue<Done, std::vector<Done>, std::greater<Done>> done_q;
  // jobs not yet ready (full misses fetching): (t_ready, job)
  std::priority_queue<Done, std::vector<Done>, std::greater<Done>> fetch_q;

  // Batched FIFO service, decided at event times <= t: the earliest-free GPU closes a batch at
  // max(free, min(time the queue held max_batch jobs, oldest ready + max_wait)) and takes every
  // ready job (up to max_batch) by then.  Fetch completions feed the ready FIFO in time order.
  auto dispatch_until = [&](double t) {
    for (;;) {
      double t_batch = 1e300;
      int g = 0;
      if (!ready.empty()) {
        g = int(std::min_element(gpu_free.begin(), gpu_free.end()) - gpu_free.begin());
        double close = out.jobs[ready.front()].t_ready + cfg.max_wait_ms;
        if ((int)ready.size() >= cfg.max_batch) close = std::min(close, out.jobs[ready[cfg.max_batch - 1]].t_ready);
        t_batch = std::max(gpu_free[g], close);
      }
      if (ready.empty() && fetch_q.empty()) return;
      const double t_fetch = fetch_q.empty() ? 1e300 : fetch_q.top().first;
      if (std::min(t_batch, t_fetch) > t) return;
      if (!fetch_q.empty() && t_fetch <= t_batch) {
        ready.push_back(fetch_q.top().second);
        fetch_q.pop();
        continue;
      }
      uint32_t b = 0, lim = (uint32_t)cfg.max_batch;
      if (cfg.cost_policy && !cfg.service_ms.empty()) {  // the live batcher's rule (lbx_batch_pick)
        uint32_t q = 0;
        while (q < ready.size() && (int)q < cfg.max_batch && out.jobs[ready[q]].t_ready <= t_batch) ++q;
        lim = lbx_batch_pick_rule(cfg.service_ms.data(), (uint32_t)cfg.service_ms.size(), q, (uint32_t)cfg.max_batch);
      }
      std::vector<int> batch;
      while (!ready.empty() && b < lim && out.jobs[ready.front()].t_ready <= t_batch) {
        batch.push_back(ready.front());
        ready.pop_front();
        ++b;
      }
      const double end = t_batch + service(b);
      gpu_free[g] = end;
      for (int j : batch) {
        Job& J = out.jobs[j];
        J.t_start = t_batch;
        J.t_end = end;
        J.gpu = g;
        J.batch = b;
        done_q.push({end + cfg.net_ms, j});
      }
    }
  };
  auto complete_until = [&](double t) {
    while (!done_q.empty() && done_q.top().first <= t) {
      const int j = done_q.top().second;
      done_q.pop();
      Job& J = out.jobs[j];
      inflight.erase(J.object_id);
      const double sample = J.t_end - J.t_ready;  // queue + batch wait + GPU, as on_job_done observes
      t_decode = seen_decode ? (1.0 - cfg.ewma) * t_decode + cfg.ewma * sample : sample;
      seen_decode = true;
    }
  };

  for (size_t i = 0; i < N; ++i) {
    const double t = double(w.trace[i].ts_ms) / cfg.time_scale;
    dispatch_until(t);
    complete_until(t);
    const uint64_t id = w.trace[i].object_id;
    auto fl = inflight.find(id);
    if (fl != inflight.end()) {  // follower: waits on the in-flight decode, never probes
      out.job_of[i] = fl->second;
      out.outcome[i] = (uint8_t)Outcome::LatentHit;
      out.coalesced++;
      continue;
    }
    const Meta& m = w.meta[id - 1];
    const Outcome o = cache.lookup(id, m);
    out.outcome[i] = (uint8_t)o;
    const bool due = ++win_lookups >= W;
    if (o == Outcome::ImageHit) {
      out.image_hits++;
    } else {
      Job J;
      J.leader = i;
      J.object_id = id;
      J.t_arrive = t;
      J.t_ready = t;
      if (o == Outcome::FullMiss) {
        out.full_misses++;
        cache.admit_latent(id, m);
        J.t_ready = t + cfg.fetch_ms;
      } else {
        out.latent_hits++;
      }
      const int j = (int)out.jobs.size();
      out.jobs.push_back(J);
      out.job_of[i] = j;
      inflight[id] = j;
      if (o == Outcome::FullMiss) fetch_q.push({J.t_ready, j});
      else ready.push_back(j);
    }
    if (due) {
      const Counters c = cache.take_counters();
      const double td = seen_decode ? t_decode : cfg.nominal_decode_ms;
      const double g = gradient_ms(c, td, cfg.fetch_ms);
      if (cfg.adaptive) cache.set_alpha(step_alpha(cache.alpha(), g, cfg.step, 0.0, 1.0));
      win_lookups = 0;
      out.windows++;
    }
  }
  dispatch_until(1e300);
  complete_until(1e300);
  out.final_alpha = cache.alpha();
  return out;
}

LatencyReport report(const ReplayOut& r, const ReplayCfg& cfg, const Workload& w) {
  const uint64_t n = w.trace.size();
  const uint64_t warm = uint64_t(std::floor(cfg.warmup_fraction * double(n)));
  std::vector<double> dec, e2e;
  double bsum = 0;
  for (const Job& J : r.jobs)
    if (J.leader >= warm) {
      dec.push_back(J.t_end - J.t_ready);
      bsum += J.batch;
    }
  for (uint64_t i = warm; i < n; ++i) {
    const double t = double(w.trace[i].ts_ms) / cfg.time_scale;
    const int64_t j = r.job_of[i];
    e2e.push_back(j < 0 ? cfg.net_ms : r.jobs[j].t_end + cfg.net_ms - t);
  }
  LatencyReport rep{};
  std::sort(dec.begin(), dec.end());
  std::sort(e2e.begin(), e2e.end());
  rep.n_decodes = dec.size();
  rep.n_requests = e2e.size();
  rep.decode_p50 = pct(dec, 0.50);
  rep.decode_p99 = pct(dec, 0.99);
  rep.decode_mean = dec.empty() ? 0 : std::accumulate(dec.begin(), dec.end(), 0.0) / double(dec.size());
  rep.e2e_p50 = pct(e2e, 0.50);
  rep.e2e_p99 = pct(e2e, 0.99);
  rep.e2e_mean = e2e.empty() ? 0 : std::accumulate(e2e.begin(), e2e.end(), 0.0) / double(e2e.size());
  rep.mean_batch = dec.empty() ? 0 : bsum / double(dec.size());
  return rep;
}

}  // namespace lbsim
