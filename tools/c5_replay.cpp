// c5_replay -- BASELINE config 5: Zipf/decaying-popularity trace replayed through the dual-format
// cache split, with decode-on-miss served by batched B200 decodes; reports nearest-rank p50/p99 of
// the decode stage (queue + batch wait + GPU) and end to end.
//
//   c5_replay sim  [opts]   whole trace in virtual time; GPU service = measured batch curve
//   c5_replay live [opts]   measure the batch curve on the local GPUs (lbx_decoder), run the
//                           virtual-time replay, then replay one window's decode jobs in wall-clock
//                           through the real multi-GPU batcher (lbx_batcher) and report both
//
// Workload defaults = SURVEY.md 8(d) C5: 100 K initial objects, 2000 arrivals/day, Zipf 1.11,
// decay 1.3, 1 M requests/day x 10 days, seed 7; cache 1% of footprint, tau 0.1, h 8, LbAdaptive.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "lb_sim.hpp"
#include "lbx/batcher.h"

namespace {

struct Opts {
  std::string mode = "sim";
  lbsim::SynthCfg synth;
  lbsim::ReplayCfg rp;
  double window_s = 20.0;      // live: wall-clock seconds of decode jobs replayed
  double window_start = 0.6;   // live: window start as a fraction of the trace duration
  int n_devices = 1;
  std::string service;         // "ms1,ms2,ms4,ms8,ms16,ms32" (sim mode); empty = defaults
  std::string policy = "cost"; // batch sizing: "cost" (lbx_batch_pick over the curve) or "greedy"
  std::string json;
  std::string dump;            // live: per-job "submit_ms start_ms end_ms batch" lines (diagnostics)
};

// Batch service curve measured on one B200 for 16x128x128 -> 1024^2 (lbx_reconstruct, host blobs,
// power-capped steady state, profiles/r1f_c5_live_1gpu_25x_cost_sustained_curve.json); sizes
// 1,2,4,8,16,32.  Used by sim mode unless --service or live measurement overrides.
const double kDefaultService[6] = {9.06, 17.85, 35.64, 73.03, 149.75, 293.35};
const int kSizes[6] = {1, 2, 4, 8, 16, 32};

std::vector<double> curve_from(const double* pts, int maxb) {
  std::vector<double> s(maxb);
  for (int b = 1; b <= maxb; ++b) {
    int k = 0;
    while (k < 5 && kSizes[k + 1] < b) ++k;
    const double b0 = kSizes[k], b1 = kSizes[k + 1];
    const double f = std::clamp((b - b0) / (b1 - b0), 0.0, 1.0);
    s[b - 1] = b <= kSizes[5] ? pts[k] + f * (pts[k + 1] - pts[k]) : pts[5] * b / 32.0;
  }
  return s;
}

bool parse(int argc, char** argv, Opts& o) {
  if (argc < 2) return false;
  o.mode = argv[1];
  o.synth.n_objects_initial = 100000;
  o.synth.arrival_rate = 2000;
  o.synth.days = 10;
  o.synth.requests_per_day = 1000000;
  o.synth.seed = 7;
  for (int i = 2; i + 1 < argc; i += 2) {
    const std::string k = argv[i], v = argv[i + 1];
    if (k == "--scale") o.rp.time_scale = std::stod(v);
    else if (k == "--gpus") o.rp.gpus = std::stoi(v);
    else if (k == "--devices") o.n_devices = std::stoi(v);
    else if (k == "--max-batch") o.rp.max_batch = std::stoi(v);
    else if (k == "--max-wait-ms") o.rp.max_wait_ms = std::stod(v);
    else if (k == "--days") o.synth.days = (uint32_t)std::stoul(v);
    else if (k == "--rpd") o.synth.requests_per_day = std::stoull(v);
    else if (k == "--objects") o.synth.n_objects_initial = std::stoull(v);
    else if (k == "--seed") o.synth.seed = std::stoull(v);
    else if (k == "--cache-frac") o.rp.cache_frac = std::stod(v);
    else if (k == "--window-s") o.window_s = std::stod(v);
    else if (k == "--window-start") o.window_start = std::stod(v);
    else if (k == "--service") o.service = v;
    else if (k == "--policy") o.policy = v;
    else if (k == "--json") o.json = v;
    else if (k == "--dump") o.dump = v;
    else {
      std::fprintf(stderr, "unknown option %s\n", k.c_str());
      return false;
    }
  }
  return o.mode == "sim" || o.mode == "live";
}

double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Synthetic 16x128x128 latents (smooth field + noise), packed lossless.
std::vector<std::vector<uint8_t>> make_blobs(int n) {
  std::vector<std::vector<uint8_t>> out;
  std::vector<uint16_t> lat(16 * 128 * 128);
  uint64_t s = 0x243F6A8885A308D3ull;
  for (int i = 0; i < n; ++i) {
    for (size_t j = 0; j < lat.size(); ++j) {
      s = s * 6364136223846793005ull + 1442695040888963407ull;
      const float f = std::sin(0.05f * float(j % 128) + float(i)) + 0.1f * (float((s >> 40) & 0xFFFF) / 65536.0f - 0.5f);
      // fp32 -> fp16 bits (values are small and normal; truncation is fine for synthetic data)
      uint32_t b;
      std::memcpy(&b, &f, 4);
      const uint32_t sign = (b >> 16) & 0x8000u;
      const int e = int((b >> 23) & 0xFF) - 127 + 15;
      lat[j] = e <= 0 ? uint16_t(sign) : uint16_t(sign | (uint32_t(e) << 10) | ((b >> 13) & 0x3FF));
    }
    size_t need = 0;
    lbx_pack(lat.data(), LBLP_LOSSLESS, 16, 128, 128, nullptr, 0, &need);
    std::vector<uint8_t> blob(need);
    lbx_pack(lat.data(), LBLP_LOSSLESS, 16, 128, 128, blob.data(), need, &need);
    out.push_back(std::move(blob));
  }
  return out;
}

bool measure_curve(int device, int maxb, const std::vector<std::vector<uint8_t>>& blobs, double* pts) {
  lbx_decoder_desc d{};
  d.family = LBX_FAMILY_SD3;
  d.latent_h = d.latent_w = 128;
  d.device = device;
  d.max_batch = (uint32_t)maxb;
  lbx_decoder* dec = nullptr;
  if (lbx_decoder_create(&d, &dec) != LBX_OK) {
    std::fprintf(stderr, "decoder: %s\n", lbx_last_error());
    return false;
  }
  uint8_t* rgb_mem = static_cast<uint8_t*>(lbx_host_alloc((size_t)maxb * 1024 * 1024 * 3));  // pinned, as live
  if (!rgb_mem) {
    std::fprintf(stderr, "pinned host allocation failed\n");
    lbx_decoder_destroy(dec);
    return false;
  }
  struct View { uint8_t* p; uint8_t* data() { return p; } } rgb{rgb_mem};
  std::vector<const uint8_t*> ptrs;
  std::vector<size_t> sizes;
  for (int i = 0; i < maxb; ++i) {
    ptrs.push_back(blobs[i % blobs.size()].data());
    sizes.push_back(blobs[i % blobs.size()].size());
  }
  for (int k = 0; k < 6; ++k)  // capture every graph first
    if (kSizes[k] <= maxb) lbx_reconstruct(dec, ptrs.data(), sizes.data(), kSizes[k], rgb.data(), nullptr);
  // steady state: a GPU that decodes back to back sits at its power cap, so warm up for 3 s and time
  // each size over >= 0.4 s (a short burst at boost clocks underestimates the service time by ~10%)
  for (const double t0 = now_ms(); now_ms() - t0 < 3000.0;)
    lbx_reconstruct(dec, ptrs.data(), sizes.data(), maxb, rgb.data(), nullptr);
  for (int k = 0; k < 6; ++k) {
    const int b = kSizes[k];
    if (b > maxb) {
      pts[k] = pts[k - 1] * b / kSizes[k - 1];
      continue;
    }
    int reps = 0;
    const double t0 = now_ms();
    while (reps < 3 || now_ms() - t0 < 400.0) {
      lbx_reconstruct(dec, ptrs.data(), sizes.data(), b, rgb.data(), nullptr);
      ++reps;
    }
    pts[k] = (now_ms() - t0) / reps;
    std::fprintf(stderr, "service b=%d: %.2f ms (%.1f img/s, %d reps)\n", b, pts[k], b * 1000.0 / pts[k], reps);
  }
  lbx_decoder_destroy(dec);
  lbx_host_free(rgb_mem);
  return true;
}

}  // namespace

int main(int argc, char** argv) {
  Opts o;
  if (!parse(argc, argv, o)) {
    std::fprintf(stderr,
                 "usage: c5_replay sim|live [--scale S] [--gpus G] [--devices D] [--max-batch B] [--max-wait-ms W]\n"
                 "       [--days N] [--rpd R] [--objects N] [--seed S] [--cache-frac F] [--window-s S]\n"
                 "       [--window-start F] [--service m1,m2,m4,m8,m16,m32] [--policy cost|greedy]\n"
                 "       [--json out.json]\n");
    return 2;
  }
  double pts[6];
  std::copy(kDefaultService, kDefaultService + 6, pts);
  std::vector<std::vector<uint8_t>> blobs;
  if (o.mode == "live") {
    blobs = make_blobs(64);
    if (!measure_curve(0, o.rp.max_batch, blobs, pts)) return 1;
    o.rp.gpus = o.n_devices;
  } else if (!o.service.empty()) {
    int k = 0;
    for (size_t p = 0; k < 6 && p <= o.service.size(); ++k) {
      const size_t q = o.service.find(',', p);
      pts[k] = std::stod(o.service.substr(p, q == std::string::npos ? std::string::npos : q - p));
      if (q == std::string::npos) break;
      p = q + 1;
    }
  }
  o.rp.service_ms = curve_from(pts, o.rp.max_batch);
  o.rp.cost_policy = o.policy == "cost";

  const double t0 = now_ms();
  const lbsim::Workload w = lbsim::synth(o.synth);
  const double t1 = now_ms();
  lbsim::ReplayOut r = lbsim::replay(w, o.rp);
  const double t2 = now_ms();
  const lbsim::LatencyReport rep = lbsim::report(r, o.rp, w);
  const double n = double(w.trace.size());
  std::fprintf(stderr, "synth %.1f s, replay %.1f s\n", (t1 - t0) / 1e3, (t2 - t1) / 1e3);

  char buf[4096];
  int len = std::snprintf(
      buf, sizeof buf,
      "{\"config\": \"c5\", \"mode\": \"%s\", \"requests\": %.0f, \"objects\": %llu, \"time_scale\": %g, \"gpus\": %d, "
      "\"max_batch\": %d, \"policy\": \"%s\", \"max_wait_ms\": %g, \"cache_frac\": %g, \"mix\": {\"image_hit\": %.4f, "
      "\"latent_hit\": %.4f, \"full_miss\": %.4f, \"coalesced\": %.4f}, \"final_alpha\": %.4f, \"windows\": %llu, "
      "\"service_ms\": [%.2f, %.2f, %.2f, %.2f, %.2f, %.2f], \"sim\": {\"decode_p50_ms\": %.2f, \"decode_p99_ms\": "
      "%.2f, \"decode_mean_ms\": %.2f, \"e2e_p50_ms\": %.2f, \"e2e_p99_ms\": %.2f, \"e2e_mean_ms\": %.2f, "
      "\"decodes\": %llu, \"mean_batch\": %.2f}",
      o.mode.c_str(), n, (unsigned long long)w.objects_total, o.rp.time_scale, o.rp.gpus, o.rp.max_batch,
      o.rp.cost_policy ? "cost" : "greedy",
      o.rp.max_wait_ms, o.rp.cache_frac, r.image_hits / n, r.latent_hits / n, r.full_misses / n, r.coalesced / n,
      r.final_alpha, (unsigned long long)r.windows, pts[0], pts[1], pts[2], pts[3], pts[4], pts[5], rep.decode_p50,
      rep.decode_p99, rep.decode_mean, rep.e2e_p50, rep.e2e_p99, rep.e2e_mean, (unsigned long long)rep.n_decodes,
      rep.mean_batch);
  std::string out(buf, len);

  if (o.mode == "live") {
    // decode jobs of the window [T0, T0 + window) in virtual ms, replayed in wall-clock
    const double T_end = double(w.trace.back().ts_ms) / o.rp.time_scale;
    const double T0 = o.window_start * T_end, T1 = T0 + o.window_s * 1000.0;
    std::vector<int> jobs;
    for (size_t j = 0; j < r.jobs.size(); ++j)
      if (r.jobs[j].t_ready >= T0 && r.jobs[j].t_ready < T1) jobs.push_back((int)j);
    std::sort(jobs.begin(), jobs.end(), [&](int a, int b) { return r.jobs[a].t_ready < r.jobs[b].t_ready; });
    std::vector<int> devs(o.n_devices);
    for (int i = 0; i < o.n_devices; ++i) devs[i] = i;
    lbx_shape shape{LBX_FAMILY_SD3, 128, 128};
    lbx_batcher_desc bd{devs.data(), o.n_devices, &shape, 1, (uint32_t)o.rp.max_batch,
                        (uint32_t)(o.rp.max_wait_ms * 1000.0), 0, o.rp.cost_policy ? 1u : 0u};
    lbx_batcher* b = nullptr;
    if (lbx_batcher_create(&bd, &b) != LBX_OK) {
      std::fprintf(stderr, "batcher: %s\n", lbx_last_error());
      return 1;
    }
    const size_t img = 1024ull * 1024 * 3;
    // output buffers in flight: enough that small batch caps never stall submission
    const int nbuf = std::max(64, 4 * o.rp.max_batch) * o.n_devices;
    // page-locked output buffers, as an integration would use (pageable memory adds a staging copy)
    uint8_t* pool_mem = static_cast<uint8_t*>(lbx_host_alloc((size_t)nbuf * img));
    std::vector<uint8_t> pool_fallback;
    if (!pool_mem) {
      pool_fallback.resize((size_t)nbuf * img);
      pool_mem = pool_fallback.data();
    }
    struct PoolView { uint8_t* p; uint8_t* data() { return p; } } pool{pool_mem};
    std::vector<int> free_bufs;
    for (int i = nbuf - 1; i >= 0; --i) free_bufs.push_back(i);
    std::vector<int> buf_of(jobs.size(), -1);
    std::vector<double> lag(jobs.size(), 0.0);  // submit - due (ms): a stalled submission still counts
    std::vector<double> live_dec, sim_dec;
    std::vector<lbx_completion> all_comp;
    std::vector<lbx_completion> comp(512);
    uint64_t backpressure = 0;
    auto drain = [&](uint32_t wait_us) {
      const int k = lbx_batcher_poll(b, comp.data(), (int)comp.size(), wait_us);
      for (int i = 0; i < k; ++i) {
        const size_t q = comp[i].request_id;
        live_dec.push_back((comp[i].t_end_us - comp[i].t_submit_us) / 1000.0 + lag[q]);
        if (!o.dump.empty()) all_comp.push_back(comp[i]);
        free_bufs.push_back(buf_of[q]);
      }
      return k;
    };
    const double wall0 = now_ms();
    for (size_t q = 0; q < jobs.size(); ++q) {
      const lbsim::Job& J = r.jobs[jobs[q]];
      const double due = wall0 + (J.t_ready - T0);
      for (;;) {
        const double now = now_ms();
        if (now >= due && !free_bufs.empty()) break;
        if (free_bufs.empty()) ++backpressure;
        drain(free_bufs.empty() ? 2000 : (uint32_t)std::max(0.0, std::min(2000.0, (due - now) * 1000.0)));
      }
      buf_of[q] = free_bufs.back();
      free_bufs.pop_back();
      lag[q] = std::max(0.0, now_ms() - due);
      const auto& blob = blobs[J.object_id % blobs.size()];
      lbx_batcher_submit(b, q, 0, blob.data(), blob.size(), pool.data() + (size_t)buf_of[q] * img);
      sim_dec.push_back(J.t_end - J.t_ready);
    }
    while (lbx_batcher_pending(b)) drain(10000);
    const double wall = (now_ms() - wall0) / 1000.0;
    lbx_batcher_destroy(b);
    if (pool_fallback.empty()) lbx_host_free(pool_mem);
    if (!o.dump.empty() && !all_comp.empty()) {
      FILE* f = std::fopen(o.dump.c_str(), "w");
      const uint64_t base = all_comp.front().t_submit_us;
      for (const auto& c : all_comp)
        if (f) std::fprintf(f, "%.3f %.3f %.3f %u\n", (c.t_submit_us - base) / 1e3, (c.t_start_us - base) / 1e3,
                            (c.t_end_us - base) / 1e3, c.batch_size);
      if (f) std::fclose(f);
    }
    std::sort(live_dec.begin(), live_dec.end());
    std::sort(sim_dec.begin(), sim_dec.end());
    len = std::snprintf(buf, sizeof buf,
                        ", \"live\": {\"devices\": %d, \"window_virtual_ms\": [%.0f, %.0f], \"jobs\": %zu, "
                        "\"wall_s\": %.2f, \"decode_p50_ms\": %.2f, \"decode_p99_ms\": %.2f, \"sim_p50_ms\": %.2f, "
                        "\"sim_p99_ms\": %.2f, \"throughput_img_s\": %.1f, \"backpressure_waits\": %llu}",
                        o.n_devices, T0, T1, jobs.size(), wall, lbsim::pct(live_dec, 0.5), lbsim::pct(live_dec, 0.99),
                        lbsim::pct(sim_dec, 0.5), lbsim::pct(sim_dec, 0.99), jobs.size() / wall,
                        (unsigned long long)backpressure);
    out += std::string(buf, len);
  }
  out += "}";
  std::printf("%s\n", out.c_str());
  if (!o.json.empty()) {
    FILE* f = std::fopen(o.json.c_str(), "w");
    if (f) {
      std::fprintf(f, "%s\n", out.c_str());
      std::fclose(f);
    }
  }
  return 0;
}
