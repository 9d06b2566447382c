// ref_binding -- the reference-side binding a LatentBox maintainer would add, compiled against the
// reference's OWN simulator sources (oracle/ref.mk -> oracle/_ref/libref_sim.a, built from
// /root/reference/proj/src, never copied) and this repo's C ABI (liblbx.so).
// describes the call-site mapping; this program is it, end to end:
//
//   1. the decode the reference models as the constant LatencyModel::decode_ms = 40
//      (proj/include/latentbox/sim.hpp:19, consumed by Engine::on_job_ready, proj/src/sim.cpp:409-429)
//      is run for real: lbx_reconstruct of one sd3 16x128x128 LBLP blob -> 1024^2 uint8 RGB in
//      page-locked host memory, batch 1 (the cost rule's choice on B200), timed per call;
//   2. the reference's own simulator (lbx::run, proj/src/sim.cpp:561) replays the reference's own
//      workload generator (lbx::generate_trace, proj/src/synth.cpp:103) twice -- stock 40 ms and the
//      measured B200 decode p50 -- and both reports' latency / GPU-queue summaries are printed.
//
//   ref_binding [--decode-ms X] [--requests-per-day N] [--days D] [--gpus G] [--time-scale S]
// --decode-ms skips the GPU measurement (CPU-only check of the binding).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "latentbox/sim.hpp"    // reference (namespace lbx)
#include "latentbox/synth.hpp"  // reference
#include "lbx/reconstruct.h"    // this repo's C ABI (extern "C", no namespace)

namespace {

double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// p50 of batch-1 lbx_reconstruct calls (host blob in, RGB in pinned host memory out).
double measure_decode_ms(int reps) {
  lbx_decoder_desc d{};
  d.family = LBX_FAMILY_SD3;
  d.latent_h = d.latent_w = 128;
  d.device = 0;
  d.max_batch = 1;
  lbx_decoder* dec = nullptr;
  if (lbx_decoder_create(&d, &dec) != LBX_OK) {
    std::fprintf(stderr, "lbx_decoder_create: %s\n", lbx_last_error());
    return -1;
  }
  std::vector<uint16_t> lat(16 * 128 * 128);
  uint64_t x = 12345;
  for (auto& v : lat) {  // fp16 values in [-2, 2): sign, exponent 13..15, random mantissa
    x = x * 6364136223846793005ull + 1442695040888963407ull;
    v = (uint16_t)(((x >> 63) << 15) | ((13 + (x >> 40) % 3) << 10) | ((x >> 20) & 0x3FF));
  }
  size_t nb = 0;
  lbx_pack(lat.data(), 1, 16, 128, 128, nullptr, 0, &nb);
  std::vector<uint8_t> blob(nb);
  lbx_pack(lat.data(), 1, 16, 128, 128, blob.data(), nb, &nb);
  uint8_t* rgb = static_cast<uint8_t*>(lbx_host_alloc(1024 * 1024 * 3));
  const uint8_t* bp = blob.data();
  std::vector<double> t;
  for (int i = 0; i < reps + 5; ++i) {
    const double t0 = now_ms();
    if (lbx_reconstruct(dec, &bp, &nb, 1, rgb, nullptr) != LBX_OK) {
      std::fprintf(stderr, "lbx_reconstruct: %s\n", lbx_last_error());
      return -1;
    }
    if (i >= 5) t.push_back(now_ms() - t0);
  }
  lbx_host_free(rgb);
  lbx_decoder_destroy(dec);
  std::sort(t.begin(), t.end());
  return t[t.size() / 2];
}

void print_report(const char* name, double decode_ms, const lbx::SimReport& r) {
  std::printf(
      "{\"model\": \"%s\", \"decode_ms\": %.3f, \"requests\": %llu, \"e2e_p50_ms\": %.2f, \"e2e_p99_ms\": %.2f, "
      "\"e2e_mean_ms\": %.2f, \"gpu_queue_p50_ms\": %.2f, \"gpu_queue_p99_ms\": %.2f, \"stage_decode_ms\": %.2f, "
      "\"decode_events\": %llu, \"frac_image_hit\": %.4f, \"frac_latent_hit\": %.4f, \"frac_full_miss\": %.4f}\n",
      name, decode_ms, (unsigned long long)r.total_requests, r.latency.p50, r.latency.p99, r.latency.mean,
      r.gpu_queue_wait.p50, r.gpu_queue_wait.p99, r.stage_decode_ms, (unsigned long long)r.decode_events,
      r.frac_image_hit, r.frac_latent_hit, r.frac_full_miss);
}

}  // namespace

int main(int argc, char** argv) {
  double decode_ms = -1;
  uint64_t rpd = 100000;
  uint32_t days = 10, gpus = 8;
  double scale = 10.0;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string k = argv[i];
    if (k == "--decode-ms") decode_ms = std::atof(argv[i + 1]);
    else if (k == "--requests-per-day") rpd = std::strtoull(argv[i + 1], nullptr, 10);
    else if (k == "--days") days = (uint32_t)std::atoi(argv[i + 1]);
    else if (k == "--gpus") gpus = (uint32_t)std::atoi(argv[i + 1]);
    else if (k == "--time-scale") scale = std::atof(argv[i + 1]);
  }
  const bool measured = decode_ms < 0;
  if (measured && (decode_ms = measure_decode_ms(50)) < 0) return 1;

  lbx::SynthConfig sc;  // SURVEY 8(d) C5 workload, scaled by --requests-per-day / --days
  sc.n_objects_initial = 100000;
  sc.arrival_rate = 2000;
  sc.zipf_exponent = 1.11;
  sc.decay_exponent = 1.3;
  sc.duration_days = days;
  sc.requests_per_day = rpd;
  sc.seed = 7;
  const lbx::SynthResult w = lbx::generate_trace(sc);
  uint64_t footprint = 0;
  for (const auto& kv : w.catalog) footprint += kv.second.image_bytes;

  lbx::ClusterConfig cfg;  // one node of `gpus` B200s, cache 1% of the footprint, LbAdaptive
  cfg.n_nodes = 1;
  cfg.gpus_per_node = gpus;
  cfg.node_cache_bytes = footprint / 100;
  cfg.policy = lbx::Policy::LbAdaptive;
  cfg.tuner.window_requests = 0;
  cfg.time_scale = scale;
  std::printf("{\"binding\": \"reference lbx::run with LatencyModel::decode_ms from lbx_reconstruct\", "
              "\"decode_measured\": %s, \"gpus_per_node\": %u, \"time_scale\": %g, \"trace_requests\": %zu}\n",
              measured ? "true" : "false", gpus, scale, w.trace.size());
  for (int k = 0; k < 2; ++k) {
    cfg.latency.decode_ms = k == 0 ? 40.0 : decode_ms;
    const lbx::SimReport r = lbx::run(w.trace, w.catalog, cfg);
    print_report(k == 0 ? "reference stock (decode_ms = 40)" : (measured ? "B200 lbx_reconstruct p50"
                                                                          : "given decode_ms"),
                 cfg.latency.decode_ms, r);
  }
  return 0;
}
