// Multi-GPU decode-on-miss request batcher (include/lbx/batcher.h).
//
// One worker thread per device owns one lbx_decoder per shape class (created on that thread's
// device).  Requests wait in per-shape FIFO queues.  An idle worker closes a batch on the shape
// whose head request is oldest.  It does so once that queue holds max_batch requests, once the head
// has waited max_wait_us, or when draining at shutdown.  Then it runs one lbx_reconstruct_v.  Pulling
// work only when idle is what makes the placement least-loaded-first (proj/src/sim.cpp:238-243);
// the FIFO order per shape mirrors the simulator's FIFO GPU (sim.cpp:413).  With policy 1 the batch
// size comes from lbx_batch_pick over the worker's own measured service curve.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "lbx/batch_pick.h"
#include "lbx/batcher.h"

namespace lbx {
lbx_status set_last_error(lbx_status s, const std::string& m);  // decoder.cu
}

namespace {

uint64_t now_us() {
  return (uint64_t)std::chrono::duration_cast<std::chrono::microseconds>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

struct Request {
  uint64_t id;
  std::vector<uint8_t> blob;
  uint8_t* rgb;
  uint64_t t_submit;
};

}  // namespace

struct lbx_batcher {
  lbx_batcher_desc desc{};
  std::vector<int> devices;
  std::vector<lbx_shape> shapes;
  std::vector<std::deque<Request>> queues;  // per shape
  std::mutex mu;
  std::condition_variable cv_work, cv_done;
  bool stopping = false;
  std::vector<lbx_completion> done;
  uint64_t pending = 0;
  std::vector<std::thread> workers;
  std::string init_error;
  int init_status = LBX_OK;
  int workers_ready = 0;

  void worker(int dev_index);
};

namespace {

// GPU time of one decode of b latents, b = 1..max_b (measured at 1, 2, 4, ... and max_b, linear in
// between): device-resident latents, so the curve is the decode alone
std::vector<double> measure_curve(lbx_decoder* dec, int fam_channels, uint32_t lh, uint32_t lw, uint32_t max_b) {
  std::vector<double> pts_b, pts_ms;
  void* lat = nullptr;
  uint8_t* rgb = nullptr;
  const size_t lat_bytes = (size_t)max_b * fam_channels * lh * lw * 2, rgb_bytes = (size_t)max_b * 64 * lh * lw * 3;
  if (cudaMalloc(&lat, lat_bytes) != cudaSuccess || cudaMalloc(reinterpret_cast<void**>(&rgb), rgb_bytes) != cudaSuccess) {
    if (lat) cudaFree(lat);
    return {};
  }
  cudaMemset(lat, 0, lat_bytes);
  for (uint32_t b = 1;; b = std::min(2 * b, max_b)) {
    lbx_decode(dec, lat, b, rgb, nullptr);  // graph already captured by lbx_decoder_prepare
    cudaDeviceSynchronize();
    const int reps = b <= 4 ? 4 : 2;
    const uint64_t t0 = now_us();
    for (int r = 0; r < reps; ++r) lbx_decode(dec, lat, b, rgb, nullptr);
    cudaDeviceSynchronize();
    pts_b.push_back(b);
    pts_ms.push_back((now_us() - t0) / 1000.0 / reps);
    if (b == max_b) break;
  }
  cudaFree(lat);
  cudaFree(rgb);
  std::vector<double> c(max_b);
  for (uint32_t b = 1; b <= max_b; ++b) {
    size_t k = 0;
    while (k + 1 < pts_b.size() && pts_b[k + 1] < b) ++k;
    if (k + 1 >= pts_b.size() || pts_b[k] == b) { c[b - 1] = pts_ms[k]; continue; }
    const double f = (b - pts_b[k]) / (pts_b[k + 1] - pts_b[k]);
    c[b - 1] = pts_ms[k] + f * (pts_ms[k + 1] - pts_ms[k]);
  }
  return c;
}

}  // namespace

void lbx_batcher::worker(int di) {
  const int device = devices[di];
  std::vector<lbx_decoder*> decs(shapes.size(), nullptr);
  std::vector<std::vector<double>> curves(shapes.size());  // policy 1: this device's service curves
  lbx_status st = LBX_OK;
  for (size_t s = 0; s < shapes.size() && st == LBX_OK; ++s) {
    lbx_decoder_desc d{};
    d.family = shapes[s].family;
    d.latent_h = shapes[s].latent_h;
    d.latent_w = shapes[s].latent_w;
    d.weight_seed = desc.weight_seed;
    d.device = device;
    d.max_batch = desc.max_batch;
    st = lbx_decoder_create(&d, &decs[s]);
    if (st == LBX_OK) st = lbx_decoder_prepare(decs[s], desc.max_batch);  // no capture on the request path
    if (st == LBX_OK && desc.policy == 1) {
      const int ch = shapes[s].family == LBX_FAMILY_SD15 ? 4 : 16;
      curves[s] = measure_curve(decs[s], ch, shapes[s].latent_h, shapes[s].latent_w, desc.max_batch);
      if (curves[s].empty()) st = LBX_E_CUDA;
    }
  }
  {
    std::lock_guard<std::mutex> g(mu);
    if (st != LBX_OK && init_status == LBX_OK) {
      init_status = st;
      init_error = std::string("device ") + std::to_string(device) + ": " + lbx_last_error();
    }
    ++workers_ready;
  }
  cv_done.notify_all();

  std::vector<Request> batch;
  std::vector<const uint8_t*> blobs;
  std::vector<size_t> sizes;
  std::vector<uint8_t*> outs;
  for (;;) {
    int shape = -1;
    {
      std::unique_lock<std::mutex> lk(mu);
      for (;;) {
        // oldest head across shapes
        uint64_t oldest = UINT64_MAX;
        shape = -1;
        for (size_t s = 0; s < queues.size(); ++s)
          if (!queues[s].empty() && queues[s].front().t_submit < oldest) {
            oldest = queues[s].front().t_submit;
            shape = (int)s;
          }
        if (shape >= 0) {
          const bool full = queues[shape].size() >= desc.max_batch;
          const uint64_t waited = now_us() - oldest;
          if (full || waited >= desc.max_wait_us || stopping || st != LBX_OK) break;
          cv_work.wait_for(lk, std::chrono::microseconds(desc.max_wait_us - waited));
          continue;
        }
        if (stopping) break;
        cv_work.wait(lk);
      }
      if (shape < 0) break;  // stopping and drained
      auto& q = queues[shape];
      const auto& cv = curves[shape];
      const size_t take = lbx_batch_pick(cv.empty() ? nullptr : cv.data(), (uint32_t)cv.size(), (uint32_t)q.size(),
                                         desc.max_batch);
      batch.clear();
      for (size_t i = 0; i < take; ++i) {
        batch.push_back(std::move(q.front()));
        q.pop_front();
      }
    }
    cv_work.notify_all();  // another idle worker may take the remainder
    const uint64_t t_start = now_us();
    lbx_status rs = st;
    if (rs == LBX_OK) {
      blobs.clear();
      sizes.clear();
      outs.clear();
      for (auto& r : batch) {
        blobs.push_back(r.blob.data());
        sizes.push_back(r.blob.size());
        outs.push_back(r.rgb);
      }
      rs = lbx_reconstruct_v(decs[shape], blobs.data(), sizes.data(), (uint32_t)batch.size(), outs.data(), nullptr);
    }
    const uint64_t t_end = now_us();
    {
      std::lock_guard<std::mutex> g(mu);
      for (auto& r : batch)
        done.push_back(lbx_completion{r.id, (int)rs, device, (uint32_t)batch.size(), r.t_submit, t_start, t_end});
    }
    cv_done.notify_all();
  }
  for (auto* d : decs)
    if (d) lbx_decoder_destroy(d);
}

extern "C" {

uint64_t lbx_now_us(void) { return now_us(); }

uint32_t lbx_batch_pick(const double* cost_ms, uint32_t n_cost, uint32_t queued, uint32_t max_batch) {
  return lbx_batch_pick_rule(cost_ms, n_cost, queued, max_batch);
}

lbx_status lbx_batcher_create(const lbx_batcher_desc* desc, lbx_batcher** out) {
  if (!desc || !out || desc->n_devices <= 0 || !desc->devices || desc->n_shapes <= 0 || !desc->shapes ||
      desc->max_batch == 0)
    return lbx::set_last_error(LBX_E_CONFIG, "lbx_batcher_create: need devices, shapes and max_batch > 0");
  *out = nullptr;
  auto* b = new lbx_batcher;
  b->desc = *desc;
  b->devices.assign(desc->devices, desc->devices + desc->n_devices);
  b->shapes.assign(desc->shapes, desc->shapes + desc->n_shapes);
  b->queues.resize(desc->n_shapes);
  for (int i = 0; i < desc->n_devices; ++i) b->workers.emplace_back(&lbx_batcher::worker, b, i);
  {
    std::unique_lock<std::mutex> lk(b->mu);
    b->cv_done.wait(lk, [&] { return b->workers_ready == desc->n_devices; });
  }
  if (b->init_status != LBX_OK) {
    const int st = b->init_status;
    const std::string msg = b->init_error;
    lbx_batcher_destroy(b);
    return lbx::set_last_error((lbx_status)st, msg);
  }
  *out = b;
  return LBX_OK;
}

lbx_status lbx_batcher_destroy(lbx_batcher* b) {
  if (!b) return LBX_E_CONFIG;
  {
    std::lock_guard<std::mutex> g(b->mu);
    b->stopping = true;
  }
  b->cv_work.notify_all();
  for (auto& t : b->workers) t.join();
  delete b;
  return LBX_OK;
}

lbx_status lbx_batcher_submit(lbx_batcher* b, uint64_t request_id, int shape, const uint8_t* blob, size_t nbytes,
                              uint8_t* rgb_out) {
  if (!b || !blob || !rgb_out || shape < 0 || shape >= (int)b->shapes.size())
    return lbx::set_last_error(LBX_E_CONFIG, "lbx_batcher_submit: bad argument");
  Request r{request_id, std::vector<uint8_t>(blob, blob + nbytes), rgb_out, now_us()};
  {
    std::lock_guard<std::mutex> g(b->mu);
    if (b->stopping) return LBX_E_RUNTIME;
    b->queues[shape].push_back(std::move(r));
    ++b->pending;
  }
  b->cv_work.notify_one();
  return LBX_OK;
}

int lbx_batcher_poll(lbx_batcher* b, lbx_completion* out, int cap, uint32_t wait_us) {
  if (!b || !out || cap <= 0) return 0;
  std::unique_lock<std::mutex> lk(b->mu);
  if (b->done.empty() && wait_us)
    b->cv_done.wait_for(lk, std::chrono::microseconds(wait_us), [&] { return !b->done.empty(); });
  const int n = (int)(b->done.size() < (size_t)cap ? b->done.size() : (size_t)cap);
  std::memcpy(out, b->done.data(), n * sizeof(lbx_completion));
  b->done.erase(b->done.begin(), b->done.begin() + n);
  b->pending -= (uint64_t)n;
  return n;
}

uint64_t lbx_batcher_pending(lbx_batcher* b) {
  if (!b) return 0;
  std::lock_guard<std::mutex> g(b->mu);
  return b->pending;
}

}  // extern "C"
