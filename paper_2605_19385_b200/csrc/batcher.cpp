// Multi-GPU decode-on-miss request batcher (include/lbx/batcher.h).
//
// One worker thread per device owns one lbx_decoder per shape class (created on that thread's
// device).  Requests wait in per-shape FIFO queues.  A worker closes a batch on a ready queue: one
// holding max_batch requests, one whose head has waited max_wait_us, (policy 1) one where more
// requests would not change the size lbx_batch_pick chooses, or any queue when draining at shutdown;
// among ready queues the oldest head goes first.  Batches run through the decoder's asynchronous
// pipeline (lbx_reconstruct_submit / _wait): a worker keeps up to two batches in flight, so batch
// k+1's host staging, H2D and unpack and batch k-1's D2H overlap batch k's decode -- the paper's
// fetch / decompress / encode pools around GPU inference.  A worker with work in
// flight takes another batch only when no worker is idle, so placement stays least-loaded-first
// (proj/src/sim.cpp:238-243); the FIFO order per shape mirrors the simulator's FIFO GPU
// (sim.cpp:413).  With policy 1 the batch size comes from lbx_batch_pick over the worker's own
// measured service curve.
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
#include <unordered_set>
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
  std::vector<uint8_t> blob;  // host blob (copied at submit) ...
  const uint8_t* blob_dev;    // ... or a blob resident in GPU memory (HBM latent tier)
  size_t dev_bytes;
  int blob_device;            // -1: host blob; else the CUDA device holding blob_dev
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
  int idle = 0;                            // workers with nothing in flight, waiting for work
  uint64_t spills = 0, spill_bytes = 0;    // device-resident blobs decoded on another GPU
  std::vector<std::vector<lbx_decoder*>> decs;  // [worker][shape], for the counters
  std::unordered_set<uint64_t> live_ids;   // submitted, not yet returned by poll
  std::vector<std::vector<std::vector<double>>> curves;  // [worker][shape] (policy 1)

  void worker(int dev_index);
  // Index of a ready shape queue (see the header comment), or -1; *next_deadline = the earliest
  // time a non-ready queue becomes ready by age.  Called with mu held.
  int ready_shape(int di, uint64_t now, uint64_t* next_deadline) const;
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

int lbx_batcher::ready_shape(int di, uint64_t now, uint64_t* next_deadline) const {
  int best = -1;
  uint64_t best_t = UINT64_MAX;
  *next_deadline = UINT64_MAX;
  for (size_t s = 0; s < queues.size(); ++s) {
    const auto& q = queues[s];
    if (q.empty()) continue;
    const uint64_t head = q.front().t_submit;
    bool ready = stopping || q.size() >= desc.max_batch || now - head >= desc.max_wait_us;
    if (!ready && desc.policy == 1) {
      // the size the rule closes now equals the size it would close from a full queue: waiting
      // for more requests cannot change the batch, only delay it
      const auto& cv = curves[di][s];
      const uint32_t now_pick = lbx_batch_pick_rule(cv.empty() ? nullptr : cv.data(), (uint32_t)cv.size(),
                                                    (uint32_t)q.size(), desc.max_batch);
      const uint32_t full_pick = lbx_batch_pick_rule(cv.empty() ? nullptr : cv.data(), (uint32_t)cv.size(),
                                                     desc.max_batch, desc.max_batch);
      ready = now_pick == full_pick;
    }
    if (ready && head < best_t) {
      best_t = head;
      best = (int)s;
    }
    if (!ready) *next_deadline = std::min(*next_deadline, head + desc.max_wait_us);
  }
  return best;
}

void lbx_batcher::worker(int di) {
  const int device = devices[di];
  std::vector<lbx_decoder*> decs(shapes.size(), nullptr);
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
    {
      std::lock_guard<std::mutex> g(mu);
      this->decs[di][s] = decs[s];
    }
    if (st == LBX_OK) st = lbx_decoder_prepare(decs[s], desc.max_batch);  // no capture on the request path
    if (st == LBX_OK && desc.policy == 1) {
      const int ch = shapes[s].family == LBX_FAMILY_SD15 ? 4 : 16;
      auto c = measure_curve(decs[s], ch, shapes[s].latent_h, shapes[s].latent_w, desc.max_batch);
      if (c.empty()) st = LBX_E_CUDA;
      std::lock_guard<std::mutex> g(mu);
      curves[di][s] = std::move(c);
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

  struct InFlight {
    uint64_t ticket;
    int shape;
    std::vector<Request> reqs;
    uint64_t t_start;
  };
  std::deque<InFlight> inflight;  // <= 2 (the decoder pipeline's depth)
  std::vector<const uint8_t*> blobs;
  std::vector<size_t> sizes;
  std::vector<int> blob_devs;
  std::vector<uint8_t*> outs;
  auto complete = [&](std::vector<Request>& reqs, lbx_status rs, uint64_t t_start) {
    const uint64_t t_end = now_us();
    {
      std::lock_guard<std::mutex> g(mu);
      for (auto& r : reqs)
        done.push_back(lbx_completion{r.id, (int)rs, device, (uint32_t)reqs.size(), r.t_submit, t_start, t_end, di});
    }
    cv_done.notify_all();
  };
  for (;;) {
    int shape = -1;
    std::vector<Request> batch;
    {
      std::unique_lock<std::mutex> lk(mu);
      if (inflight.empty()) {
        ++idle;
        for (;;) {
          uint64_t deadline = UINT64_MAX;
          const uint64_t now = now_us();
          shape = ready_shape(di, now, &deadline);
          if (shape >= 0 || (stopping && deadline == UINT64_MAX)) break;
          if (st != LBX_OK && deadline != UINT64_MAX) {  // failed worker: drain with errors
            for (size_t s = 0; s < queues.size() && shape < 0; ++s)
              if (!queues[s].empty()) shape = (int)s;
            break;
          }
          if (deadline == UINT64_MAX) cv_work.wait(lk);
          else cv_work.wait_for(lk, std::chrono::microseconds(deadline - now));
        }
        --idle;
      } else if (inflight.size() < 2 && idle == 0) {
        uint64_t deadline;
        shape = ready_shape(di, now_us(), &deadline);
      }
      if (shape >= 0) {
        auto& q = queues[shape];
        const auto& cv = curves[di][shape];
        const size_t take = lbx_batch_pick_rule(cv.empty() ? nullptr : cv.data(), (uint32_t)cv.size(),
                                                (uint32_t)q.size(), desc.max_batch);
        for (size_t i = 0; i < take; ++i) {
          batch.push_back(std::move(q.front()));
          q.pop_front();
        }
      }
    }
    if (shape >= 0) {
      cv_work.notify_all();  // another idle worker may take the remainder
      const uint64_t t_start = now_us();
      lbx_status rs = st;
      uint64_t ticket = 0;
      if (rs == LBX_OK) {
        blobs.clear();
        sizes.clear();
        blob_devs.clear();
        outs.clear();
        bool any_dev = false;
        uint64_t sp = 0, sp_bytes = 0;
        for (auto& r : batch) {
          const bool on_dev = r.blob_device >= 0;
          blobs.push_back(on_dev ? r.blob_dev : r.blob.data());
          sizes.push_back(on_dev ? r.dev_bytes : r.blob.size());
          blob_devs.push_back(r.blob_device);
          outs.push_back(r.rgb);
          any_dev |= on_dev;
          if (on_dev && r.blob_device != device) {
            ++sp;
            sp_bytes += r.dev_bytes;
          }
        }
        if (sp) {
          std::lock_guard<std::mutex> g(mu);
          spills += sp;
          spill_bytes += sp_bytes;
        }
        rs = any_dev ? lbx_reconstruct_submit_dev(decs[shape], blobs.data(), blob_devs.data(), sizes.data(),
                                                  (uint32_t)batch.size(), outs.data(), &ticket)
                     : lbx_reconstruct_submit(decs[shape], blobs.data(), sizes.data(), (uint32_t)batch.size(),
                                              outs.data(), &ticket);
      }
      if (rs == LBX_OK) inflight.push_back(InFlight{ticket, shape, std::move(batch), t_start});
      else complete(batch, rs, t_start);
      continue;
    }
    if (inflight.empty()) break;  // stopping and drained
    InFlight& f = inflight.front();
    const lbx_status rs = lbx_reconstruct_wait(decs[f.shape], f.ticket);
    complete(f.reqs, rs, f.t_start);
    inflight.pop_front();
  }
  {
    std::lock_guard<std::mutex> g(mu);
    for (auto*& d : this->decs[di]) d = nullptr;
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
  b->curves.assign(desc->n_devices, std::vector<std::vector<double>>(desc->n_shapes));
  b->decs.assign(desc->n_devices, std::vector<lbx_decoder*>(desc->n_shapes, nullptr));
  // NVLink peer access between the batcher's GPUs, for device-resident blobs decoded elsewhere
  // (cudaMemcpyPeerAsync also works without it, through the copy engines)
  for (int i = 0; i < desc->n_devices; ++i)
    for (int j = 0; j < desc->n_devices; ++j) {
      int can = 0;
      const int a = desc->devices[i], c = desc->devices[j];
      if (a != c && cudaDeviceCanAccessPeer(&can, a, c) == cudaSuccess && can) {
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(a);
        if (cudaDeviceEnablePeerAccess(c, 0) != cudaSuccess) cudaGetLastError();  // already enabled: fine
        cudaSetDevice(cur);
      }
    }
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
  Request r{request_id, std::vector<uint8_t>(blob, blob + nbytes), nullptr, 0, -1, rgb_out, now_us()};
  {
    std::lock_guard<std::mutex> g(b->mu);
    if (b->stopping) return lbx::set_last_error(LBX_E_RUNTIME, "lbx_batcher_submit: batcher is stopping");
    if (!b->live_ids.insert(request_id).second)
      return lbx::set_last_error(LBX_E_CONFIG, "lbx_batcher_submit: request_id " + std::to_string(request_id) +
                                                   " is already in flight");
    b->queues[shape].push_back(std::move(r));
    ++b->pending;
  }
  b->cv_work.notify_one();
  return LBX_OK;
}

lbx_status lbx_batcher_submit_device(lbx_batcher* b, uint64_t request_id, int shape, const uint8_t* blob_dev,
                                     size_t nbytes, int blob_device, uint8_t* rgb_out) {
  if (!b || !blob_dev || !rgb_out || shape < 0 || shape >= (int)b->shapes.size() || nbytes == 0 || blob_device < 0)
    return lbx::set_last_error(LBX_E_CONFIG, "lbx_batcher_submit_device: bad argument");
  Request r{request_id, {}, blob_dev, nbytes, blob_device, rgb_out, now_us()};
  {
    std::lock_guard<std::mutex> g(b->mu);
    if (b->stopping) return lbx::set_last_error(LBX_E_RUNTIME, "lbx_batcher_submit_device: batcher is stopping");
    if (!b->live_ids.insert(request_id).second)
      return lbx::set_last_error(LBX_E_CONFIG, "lbx_batcher_submit_device: request_id " + std::to_string(request_id) +
                                                   " is already in flight");
    b->queues[shape].push_back(std::move(r));
    ++b->pending;
  }
  b->cv_work.notify_one();
  return LBX_OK;
}

lbx_status lbx_batcher_get_stats(lbx_batcher* b, lbx_batcher_stats* out) {
  if (!b || !out) return lbx::set_last_error(LBX_E_CONFIG, "lbx_batcher_get_stats: null argument");
  std::lock_guard<std::mutex> g(b->mu);
  *out = lbx_batcher_stats{};
  out->spills = b->spills;
  out->spill_bytes = b->spill_bytes;
  for (auto& row : b->decs)
    for (auto* d : row) {
      lbx_decoder_counters c{};
      if (d && lbx_decoder_get_counters(d, &c) == LBX_OK) {
        out->peer_copies += c.peer_copies;
        out->peer_ms += c.peer_ms;
        out->graph_captures += c.graph_captures;
      }
    }
  return LBX_OK;
}

int lbx_batcher_poll(lbx_batcher* b, lbx_completion* out, int cap, uint32_t wait_us) {
  if (!b || !out || cap <= 0) return 0;
  std::unique_lock<std::mutex> lk(b->mu);
  if (b->done.empty() && wait_us)
    b->cv_done.wait_for(lk, std::chrono::microseconds(wait_us), [&] { return !b->done.empty(); });
  const int n = (int)(b->done.size() < (size_t)cap ? b->done.size() : (size_t)cap);
  std::memcpy(out, b->done.data(), n * sizeof(lbx_completion));
  for (int i = 0; i < n; ++i) b->live_ids.erase(out[i].request_id);
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
