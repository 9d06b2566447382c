/*
 * lbx/batcher.h -- multi-GPU decode-on-miss request batcher (north_star item 3).
 *
 * Replaces the simulator's GPU placement and FIFO service (proj/src/sim.cpp:238-243, 409-442) with
 * real per-GPU queues.  One worker thread per device owns one lbx_decoder per latent shape class
 * ("groups cache-miss decodes by latent shape").  An idle worker pulls the next batch, so a request
 * goes to the least-loaded GPU, as least_loaded_gpu() picks the GPU with the smallest depth; a worker
 * that already has a batch in flight pre-stages a second one (lbx_reconstruct_submit) only while no
 * worker is idle.  A batch closes when its queue holds max_batch requests, its oldest request has
 * waited max_wait_us, or (policy 1) more requests would not change the size lbx_batch_pick chooses;
 * any ready queue is served oldest-head first.  Whole requests are never split across GPUs and there
 * is no collective: one process drives all GPUs of a box, and requests are independent.
 *
 * Each completion carries the timestamps that Engine::on_job_done feeds to observe_latency:
 * queue + batch wait = t_start - t_submit, and service = t_end - t_start (sim.cpp:438-440); with a
 * pre-staged batch the service includes the wait behind the batch ahead of it on the same GPU.
 */
#ifndef LBX_BATCHER_H
#define LBX_BATCHER_H

#include <stddef.h>
#include <stdint.h>

#include "lbx/reconstruct.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int family;                  /* lbx_family */
  uint32_t latent_h, latent_w; /* latent shape of this class */
} lbx_shape;

typedef struct {
  const int* devices;          /* CUDA ordinals, one worker per entry */
  int n_devices;
  const lbx_shape* shapes;     /* shape classes; a request names its class by index */
  int n_shapes;
  uint32_t max_batch;          /* per-launch batch cap (also the decoders' arena size) */
  uint32_t max_wait_us;        /* close a partial batch once its oldest request waited this long */
  uint64_t weight_seed;        /* decoder weights (deterministic generator) */
  uint32_t policy;             /* 0 (default): close batches of up to max_batch (greedy); 1: each worker
                                  measures its device's service curve at creation and closes the batch
                                  size lbx_batch_pick chooses (no batching when it does not pay) */
} lbx_batcher_desc;

typedef struct {
  uint64_t request_id;
  int status;                  /* lbx_status of the batch that carried the request */
  int device;                  /* CUDA ordinal that decoded it */
  uint32_t batch_size;         /* requests in that batch */
  uint64_t t_submit_us, t_start_us, t_end_us; /* steady-clock microseconds */
  int worker;                  /* index into desc.devices of the worker that decoded it */
} lbx_completion;

typedef struct lbx_batcher lbx_batcher;

LBX_API lbx_status lbx_batcher_create(const lbx_batcher_desc* desc, lbx_batcher** out);
/* Stops the workers after draining queued requests, then frees everything. */
LBX_API lbx_status lbx_batcher_destroy(lbx_batcher* b);

/* Enqueue one request.  The blob is copied.  rgb_out (8h x 8w x 3 bytes, host memory; pinned is
 * fastest) must stay valid until the request's completion is returned by lbx_batcher_poll.  A
 * request_id still in flight (submitted, completion not yet polled) is rejected with LBX_E_CONFIG. */
LBX_API lbx_status lbx_batcher_submit(lbx_batcher* b, uint64_t request_id, int shape, const uint8_t* blob, size_t nbytes,
                              uint8_t* rgb_out);

/* Enqueue one request whose blob is resident in GPU memory (an HBM latent tier): nbytes at device
 * pointer blob_dev on CUDA device blob_device, valid until the completion is polled.  Whichever
 * worker takes it copies the blob D2D (same GPU) or fetches it over NVLink with a peer copy (another
 * GPU): a spilled decode's latent shipping, LatencyModel::intra_cluster_ms = 5 in the reference
 * (proj/include/latentbox/sim.hpp:20, proj/src/router.cpp:99-114).  Headers are checked by the
 * device unpack (the completion's status is LBX_E_FORMAT for a malformed blob). */
LBX_API lbx_status lbx_batcher_submit_device(lbx_batcher* b, uint64_t request_id, int shape, const uint8_t* blob_dev,
                                     size_t nbytes, int blob_device, uint8_t* rgb_out);

typedef struct {
  uint64_t spills;         /* device-resident blobs decoded on a GPU other than their own */
  uint64_t spill_bytes;    /* their bytes */
  uint64_t peer_copies;    /* peer copies the decoders issued (== spills) */
  double peer_ms;          /* device time of the batches' peer-copy phases, summed */
  uint64_t graph_captures; /* CUDA graphs captured by the workers' decoders */
} lbx_batcher_stats;
LBX_API lbx_status lbx_batcher_get_stats(lbx_batcher* b, lbx_batcher_stats* out);

/* Up to cap completions.  Waits up to wait_us for the first one.  Returns the count (>= 0). */
LBX_API int lbx_batcher_poll(lbx_batcher* b, lbx_completion* out, int cap, uint32_t wait_us);

/* Requests submitted but not yet returned by poll. */
LBX_API uint64_t lbx_batcher_pending(lbx_batcher* b);

/* Batch size to close from `queued` waiting requests, 1 <= result <= min(queued, max_batch) (0 if
 * queued == 0), given a service curve cost_ms[b-1] = GPU time of a batch of b, b = 1..n_cost
 * (extended linearly past n_cost): the size that minimises the mean completion time of the queued
 * requests served FIFO in batches of that size.  cost_ms == NULL: min(queued, max_batch) (greedy).
 * On B200 the decode's time per image is nearly flat in the batch size, so this returns 1 until a
 * deep backlog (batching would make early requests wait for late ones); on engines with a fixed
 * per-launch cost it batches. */
LBX_API uint32_t lbx_batch_pick(const double* cost_ms, uint32_t n_cost, uint32_t queued, uint32_t max_batch);

/* Steady-clock microseconds, the time base of lbx_completion. */
LBX_API uint64_t lbx_now_us(void);

#ifdef __cplusplus
}
#endif
#endif /* LBX_BATCHER_H */
