// Decoder runtime + C ABI (include/lbx/reconstruct.h).
//
// One lbx_decoder per GPU owns: device weights in GEMM-ready layouts (fp16 K-major, conv taps
// (ky,kx,ci) innermost-ci, upsample convs pre-folded into 4 sub-pixel 2x2 kernels), an activation
// arena sized for max_batch (NHWC fp16), and one CUDA graph per batch size n, captured once on the
// decoder's own latent / RGB buffers (caller buffers are copied in and out, so new caller pointers
// never trigger a capture) -- the paper wraps its TensorRT engine in a CUDA graph the same way
// (PAPER.md:675).  Two asynchronous slots (lbx_reconstruct_submit / _wait) pipeline host blobs
// through three streams: H2D + unpack of batch k+1 and the D2H of batch k-1 overlap batch k's graph
// (the paper's fetch / decompress / encode pools around GPU inference).
//
// Layer plan per micro-batch, buffers X (residual stream), A (normalised
// activations / shortcut / upsample output), H (conv1 output, normalised in place; attention QKV):
//   prep(latents) -> A ; conv_in(A) -> X
//   Res: A = SiLU(GN1(X)); H = conv1(A); H = SiLU(GN2(H)); [A = shortcut(X)]; X = conv2(H) + X|A
//   Attn: A = GN(X); H = A Wqkv^T; per group of up to 8 images (one launch each): S = QK^T/sqrt(d);
//         P = exp(S - max); O = P V / sum (V read in place, MN-major) -> A; X = A Wo^T + bo + X
//   Up:   A = subpixel_conv(X) (nearest-2x + conv3x3 in 4 phases); swap(X, A)
//   tail: rgb = u8(conv_out(SiLU(GN(X))))
// Every conv epilogue accumulates the GroupNorm-32 statistics its consumer needs.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "codec.h"
#include "gemm_tc.cuh"
#include "gnfix.cuh"
#include "kernels.cuh"
#include "lbx/reconstruct.h"
#include "model.h"

namespace lbx {

static thread_local std::string g_err;
static lbx_status set_err(lbx_status s, const std::string& m) {
  g_err = m;
  return s;
}
// For other translation units of the library (batcher.cpp): record an error on this thread.
lbx_status set_last_error(lbx_status s, const std::string& m) { return set_err(s, m); }

#define LBX_CUDA_TRY(expr)                                                                      \
  do {                                                                                          \
    cudaError_t _e = (expr);                                                                    \
    if (_e != cudaSuccess)                                                                      \
      return set_err(LBX_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));           \
  } while (0)

struct ConvW {
  __half* w = nullptr;
  float* b = nullptr;
};
struct NormW {
  float* g = nullptr;
  float* b = nullptr;
};
struct ResW {
  int cin = 0, cout = 0;
  NormW n1, n2;
  ConvW c1, c2, sc;
};

class Decoder {
 public:
  lbx_decoder_desc desc{};
  FamilyInfo fi{};
  int h = 0, w = 0, cl = 0, max_batch = 0;
  cudaStream_t stream = nullptr;

  // weights
  void* wblock = nullptr;
  float *pq_w = nullptr, *pq_b = nullptr;
  ConvW conv_in;
  ResW res[14];
  NormW attn_gn;
  __half* wqkv = nullptr;
  float* bqkv = nullptr;
  __half* wo = nullptr;
  float* bo = nullptr;
  ConvW up[3];
  NormW norm_out;
  float *wout = nullptr, *bout = nullptr;

  // arena
  void* arena = nullptr;
  __half *X = nullptr, *A = nullptr, *Hb = nullptr, *S = nullptr, *Vt = nullptr, *lat = nullptr;
  float* rowscale = nullptr;
  float* rowmax = nullptr;    // fused-exp attention: sampled row maxima, 2 per row of a group
  float* rowpart = nullptr;   // fused-exp attention: row partial sums, 2 per (row, 256-key tile)
  int* attn_flag = nullptr;   // fused-exp attention: per-image overflow flags (fallback runs if set)
  unsigned long long* attn_fallbacks = nullptr;  // flagged images so far (never reset; counters API)
  unsigned long long* stats = nullptr;  // GroupNorm sites, gnfix.cuh layout
  float2* ss = nullptr;
  uint8_t* rgb = nullptr;
  int* err = nullptr;
  static constexpr int kMaxSites = 64;
  int s_imgs = 1;                 // images whose attention scores fit the S buffer at once

  // host-blob staging: pinned host copy -> one H2D -> device blobs + offset/size table
  struct Staging {
    uint8_t* host = nullptr;  // pinned
    uint8_t* dev = nullptr;
    size_t cap = 0;
    unsigned long long* offs_dev = nullptr;  // [max_batch] offsets, then [max_batch] u32 sizes
    unsigned int* sizes_dev = nullptr;
    unsigned long long* table_host = nullptr;  // pinned mirror of the table
    cudaEvent_t copied = nullptr;  // the last H2D out of `host` has completed: host may be rewritten
  };
  Staging sync_st;        // the synchronous calls (lbx_unpack / lbx_reconstruct*)
  int* err_host = nullptr;  // pinned
  // asynchronous pipeline (lbx_reconstruct_submit / lbx_reconstruct_wait): two slots, three streams
  struct Slot {
    Staging st;
    __half* lat = nullptr;
    uint8_t* rgb = nullptr;
    int* err = nullptr;
    int* err_host = nullptr;  // pinned
    cudaEvent_t unpacked = nullptr, computed = nullptr, drained = nullptr;
    cudaEvent_t peer0 = nullptr, peer1 = nullptr;  // timing: around this batch's peer copies
    bool busy = false, timed_peer = false;
    uint64_t ticket = 0;
  };
  Slot slots[2];
  cudaStream_t in_stream = nullptr, out_stream = nullptr;
  uint64_t next_ticket = 1;
  // cross-stream ordering of the work that touches decoder-owned device buffers: a call on a
  // different stream than the previous one first waits for the previous call's last enqueued work
  cudaEvent_t last_ev = nullptr;
  cudaStream_t last_stream = nullptr;
  bool last_valid = false;
  uint64_t captures = 0;  // CUDA graphs captured so far (one per batch size n)
  // HBM-resident blobs fetched from another GPU (latent spillover over NVLink): counters, and a
  // timing event pair per slot around its peer copies
  uint64_t peer_copies = 0, peer_bytes = 0;
  double peer_ms = 0.0;

  // return path (lbx_reconstruct_png), allocated on first use
  uint8_t* png_dev = nullptr;    // max_batch PNGs back to back
  uint8_t* png_work = nullptr;   // png_workspace(max_batch)
  uint32_t* png_sizes = nullptr;
  uint32_t* png_sizes_host = nullptr;  // pinned

  std::map<int, cudaGraphExec_t> graphs;
  std::map<int, int> launch_counts;
  struct ProfRec {
    std::string name;
    double flops, algo_flops, bytes;
    cudaEvent_t ev;
  };
  std::vector<ProfRec>* prof = nullptr;

  ~Decoder() { release(); }

  void release() {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(desc.device);
    if (stream) cudaStreamSynchronize(stream);
    if (in_stream) cudaStreamSynchronize(in_stream);
    if (out_stream) cudaStreamSynchronize(out_stream);
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    graphs.clear();
    if (wblock) cudaFree(wblock);
    if (arena) cudaFree(arena);
    free_staging(sync_st);
    for (Slot& sl : slots) {
      free_staging(sl.st);
      if (sl.lat) cudaFree(sl.lat);
      if (sl.err_host) cudaFreeHost(sl.err_host);
      for (cudaEvent_t e : {sl.unpacked, sl.computed, sl.drained, sl.peer0, sl.peer1})
        if (e) cudaEventDestroy(e);
      sl = Slot{};
    }
    if (err_host) cudaFreeHost(err_host);
    err_host = nullptr;
    if (last_ev) cudaEventDestroy(last_ev);
    last_ev = nullptr;
    if (in_stream) cudaStreamDestroy(in_stream);
    if (out_stream) cudaStreamDestroy(out_stream);
    in_stream = out_stream = nullptr;
    if (png_dev) cudaFree(png_dev);
    if (png_work) cudaFree(png_work);
    if (png_sizes) cudaFree(png_sizes);
    if (png_sizes_host) cudaFreeHost(png_sizes_host);
    png_dev = png_work = nullptr;
    png_sizes = png_sizes_host = nullptr;
    if (stream) cudaStreamDestroy(stream);
    wblock = arena = nullptr;
    stream = nullptr;
    cudaSetDevice(cur);
  }

  size_t lat_elems(int n) const { return (size_t)n * cl * h * w; }
  size_t rgb_bytes(int n) const { return (size_t)n * 64 * h * w * 3; }

  lbx_status init(const lbx_decoder_desc& d);
  lbx_status upload_weights(const std::vector<float>& p);
  lbx_status alloc_arena();
  lbx_status plan(int n, const __half* lat_in, uint8_t* rgb_out, cudaStream_t s, bool counting);
  lbx_status run(int n, const __half* lat_in, uint8_t* rgb_out, cudaStream_t s);
  lbx_status graph_for(int n, cudaStream_t s, cudaGraphExec_t* out);
  lbx_status validate_blobs(const uint8_t* const* blobs, const size_t* nbytes, uint32_t n, size_t* total);
  lbx_status stage_blobs(Staging& st, const uint8_t* const* blobs, const size_t* nbytes, uint32_t n,
                         cudaStream_t s, __half* lat_out, int* err_dev, const int* blob_devs = nullptr,
                         cudaEvent_t after_copies = nullptr);
  lbx_status grow_staging(Staging& st, size_t total);
  lbx_status alloc_slot(Slot& sl);
  static void free_staging(Staging& st) {
    if (st.host) cudaFreeHost(st.host);
    if (st.dev) cudaFree(st.dev);
    if (st.table_host) cudaFreeHost(st.table_host);
    if (st.copied) cudaEventDestroy(st.copied);
    st = Staging{};
  }
  // call-ordering helpers (see last_ev)
  void order(cudaStream_t s) {
    if (last_valid && last_stream != s) cudaStreamWaitEvent(s, last_ev, 0);
  }
  void mark(cudaStream_t s) {
    cudaEventRecord(last_ev, s);
    last_stream = s;
    last_valid = true;
  }
};

// --------------------------------------------------------------------------- weights
namespace {
struct Bump {
  uint8_t* base;
  size_t off = 0;
  template <class T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(base + off);
    off += count * sizeof(T);
    return p;
  }
};
}  // namespace

lbx_status Decoder::upload_weights(const std::vector<float>& p) {
  const auto specs = param_specs(fi.latent_channels, fi.post_quant);
  std::unordered_map<std::string, const float*> by_name;
  size_t pos = 0;
  for (const auto& s : specs) {
    by_name[s.name] = p.data() + pos;
    pos += s.count();
  }
  auto get = [&](const std::string& n) { return by_name.at(n); };

  // host staging buffer mirrors the device block
  std::vector<uint8_t> host(160u << 20, 0);
  Bump hb{host.data()};
  std::vector<std::pair<size_t, size_t>> dummy;
  struct Fix {
    size_t off;
    void** dst;
  };
  std::vector<Fix> fixes;
  auto f32 = [&](const float* src, size_t n, float** dst) {
    float* q = hb.take<float>(n);
    std::memcpy(q, src, n * 4);
    fixes.push_back({(size_t)((uint8_t*)q - host.data()), (void**)dst});
  };
  auto h16 = [&](size_t n, __half** dst) -> uint16_t* {
    uint16_t* q = hb.take<uint16_t>(n);
    fixes.push_back({(size_t)((uint8_t*)q - host.data()), (void**)dst});
    return q;
  };
  // conv3x3 [cout][cin][3][3] -> [cout][ky][kx][cin_pad]
  auto conv3 = [&](const std::string& n, int cin, int cout, int cin_pad, ConvW* cw) {
    const float* W = get(n + ".weight");
    uint16_t* q = h16((size_t)cout * 9 * cin_pad, &cw->w);
    for (int o = 0; o < cout; ++o)
      for (int t = 0; t < 9; ++t)
        for (int c = 0; c < cin; ++c) q[((size_t)o * 9 + t) * cin_pad + c] = f32_to_f16_bits(W[((size_t)o * cin + c) * 9 + t]);
    f32(get(n + ".bias"), cout, &cw->b);
  };
  auto norm = [&](const std::string& n, int c, NormW* nw) {
    f32(get(n + ".weight"), c, &nw->g);
    f32(get(n + ".bias"), c, &nw->b);
  };
  auto lin = [&](const float* W, int cout, int cin, uint16_t* q) {
    for (size_t i = 0; i < (size_t)cout * cin; ++i) q[i] = f32_to_f16_bits(W[i]);
  };

  if (fi.post_quant) {
    f32(get("post_quant_conv.weight"), (size_t)cl * cl, &pq_w);
    f32(get("post_quant_conv.bias"), cl, &pq_b);
  }
  conv3("decoder.conv_in", cl, 512, 64, &conv_in);
  const int chans[4] = {512, 512, 256, 128};
  std::vector<std::string> rnames = {"decoder.mid_block.resnets.0", "decoder.mid_block.resnets.1"};
  std::vector<std::pair<int, int>> rio = {{512, 512}, {512, 512}};
  int prev = 512;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 3; ++j) {
      rnames.push_back("decoder.up_blocks." + std::to_string(i) + ".resnets." + std::to_string(j));
      rio.push_back({j == 0 ? prev : chans[i], chans[i]});
      if (j == 2) prev = chans[i];
    }
  for (int r = 0; r < 14; ++r) {
    ResW& R = res[r];
    R.cin = rio[r].first;
    R.cout = rio[r].second;
    norm(rnames[r] + ".norm1", R.cin, &R.n1);
    conv3(rnames[r] + ".conv1", R.cin, R.cout, R.cin, &R.c1);
    norm(rnames[r] + ".norm2", R.cout, &R.n2);
    {
      // conv2 with the residual folded into K: [Cout][9*Cout + Cin] = [W2 taps | W_sc or identity],
      // bias b2 (+ b_sc); the tensor core adds x (or shortcut(x)) into the conv2 accumulator.
      const int K = 9 * R.cout + R.cin;
      const float* W = get(rnames[r] + ".conv2.weight");
      uint16_t* q = h16((size_t)R.cout * K, &R.c2.w);
      const float* Wsc = R.cin != R.cout ? get(rnames[r] + ".conv_shortcut.weight") : nullptr;
      for (int o = 0; o < R.cout; ++o) {
        for (int t = 0; t < 9; ++t)
          for (int c = 0; c < R.cout; ++c)
            q[(size_t)o * K + t * R.cout + c] = f32_to_f16_bits(W[((size_t)o * R.cout + c) * 9 + t]);
        for (int c = 0; c < R.cin; ++c)
          q[(size_t)o * K + 9 * R.cout + c] =
              Wsc ? f32_to_f16_bits(Wsc[(size_t)o * R.cin + c]) : (uint16_t)(c == o ? 0x3C00 : 0);
      }
      float* bq = hb.take<float>(R.cout);
      const float* b2 = get(rnames[r] + ".conv2.bias");
      const float* bsc = R.cin != R.cout ? get(rnames[r] + ".conv_shortcut.bias") : nullptr;
      for (int o = 0; o < R.cout; ++o) bq[o] = bsc ? b2[o] + bsc[o] : b2[o];
      fixes.push_back({(size_t)((uint8_t*)bq - host.data()), (void**)&R.c2.b});
    }
  }
  const std::string an = "decoder.mid_block.attentions.0";
  norm(an + ".group_norm", 512, &attn_gn);
  {
    uint16_t* q = h16((size_t)1536 * 512, &wqkv);
    lin(get(an + ".to_q.weight"), 512, 512, q);
    lin(get(an + ".to_k.weight"), 512, 512, q + 512 * 512);
    lin(get(an + ".to_v.weight"), 512, 512, q + 2 * 512 * 512);
    float* bq = hb.take<float>(1536);
    std::memcpy(bq, get(an + ".to_q.bias"), 512 * 4);
    std::memcpy(bq + 512, get(an + ".to_k.bias"), 512 * 4);
    std::memcpy(bq + 1024, get(an + ".to_v.bias"), 512 * 4);
    fixes.push_back({(size_t)((uint8_t*)bq - host.data()), (void**)&bqkv});
    uint16_t* qo = h16((size_t)512 * 512, &wo);
    lin(get(an + ".to_out.0.weight"), 512, 512, qo);
    f32(get(an + ".to_out.0.bias"), 512, &bo);
  }
  for (int i = 0; i < 3; ++i) {
    const std::string n = "decoder.up_blocks." + std::to_string(i) + ".upsamplers.0.conv";
    const int c = chans[i];
    const float* W = get(n + ".weight");  // [c][c][3][3]
    uint16_t* q = h16((size_t)4 * c * 4 * c, &up[i].w);
    // phase (a,b): 2x2 taps (r,s); row r gathers original ky in S_a[r], S_0 = {{0},{1,2}}, S_1 = {{0,1},{2}}
    static const int kset[2][2][2] = {{{0, -1}, {1, 2}}, {{0, 1}, {2, -1}}};
    for (int ph = 0; ph < 4; ++ph) {
      const int a = ph >> 1, bb = ph & 1;
      for (int o = 0; o < c; ++o)
        for (int t = 0; t < 4; ++t) {
          const int r = t >> 1, s = t & 1;
          for (int ci = 0; ci < c; ++ci) {
            float acc = 0.f;
            for (int u = 0; u < 2; ++u) {
              const int ky = kset[a][r][u];
              if (ky < 0) continue;
              for (int v = 0; v < 2; ++v) {
                const int kx = kset[bb][s][v];
                if (kx < 0) continue;
                acc += W[(((size_t)o * c + ci) * 3 + ky) * 3 + kx];
              }
            }
            q[(((size_t)ph * c + o) * 4 + t) * c + ci] = f32_to_f16_bits(acc);
          }
        }
    }
    f32(get(n + ".bias"), c, &up[i].b);
  }
  norm("decoder.conv_norm_out", 128, &norm_out);
  {
    const float* W = get("decoder.conv_out.weight");  // [3][128][3][3] -> [3][ky][kx][128]
    float* q = hb.take<float>(3 * 9 * 128);
    for (int o = 0; o < 3; ++o)
      for (int t = 0; t < 9; ++t)
        for (int c = 0; c < 128; ++c) q[(o * 9 + t) * 128 + c] = W[(o * 128 + c) * 9 + t];
    fixes.push_back({(size_t)((uint8_t*)q - host.data()), (void**)&wout});
    f32(get("decoder.conv_out.bias"), 3, &bout);
  }
  const size_t bytes = (hb.off + 255) & ~size_t(255);
  if (bytes > host.size()) return set_err(LBX_E_RUNTIME, "weight staging overflow");
  LBX_CUDA_TRY(cudaMalloc(&wblock, bytes));
  LBX_CUDA_TRY(cudaMemcpy(wblock, host.data(), bytes, cudaMemcpyHostToDevice));
  for (const auto& f : fixes) *f.dst = (uint8_t*)wblock + f.off;
  return LBX_OK;
}

// Images per conv launch.  LBX_CONV_CHUNK = k > 0 fixes k images (0: one launch per conv); by
// default (-1) each launch gets about LBX_CONV_CHUNK_ELEMS output elements (2^28: 8 images of a
// c512 @256^2 conv, 2 of a c128 @1024^2 conv, the whole batch of the small 128^2 layers).  A fixed 8
// measured 285.7 against 292.1 ms per batch-32 step with one launch per conv, bit-identical; the
// 2^28-element rule 278.0 against 279.8 for the fixed 8 (2^27 and 2^29 in between).
static int conv_chunk_fixed() {
  static const int v = [] {
    const char* e = std::getenv("LBX_CONV_CHUNK");
    return e ? std::atoi(e) : -1;
  }();
  return v;
}
static int conv_chunk_images(size_t out_elems_per_image) {
  const int fixed = conv_chunk_fixed();
  if (fixed >= 0) return fixed;
  static const double target = [] {
    const char* e = std::getenv("LBX_CONV_CHUNK_ELEMS");
    return e ? std::atof(e) : 268435456.0;
  }();
  return std::max(1, (int)(target / (double)std::max<size_t>(1, out_elems_per_image)));
}

// --------------------------------------------------------------------------- arena
lbx_status Decoder::alloc_arena() {
  const size_t hw = (size_t)h * w;
  const size_t nb = (size_t)max_batch;
  const size_t x_el = nb * hw * 64 * 256;  // max residual-stream tensor: 8h x 8w x 256
  const size_t h_el = nb * hw * 64 * 128;  // max conv1 output: 8h x 8w x 128 (>= QKV hw x 1536)
  // attention scores of up to 8 images at once (LBX_ATTN_GROUP overrides, diagnostics)
  int group = 8;
  if (const char* e = std::getenv("LBX_ATTN_GROUP")) group = std::max(1, std::atoi(e));
  s_imgs = std::max(1, std::min(max_batch, group));
  const size_t s_el = hw * hw * (size_t)s_imgs;
  const size_t vt_el = 512 * hw;
  size_t off = 0;
  auto slot = [&](size_t bytes) {
    size_t o = (off + 1023) & ~size_t(1023);
    off = o + bytes;
    return o;
  };
  const size_t oX = slot(x_el * 2), oA = slot(x_el * 2), oH = slot(h_el * 2), oS = slot(s_el * 2),
               oVt = slot(vt_el * 2), oR = slot(hw * 4 * (size_t)s_imgs), oRm = slot(hw * 8 * (size_t)s_imgs),
               oRp = slot(hw * (size_t)s_imgs * (hw / 256 + 1) * 8), oFl = slot(4 * (size_t)(nb + 1)), oCnt = slot(8), oSt = slot((size_t)kMaxSites * nb * 32 * kGnStatWords * 8),
               oSs = slot(nb * 512 * 8), oLat = slot(nb * cl * hw * 2), oRgb = slot(nb * hw * 64 * 3),
               oErr = slot(64);
  LBX_CUDA_TRY(cudaMalloc(&arena, off));
  uint8_t* b = (uint8_t*)arena;
  X = (__half*)(b + oX);
  A = (__half*)(b + oA);
  Hb = (__half*)(b + oH);
  S = (__half*)(b + oS);
  Vt = (__half*)(b + oVt);
  rowscale = (float*)(b + oR);
  rowmax = (float*)(b + oRm);
  rowpart = (float*)(b + oRp);
  attn_flag = (int*)(b + oFl);
  attn_fallbacks = (unsigned long long*)(b + oCnt);
  LBX_CUDA_TRY(cudaMemset(attn_fallbacks, 0, 8));
  stats = (unsigned long long*)(b + oSt);
  ss = (float2*)(b + oSs);
  lat = (__half*)(b + oLat);
  rgb = b + oRgb;
  err = (int*)(b + oErr);
  LBX_CUDA_TRY(cudaMemset(err, 0, 64));
  LBX_CUDA_TRY(cudaMallocHost(&err_host, 64));
  LBX_CUDA_TRY(cudaMallocHost(&sync_st.table_host, nb * 16));
  LBX_CUDA_TRY(cudaEventCreateWithFlags(&sync_st.copied, cudaEventDisableTiming));
  LBX_CUDA_TRY(cudaEventCreateWithFlags(&last_ev, cudaEventDisableTiming));
  return LBX_OK;
}

// An asynchronous slot: its own staging, latents, RGB and status word (allocated on first use).
lbx_status Decoder::alloc_slot(Slot& sl) {
  if (sl.lat) return LBX_OK;
  const size_t lat_b = (lat_elems(max_batch) * 2 + 1023) & ~size_t(1023);
  void* p = nullptr;
  LBX_CUDA_TRY(cudaMalloc(&p, lat_b + rgb_bytes(max_batch) + 64));
  sl.lat = reinterpret_cast<__half*>(p);
  sl.rgb = reinterpret_cast<uint8_t*>(p) + lat_b;
  sl.err = reinterpret_cast<int*>(sl.rgb + rgb_bytes(max_batch));
  LBX_CUDA_TRY(cudaMemset(sl.err, 0, 64));
  LBX_CUDA_TRY(cudaMallocHost(&sl.err_host, 64));
  LBX_CUDA_TRY(cudaMallocHost(&sl.st.table_host, (size_t)max_batch * 16));
  for (cudaEvent_t* e : {&sl.st.copied, &sl.unpacked, &sl.computed, &sl.drained})
    LBX_CUDA_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  LBX_CUDA_TRY(cudaEventCreate(&sl.peer0));
  LBX_CUDA_TRY(cudaEventCreate(&sl.peer1));
  if (!in_stream) {
    LBX_CUDA_TRY(cudaStreamCreateWithFlags(&in_stream, cudaStreamNonBlocking));
    LBX_CUDA_TRY(cudaStreamCreateWithFlags(&out_stream, cudaStreamNonBlocking));
  }
  return LBX_OK;
}

lbx_status Decoder::init(const lbx_decoder_desc& d) {
  desc = d;
  if (!family_info(d.family, &fi)) return set_err(LBX_E_CONFIG, "desc.family: unknown family");
  cl = fi.latent_channels;
  h = (int)d.latent_h;
  w = (int)d.latent_w;
  max_batch = (int)d.max_batch;
  if (max_batch <= 0 || max_batch > 4096) return set_err(LBX_E_CONFIG, "desc.max_batch: must be in [1, 4096]");
  if (h < 8 || w < 8 || h > 512 || w > 512) return set_err(LBX_E_CONFIG, "desc.latent_h/latent_w: out of range");
  // tile geometry: every resolution's width must be 64 or a multiple of 128, heights even
  if (!((w == 64) || (w % 128 == 0)) || h % 2) return set_err(LBX_E_CONFIG, "desc.latent_w: must be 64 or a multiple of 128 (latent_h even)");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return set_err(LBX_E_CUDA, "no CUDA device");
  if (d.device < 0 || d.device >= ndev) return set_err(LBX_E_CONFIG, "desc.device: no such device");
  LBX_CUDA_TRY(cudaSetDevice(d.device));
  cudaDeviceProp prop;
  LBX_CUDA_TRY(cudaGetDeviceProperties(&prop, d.device));
  if (prop.major != 10) return set_err(LBX_E_CUDA, "device is not sm_100 (B200); this build has no other code path");
  if (!gemm_tc_prepare()) return set_err(LBX_E_CUDA, "tcgen05 GEMM setup failed (cuTensorMapEncodeTiled / smem attribute)");
  LBX_CUDA_TRY(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  std::vector<float> params;
  const size_t expect = param_specs(fi.latent_channels, fi.post_quant).size();
  (void)expect;
  size_t count = 0;
  for (const auto& s : param_specs(fi.latent_channels, fi.post_quant)) count += s.count();
  if (d.weights) {
    if (d.weights_count != count) return set_err(LBX_E_CONFIG, "desc.weights_count: != lbx_param_count(family)");
    params.assign(d.weights, d.weights + count);
  } else {
    params = generate_params(d.family, d.weight_seed);
  }
  lbx_status st = upload_weights(params);
  if (st != LBX_OK) return st;
  return alloc_arena();
}

// --------------------------------------------------------------------------- plan
lbx_status Decoder::plan(int n, const __half* lat_in, uint8_t* rgb_out, cudaStream_t s, bool counting) {
  int launches = 0;
  int site = 0;
  const size_t site_stride = (size_t)max_batch * 32 * kGnStatWords;
  auto site_ptr = [&](int i) { return stats + (size_t)i * site_stride; };
  auto chk = [&](cudaError_t e, const std::string& what) -> lbx_status {
    if (e != cudaSuccess) return set_err(LBX_E_CUDA, what + ": " + cudaGetErrorString(e));
    return LBX_OK;
  };
#define LBX_STEP(expr, what)                       \
  do {                                             \
    lbx_status _s = chk((expr), what);             \
    if (_s != LBX_OK) return _s;                   \
  } while (0)
  auto mark = [&](const std::string& name, double flops, double algo, double bytes) {
    if (!prof) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    prof->push_back({name, flops, algo, bytes, e});
  };
#define LBX_LAUNCH(stmt, what, bytes)              \
  do {                                             \
    stmt;                                          \
    ++launches;                                    \
    LBX_STEP(cudaPeekAtLastError(), what);         \
    mark(what, 0.0, 0.0, (double)(bytes));         \
  } while (0)

  __half* X_ = X;
  __half* A_ = A;
  const bool h2 = desc.precise_activations == 0;  // packed-half SiLU unless the caller asked for fp32
  if (prof) mark("start", 0, 0, 0);
  LBX_STEP(cudaMemsetAsync(stats, 0, (size_t)kMaxSites * site_stride * 8, s), "memset stats");

  // one kernel launch, and (profiling) its entry: executed / algorithmic FLOPs and bytes of this launch
  auto launch1 = [&](const GemmArgs& ga, const char* what) -> lbx_status {
    ++launches;
    const lbx_status e = chk(gemm_tc_launch(ga, s), what);
    if (e == LBX_OK && prof) {
      const double fl_main = 2.0 * ga.M * (double)ga.N * ga.K * (ga.mode == GEMM_SUBPIX ? 4 : 1);  // 4 phases
      const double fl = fl_main + 2.0 * ga.M * (double)ga.N * ga.K2;  // executed, incl. the folded K
      // algorithmic (standard) FLOPs: the sub-pixel form stands for nearest-2x + a full 3x3 conv
      double algo = ga.mode == GEMM_SUBPIX ? 2.0 * 4.0 * ga.M * (double)ga.N * 9.0 * ga.C : fl_main;
      // folded extra K: a 1x1 shortcut (K2 != N) is real algorithmic work; an identity residual is not
      if (ga.K2 && ga.K2 != ga.N) algo += 2.0 * ga.M * (double)ga.N * ga.K2;
      if (ga.rowred == 1) algo = 0;  // the sampled row maxima are extra work, not the algorithm's
      double fl_ex = fl;
      if (ga.run_if) fl_ex = algo = 0;  // the fallback runs only when flagged (normally an early exit)
      char nm[160];
      if (ga.mode == GEMM_PLAIN)
        snprintf(nm, sizeof nm, "%s gemm M%d N%d K%d", what, ga.M, ga.N, ga.K);
      else  // named per layer (not per chunk): the launches of one conv group together
        snprintf(nm, sizeof nm, "%s %s c%d->%d @%dx%d", what, ga.mode == GEMM_CONV3X3 ? "conv3x3" : "subpix2x2",
                 ga.C, ga.N, ga.mode == GEMM_SUBPIX ? 2 * ga.H : ga.H, ga.mode == GEMM_SUBPIX ? 2 * ga.W : ga.W);
      const double by = 2.0 * ((double)ga.M * ga.K / (ga.mode == GEMM_PLAIN ? 1 : (ga.mode == GEMM_CONV3X3 ? 9 : 4)) +
                               (double)ga.N * ga.K * (ga.mode == GEMM_SUBPIX ? 4 : 1) +
                               (double)ga.M * ga.N * (ga.mode == GEMM_SUBPIX ? 4 : 1) * (ga.resid ? 2 : 1));
      mark(nm, fl_ex, algo, ga.run_if ? 0.0 : by);
    }
    return e;
  };
  auto gemm = [&](GemmArgs ga, const char* what) -> lbx_status {
    if (ga.mode == GEMM_PLAIN) return launch1(ga, what);
    const int chunk = conv_chunk_images((size_t)ga.H * ga.W * ga.N * (ga.mode == GEMM_SUBPIX ? 4 : 1));
    if (chunk <= 0 || ga.B_img <= chunk) return launch1(ga, what);
    // a long conv launch as several launches of `chunk` whole images: the persistent clusters
    // drift apart over hundreds of tiles, and vertically adjacent tiles -- which share halo rows --
    // then run too far apart for the rows to survive in L2.  Each launch starts the
    // clusters in step again.  Image tiles map to clusters exactly as in one launch, so the
    // GroupNorm partial sums (and the decode) are bit-identical.
    const size_t hw = (size_t)ga.H * ga.W, ohw = ga.mode == GEMM_SUBPIX ? 4 * hw : hw;
    lbx_status e = LBX_OK;
    for (int i0 = 0; i0 < ga.B_img && e == LBX_OK; i0 += chunk) {
      GemmArgs c = ga;
      const int cnt = std::min(chunk, ga.B_img - i0);
      c.B_img = cnt;
      c.M = (int)(cnt * hw);
      c.A = ga.A + i0 * hw * ga.C;
      if (ga.A2) c.A2 = ga.A2 + i0 * hw * ga.lda2;
      c.out = ga.out + i0 * ohw * ga.ldo;
      if (ga.resid) c.resid = ga.resid + i0 * hw * ga.ldr;
      if (ga.gn_stats) c.gn_stats = ga.gn_stats + (size_t)i0 * 32 * kGnStatWords;
      if (ga.gn_ss) c.gn_ss = ga.gn_ss + (size_t)i0 * ga.C;
      e = launch1(c, what);
    }
    return e;
  };
  auto gn = [&](int st_site, const NormW& nw, const __half* x, __half* y, int C, int hw, bool silu) -> lbx_status {
    const GnSrc gs{site_ptr(st_site), nw.g, nw.b, 1.0 / ((double)hw * (C / 32)), 1e-6f};
    LBX_LAUNCH(launch_gn_apply(x, y, gs, (long long)n * hw, hw, C, silu, h2, s),
               std::string(silu ? "gn_apply_silu c" : "gn_apply c") + std::to_string(C) + " hw" + std::to_string(hw),
               4.0 * n * (double)hw * C);
    return LBX_OK;
  };
  auto conv3 = [&](const __half* in, int H, int W, int C, const ConvW& cw, int N, __half* out, const __half* resid,
                   int out_site, const char* what) -> lbx_status {
    GemmArgs g;
    g.mode = GEMM_CONV3X3;
    g.M = n * H * W; g.N = N; g.K = 9 * C;
    g.A = in; g.B_img = n; g.H = H; g.W = W; g.C = C;
    g.Bw = cw.w; g.ldb = 9 * C;
    g.out = out; g.ldo = N; g.bias = cw.b;
    g.resid = resid; g.ldr = N;
    g.gn_stats = out_site >= 0 ? site_ptr(out_site) : nullptr;
    g.gn_cpg = N / 32; g.rows_per_img = H * W;
    return gemm(g, what);
  };
  lbx_status st;

  // prep + conv_in
  LBX_LAUNCH(launch_latent_prep(lat_in, A_, n, cl, h, w, fi.scaling, fi.shift, pq_w, pq_b, s), "latent_prep",
             2.0 * n * h * w * (cl + 64));
  int x_site = site++;
  if ((st = conv3(A_, h, w, 64, conv_in, 512, X_, nullptr, x_site, "conv_in")) != LBX_OK) return st;

  // GroupNorm + SiLU of a conv input: fused into the conv's A operand where the kernel supports it
  // (halo staging, 256-wide N tiles, >= 256 input channels), else a separate apply pass.
  auto gn_for_conv = [&](int st_site, const NormW& nw, const __half* x, __half* scratch, int C, int H, int W,
                         int N, GemmArgs* g) -> lbx_status {
    GemmArgs probe;
    probe.mode = GEMM_CONV3X3;
    probe.M = n * H * W; probe.N = N; probe.C = C; probe.W = W;
    if (gemm_tc_can_fuse_gn(probe)) {
      LBX_LAUNCH(launch_gn_finalize(site_ptr(st_site), nw.g, nw.b, ss, n, C, (double)H * W * (C / 32), 1e-6f, s),
                 "gn_finalize", n * C * 8.0);
      g->A = x;
      g->gn_ss = ss;
      return LBX_OK;
    }
    g->A = scratch;
    return gn(st_site, nw, x, scratch, C, H * W, true);
  };

  auto resnet = [&](const ResW& R, int H, int W) -> lbx_status {
    const int hw = H * W;
    lbx_status e;
    const int mid = site++;
    {  // conv1(SiLU(GN1(x)))
      GemmArgs g;
      g.mode = GEMM_CONV3X3;
      g.M = n * hw; g.N = R.cout; g.K = 9 * R.cin;
      g.B_img = n; g.H = H; g.W = W; g.C = R.cin;
      g.Bw = R.c1.w; g.ldb = 9 * R.cin;
      g.out = Hb; g.ldo = R.cout; g.bias = R.c1.b;
      g.gn_stats = site_ptr(mid); g.gn_cpg = R.cout / 32; g.rows_per_img = hw;
      if ((e = gn_for_conv(x_site, R.n1, X_, A_, R.cin, H, W, R.cout, &g)) != LBX_OK) return e;
      if ((e = gemm(g, g.gn_ss ? "resnet.conv1+gn" : "resnet.conv1")) != LBX_OK) return e;
    }
    // conv2(SiLU(GN2(h))) + (x or shortcut(x)): the residual is an extra K segment of the same
    // tcgen05 GEMM.  Same width: the output overwrites X in place (each tile reads only its own X
    // rows, via TMA, before its epilogue writes them).  Cin != Cout: row strides differ, so a tile's
    // output rows would land on other tiles' unread input rows -- write to A and swap.
    const int out_site = site++;
    {
      GemmArgs g;
      g.mode = GEMM_CONV3X3;
      g.M = n * hw; g.N = R.cout; g.K = 9 * R.cout;
      g.B_img = n; g.H = H; g.W = W; g.C = R.cout;
      // identity residual: preloaded into the TMEM accumulator by the epilogue warps before the
      // tile's MMAs (gemm_tc rpf; in place: a tile's residual rows are read before its outputs are
      // written).  Without the preload (debug bit 10) it is added in the epilogue at >= 256
      // channels and folded as extra K at 128.  A 1x1 shortcut is always folded.
      const bool epi_resid =
          R.cin == R.cout && !resid_fold_always() && !(resid_rbuf() && R.cout <= 128) &&
          (resid_preload() || R.cout >= 256 || resid_epilogue_all());
      if (epi_resid) {
        g.resid = X_; g.ldr = R.cout;
      } else {
        g.A2 = X_; g.lda2 = R.cin; g.K2 = R.cin;
      }
      g.Bw = R.c2.w; g.ldb = 9 * R.cout + R.cin;
      g.out = R.cin == R.cout ? X_ : A_; g.ldo = R.cout; g.bias = R.c2.b;
      g.gn_stats = site_ptr(out_site); g.gn_cpg = R.cout / 32; g.rows_per_img = hw;
      if ((e = gn_for_conv(mid, R.n2, Hb, Hb, R.cout, H, W, R.cout, &g)) != LBX_OK) return e;
      if ((e = gemm(g, g.gn_ss ? "resnet.conv2+gn+residual" : "resnet.conv2+residual")) != LBX_OK) return e;
      if (R.cin != R.cout) std::swap(X_, A_);
    }
    x_site = out_site;
    return LBX_OK;
  };

  // mid block
  if ((st = resnet(res[0], h, w)) != LBX_OK) return st;
  {
    const int L = h * w;
    if ((st = gn(x_site, attn_gn, X_, A_, 512, L, false)) != LBX_OK) return st;
    GemmArgs g;
    g.mode = GEMM_PLAIN;
    g.M = n * L; g.N = 1536; g.K = 512;
    g.A = A_; g.lda = 512; g.Bw = wqkv; g.ldb = 512;
    g.out = Hb; g.ldo = 1536; g.bias = bqkv;
    if ((st = gemm(g, "attn.qkv")) != LBX_OK) return st;
    // groups of up to s_imgs images: one scores GEMM, one softmax and one P.V launch per group
    // (batched plain GEMMs; the P.V of a single image is only 128 pair-tiles, < 2 waves)
    const int gsz = v_transpose_legacy() ? 1 : s_imgs;
    const bool fused_exp = attn_fused_exp() && L % 256 == 0 && L >= 256;
    if (fused_exp) LBX_STEP(cudaMemsetAsync(attn_flag, 0, sizeof(int) * (size_t)n, s), "memset attn flags");
    for (int i0 = 0; i0 < n; i0 += gsz) {
      const int g = std::min(gsz, n - i0);
      const __half* base = Hb + (size_t)i0 * L * 1536;
      GemmArgs sq;
      sq.mode = GEMM_PLAIN;
      sq.M = g * L; sq.N = L; sq.K = 512;
      sq.A = base; sq.lda = 1536;
      sq.Bw = base + 512; sq.ldb = 1536;
      sq.out = S; sq.ldo = L;
      sq.alpha = 1.0f / std::sqrt(512.0f);
      if (g > 1) { sq.batch_m = L; sq.batch_b = L; sq.b_rows_total = g * L; }
      if (fused_exp) {
        // softmax folded into the score GEMM: r_m = max of S over 256 keys sampled at stride L/256
        // (a small GEMM whose epilogue keeps only row maxima), then E = exp(S - r_m) straight from
        // the fp32 accumulator with per-row partial sums, then row_scale = 1 / sum.  An E that may
        // overflow fp16 (a score ~11 above r_m) flags the group; the fallback below -- launched
        // always, running only when flagged -- takes the exact row maximum over all keys (the same
        // GEMM with N = L) and recomputes E against it, so every E <= 1.
        int* flag = attn_flag + i0;  // one flag per image: a flagged image never changes another's pixels
        const int nparts = 2 * (L / 256);
        GemmArgs mx = sq;
        mx.N = 256;
        mx.Bw = base + 512; mx.ldb = 1536 * (L / 256);  // every (L/256)-th key row of each image
        if (g > 1) { mx.batch_b = 256; mx.b_rows_total = g * 256; }
        mx.out = S; mx.ldo = 256;                        // not written (rowred 1)
        mx.rowred = 1; mx.row_part = rowmax;
        if ((st = gemm(mx, "attn.score_sample")) != LBX_OK) return st;
        GemmArgs ex = sq;
        ex.rowred = 2; ex.row_max = rowmax; ex.row_part = rowpart; ex.exp_flag = flag;
        ex.exp_force = attn_force_fallback() ? 1 : 0;  // tests: every group takes the fallback
        if ((st = gemm(ex, "attn.scores+exp")) != LBX_OK) return st;
        LBX_LAUNCH(launch_attn_rowsum(rowpart, nparts, rowscale, g * L, s), "attn.rowsum",
                   4.0 * g * L * nparts + 4.0 * g * L);
        GemmArgs fmx = sq;  // fallback: exact row maxima over all keys (nothing stored)
        fmx.rowred = 1; fmx.row_part = rowpart; fmx.run_if = flag; fmx.run_if_n = g;
        if ((st = gemm(fmx, "attn.score_max(fallback)")) != LBX_OK) return st;
        LBX_LAUNCH(launch_attn_rowmax(rowpart, nparts, rowmax, g * L, s, flag, L), "attn.rowmax(fallback)", 0.0);
        GemmArgs fex = ex;
        fex.exp_force = 0; fex.run_if = flag; fex.run_if_n = g;
        if ((st = gemm(fex, "attn.scores+exp(fallback)")) != LBX_OK) return st;
        LBX_LAUNCH(launch_attn_rowsum(rowpart, nparts, rowscale, g * L, s, flag, L), "attn.rowsum(fallback)", 0.0);
      } else {
        if ((st = gemm(sq, "attn.scores")) != LBX_OK) return st;
        LBX_LAUNCH(launch_softmax_rows(S, rowscale, g * L, L, s), "attn.softmax", 4.0 * g * L * (double)L);
      }
      GemmArgs pv;
      pv.mode = GEMM_PLAIN;
      pv.M = g * L; pv.N = 512; pv.K = L;
      pv.A = S; pv.lda = L;
      if (v_transpose_legacy()) {
        LBX_LAUNCH(launch_transpose(base + 1024, 1536, Vt, L, L, 512, s), "attn.v_transpose", 4.0 * L * 512.0);
        pv.Bw = Vt; pv.ldb = L;
      } else {  // V read in place from the QKV buffer as an MN-major B operand (no transpose)
        pv.Bw = base + 1024; pv.ldb = 1536; pv.b_mn_major = 1;
        if (g > 1) { pv.batch_m = L; pv.batch_b = L; pv.b_rows_total = g * L; }
      }
      pv.out = A_ + (size_t)i0 * L * 512; pv.ldo = 512;
      pv.row_scale = rowscale;
      if ((st = gemm(pv, "attn.pv")) != LBX_OK) return st;
    }
    if (fused_exp)
      LBX_LAUNCH(launch_attn_count(attn_flag, n, attn_fallbacks, s), "attn.count", 0.0);
    GemmArgs o;
    o.mode = GEMM_PLAIN;
    o.M = n * L; o.N = 512; o.K = 512;
    o.A = A_; o.lda = 512; o.Bw = wo; o.ldb = 512;
    o.out = X_; o.ldo = 512; o.bias = bo; o.resid = X_; o.ldr = 512;
    const int out_site = site++;
    o.gn_stats = site_ptr(out_site); o.gn_cpg = 16; o.rows_per_img = L;
    if ((st = gemm(o, "attn.out")) != LBX_OK) return st;
    x_site = out_site;
  }
  if ((st = resnet(res[1], h, w)) != LBX_OK) return st;

  // up blocks
  int H = h, W = w;
  const int chans[4] = {512, 512, 256, 128};
  for (int i = 0; i < 4; ++i) {
    for (int j = 0; j < 3; ++j)
      if ((st = resnet(res[2 + 3 * i + j], H, W)) != LBX_OK) return st;
    if (i < 3) {
      const int c = chans[i];
      GemmArgs g;
      g.mode = GEMM_SUBPIX;
      g.M = n * H * W; g.N = c; g.K = 4 * c;
      g.A = X_; g.B_img = n; g.H = H; g.W = W; g.C = c;
      g.Bw = up[i].w; g.ldb = 4 * c;
      g.out = A_; g.ldo = c; g.bias = up[i].b;
      const int out_site = site++;
      g.gn_stats = site_ptr(out_site); g.gn_cpg = c / 32; g.rows_per_img = H * W;
      if ((st = gemm(g, "upsample.subpixel_conv")) != LBX_OK) return st;
      x_site = out_site;
      std::swap(X_, A_);
      H *= 2;
      W *= 2;
    }
  }
  // tail
  LBX_LAUNCH(launch_gn_finalize(site_ptr(x_site), norm_out.g, norm_out.b, ss, n, 128, (double)H * W * 4, 1e-6f, s),
             "norm_out.finalize", n * 128 * 8.0);
  if (W % 128 == 0 && !kernels_conv_out_legacy()) {
    LBX_STEP(launch_conv_out_tc(X_, ss, wout, bout, rgb_out, n, H, W, h2, s), "conv_out_tc");
    ++launches;
    mark("conv_out_tc", 2.0 * n * H * W * 16 * 1152, 2.0 * n * H * W * 3 * 1152, (double)n * H * W * (128 * 2 + 3));
  } else {
    LBX_LAUNCH(launch_conv_out_u8(X_, ss, wout, bout, rgb_out, n, H, W, s), "conv_out_u8",
               (double)n * H * W * (128 * 2 + 3));
  }
  if (site > kMaxSites) return set_err(LBX_E_RUNTIME, "too many GroupNorm sites");
  if (counting) launch_counts[n] = launches;
  return LBX_OK;
#undef LBX_STEP
#undef LBX_LAUNCH
}

lbx_status Decoder::graph_for(int n, cudaStream_t s, cudaGraphExec_t* out) {
  auto it = graphs.find(n);
  if (it == graphs.end()) {
    // one graph per batch size, on the decoder's own buffers (lat -> rgb): at most max_batch graphs
    cudaGraph_t g = nullptr;
    LBX_CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    lbx_status st = plan(n, lat, rgb, s, true);
    cudaError_t ce = cudaStreamEndCapture(s, &g);
    if (st != LBX_OK) {
      if (g) cudaGraphDestroy(g);
      return st;
    }
    if (ce != cudaSuccess) return set_err(LBX_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
    cudaGraphExec_t ex = nullptr;
    ce = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (ce != cudaSuccess) return set_err(LBX_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ce));
    ++captures;
    it = graphs.emplace(n, ex).first;
  }
  *out = it->second;
  return LBX_OK;
}

// Decode n latents: caller latents are copied into the graph's input buffer and the RGB out of its
// output buffer (D2D; 0.1% of a 1024^2 decode) unless they already are those buffers.
lbx_status Decoder::run(int n, const __half* lat_in, uint8_t* rgb_out, cudaStream_t s) {
  cudaGraphExec_t ex = nullptr;
  lbx_status st = graph_for(n, s, &ex);
  if (st != LBX_OK) return st;
  if (lat_in != lat) LBX_CUDA_TRY(cudaMemcpyAsync(lat, lat_in, lat_elems(n) * 2, cudaMemcpyDeviceToDevice, s));
  LBX_CUDA_TRY(cudaGraphLaunch(ex, s));
  if (rgb_out != rgb) LBX_CUDA_TRY(cudaMemcpyAsync(rgb_out, rgb, rgb_bytes(n), cudaMemcpyDeviceToDevice, s));
  return LBX_OK;
}

lbx_status Decoder::validate_blobs(const uint8_t* const* blobs, const size_t* nbytes, uint32_t n, size_t* total) {
  *total = 0;
  if (!blobs || !nbytes) return set_err(LBX_E_CONFIG, "blobs: null pointer");
  for (uint32_t i = 0; i < n; ++i) {
    std::string why;
    if (!blobs[i]) return set_err(LBX_E_CONFIG, "blobs: null pointer");
    if (!lblp_validate(blobs[i], nbytes[i], cl, h, w, &why))
      return set_err(LBX_E_FORMAT, "blob " + std::to_string(i) + ": " + why);
    *total += (nbytes[i] + 15) & ~size_t(15);
  }
  return LBX_OK;
}

lbx_status Decoder::grow_staging(Staging& st, size_t total) {
  if (total <= st.cap) return LBX_OK;
  if (st.host) cudaFreeHost(st.host);
  if (st.dev) cudaFree(st.dev);
  st.host = st.dev = nullptr;
  st.cap = (total + (total >> 2) + 4096 + 255) & ~size_t(255);  // the table follows: keep 8B+ alignment
  LBX_CUDA_TRY(cudaMallocHost(&st.host, st.cap));
  LBX_CUDA_TRY(cudaMalloc(&st.dev, st.cap + (size_t)max_batch * 16));
  st.offs_dev = reinterpret_cast<unsigned long long*>(st.dev + st.cap);
  st.sizes_dev = reinterpret_cast<unsigned int*>(st.offs_dev + max_batch);
  return LBX_OK;
}

// Gather n blobs into device staging and unpack them into lat_out (status into err_dev), all on s.
// Host blobs (blob_devs == NULL): headers validated here, copied into pinned staging, one H2D.
// Device blobs (blob_devs[i] = the GPU holding blob i, an HBM-resident latent tier): a D2D copy,
// or a peer copy over NVLink when the blob lives on another GPU (the reference ships such a latent
// to the executing node at LatencyModel::intra_cluster_ms, proj/include/latentbox/sim.hpp:20,
// proj/src/sim.cpp:369-373); their headers are validated by the device unpack (err_dev).
lbx_status Decoder::stage_blobs(Staging& st, const uint8_t* const* blobs, const size_t* nbytes, uint32_t n,
                                cudaStream_t s, __half* lat_out, int* err_dev, const int* blob_devs,
                                cudaEvent_t after_copies) {
  size_t total = 0;
  if (!blob_devs) {
    lbx_status vs = validate_blobs(blobs, nbytes, n, &total);
    if (vs != LBX_OK) return vs;
  } else {  // per blob: host (blob_devs[i] < 0, validated here) or device memory
    if (!blobs || !nbytes) return set_err(LBX_E_CONFIG, "blobs: null pointer");
    for (uint32_t i = 0; i < n; ++i) {
      if (!blobs[i] || nbytes[i] == 0 || nbytes[i] > 0xFFFFFFFFull)
        return set_err(LBX_E_CONFIG, "blob " + std::to_string(i) + ": null or bad size");
      std::string why;
      if (blob_devs[i] < 0 && !lblp_validate(blobs[i], nbytes[i], cl, h, w, &why))
        return set_err(LBX_E_FORMAT, "blob " + std::to_string(i) + ": " + why);
      total += (nbytes[i] + 15) & ~size_t(15);
    }
  }
  // the previous H2D out of the pinned buffer must be complete before it is rewritten or replaced
  LBX_CUDA_TRY(cudaEventSynchronize(st.copied));
  lbx_status gs = grow_staging(st, total);
  if (gs != LBX_OK) return gs;
  size_t off = 0;
  unsigned int* sizes_host = reinterpret_cast<unsigned int*>(st.table_host + max_batch);
  for (uint32_t i = 0; i < n; ++i) {
    if (!blob_devs || blob_devs[i] < 0) std::memcpy(st.host + off, blobs[i], nbytes[i]);
    st.table_host[i] = off;
    sizes_host[i] = (unsigned int)nbytes[i];
    off += (nbytes[i] + 15) & ~size_t(15);
  }
  bool any_host = !blob_devs;
  for (uint32_t i = 0; blob_devs && i < n; ++i) any_host |= blob_devs[i] < 0;
  // host blobs: one H2D of the whole staging region (device blobs' slots are overwritten below,
  // in stream order)
  if (any_host) LBX_CUDA_TRY(cudaMemcpyAsync(st.dev, st.host, off, cudaMemcpyHostToDevice, s));
  if (blob_devs) {
    for (uint32_t i = 0; i < n; ++i) {
      uint8_t* dst = st.dev + st.table_host[i];
      if (blob_devs[i] < 0) continue;
      if (blob_devs[i] == desc.device) {
        LBX_CUDA_TRY(cudaMemcpyAsync(dst, blobs[i], nbytes[i], cudaMemcpyDeviceToDevice, s));
      } else {
        LBX_CUDA_TRY(cudaMemcpyPeerAsync(dst, desc.device, blobs[i], blob_devs[i], nbytes[i], s));
        ++peer_copies;
        peer_bytes += nbytes[i];
      }
    }
  }
  if (after_copies) LBX_CUDA_TRY(cudaEventRecord(after_copies, s));
  LBX_CUDA_TRY(cudaMemcpyAsync(st.offs_dev, st.table_host, (size_t)max_batch * 12, cudaMemcpyHostToDevice, s));
  LBX_CUDA_TRY(cudaEventRecord(st.copied, s));
  launch_lblp_unpack(st.dev, st.offs_dev, st.sizes_dev, (int)n, cl, h, w, lat_out, err_dev, s);
  LBX_CUDA_TRY(cudaPeekAtLastError());
  return LBX_OK;
}

}  // namespace lbx

// =========================================================================== C ABI
using lbx::Decoder;
using lbx::set_err;

struct lbx_decoder {
  Decoder d;
  std::mutex mu;  // defensive: the contract is single-owner per decoder
};

static cudaStream_t pick(lbx_decoder* dec, lbx_stream s) {
  return s ? reinterpret_cast<cudaStream_t>(s) : dec->d.stream;
}

extern "C" {

const char* lbx_last_error(void) { return lbx::g_err.c_str(); }

size_t lbx_param_count(int family) {
  lbx::FamilyInfo fi;
  if (!lbx::family_info(family, &fi)) return 0;
  size_t n = 0;
  for (const auto& s : lbx::param_specs(fi.latent_channels, fi.post_quant)) n += s.count();
  return n;
}

lbx_status lbx_generate_params(int family, uint64_t seed, float* out, size_t count) {
  if (!out || count != lbx_param_count(family) || count == 0)
    return set_err(LBX_E_CONFIG, "lbx_generate_params: count != lbx_param_count(family)");
  const std::vector<float> p = lbx::generate_params(family, seed);
  std::memcpy(out, p.data(), count * sizeof(float));
  return LBX_OK;
}

lbx_status lbx_decoder_create(const lbx_decoder_desc* desc, lbx_decoder** out) {
  if (!desc || !out) return set_err(LBX_E_CONFIG, "lbx_decoder_create: null argument");
  *out = nullptr;
  auto* dec = new (std::nothrow) lbx_decoder;
  if (!dec) return set_err(LBX_E_RUNTIME, "out of host memory");
  lbx_status st = dec->d.init(*desc);
  if (st != LBX_OK) {
    delete dec;
    return st;
  }
  *out = dec;
  lbx::g_err.clear();
  return LBX_OK;
}

lbx_status lbx_decoder_prepare(lbx_decoder* dec, uint32_t n_max) {
  if (!dec) return set_err(LBX_E_CONFIG, "lbx_decoder_prepare: null decoder");
  std::lock_guard<std::mutex> g(dec->mu);
  Decoder& d = dec->d;
  if (n_max == 0 || (int)n_max > d.max_batch) return set_err(LBX_E_CONFIG, "n_max: must be in [1, desc.max_batch]");
  cudaSetDevice(d.desc.device);
  d.order(d.stream);
  for (uint32_t n = 1; n <= n_max; ++n) {
    cudaGraphExec_t ex = nullptr;
    lbx_status st = d.graph_for((int)n, d.stream, &ex);
    if (st != LBX_OK) return st;
  }
  return LBX_OK;
}

uint64_t lbx_graph_captures(lbx_decoder* dec) { return dec ? dec->d.captures : 0; }

lbx_status lbx_decoder_destroy(lbx_decoder* dec) {
  if (!dec) return set_err(LBX_E_CONFIG, "lbx_decoder_destroy: null decoder");
  delete dec;
  return LBX_OK;
}

lbx_status lbx_unpack(lbx_decoder* dec, const uint8_t* const* blobs, const size_t* nbytes, uint32_t n,
                      void* latents_dev, lbx_stream stream) {
  if (!dec || !latents_dev) return set_err(LBX_E_CONFIG, "lbx_unpack: null argument");
  std::lock_guard<std::mutex> g(dec->mu);
  Decoder& d = dec->d;
  if (n == 0) return LBX_OK;
  if ((int)n > d.max_batch) return set_err(LBX_E_CONFIG, "n: exceeds desc.max_batch");
  cudaSetDevice(d.desc.device);
  cudaStream_t s = pick(dec, stream);
  d.order(s);
  lbx_status st = d.stage_blobs(d.sync_st, blobs, nbytes, n, s, reinterpret_cast<__half*>(latents_dev), d.err);
  d.mark(s);
  return st;
}

lbx_status lbx_decode(lbx_decoder* dec, const void* latents_dev, uint32_t n, uint8_t* rgb_dev, lbx_stream stream) {
  if (!dec || !latents_dev || !rgb_dev) return set_err(LBX_E_CONFIG, "lbx_decode: null argument");
  std::lock_guard<std::mutex> g(dec->mu);
  Decoder& d = dec->d;
  if (n == 0) return LBX_OK;
  if ((int)n > d.max_batch) return set_err(LBX_E_CONFIG, "n: exceeds desc.max_batch");
  cudaSetDevice(d.desc.device);
  cudaStream_t s = pick(dec, stream);
  d.order(s);
  lbx_status st = d.run((int)n, reinterpret_cast<const __half*>(latents_dev), rgb_dev, s);
  d.mark(s);
  return st;
}

// Decode d.lat (already staged on s), D2H the RGB, wait, check the device status word.
static lbx_status finish_reconstruct(Decoder& d, uint32_t n, uint8_t* rgb_host, cudaStream_t s,
                                     uint8_t* const* rgb_hosts = nullptr) {
  lbx_status st = d.run((int)n, d.lat, d.rgb, s);
  if (st != LBX_OK) return st;
  if (rgb_hosts) {
    const size_t per = d.rgb_bytes(1);
    for (uint32_t i = 0; i < n; ++i)
      if (cudaMemcpyAsync(rgb_hosts[i], d.rgb + i * per, per, cudaMemcpyDeviceToHost, s) != cudaSuccess)
        return set_err(LBX_E_CUDA, "D2H of rgb failed");
  } else if (cudaMemcpyAsync(rgb_host, d.rgb, d.rgb_bytes(n), cudaMemcpyDeviceToHost, s) != cudaSuccess) {
    return set_err(LBX_E_CUDA, "D2H of rgb failed");
  }
  if (cudaMemcpyAsync(d.err_host, d.err, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return set_err(LBX_E_CUDA, "D2H of status failed");
  d.mark(s);
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return set_err(LBX_E_CUDA, std::string("reconstruct: ") + cudaGetErrorString(e));
  if (*d.err_host) {
    cudaMemset(d.err, 0, 4);
    return set_err(LBX_E_FORMAT, "device unpack reported a malformed blob (code " + std::to_string(*d.err_host) + ")");
  }
  return LBX_OK;
}

lbx_status lbx_reconstruct(lbx_decoder* dec, const uint8_t* const* blobs, const size_t* nbytes, uint32_t n,
                           uint8_t* rgb_host, lbx_stream stream) {
  if (!dec || !rgb_host) return set_err(LBX_E_CONFIG, "lbx_reconstruct: null argument");
  std::lock_guard<std::mutex> g(dec->mu);
  Decoder& d = dec->d;
  if (n == 0) return LBX_OK;
  if ((int)n > d.max_batch) return set_err(LBX_E_CONFIG, "n: exceeds desc.max_batch");
  cudaSetDevice(d.desc.device);
  cudaStream_t s = pick(dec, stream);
  d.order(s);
  lbx_status st = d.stage_blobs(d.sync_st, blobs, nbytes, n, s, d.lat, d.err);
  if (st != LBX_OK) return st;
  return finish_reconstruct(d, n, rgb_host, s);
}

lbx_status lbx_reconstruct_v(lbx_decoder* dec, const uint8_t* const* blobs, const size_t* nbytes, uint32_t n,
                             uint8_t* const* rgb_hosts, lbx_stream stream) {
  if (!dec || !rgb_hosts) return set_err(LBX_E_CONFIG, "lbx_reconstruct_v: null argument");
  for (uint32_t i = 0; i < n; ++i)
    if (!rgb_hosts[i]) return set_err(LBX_E_CONFIG, "rgb_hosts: null entry");
  std::lock_guard<std::mutex> g(dec->mu);
  Decoder& d = dec->d;
  if (n == 0) return LBX_OK;
  if ((int)n > d.max_batch) return set_err(LBX_E_CONFIG, "n: exceeds desc.max_batch");
  cudaSetDevice(d.desc.device);
  cudaStream_t s = pick(dec, stream);
  d.order(s);
  lbx_status st = d.stage_blobs(d.sync_st, blobs, nbytes, n, s, d.lat, d.err);
  if (st != LBX_OK) return st;
  return finish_reconstruct(d, n, nullptr, s, rgb_hosts);
}

// Asynchronous pipeline.  Slot k % 2 carries ticket k:
//   in_stream : H2D blobs -> unpack into slot.lat                               -> [unpacked]
//   stream    : wait unpacked; lat <- slot.lat; graph; wait drained(previous use of the slot);
//               slot.rgb <- rgb                                                  -> [computed]
//   out_stream: wait computed; D2H slot.rgb -> rgb_hosts[i]; status word         -> [drained]
// so batch k+1's copy-in and batch k-1's copy-out overlap batch k's graph.
static lbx_status submit_impl(lbx_decoder* dec, const uint8_t* const* blobs, const int* blob_devs,
                              const size_t* nbytes, uint32_t n, uint8_t* const* rgb_hosts, uint64_t* ticket) {
  if (!dec || !rgb_hosts || !ticket) return set_err(LBX_E_CONFIG, "lbx_reconstruct_submit: null argument");
  for (uint32_t i = 0; i < n; ++i)
    if (!rgb_hosts[i]) return set_err(LBX_E_CONFIG, "rgb_hosts: null entry");
  *ticket = 0;
  lbx_status st = LBX_OK;
  std::lock_guard<std::mutex> g(dec->mu);
  Decoder& d = dec->d;
  if (n == 0 || (int)n > d.max_batch) return set_err(LBX_E_CONFIG, "n: must be in [1, desc.max_batch]");
  cudaSetDevice(d.desc.device);
  Decoder::Slot& sl = d.slots[d.next_ticket & 1];
  if (sl.busy)
    return set_err(LBX_E_RUNTIME, "lbx_reconstruct_submit: two batches in flight; wait for ticket " +
                                      std::to_string(sl.ticket) + " first");
  if ((st = d.alloc_slot(sl)) != LBX_OK) return st;
  cudaGraphExec_t ex = nullptr;
  d.order(d.stream);
  if ((st = d.graph_for((int)n, d.stream, &ex)) != LBX_OK) return st;  // captured once per n
  // the slot's latents were last read by its previous batch's copy on `stream`
  LBX_CUDA_TRY(cudaStreamWaitEvent(d.in_stream, sl.computed, 0));
  sl.timed_peer = false;
  if (blob_devs)
    for (uint32_t i = 0; i < n; ++i) sl.timed_peer |= blob_devs[i] >= 0 && blob_devs[i] != d.desc.device;
  if (sl.timed_peer) LBX_CUDA_TRY(cudaEventRecord(sl.peer0, d.in_stream));
  // peer1 is recorded right after the blob copies (before the table upload and the unpack)
  if ((st = d.stage_blobs(sl.st, blobs, nbytes, n, d.in_stream, sl.lat, sl.err, blob_devs,
                          sl.timed_peer ? sl.peer1 : nullptr)) != LBX_OK)
    return st;
  LBX_CUDA_TRY(cudaEventRecord(sl.unpacked, d.in_stream));
  LBX_CUDA_TRY(cudaStreamWaitEvent(d.stream, sl.unpacked, 0));
  LBX_CUDA_TRY(cudaMemcpyAsync(d.lat, sl.lat, d.lat_elems(n) * 2, cudaMemcpyDeviceToDevice, d.stream));
  LBX_CUDA_TRY(cudaGraphLaunch(ex, d.stream));
  LBX_CUDA_TRY(cudaStreamWaitEvent(d.stream, sl.drained, 0));
  LBX_CUDA_TRY(cudaMemcpyAsync(sl.rgb, d.rgb, d.rgb_bytes(n), cudaMemcpyDeviceToDevice, d.stream));
  LBX_CUDA_TRY(cudaEventRecord(sl.computed, d.stream));
  d.mark(d.stream);
  LBX_CUDA_TRY(cudaStreamWaitEvent(d.out_stream, sl.computed, 0));
  const size_t per = d.rgb_bytes(1);
  for (uint32_t i = 0; i < n; ++i)
    LBX_CUDA_TRY(cudaMemcpyAsync(rgb_hosts[i], sl.rgb + i * per, per, cudaMemcpyDeviceToHost, d.out_stream));
  LBX_CUDA_TRY(cudaMemcpyAsync(sl.err_host, sl.err, 4, cudaMemcpyDeviceToHost, d.out_stream));
  LBX_CUDA_TRY(cudaEventRecord(sl.drained, d.out_stream));
  sl.busy = true;
  sl.ticket = d.next_ticket++;
  *ticket = sl.ticket;
  return LBX_OK;
}

lbx_status lbx_reconstruct_submit(lbx_decoder* dec, const uint8_t* const* blobs, const size_t* nbytes, uint32_t n,
                                  uint8_t* const* rgb_hosts, uint64_t* ticket) {
  return submit_impl(dec, blobs, nullptr, nbytes, n, rgb_hosts, ticket);
}

lbx_status lbx_reconstruct_submit_dev(lbx_decoder* dec, const uint8_t* const* blobs_dev, const int* blob_devices,
                                      const size_t* nbytes, uint32_t n, uint8_t* const* rgb_hosts, uint64_t* ticket) {
  if (!blob_devices) return set_err(LBX_E_CONFIG, "lbx_reconstruct_submit_dev: null blob_devices");
  return submit_impl(dec, blobs_dev, blob_devices, nbytes, n, rgb_hosts, ticket);
}

lbx_status lbx_decoder_get_counters(lbx_decoder* dec, lbx_decoder_counters* out) {
  if (!dec || !out) return set_err(LBX_E_CONFIG, "lbx_decoder_get_counters: null argument");
  std::lock_guard<std::mutex> g(dec->mu);
  out->graph_captures = dec->d.captures;
  out->peer_copies = dec->d.peer_copies;
  out->peer_bytes = dec->d.peer_bytes;
  out->peer_ms = dec->d.peer_ms;
  out->attn_fallbacks = 0;
  if (dec->d.attn_fallbacks) {
    LBX_CUDA_TRY(cudaSetDevice(dec->d.desc.device));
    LBX_CUDA_TRY(cudaMemcpy(&out->attn_fallbacks, dec->d.attn_fallbacks, 8, cudaMemcpyDeviceToHost));
  }
  return LBX_OK;
}

lbx_status lbx_reconstruct_wait(lbx_decoder* dec, uint64_t ticket) {
  if (!dec) return set_err(LBX_E_CONFIG, "lbx_reconstruct_wait: null decoder");
  cudaEvent_t ev = nullptr;
  int slot = -1;
  {
    std::lock_guard<std::mutex> g(dec->mu);
    Decoder& d = dec->d;
    for (int i = 0; i < 2; ++i)
      if (d.slots[i].busy && d.slots[i].ticket == ticket) slot = i;
    if (slot < 0) return set_err(LBX_E_CONFIG, "lbx_reconstruct_wait: unknown or already retired ticket");
    ev = d.slots[slot].drained;
  }
  const cudaError_t e = cudaEventSynchronize(ev);  // outside the lock: the next batch may be submitted
  std::lock_guard<std::mutex> g(dec->mu);
  Decoder::Slot& sl = dec->d.slots[slot];
  sl.busy = false;
  if (sl.timed_peer && e == cudaSuccess) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, sl.peer0, sl.peer1) == cudaSuccess) dec->d.peer_ms += ms;
  }
  if (e != cudaSuccess) return set_err(LBX_E_CUDA, std::string("reconstruct: ") + cudaGetErrorString(e));
  if (*sl.err_host) {
    const int code = *sl.err_host;
    *sl.err_host = 0;
    cudaMemsetAsync(sl.err, 0, 4, dec->d.in_stream);
    return set_err(LBX_E_FORMAT, "device unpack reported a malformed blob (code " + std::to_string(code) + ")");
  }
  return LBX_OK;
}

lbx_status lbx_reconstruct_png(lbx_decoder* dec, const uint8_t* const* blobs, const size_t* nbytes, uint32_t n,
                               uint8_t* png_host, size_t cap, size_t* png_sizes, lbx_stream stream) {
  if (!dec || !png_host || !png_sizes) return set_err(LBX_E_CONFIG, "lbx_reconstruct_png: null argument");
  std::lock_guard<std::mutex> g(dec->mu);
  Decoder& d = dec->d;
  if (n == 0) return LBX_OK;
  if ((int)n > d.max_batch) return set_err(LBX_E_CONFIG, "n: exceeds desc.max_batch");
  cudaSetDevice(d.desc.device);
  cudaStream_t s = pick(dec, stream);
  const int H = 8 * d.h, W = 8 * d.w;
  if (!d.png_dev) {
    const size_t out_bytes = (size_t)d.max_batch * lbx::png_bound(H, W);
    if (cudaMalloc(&d.png_dev, out_bytes) != cudaSuccess ||
        cudaMalloc(&d.png_work, lbx::png_workspace(d.max_batch, H, W)) != cudaSuccess ||
        cudaMalloc(&d.png_sizes, 4 * (size_t)d.max_batch) != cudaSuccess ||
        cudaMallocHost(&d.png_sizes_host, 4 * (size_t)d.max_batch) != cudaSuccess)
      return set_err(LBX_E_CUDA, "lbx_reconstruct_png: PNG buffers");
  }
  d.order(s);
  lbx_status st = d.stage_blobs(d.sync_st, blobs, nbytes, n, s, d.lat, d.err);
  if (st != LBX_OK) return st;
  if ((st = d.run((int)n, d.lat, d.rgb, s)) != LBX_OK) return st;
  cudaError_t e = lbx::launch_png_encode(d.rgb, (int)n, H, W, d.png_dev, 0, d.png_sizes, d.png_work, s, true);
  if (e != cudaSuccess) return set_err(LBX_E_CUDA, std::string("lbx_reconstruct_png: ") + cudaGetErrorString(e));
  if (cudaMemcpyAsync(d.png_sizes_host, d.png_sizes, 4 * (size_t)n, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaMemcpyAsync(d.err_host, d.err, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return set_err(LBX_E_CUDA, "D2H of PNG sizes failed");
  d.mark(s);
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess)
    return set_err(LBX_E_CUDA, std::string("reconstruct_png: ") + cudaGetErrorString(e));
  if (*d.err_host) {
    cudaMemset(d.err, 0, 4);
    return set_err(LBX_E_FORMAT, "device unpack reported a malformed blob (code " + std::to_string(*d.err_host) + ")");
  }
  size_t total = 0;
  for (uint32_t i = 0; i < n; ++i) total += (png_sizes[i] = d.png_sizes_host[i]);
  if (total > cap)
    return set_err(LBX_E_CONFIG, "cap: the PNGs need " + std::to_string(total) + " bytes (sizes returned)");
  if (cudaMemcpyAsync(png_host, d.png_dev, total, cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return set_err(LBX_E_CUDA, "D2H of PNGs failed");
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess)
    return set_err(LBX_E_CUDA, std::string("reconstruct_png: ") + cudaGetErrorString(e));
  return LBX_OK;
}

lbx_status lbx_reconstruct_latents(lbx_decoder* dec, const void* latents_host, uint32_t n, uint8_t* rgb_host,
                                   lbx_stream stream) {
  if (!dec || !latents_host || !rgb_host) return set_err(LBX_E_CONFIG, "lbx_reconstruct_latents: null argument");
  std::lock_guard<std::mutex> g(dec->mu);
  Decoder& d = dec->d;
  if (n == 0) return LBX_OK;
  if ((int)n > d.max_batch) return set_err(LBX_E_CONFIG, "n: exceeds desc.max_batch");
  cudaSetDevice(d.desc.device);
  cudaStream_t s = pick(dec, stream);
  d.order(s);
  if (cudaMemcpyAsync(d.lat, latents_host, d.lat_elems(n) * 2, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return set_err(LBX_E_CUDA, "H2D of latents failed");
  return finish_reconstruct(d, n, rgb_host, s);
}

lbx_status lbx_pack(const uint16_t* latent, int mode, uint32_t c, uint32_t h, uint32_t w, uint8_t* out, size_t cap,
                    size_t* out_bytes) {
  std::vector<uint8_t> blob;
  std::string why;
  if (!lbx::lblp_pack(latent, mode, c, h, w, &blob, &why)) return set_err(LBX_E_CONFIG, why);
  if (out_bytes) *out_bytes = blob.size();
  if (out) {
    if (cap < blob.size()) return set_err(LBX_E_CONFIG, "cap: smaller than the encoded blob");
    std::memcpy(out, blob.data(), blob.size());
  }
  return LBX_OK;
}

// ------------------------------------------------------------------ op-level entry points
lbx_status lbx_op_gemm(int mode, int M, int N, int K, const void* A, int lda, int b, int h, int w, int c,
                       const void* Bw, int ldb, void* out, int ldo, const float* bias, const void* resid, int ldr,
                       const float* row_scale, float alpha, uint64_t* gn_stats, int cta_group, int bn,
                       lbx_stream stream) {
  lbx::GemmArgs g;
  g.mode = mode;
  g.M = M; g.N = N; g.K = K;
  g.A = reinterpret_cast<const __half*>(A); g.lda = lda;
  g.B_img = b; g.H = h; g.W = w; g.C = c;
  g.Bw = reinterpret_cast<const __half*>(Bw); g.ldb = ldb;
  g.out = reinterpret_cast<__half*>(out); g.ldo = ldo;
  g.bias = bias;
  g.resid = reinterpret_cast<const __half*>(resid); g.ldr = ldr;
  g.row_scale = row_scale; g.alpha = alpha;
  g.gn_stats = reinterpret_cast<unsigned long long*>(gn_stats); g.gn_cpg = N / 32; g.rows_per_img = (mode == 0) ? (b > 0 ? M / b : M) : h * w;
  cudaError_t e = lbx::gemm_tc_launch(g, reinterpret_cast<cudaStream_t>(stream), cta_group, bn);
  if (e != cudaSuccess) return set_err(e == cudaErrorInvalidValue ? LBX_E_CONFIG : LBX_E_CUDA,
                                       std::string("lbx_op_gemm: ") + cudaGetErrorString(e));
  return LBX_OK;
}

lbx_status lbx_op_gemm_desc(const lbx_gemm_desc* d, lbx_stream stream) {
  if (!d) return set_err(LBX_E_CONFIG, "lbx_op_gemm_desc: null descriptor");
  lbx::GemmArgs g;
  g.mode = d->mode;
  g.M = d->M; g.N = d->N; g.K = d->K;
  g.A = reinterpret_cast<const __half*>(d->A); g.lda = d->lda;
  g.B_img = d->b; g.H = d->h; g.W = d->w; g.C = d->c;
  g.A2 = reinterpret_cast<const __half*>(d->A2); g.lda2 = d->lda2; g.K2 = d->K2;
  g.Bw = reinterpret_cast<const __half*>(d->B); g.ldb = d->ldb;
  g.out = reinterpret_cast<__half*>(d->out); g.ldo = d->ldo;
  g.bias = d->bias;
  g.resid = reinterpret_cast<const __half*>(d->resid); g.ldr = d->ldr;
  g.row_scale = d->row_scale; g.alpha = d->alpha;
  g.gn_stats = reinterpret_cast<unsigned long long*>(d->gn_stats); g.gn_cpg = d->N / 32;
  g.gn_ss = reinterpret_cast<const float2*>(d->gn_ss);
  g.b_mn_major = d->b_mn_major;
  g.rows_per_img = (d->mode == 0) ? (d->b > 0 ? d->M / d->b : d->M) : d->h * d->w;
  cudaError_t e = lbx::gemm_tc_launch(g, reinterpret_cast<cudaStream_t>(stream), d->cta_group, d->bn);
  if (e != cudaSuccess) return set_err(e == cudaErrorInvalidValue ? LBX_E_CONFIG : LBX_E_CUDA,
                                       std::string("lbx_op_gemm_desc: ") + cudaGetErrorString(e));
  return LBX_OK;
}

lbx_status lbx_op_attention(const void* qkv, void* out, int n, int L, lbx_stream stream) {
  if (!qkv || !out || n <= 0 || L <= 0 || L % 128) return set_err(LBX_E_CONFIG, "lbx_op_attention: bad argument");
  cudaError_t e = lbx::launch_attn_fa(reinterpret_cast<const __half*>(qkv), reinterpret_cast<__half*>(out), n, L,
                                      reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess)
    return set_err(e == cudaErrorInvalidValue ? LBX_E_CONFIG : LBX_E_CUDA,
                   std::string("lbx_op_attention: ") + cudaGetErrorString(e));
  return LBX_OK;
}

size_t lbx_pack_bound(uint32_t c, uint32_t h, uint32_t w) {
  if (c == 0 || h == 0 || w == 0 || w % 32) return 0;
  return lbx::lblp_pack_bound((int)c, (int)h, (int)w);
}

lbx_status lbx_pack_device(const void* latents_dev, uint32_t n, uint32_t c, uint32_t h, uint32_t w, uint8_t* out_dev,
                           size_t stride, uint32_t* sizes_dev, lbx_stream stream) {
  if (n == 0) return LBX_OK;
  if (!latents_dev || !out_dev || !sizes_dev) return set_err(LBX_E_CONFIG, "lbx_pack_device: null pointer");
  if (c == 0 || h == 0 || w == 0 || w % 32 || c > 65535 || h > 65535 || w > 65535)
    return set_err(LBX_E_CONFIG, "lbx_pack_device: shape must be nonzero, <= 65535, w % 32 == 0");
  if (stride < lbx::lblp_pack_bound((int)c, (int)h, (int)w) || stride % 4)
    return set_err(LBX_E_CONFIG, "lbx_pack_device: stride must be >= lbx_pack_bound and a multiple of 4");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t rows = (size_t)n * c * h;
  uint8_t* tmp = nullptr;
  const size_t wbytes = (rows * (w / 32) + 15) & ~size_t(15);
  if (cudaMallocAsync(reinterpret_cast<void**>(&tmp), wbytes + rows * 4, s) != cudaSuccess)
    return set_err(LBX_E_CUDA, "lbx_pack_device: cudaMallocAsync");
  cudaError_t e = lbx::launch_lblp_pack(reinterpret_cast<const uint16_t*>(latents_dev), (int)n, (int)c, (int)h, (int)w,
                                        out_dev, (long long)stride, sizes_dev, tmp,
                                        reinterpret_cast<uint32_t*>(tmp + wbytes), s);
  cudaFreeAsync(tmp, s);
  if (e != cudaSuccess) return set_err(LBX_E_CUDA, std::string("lbx_pack_device: ") + cudaGetErrorString(e));
  return LBX_OK;
}

size_t lbx_png_bound(uint32_t h, uint32_t w) {
  if (h == 0 || w == 0 || w > 8192 || h > 65535) return 0;
  return lbx::png_bound((int)h, (int)w);
}

lbx_status lbx_png_encode_device(const uint8_t* rgb_dev, uint32_t n, uint32_t h, uint32_t w, uint8_t* out_dev,
                                 size_t stride, uint32_t* sizes_dev, lbx_stream stream) {
  if (n == 0) return LBX_OK;
  if (!rgb_dev || !out_dev || !sizes_dev) return set_err(LBX_E_CONFIG, "lbx_png_encode_device: null pointer");
  if (h == 0 || w == 0 || w > 8192 || h > 65535)
    return set_err(LBX_E_CONFIG, "lbx_png_encode_device: shape must be nonzero, w <= 8192, h <= 65535");
  if (stride < lbx::png_bound((int)h, (int)w))
    return set_err(LBX_E_CONFIG, "lbx_png_encode_device: stride must be >= lbx_png_bound(h, w)");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* work = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&work), lbx::png_workspace((int)n, (int)h, (int)w), s) != cudaSuccess)
    return set_err(LBX_E_CUDA, "lbx_png_encode_device: cudaMallocAsync");
  cudaError_t e = lbx::launch_png_encode(rgb_dev, (int)n, (int)h, (int)w, out_dev, (long long)stride, sizes_dev, work, s);
  cudaFreeAsync(work, s);
  if (e != cudaSuccess) return set_err(LBX_E_CUDA, std::string("lbx_png_encode_device: ") + cudaGetErrorString(e));
  return LBX_OK;
}

lbx_status lbx_op_unpack(const uint8_t* blobs_dev, const unsigned long long* offs_dev, const uint32_t* sizes_dev,
                         uint32_t n, uint32_t c, uint32_t h, uint32_t w, void* out_dev, int* err_dev,
                         lbx_stream stream) {
  if (n == 0) return LBX_OK;
  if (!blobs_dev || !offs_dev || !sizes_dev || !out_dev || !err_dev)
    return set_err(LBX_E_CONFIG, "lbx_op_unpack: null pointer");
  if (c == 0 || h == 0 || w == 0 || w % 32 || c > 65535 || h > 65535 || w > 65535)
    return set_err(LBX_E_CONFIG, "lbx_op_unpack: shape must be nonzero, <= 65535, w % 32 == 0");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  lbx::launch_lblp_unpack(blobs_dev, offs_dev, reinterpret_cast<const unsigned int*>(sizes_dev), (int)n, (int)c,
                          (int)h, (int)w, reinterpret_cast<__half*>(out_dev), err_dev, s);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(LBX_E_CUDA, std::string("lbx_op_unpack: ") + cudaGetErrorString(e));
  return LBX_OK;
}

lbx_status lbx_op_conv_out(const void* x, const float* ss, const float* w, const float* b, uint8_t* rgb, int n,
                           int H, int W, int impl, lbx_stream stream) {
  if (!x || !ss || !w || !b || !rgb || n <= 0 || H <= 0 || W <= 0)
    return set_err(LBX_E_CONFIG, "lbx_op_conv_out: bad argument");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const __half* xh = reinterpret_cast<const __half*>(x);
  const float2* s2 = reinterpret_cast<const float2*>(ss);
  cudaError_t e;
  if (impl == 1) {
    lbx::launch_conv_out_u8(xh, s2, w, b, rgb, n, H, W, s);
    e = cudaGetLastError();
  } else {
    e = lbx::launch_conv_out_tc(xh, s2, w, b, rgb, n, H, W, impl == 2, s);
  }
  if (e != cudaSuccess)
    return set_err(e == cudaErrorInvalidValue ? LBX_E_CONFIG : LBX_E_CUDA,
                   std::string("lbx_op_conv_out: ") + cudaGetErrorString(e));
  return LBX_OK;
}

lbx_status lbx_op_set_debug(int halo_policy, int desc_base_mode) {
  lbx::gemm_tc_set_debug(halo_policy, desc_base_mode);
  lbx::kernels_set_conv_out_legacy((halo_policy >> 4) & 1);
  lbx::kernels_set_apply_bulk(!((halo_policy >> 8) & 1));
  lbx::kernels_set_unpack_rows((halo_policy >> 24) & 1);
  return LBX_OK;
}

void* lbx_host_alloc(size_t bytes) {
  void* p = nullptr;
  return cudaMallocHost(&p, bytes) == cudaSuccess ? p : nullptr;
}

void lbx_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

lbx_status lbx_op_set_grid_limits(int gemm_sms, int apply_sms) {
  lbx::gemm_tc_set_max_sms(gemm_sms);
  lbx::kernels_set_apply_max_sms(apply_sms);
  return LBX_OK;
}

lbx_status lbx_subpixel_weights(const float* w3, int N, int C, uint16_t* out) {
  if (!w3 || !out || N <= 0 || C <= 0) return set_err(LBX_E_CONFIG, "lbx_subpixel_weights: bad argument");
  static const int kset[2][2][2] = {{{0, -1}, {1, 2}}, {{0, 1}, {2, -1}}};
  for (int ph = 0; ph < 4; ++ph) {
    const int a = ph >> 1, bb = ph & 1;
    for (int o = 0; o < N; ++o)
      for (int t = 0; t < 4; ++t)
        for (int ci = 0; ci < C; ++ci) {
          float acc = 0.f;
          for (int u = 0; u < 2; ++u) {
            const int ky = kset[a][t >> 1][u];
            if (ky < 0) continue;
            for (int v = 0; v < 2; ++v) {
              const int kx = kset[bb][t & 1][v];
              if (kx < 0) continue;
              acc += w3[(((size_t)o * 3 + ky) * 3 + kx) * C + ci];
            }
          }
          out[(((size_t)ph * N + o) * 4 + t) * C + ci] = lbx::f32_to_f16_bits(acc);
        }
  }
  return LBX_OK;
}

lbx_status lbx_op_groupnorm(const void* x, void* y, const uint64_t* stats, const float* gamma, const float* beta, int b,
                            int hw, int c, int silu, float eps, lbx_stream stream) {
  if (!x || !y || !stats || !gamma || !beta || !(c == 128 || c == 256 || c == 512))
    return set_err(LBX_E_CONFIG, "lbx_op_groupnorm: bad argument");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const lbx::GnSrc gs{reinterpret_cast<const unsigned long long*>(stats), gamma, beta, 1.0 / ((double)hw * (c / 32)), eps};
  lbx::launch_gn_apply(reinterpret_cast<const __half*>(x), reinterpret_cast<__half*>(y), gs, (long long)b * hw, hw, c,
                       silu != 0, silu == 2, s);
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return set_err(LBX_E_CUDA, cudaGetErrorString(e));
  return LBX_OK;
}

lbx_status lbx_op_gn_stats(const void* x, uint64_t* stats, int b, int hw, int c, lbx_stream stream) {
  if (!x || !stats || c % 32 || c > 512 || b <= 0 || hw <= 0) return set_err(LBX_E_CONFIG, "lbx_op_gn_stats: bad argument");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(stats, 0, (size_t)b * 32 * lbx::kGnStatWords * 8, s) != cudaSuccess)
    return set_err(LBX_E_CUDA, "memset");
  lbx::launch_gn_stats(reinterpret_cast<const __half*>(x), reinterpret_cast<unsigned long long*>(stats), b, hw, c, s);
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return set_err(LBX_E_CUDA, cudaGetErrorString(e));
  return LBX_OK;
}

lbx_status lbx_profile(lbx_decoder* dec, uint32_t n, lbx_prof_entry* out, int cap, int* count) {
  if (!dec || !out || !count) return set_err(LBX_E_CONFIG, "lbx_profile: null argument");
  std::lock_guard<std::mutex> g(dec->mu);
  Decoder& d = dec->d;
  if (n == 0 || (int)n > d.max_batch) return set_err(LBX_E_CONFIG, "n: must be in [1, desc.max_batch]");
  cudaSetDevice(d.desc.device);
  std::vector<Decoder::ProfRec> recs;
  d.order(d.stream);
  d.prof = &recs;
  lbx_status st = d.plan((int)n, d.lat, d.rgb, d.stream, false);
  d.prof = nullptr;
  d.mark(d.stream);
  cudaError_t e = cudaStreamSynchronize(d.stream);
  int k = 0;
  for (size_t i = 1; i < recs.size(); ++i) {
    if (st == LBX_OK && e == cudaSuccess && k < cap) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, recs[i - 1].ev, recs[i].ev);
      lbx_prof_entry& o = out[k++];
      std::memset(&o, 0, sizeof o);
      std::snprintf(o.name, sizeof o.name, "%s", recs[i].name.c_str());
      o.ms = ms;
      o.flops = recs[i].flops;
      o.algo_flops = recs[i].algo_flops;
      o.bytes = recs[i].bytes;
    }
  }
  for (auto& r : recs) cudaEventDestroy(r.ev);
  *count = k;
  if (st != LBX_OK) return st;
  if (e != cudaSuccess) return set_err(LBX_E_CUDA, std::string("lbx_profile: ") + cudaGetErrorString(e));
  return LBX_OK;
}

int lbx_launch_count(lbx_decoder* dec, uint32_t n) {
  if (!dec) return -1;
  auto it = dec->d.launch_counts.find((int)n);
  return it == dec->d.launch_counts.end() ? -1 : it->second;
}

}  // extern "C"
