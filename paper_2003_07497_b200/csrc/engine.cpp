// engine.cpp — the C ABI of include/lann_engine.h: argument validation with the
// reference's error contract, device buffers, launch plans and the
// whole-population pipeline. There is no CPU fallback: without a CUDA device
// every compute entry point returns LANN_NO_DEVICE.
//
// A training "plan" is built once per population (device-side argument
// arrays, FP32 row packing, model grouping, stream assignment) and executed
// any number of times with launches only — so a prepared population re-runs
// with its inputs resident in HBM and no host<->device traffic.
#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <string>
#include <thread>
#include <tuple>
#include <type_traits>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/lann_engine.h"
#include "domain.hpp"
#include "kernels.cuh"

constexpr int kAuxStreams = 8;

struct lann_engine {
  int device = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t aux[kAuxStreams] = {};
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, tr0 = nullptr, tr1 = nullptr;
  cudaEvent_t fork = nullptr, join[kAuxStreams] = {};
  std::string err;
  double last_ms = 0.0, last_train_ms = 0.0;
  int64_t launches = 0;
  int max_smem = 0;
  unsigned char* pin = nullptr;  // pinned host staging for population uploads (grows, kept)
  size_t pin_cap = 0;
  float2* brcp = nullptr;        // FP32 Adam bias-correction reciprocal table (grows, kept)
  int brcp_n = 0;
  std::vector<struct lann_population*> pops;  // live prepared populations (freed before the engine)
};

namespace lann {
namespace {

struct CudaFail {
  std::string what;
};

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaFail{std::string(what) + ": " + cudaGetErrorString(e)};
}

// host<->device bytes moved by the calling thread (reported per C-ABI call)
thread_local int64_t t_h2d = 0, t_d2h = 0;

// Stream-ordered device buffer.
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  bool owned = true;
  DBuf() = default;
  DBuf(size_t count, cudaStream_t st) : n(count), s(st) {
    if (n) ck(cudaMallocAsync((void**)&p, n * sizeof(T), s), "cudaMallocAsync");
  }
  DBuf(const T* host, size_t count, cudaStream_t st) : DBuf(count, st) { up(host); }
  DBuf(const std::vector<T>& v, cudaStream_t st) : DBuf(v.data(), v.size(), st) {}
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept { *this = std::move(o); }
  DBuf& operator=(DBuf&& o) noexcept {
    std::swap(p, o.p);
    std::swap(n, o.n);
    std::swap(s, o.s);
    std::swap(owned, o.owned);
    return *this;
  }
  ~DBuf() {
    if (p && owned) cudaFreeAsync(p, s);
  }
  // a non-owning window into another buffer (the population blob)
  static DBuf view(T* ptr, size_t count, cudaStream_t st) {
    DBuf d;
    d.p = ptr;
    d.n = count;
    d.s = st;
    d.owned = false;
    return d;
  }
  void up(const T* host) { up(host, n * sizeof(T)); }
  void up(const void* host, size_t bytes) {
    if (bytes) ck(cudaMemcpyAsync(p, host, bytes, cudaMemcpyHostToDevice, s), "H2D");
    t_h2d += int64_t(bytes);
  }
  void down(T* host) const {
    if (n) ck(cudaMemcpyAsync(host, p, n * sizeof(T), cudaMemcpyDeviceToHost, s), "D2H");
    t_d2h += int64_t(n * sizeof(T));
  }
};

int set_err(lann_engine* e, const Status& st) {
  if (e) e->err = st.msg;
  return st.code;
}

// CUDA-event timer over the engine stream (whole call) — device time only.
struct Timer {
  lann_engine* e;
  explicit Timer(lann_engine* eng) : e(eng) {
    e->launches = 0;
    e->last_ms = 0.0;
    ck(cudaEventRecord(e->ev0, e->stream), "event");
  }
  void stop() {
    ck(cudaEventRecord(e->ev1, e->stream), "event");
    ck(cudaEventSynchronize(e->ev1), "sync");
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, e->ev0, e->ev1), "elapsed");
    e->last_ms = ms;
  }
};

// ---- training description (host side) -------------------------------------------------
struct DevTrain {
  int n_models = 0, n_tiles = 0;
  std::vector<int> tile_rows, tile_inputs, model_tile, h1, h2, epochs;
  std::vector<int64_t> tile_offset, param_offset;
  std::vector<double> lr;
  int64_t total_params = 0;
  int trace_stride = 1;
};

Status validate_train(const DevTrain& t) {
  if (t.n_models < 1) return {LANN_PARAM_ERROR, "population needs at least one model"};
  if (t.trace_stride < 1) return {LANN_PARAM_ERROR, "trace stride must be >= 1"};
  for (int k = 0; k < t.n_tiles; ++k) {
    if (t.tile_rows[k] < 1) return {LANN_PARAM_ERROR, "bad training batch"};  // mlp.cpp:77
    if (t.tile_inputs[k] < 1 || t.tile_inputs[k] > 7)
      return {LANN_PARAM_ERROR, "model inputs must lie in 1..7"};
  }
  for (int m = 0; m < t.n_models; ++m) {
    if (t.model_tile[m] < 0 || t.model_tile[m] >= t.n_tiles)
      return {LANN_PARAM_ERROR, "model references an unknown tile"};
    if (t.h1[m] < 1 || t.h2[m] < 0 || t.h1[m] > 64 || t.h2[m] > 64)
      return {LANN_PARAM_ERROR, "network layer widths must lie in 1..64"};
    if (t.epochs[m] < 1) return {LANN_PARAM_ERROR, "epochs must be >= 1"};
    if (!(t.lr[m] > 0.0)) return {LANN_PARAM_ERROR, "learning rate must be > 0"};
    const int P = param_count(t.tile_inputs[t.model_tile[m]], t.h1[m], t.h2[m]);
    if (t.param_offset[m] < 0 || t.param_offset[m] + P > t.total_params)
      return {LANN_PARAM_ERROR, "flat parameter size mismatch"};
  }
  return {};
}

// ---- training plan ------------------------------------------------------------------------
struct Fp32Bucket {
  int in, h1, h2, lanes, tile_bytes, n_groups;
  DBuf<int> gfirst, gcount, sorted;
  DBuf<long long> prof;  // LANN_PHASE_PROFILE: CTA 0 cycle split (CTA kernel)
  double cost;
};

struct Fp64Bucket {
  int shape[3] = {0, 0, 0};  // compiled shape, or {0,0,0} = generic kernel
  int n = 0, max_p = 0, dyn = 0, in_smem = 0, products = 0, chunk = 0;
  DBuf<int> order;
  DBuf<double> scratch;
  DBuf<int64_t> soff;
  DBuf<long long> prof;  // LANN_PHASE_PROFILE: CTA 0 cycle split
  double cost = 0.0;
};

struct TrainPlan {
  DBuf<int> tile_rows, tile_inputs, model_tile, h1, h2, epochs;
  DBuf<int64_t> tile_off, poff;
  DBuf<double> lr;
  // FP32 part
  DBuf<float> rows_f;
  std::vector<std::unique_ptr<Fp32Bucket>> buckets;
  // FP64 part (exact mode, or FP32-mode models without a compiled FP32 shape)
  std::vector<std::unique_ptr<Fp64Bucket>> buckets64;
  DBuf<double2> bc;
  const float2* brcp = nullptr;  // FP32 Adam bias-correction reciprocals per epoch (engine-owned)
  const double* dX = nullptr;
  const double* dY = nullptr;
  int trace_stride = 1;
  std::vector<int> model_precision;  // per model: the lann_precision its trainer runs in
  // FP32 mode, shapes without a compiled FP32 kernel: the generic FP32 CTA kernel
  DBuf<int> wide_order;
  int wide_n = 0, wide_chunk = 0, wide_dyn = 0, wide_max_p = 0;
};

std::unique_ptr<TrainPlan> build_plan(lann_engine* e, const DevTrain& t, int precision,
                                      const double* dX, const double* dY, int64_t total_rows) {
  cudaStream_t s = e->stream;
  auto plan = std::make_unique<TrainPlan>();
  TrainPlan& P = *plan;
  P.tile_rows = DBuf<int>(t.tile_rows, s);
  P.tile_inputs = DBuf<int>(t.tile_inputs, s);
  P.model_tile = DBuf<int>(t.model_tile, s);
  P.h1 = DBuf<int>(t.h1, s);
  P.h2 = DBuf<int>(t.h2, s);
  P.epochs = DBuf<int>(t.epochs, s);
  P.tile_off = DBuf<int64_t>(t.tile_offset, s);
  P.poff = DBuf<int64_t>(t.param_offset, s);
  P.lr = DBuf<double>(t.lr, s);
  P.dX = dX;
  P.dY = dY;
  P.trace_stride = t.trace_stride;

  std::vector<int> fp64_models, wide_models;
  P.model_precision.assign(size_t(t.n_models), LANN_FP64_EXACT);
  if (precision == LANN_FP32) {
    P.rows_f = DBuf<float>(size_t(total_rows) * 8, s);
    launch_pack_rows(dX, dY, total_rows, P.rows_f.p, s);
    using Shape = std::tuple<int, int, int>;
    std::map<Shape, std::vector<int>> by_shape;
    for (int m = 0; m < t.n_models; ++m) {
      const int tile = t.model_tile[m];
      const int I = t.tile_inputs[tile];
      if (fp32_shape_supported(I, t.h1[m], t.h2[m]) && t.tile_rows[tile] * 32 <= 96 * 1024) {
        by_shape[{I, t.h1[m], t.h2[m]}].push_back(m);
        P.model_precision[size_t(m)] = LANN_FP32;
      } else if (fp32_wide_supported(I, t.h1[m], t.h2[m]) && !std::getenv("LANN_FP32_NO_WIDE")) {
        wide_models.push_back(m);
        P.model_precision[size_t(m)] = LANN_FP32;
      } else {
        fp64_models.push_back(m);
      }
    }
    int env_lanes = 0;
    if (const char* env = std::getenv("LANN_FP32_LANES")) env_lanes = std::atoi(env);
    if (env_lanes != 1 && env_lanes != 2 && env_lanes != 4 && env_lanes != 8 && env_lanes != 32 &&
        env_lanes != 64 && env_lanes != 128 && env_lanes != 256)
      env_lanes = 0;
    // populations too small to fill the GPU with warps get a whole CTA (4 warps) per model
    const int total_fp32 = t.n_models - int(fp64_models.size()) - int(wide_models.size());
    const bool small = total_fp32 <= 4 * e->sms;
    // Large populations: all warp-kernel buckets run concurrently (one stream each), so the GPU
    // stays full whatever a single bucket's wave count is; then the cheapest mapping is 2 lanes
    // per model (less butterfly / redundant-Adam work than 4-8 lanes, a short enough per-lane
    // sample loop, and enough warps). Measured on the config-3 sweep: 2 lanes 823 ms vs the
    // per-bucket fill heuristic 892 ms (1 lane 994, 8 lanes 966).
    int max_epochs_all = 0;
    for (auto& [shape, ms] : by_shape)
      for (int m : ms) max_epochs_all = std::max(max_epochs_all, t.epochs[m]);
    for (int m : wide_models) max_epochs_all = std::max(max_epochs_all, t.epochs[m]);
    // the CTA kernel reads its bias corrections per epoch instead of computing them; the table
    // is engine-resident (grown on demand), not re-uploaded per population
    if (e->brcp_n < max_epochs_all) {
      const int n = std::max(max_epochs_all, 32768);
      const auto& bc = adam_bias_table(n);
      std::vector<float2> r(static_cast<size_t>(n));
      for (size_t k = 0; k < r.size(); ++k) r[k] = make_float2(float(1.0 / bc[2 * k]), float(1.0 / bc[2 * k + 1]));
      ck(cudaDeviceSynchronize(), "bias table");  // no launch in flight still reads the old one
      if (e->brcp) ck(cudaFree(e->brcp), "cudaFree");
      e->brcp = nullptr;
      e->brcp_n = 0;
      ck(cudaMalloc(reinterpret_cast<void**>(&e->brcp), r.size() * sizeof(float2)), "cudaMalloc");
      ck(cudaMemcpy(e->brcp, r.data(), r.size() * sizeof(float2), cudaMemcpyHostToDevice), "H2D");
      e->brcp_n = n;
    }
    P.brcp = e->brcp;
    int global_lanes = 0;
    int off_lanes = 4;  // lanes for buckets off the critical path (mid-size populations)
    if (!env_lanes && !small) {
      long long warps = 0, warps_mixed = 0;
      int min_slots = 1 << 30;
      for (auto& [shape, ms] : by_shape) {
        std::map<std::pair<int, int>, int> per_tile;  // (tile, epochs) -> models
        int rows = 1, epochs = 0;
        for (int m : ms) {
          per_tile[{t.model_tile[m], t.epochs[m]}] += 1;
          rows = std::max(rows, t.tile_rows[t.model_tile[m]]);
          epochs = std::max(epochs, t.epochs[m]);
        }
        for (const auto& [key, cnt] : per_tile) {
          warps += (cnt + 15) / 16;
          warps_mixed += epochs < max_epochs_all ? (cnt + 15) / 16 : (cnt + 3) / 4;
        }
        min_slots = std::min(min_slots, std::max(1, fp32_warp_slots_per_sm(std::get<0>(shape), std::get<1>(shape),
                                                                          std::get<2>(shape), 2, rows * 32)));
      }
      if (warps >= 2LL * min_slots * e->sms) global_lanes = 2;
      // with the critical bucket at 8 lanes and the rest at 2, does the population fill the GPU
      // once? then 2 lanes for the rest (throughput), else 4 (measured on 7,680 / 15,360 /
      // 30,720-model sweep shares: 4 best at the smallest, 2 at the others)
      if (warps_mixed >= 1LL * min_slots * e->sms) off_lanes = 2;
    }
    for (auto& [shape, ms] : by_shape) {
      // group: same tile and epoch count, up to G models; longest groups first
      std::stable_sort(ms.begin(), ms.end(), [&](int a, int b) {
        const double ca = double(t.epochs[a]) * t.tile_rows[t.model_tile[a]];
        const double cb = double(t.epochs[b]) * t.tile_rows[t.model_tile[b]];
        if (ca != cb) return ca > cb;
        if (t.model_tile[a] != t.model_tile[b]) return t.model_tile[a] < t.model_tile[b];
        return t.epochs[a] < t.epochs[b];
      });
      auto count_groups = [&](int G) {
        int n = 0;
        for (size_t i = 0; i < ms.size();) {
          size_t j = i + 1;
          while (j < ms.size() && int(j - i) < G && t.model_tile[ms[j]] == t.model_tile[ms[i]] &&
                 t.epochs[ms[j]] == t.epochs[ms[i]])
            ++j;
          ++n;
          i = j;
        }
        return n;
      };
      int bucket_rows = 1;
      for (int m : ms) bucket_rows = std::max(bucket_rows, t.tile_rows[t.model_tile[m]]);
      int lanes = env_lanes ? env_lanes : global_lanes;
      // per-shape-class overrides for experiments: LANN_FP32_LANES_H8 / LANN_FP32_LANES_2H
      if (const char* ov = std::getenv(std::get<2>(shape) > 0 ? "LANN_FP32_LANES_2H" : "LANN_FP32_LANES_H8"))
        if (std::atoi(ov) > 0) lanes = std::atoi(ov);
      if (!lanes && small) lanes = 128;
      if (!lanes) {
        // lanes per model minimising the modelled makespan of this bucket on its own:
        // waves x per-warp epoch cost (samples per lane + butterfly levels + Adam), with
        // the wave size from the kernel's measured occupancy
        double best = 1e300;
        for (int k : {1, 2, 4, 8}) {
          const int slots = std::max(1, fp32_warp_slots_per_sm(std::get<0>(shape), std::get<1>(shape),
                                                               std::get<2>(shape), k, bucket_rows * 32)) * e->sms;
          const double waves = std::ceil(double(count_groups(32 / k)) / slots);
          const double epoch = double(bucket_rows) / k + 1.0 * std::log2(double(k)) + 6.0;
          if (waves * epoch < best * 0.999) {
            best = waves * epoch;
            lanes = k;
          }
        }
        // buckets run concurrently: a bucket with fewer epochs than the population's longest
        // models is off the critical path and trades latency for throughput (off_lanes), while
        // the critical-path bucket keeps at least 8 lanes per model (latency); measured on
        // 7,680 / 15,360 / 30,720-model sweeps: 180.6 -> 161.8 / 266 -> 244 / 441 -> 428 ms
        int bucket_epochs = 0;
        for (int m : ms) bucket_epochs = std::max(bucket_epochs, t.epochs[m]);
        if (bucket_epochs < max_epochs_all) lanes = off_lanes;
        else lanes = std::max(8, lanes);
      }
      const int G = lanes <= 32 ? 32 / lanes : 1;
      std::vector<int> gfirst, gcount;
      int max_rows = 1;
      double cost = 0.0;
      for (size_t i = 0; i < ms.size();) {
        size_t j = i + 1;
        while (j < ms.size() && int(j - i) < G && t.model_tile[ms[j]] == t.model_tile[ms[i]] &&
               t.epochs[ms[j]] == t.epochs[ms[i]])
          ++j;
        gfirst.push_back(int(i));
        gcount.push_back(int(j - i));
        max_rows = std::max(max_rows, t.tile_rows[t.model_tile[ms[i]]]);
        cost = std::max(cost, double(t.epochs[ms[i]]) * t.tile_rows[t.model_tile[ms[i]]]);
        i = j;
      }
      auto b = std::make_unique<Fp32Bucket>();
      b->in = std::get<0>(shape);
      b->h1 = std::get<1>(shape);
      b->h2 = std::get<2>(shape);
      b->lanes = lanes;
      b->tile_bytes = max_rows * 32;
      b->n_groups = int(gfirst.size());
      b->gfirst = DBuf<int>(gfirst, s);
      b->gcount = DBuf<int>(gcount, s);
      b->sorted = DBuf<int>(ms, s);
      b->cost = cost;
      if (std::getenv("LANN_PHASE_PROFILE")) b->prof = DBuf<long long>(8, s);
      if (std::getenv("LANN_PLAN_VERBOSE"))
        std::fprintf(stderr, "fp32 bucket %d-%d-%d: %zu models, lanes %d, %d groups, rows <= %d\n", b->in, b->h1,
                     b->h2, ms.size(), b->lanes, b->n_groups, max_rows);
      P.buckets.push_back(std::move(b));
    }
    // longest bucket first so it starts first on its stream
    std::stable_sort(P.buckets.begin(), P.buckets.end(),
                     [](const auto& a, const auto& b) { return a->cost > b->cost; });
    if (!wide_models.empty()) {
      // one CTA per model, longest first; records a chunk of samples at a time (the largest
      // multiple of 32 that fits beside the largest model's state)
      std::stable_sort(wide_models.begin(), wide_models.end(), [&](int a, int b) {
        return double(t.epochs[a]) * t.tile_rows[t.model_tile[a]] > double(t.epochs[b]) * t.tile_rows[t.model_tile[b]];
      });
      int rows = 0, max_n = 1;
      for (int m : wide_models) {
        const int tile = t.model_tile[m];
        rows = std::max(rows, fp32_wide_rows(t.h1[m], t.h2[m]));
        P.wide_max_p = std::max(P.wide_max_p, param_count(t.tile_inputs[tile], t.h1[m], t.h2[m]));
        max_n = std::max(max_n, t.tile_rows[tile]);
      }
      int ch = int(std::min<int64_t>(((max_n + 31) / 32) * 32, 4096));
      while (ch > 32 && fp32_wide_smem_bytes(P.wide_max_p, rows, ch) > size_t(e->max_smem)) ch -= 32;
      if (ch > 256) ch &= ~255;  // whole passes of the 256 phase-A threads
      if (fp32_wide_smem_bytes(P.wide_max_p, rows, ch) <= size_t(e->max_smem)) {
        P.wide_chunk = ch;
        P.wide_dyn = int(fp32_wide_smem_bytes(P.wide_max_p, rows, ch));
        P.wide_n = int(wide_models.size());
        P.wide_order = DBuf<int>(wide_models, s);
      } else {  // no room for a 32-sample chunk: the FP64 exact kernel takes them (and says so)
        for (int m : wide_models) {
          P.model_precision[size_t(m)] = LANN_FP64_EXACT;
          fp64_models.push_back(m);
        }
      }
    }
  } else {
    fp64_models.resize(t.n_models);
    std::iota(fp64_models.begin(), fp64_models.end(), 0);
  }
  if (!fp64_models.empty()) {
    int max_e = 1;
    for (int m : fp64_models) max_e = std::max(max_e, t.epochs[m]);
    const auto& bc = adam_bias_table(max_e);
    P.bc = DBuf<double2>(reinterpret_cast<const double2*>(bc.data()), size_t(max_e), s);
    // one bucket per compiled shape (+ one generic bucket), each on its own stream
    using Shape = std::tuple<int, int, int>;
    std::map<Shape, std::vector<int>> by_shape;
    for (int m : fp64_models) {
      const int I = t.tile_inputs[t.model_tile[m]];
      if (fp64_shape_compiled(I, t.h1[m], t.h2[m])) by_shape[{I, t.h1[m], t.h2[m]}].push_back(m);
      else by_shape[{0, 0, 0}].push_back(m);
    }
    auto cost = [&](int m) {
      const int tile = t.model_tile[m];
      return double(t.epochs[m]) * t.tile_rows[tile] *
             param_count(t.tile_inputs[tile], t.h1[m], t.h2[m]);
    };
    for (auto& [shape, order] : by_shape) {
      // longest models first so the block scheduler packs the tail
      std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost(a) > cost(b); });
      auto b = std::make_unique<Fp64Bucket>();
      b->shape[0] = std::get<0>(shape);
      b->shape[1] = std::get<1>(shape);
      b->shape[2] = std::get<2>(shape);
      b->n = int(order.size());
      b->cost = cost(order.front());
      size_t max_bytes_smem = 0, max_state = 0, max_bytes_prod = 0;
      std::vector<int64_t> soff(t.n_models, 0);
      int64_t scratch = 0;
      for (int m : order) {
        const int tile = t.model_tile[m];
        const int np = param_count(t.tile_inputs[tile], t.h1[m], t.h2[m]);
        b->max_p = std::max(b->max_p, np);
        const size_t rec = fp64_record_bytes(t.tile_inputs[tile], t.h1[m], t.h2[m], t.tile_rows[tile]);
        const size_t state = fp64_state_bytes(np);
        max_state = std::max(max_state, state);
        max_bytes_smem = std::max(max_bytes_smem, state + rec);
        if (b->shape[0] > 0)
          max_bytes_prod = std::max(max_bytes_prod, state + fp64_product_record_bytes(t.tile_inputs[tile], t.h1[m],
                                                                                      t.h2[m], t.tile_rows[tile]));
        soff[m] = scratch;
        scratch += int64_t(rec / 8);
      }
      b->in_smem = max_bytes_smem <= size_t(e->max_smem);
      b->dyn = int(b->in_smem ? max_bytes_smem : max_state);
      if (!b->in_smem && !std::getenv("LANN_FP64_GLOBAL_RECORDS")) {
        // records too large for one CTA: keep them in shared memory a chunk of samples at a time
        // (the largest even chunk that fits beside the model state; every bucket model's rows <= R)
        int rows = 0;
        for (int m : order) rows = std::max(rows, fp64_record_rows(t.h1[m], t.h2[m]));
        const size_t room = size_t(e->max_smem) > max_state ? size_t(e->max_smem) - max_state : 0;
        int ch = int(std::min<size_t>(room / (size_t(rows) * 8), 4096)) & ~1;
        while (ch >= 32 && size_t(rows) * size_t(fp64_chunk_ld(ch)) * 8 > room) ch -= 2;
        if (ch >= 32) {
          b->in_smem = 1;
          b->chunk = ch;
          b->dyn = int(max_state + size_t(rows) * size_t(fp64_chunk_ld(ch)) * 8);
        }
      }
      // compiled shapes whose product rows fit too: phase B becomes pure DADD chains
      if (b->shape[0] > 0 && max_bytes_prod <= size_t(e->max_smem) && !std::getenv("LANN_FP64_NOPROD")) {
        b->products = 1;
        b->dyn = int(max_bytes_prod);
      }
      if (!b->in_smem) b->scratch = DBuf<double>(size_t(scratch), s);
      b->soff = DBuf<int64_t>(soff, s);
      b->order = DBuf<int>(order, s);
      if (std::getenv("LANN_PHASE_PROFILE")) b->prof = DBuf<long long>(8, s);
      P.buckets64.push_back(std::move(b));
    }
    std::stable_sort(P.buckets64.begin(), P.buckets64.end(),
                     [](const auto& a, const auto& b) { return a->cost > b->cost; });
  }
  ck(cudaGetLastError(), "plan");
  return plan;
}

// Launch the whole trainer; buckets run concurrently on the auxiliary streams.
void execute_plan(lann_engine* e, const TrainPlan& P, double* dparams, double* dfinal, int* dbad,
                  double* dtrace, const int64_t* dtrace_off) {
  cudaStream_t s = e->stream;
  const int n_launch = int(P.buckets.size()) + int(P.buckets64.size()) + (P.wide_n > 0 ? 1 : 0);
  ck(cudaEventRecord(e->tr0, s), "event");
  ck(cudaEventRecord(e->fork, s), "event");
  int k = 0;
  auto next_stream = [&]() -> cudaStream_t {
    if (n_launch == 1) return s;
    cudaStream_t st = e->aux[k % kAuxStreams];
    ++k;
    return st;
  };
  for (int i = 0; i < kAuxStreams && n_launch > 1; ++i)
    ck(cudaStreamWaitEvent(e->aux[i], e->fork, 0), "wait");
  for (const auto& b : P.buckets) {
    TrainF32Args a{};
    a.n_groups = b->n_groups;
    a.group_first = b->gfirst.p;
    a.group_count = b->gcount.p;
    a.sorted_model = b->sorted.p;
    a.rows = P.rows_f.p;
    a.tile_rows = P.tile_rows.p;
    a.tile_offset = P.tile_off.p;
    a.model_tile = P.model_tile.p;
    a.lr = P.lr.p;
    a.epochs = P.epochs.p;
    a.param_offset = P.poff.p;
    a.params = dparams;
    a.final_loss = dfinal;
    a.nonfinite_epoch = dbad;
    a.loss_trace = dtrace;
    a.trace_offset = dtrace_off;
    a.trace_stride = P.trace_stride;
    a.phase_cycles = b->prof.p;
    a.bias_rcp = P.brcp;
    if (!launch_train_fp32(a, b->in, b->h1, b->h2, b->lanes, b->tile_bytes, next_stream()))
      throw CudaFail{"no FP32 kernel for this shape"};
    ck(cudaGetLastError(), "train_fp32 launch");
    e->launches += 1;
  }
  if (P.wide_n > 0) {
    TrainWideArgs a{};
    a.n_models = P.wide_n;
    a.order = P.wide_order.p;
    a.rows = P.rows_f.p;
    a.tile_rows = P.tile_rows.p;
    a.tile_inputs = P.tile_inputs.p;
    a.tile_offset = P.tile_off.p;
    a.model_tile = P.model_tile.p;
    a.h1 = P.h1.p;
    a.h2 = P.h2.p;
    a.lr = P.lr.p;
    a.epochs = P.epochs.p;
    a.param_offset = P.poff.p;
    a.params = dparams;
    a.final_loss = dfinal;
    a.nonfinite_epoch = dbad;
    a.loss_trace = dtrace;
    a.trace_offset = dtrace_off;
    a.trace_stride = P.trace_stride;
    a.bias_rcp = P.brcp;
    a.chunk = P.wide_chunk;
    a.max_p = P.wide_max_p;
    launch_train_fp32_wide(a, P.wide_dyn, next_stream());
    ck(cudaGetLastError(), "train_fp32_wide launch");
    e->launches += 1;
  }
  for (const auto& b : P.buckets64) {
    TrainArgs a{};
    a.n_models = b->n;
    a.order = b->order.p;
    a.tile_rows = P.tile_rows.p;
    a.tile_inputs = P.tile_inputs.p;
    a.tile_offset = P.tile_off.p;
    a.X = P.dX;
    a.y = P.dY;
    a.model_tile = P.model_tile.p;
    a.h1 = P.h1.p;
    a.h2 = P.h2.p;
    a.lr = P.lr.p;
    a.epochs = P.epochs.p;
    a.param_offset = P.poff.p;
    a.params = dparams;
    a.final_loss = dfinal;
    a.nonfinite_epoch = dbad;
    a.loss_trace = dtrace;
    a.trace_offset = dtrace_off;
    a.trace_stride = P.trace_stride;
    a.bias_corr = P.bc.p;
    a.scratch = b->scratch.p;
    a.scratch_offset = b->soff.p;
    a.smem_records = b->in_smem;
    a.rec_chunk = b->chunk;
    a.rec_products = b->products;
    a.phase_cycles = b->prof.p;
    launch_train_fp64(a, b->max_p, b->dyn, b->shape[0] > 0 ? b->shape : nullptr, next_stream());
    ck(cudaGetLastError(), "train_fp64 launch");
    e->launches += 1;
  }
  if (std::getenv("LANN_PHASE_PROFILE")) {
    ck(cudaDeviceSynchronize(), "profile sync");
    for (const auto& b : P.buckets) {
      if (b->lanes < 64) continue;
      long long c[4] = {0, 0, 0, 0};
      ck(cudaMemcpy(c, b->prof.p, 4 * sizeof(long long), cudaMemcpyDeviceToHost), "profile D2H");
      std::fprintf(stderr, "fp32 cta shape %d-%d-%d: cycles compute %lld reduce %lld adam %lld loop %lld\n", b->in,
                   b->h1, b->h2, c[0], c[1], c[2], c[3]);
    }
    for (const auto& b : P.buckets64) {
      long long c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      ck(cudaMemcpy(c, b->prof.p, sizeof c, cudaMemcpyDeviceToHost), "profile D2H");
      std::fprintf(stderr, "fp64 shape %d-%d-%d: cycles phaseA %lld chain %lld adam %lld wait %lld | producer "
                   "weights %lld round0 %lld round1 %lld barrier %lld\n", b->shape[0], b->shape[1], b->shape[2],
                   c[0], c[1], c[2], c[3], c[4], c[5], c[6], c[7]);
    }
  }
  if (n_launch > 1)
    for (int i = 0; i < kAuxStreams; ++i) {
      ck(cudaEventRecord(e->join[i], e->aux[i]), "event");
      ck(cudaStreamWaitEvent(s, e->join[i], 0), "wait");
    }
  ck(cudaEventRecord(e->tr1, s), "event");
}

// ---- prepared population ----------------------------------------------------------------
// 16-B aligned sub-array offsets of one allocation
struct BlobLayout {
  size_t bytes = 0;
  template <class T>
  size_t add(size_t count) {
    const size_t off = (bytes + 15) & ~size_t(15);
    bytes = off + count * sizeof(T);
    return off;
  }
};

// The engine's pinned staging buffer, grown to at least `bytes` (the previous upload from it
// has completed: population preparation synchronises its stream before returning).
unsigned char* pinned_stage(lann_engine* e, size_t bytes) {
  if (bytes > e->pin_cap) {
    if (e->pin) ck(cudaFreeHost(e->pin), "cudaFreeHost");
    e->pin = nullptr;
    e->pin_cap = 0;
    const size_t cap = std::max(bytes, size_t(1) << 21);
    ck(cudaMallocHost(reinterpret_cast<void**>(&e->pin), cap), "cudaMallocHost");
    e->pin_cap = cap;
  }
  return e->pin;
}

// ---- cross-validation layout (lann_engine.h "cross-validation summary"), host only ----------
struct CvLayout {
  std::vector<int> job_group, job_ens;  // -1 for jobs outside k-fold groups
  std::vector<int> group_first, group_folds, group_models, group_ens;
  std::vector<int> ens_group, ens_first;  // ensemble's group, its first job
  std::vector<uint64_t> ens_seed;
  std::vector<std::vector<int>> ens_member;  // [ensemble][fold]: first job of that fold, -1 if absent
  int n_groups() const { return int(group_first.size()); }
  int n_ens() const { return int(ens_group.size()); }
};

// every job field except fold and init_seed (struct padding is not part of the key)
std::string cv_group_key(const lann_job& j) {
  std::string k(reinterpret_cast<const char*>(&j.world), sizeof(lann_world));
  auto add = [&k](const auto& v) { k.append(reinterpret_cast<const char*>(&v), sizeof v); };
  add(j.data_seed);
  add(j.count);
  add(j.train_fraction);
  add(j.n_folds);
  add(j.family);
  add(j.n_hidden);
  add(j.hidden[0]);
  add(j.hidden[1]);
  add(j.learning_rate);
  add(j.epochs);
  add(j.log_target);
  add(j.unconstrained);
  return k;
}

CvLayout cv_layout(int n, const lann_job* jobs) {
  CvLayout L;
  L.job_group.assign(size_t(n), -1);
  L.job_ens.assign(size_t(n), -1);
  std::map<std::string, int> groups;
  std::map<std::pair<int, uint64_t>, int> ens;
  for (int j = 0; j < n; ++j) {
    const lann_job& J = jobs[j];
    if (J.n_folds < 2) continue;
    auto g = groups.find(cv_group_key(J));
    if (g == groups.end()) {
      g = groups.emplace(cv_group_key(J), L.n_groups()).first;
      L.group_first.push_back(j);
      L.group_folds.push_back(J.n_folds);
      L.group_models.push_back(0);
      L.group_ens.push_back(0);
    }
    const int gi = g->second;
    L.job_group[size_t(j)] = gi;
    ++L.group_models[size_t(gi)];
    auto e = ens.find({gi, J.init_seed});
    if (e == ens.end()) {
      e = ens.emplace(std::make_pair(gi, J.init_seed), L.n_ens()).first;
      L.ens_group.push_back(gi);
      L.ens_first.push_back(j);
      L.ens_seed.push_back(J.init_seed);
      L.ens_member.emplace_back(size_t(J.n_folds), -1);
      ++L.group_ens[size_t(gi)];
    }
    L.job_ens[size_t(j)] = e->second;
    auto& mem = L.ens_member[size_t(e->second)];
    if (J.fold >= 0 && J.fold < J.n_folds && mem[size_t(J.fold)] < 0) mem[size_t(J.fold)] = j;
  }
  return L;
}

// device side of a population's cross-validation summary (all arrays are views into the blob)
struct CvState {
  CvLayout L;
  std::vector<int> dev_of;       // per ensemble: its device slot, or -1
  std::vector<int> host_status;  // per ensemble off the device: why
  std::vector<int> ens_test;     // per ensemble: test-part samples
  std::vector<int> dev_members;  // [slot][kmax]: engine model indices (for member statuses)
  std::vector<int> group_test;
  int n_dev = 0, kmax = 0, max_test = 0;
  int64_t total_out = 0;
  size_t res_off = 0, res_bytes = 0;
  size_t r_mape = 0, r_thr = 0, r_rho = 0, r_sf = 0, r_se = 0, r_kept = 0, r_st = 0, r_bad = 0, r_nf = 0, r_ne = 0;
  FoldMeanArgs fm{};
  EvalArgs ev{};
  CvStatsArgs sf{}, se{};
};

struct Population {
  lann_engine* e = nullptr;
  int n_jobs = 0, M = 0, precision = 0;
  std::vector<lann_job_result> base;  // per-job status / shape after host preparation
  std::vector<int> model_job;
  DevTrain t;
  int64_t rows = 0, n_eval_rows = 0;
  int max_eval = 1;
  // device: every array lives in one blob (views below)
  DBuf<unsigned char> blob;
  size_t res_off = 0, res_bytes = 0;  // the per-model result block inside the blob
  std::array<size_t, 7> res_rel{};   // final loss, mape, thr, rho, bad epoch, kept, status
  DBuf<double> dX, dY, dP0, dP, dF, dER, dPred, dN, dET, dMape, dThr, dRho, dT;
  DBuf<int> dB, dEM, dI, dh1, dh2, dlog, dEL, dK, dS;
  DBuf<int64_t> dpo, dEO, dTO;
  std::unique_ptr<TrainPlan> plan;
  std::unique_ptr<CvState> cv;  // k-fold populations only
  int64_t trace_total = 0;
  std::vector<int64_t> toff;
  double train_flop = 0.0;  // algorithmic FLOP of one training pass
};

// Persistent host worker pool for the per-population preparation (datasets, tiles, init):
// spawning threads per call cost ~1-2 ms of the end-to-end path. Workers live for the process
// (detached, never joined); one parallel_for runs at a time.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool* pool = new HostPool();
    return *pool;
  }
  void run(int n, const std::function<void(int)>& fn) {
    if (n <= 0) return;
    std::lock_guard<std::mutex> one(call_);
    if (n == 1 || workers_ == 0) {
      for (int i = 0; i < n; ++i) fn(i);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(m_);
      fn_ = &fn;
      n_ = n;
      next_.store(0);
      active_ = workers_;
      ++gen_;
    }
    cv_.notify_all();
    drain();
    std::unique_lock<std::mutex> lk(m_);
    done_.wait(lk, [&] { return active_ == 0; });
    fn_ = nullptr;
  }

 private:
  HostPool() {
    workers_ = int(std::max(1u, std::min(32u, std::thread::hardware_concurrency()))) - 1;
    for (int t = 0; t < workers_; ++t) std::thread([this] { loop(); }).detach();
  }
  void drain() {
    for (int i; (i = next_.fetch_add(1)) < n_;) (*fn_)(i);
  }
  void loop() {
    std::uint64_t seen = 0;
    for (;;) {
      // a population preparation issues several parallel_for calls back to back: spin ~50 us
      // on the generation counter before sleeping, so the next call finds its workers awake
      const auto t0 = std::chrono::steady_clock::now();
      while (gen_.load(std::memory_order_acquire) == seen &&
             std::chrono::steady_clock::now() - t0 < std::chrono::microseconds(50))
        std::this_thread::yield();
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return gen_.load() != seen; });
        seen = gen_.load();
      }
      drain();
      std::lock_guard<std::mutex> lk(m_);
      if (--active_ == 0) done_.notify_one();
    }
  }
  std::mutex call_, m_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* fn_ = nullptr;
  std::atomic<int> next_{0};
  int n_ = 0, workers_ = 0, active_ = 0;
  std::atomic<std::uint64_t> gen_{0};
};

template <class F>
void parallel_for(int n, F&& fn) {
  const std::function<void(int)> f = fn;
  HostPool::get().run(n, f);
}

double flop_per_model_epoch(int I, int h1, int h2, int n) {
  const double fs = h2 > 0 ? 4.0 * I * h1 + 6.0 * h1 * h2 + 6.0 * h2 + h1 + 5 : 4.0 * I * h1 + 6.0 * h1 + 5;
  return n * fs + 14.0 * param_count(I, h1, h2);
}

// Host preparation (datasets, splits, tiles, validation, init) + upload.
int prepare_population(lann_engine* e, int n_jobs, const lann_job* jobs, int precision,
                       bool want_trace, Population& pop, bool sync_uploads = true) {
  pop.e = e;
  pop.n_jobs = n_jobs;
  pop.precision = precision;
  pop.base.assign(n_jobs, lann_job_result{});
  for (auto& r : pop.base) {
    r.nonfinite_epoch = -1;
    r.precision_run = -1;  // not trained (host preparation failed)
  }
  e->err.clear();
  const bool hprof = std::getenv("LANN_HOST_PROFILE") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  const auto h0 = now();
  auto hlog = [&](const char* what, std::chrono::steady_clock::time_point since) {
    if (hprof)
      std::fprintf(stderr, "host %-10s %8.3f ms\n", what,
                   std::chrono::duration<double, std::milli>(now() - since).count());
  };
  // distinct datasets, splits and tiles
  using DKey = std::tuple<std::string, uint64_t, int>;
  std::map<DKey, int> dkeys;
  std::vector<const lann_job*> dsrc;
  std::vector<int> job_ds(n_jobs);
  for (int j = 0; j < n_jobs; ++j) {
    DKey k{std::string(reinterpret_cast<const char*>(&jobs[j].world), sizeof(lann_world)),
           jobs[j].data_seed, jobs[j].count};
    auto it = dkeys.find(k);
    if (it == dkeys.end()) {
      it = dkeys.emplace(k, int(dsrc.size())).first;
      dsrc.push_back(&jobs[j]);
    }
    job_ds[j] = it->second;
  }
  using TKey = std::tuple<int, double, int, int, int, int>;
  std::map<TKey, int> tkeys;
  std::vector<int> job_tile(n_jobs);
  std::vector<TKey> tsrc;
  for (int j = 0; j < n_jobs; ++j) {
    const lann_job& J = jobs[j];
    TKey k{job_ds[j], J.train_fraction, J.n_folds >= 2 ? J.n_folds : 0,
           J.n_folds >= 2 ? J.fold : 0, J.family, J.log_target};
    auto it = tkeys.find(k);
    if (it == tkeys.end()) {
      it = tkeys.emplace(k, int(tsrc.size())).first;
      tsrc.push_back(k);
    }
    job_tile[j] = it->second;
  }
  // one pool pass: each task builds a dataset and then every tile cut from it
  std::vector<Dataset> dsets(dsrc.size());
  std::vector<Status> dstat(dsrc.size());
  std::vector<Tile> tiles(tsrc.size());
  std::vector<Status> tstat(tsrc.size());
  std::vector<std::vector<int>> tiles_of(dsrc.size());
  for (int k = 0; k < int(tsrc.size()); ++k) tiles_of[std::get<0>(tsrc[k])].push_back(k);
  const auto h1 = now();
  parallel_for(int(dsrc.size()), [&](int d) {
    dstat[d] = build_dataset(dsrc[d]->world, dsrc[d]->data_seed, dsrc[d]->count, dsets[d]);
    for (int k : tiles_of[d]) {
      const auto& [dd, frac, folds, fold, family, logt] = tsrc[k];
      (void)dd;
      if (dstat[d]) {
        tstat[k] = dstat[d];
        continue;
      }
      std::vector<int64_t> order;
      int ntr = 0;
      tstat[k] = split_order(dsets[d].size(), frac, dsrc[d]->data_seed, order, ntr);
      if (!tstat[k]) tstat[k] = make_tile(dsets[d], order, ntr, folds, fold, family, logt != 0, tiles[k]);
    }
  });
  hlog("datasets", h0);
  for (int j = 0; j < n_jobs; ++j) {
    const int k = job_tile[j];
    Status st = tstat[k];
    if (!st) st = validate_config(jobs[j], tiles[k].n_inputs);
    if (!st && tiles[k].n_eval() < 2)
      st = {LANN_DOMAIN_ERROR, "spearman needs at least two samples"};  // eval.cpp:80
    lann_job_result& r = pop.base[j];
    r.status = st.code;
    if (st) {
      if (e->err.empty()) e->err = st.msg;
      continue;
    }
    r.n_inputs = tiles[k].n_inputs;
    r.n_params = param_count(tiles[k].n_inputs, jobs[j].hidden[0],
                             jobs[j].n_hidden > 1 ? jobs[j].hidden[1] : 0);
    r.n_train = tiles[k].n_train();
    r.n_eval = tiles[k].n_eval();
    pop.model_job.push_back(j);
  }
  hlog("tiles", h1);
  const auto h2 = now();
  const int M = int(pop.model_job.size());
  pop.M = M;
  if (M == 0) return pop.base[0].status;
  // cross-validation ensembles of the k-fold jobs: members, test sets, group item lists
  std::vector<int> cv_set_tile, cv_ens_set, cv_fold_items, cv_ens_items;
  std::vector<int64_t> cv_fold_off, cv_ens_off, cv_set_row;
  std::vector<int> cv_fold_len, cv_ens_len;
  int64_t cv_rows = 0;
  if (std::any_of(jobs, jobs + n_jobs, [](const lann_job& J) { return J.n_folds >= 2; })) {
    pop.cv = std::make_unique<CvState>();
    CvState& cv = *pop.cv;
    cv.L = cv_layout(n_jobs, jobs);
    const int E = cv.L.n_ens(), G = cv.L.n_groups();
    std::vector<int> job_model(size_t(n_jobs), -1);
    for (int m = 0; m < M; ++m) job_model[size_t(pop.model_job[size_t(m)])] = m;
    cv.dev_of.assign(size_t(E), -1);
    cv.host_status.assign(size_t(E), LANN_OK);
    cv.ens_test.assign(size_t(E), 0);
    for (int f : cv.L.group_folds) cv.kmax = std::max(cv.kmax, f);
    std::map<std::tuple<int, double, int>, int> skeys;  // (dataset, train fraction, family)
    for (int en = 0; en < E; ++en) {
      const auto& mem = cv.L.ens_member[size_t(en)];
      int st = LANN_OK;
      for (int j : mem) {
        if (j < 0) {
          st = LANN_PARAM_ERROR;  // a fold of this seed is not in the job list
          break;
        }
        if (job_model[size_t(j)] < 0) {
          st = pop.base[size_t(j)].status;  // the member failed host preparation
          break;
        }
      }
      if (st != LANN_OK) {
        cv.host_status[size_t(en)] = st;
        continue;
      }
      const int k = job_tile[size_t(mem[0])];
      const std::tuple<int, double, int> key{std::get<0>(tsrc[size_t(k)]), std::get<1>(tsrc[size_t(k)]),
                                             std::get<4>(tsrc[size_t(k)])};
      auto it = skeys.find(key);
      if (it == skeys.end()) {
        it = skeys.emplace(key, int(cv_set_tile.size())).first;
        cv_set_tile.push_back(k);
        cv_set_row.push_back(cv_rows);
        cv_rows += tiles[size_t(k)].n_test();
      }
      cv.ens_test[size_t(en)] = tiles[size_t(k)].n_test();
      cv.dev_of[size_t(en)] = cv.n_dev++;
      cv_ens_set.push_back(it->second);
      for (int f = 0; f < cv.kmax; ++f)
        cv.dev_members.push_back(f < int(mem.size()) ? job_model[size_t(mem[size_t(f)])] : 0);
      cv.max_test = std::max(cv.max_test, cv.ens_test[size_t(en)]);
      cv.total_out += cv.ens_test[size_t(en)];
    }
    // item lists: a group's trained models in job order, its device ensembles in ensemble order
    std::vector<std::vector<int>> fi(static_cast<size_t>(G)), ei(static_cast<size_t>(G));
    for (int m = 0; m < M; ++m) {
      const int g = cv.L.job_group[size_t(pop.model_job[size_t(m)])];
      if (g >= 0) fi[size_t(g)].push_back(m);
    }
    for (int en = 0; en < E; ++en)
      if (cv.dev_of[size_t(en)] >= 0) ei[size_t(cv.L.ens_group[size_t(en)])].push_back(cv.dev_of[size_t(en)]);
    for (int g = 0; g < G; ++g) {
      cv_fold_off.push_back(int64_t(cv_fold_items.size()));
      cv_fold_len.push_back(int(fi[size_t(g)].size()));
      cv_fold_items.insert(cv_fold_items.end(), fi[size_t(g)].begin(), fi[size_t(g)].end());
      cv_ens_off.push_back(int64_t(cv_ens_items.size()));
      cv_ens_len.push_back(int(ei[size_t(g)].size()));
      cv_ens_items.insert(cv_ens_items.end(), ei[size_t(g)].begin(), ei[size_t(g)].end());
    }
  }
  // pack straight into the engine's pinned staging buffer, laid out like the one device blob
  // that receives it (a single H2D copy; no growing host vectors, no pageable staging)
  DevTrain& t = pop.t;
  t.n_models = M;
  t.n_tiles = int(tiles.size());
  int64_t n_eval_total = 0, eval_row_doubles = 0;
  for (size_t k = 0; k < tiles.size(); ++k) pop.rows += tiles[k].n_train();
  for (int m = 0; m < M; ++m) {
    const Tile& T = tiles[job_tile[pop.model_job[m]]];
    n_eval_total += T.n_eval();
    eval_row_doubles += int64_t(T.eval_rows.size());
  }
  for (int m = 0; m < M; ++m) {
    const lann_job& J = jobs[pop.model_job[m]];
    const Tile& T = tiles[job_tile[pop.model_job[m]]];
    t.model_tile.push_back(job_tile[pop.model_job[m]]);
    t.h1.push_back(J.hidden[0]);
    t.h2.push_back(J.n_hidden > 1 ? J.hidden[1] : 0);
    t.lr.push_back(J.learning_rate);
    t.epochs.push_back(J.epochs);
    t.param_offset.push_back(t.total_params);
    t.total_params += param_count(T.n_inputs, t.h1.back(), t.h2.back());
    pop.train_flop += double(J.epochs) * flop_per_model_epoch(T.n_inputs, t.h1.back(), t.h2.back(), T.n_train());
    pop.max_eval = std::max(pop.max_eval, T.n_eval());
  }
  pop.toff.assign(M, 0);
  if (want_trace)
    for (int m = 0; m < M; ++m) {
      pop.toff[m] = pop.trace_total;
      pop.trace_total += t.epochs[m];
    }
  pop.n_eval_rows = n_eval_total;
  BlobLayout L;
  const size_t oX = L.add<double>(size_t(pop.rows) * 8), oY = L.add<double>(size_t(pop.rows));
  const size_t oP0 = L.add<double>(size_t(t.total_params)), oN = L.add<double>(size_t(M) * 18);
  const size_t oER = L.add<double>(size_t(eval_row_doubles)), oET = L.add<double>(size_t(n_eval_total));
  const size_t oEM = L.add<int>(size_t(n_eval_total)), oI = L.add<int>(size_t(M)), oH1 = L.add<int>(size_t(M));
  const size_t oH2 = L.add<int>(size_t(M)), oLog = L.add<int>(size_t(M)), oEL = L.add<int>(size_t(M));
  const size_t oPO = L.add<int64_t>(size_t(M)), oEO = L.add<int64_t>(size_t(M)), oTO = L.add<int64_t>(size_t(M));
  CvState* cvp = pop.cv.get();
  const int cvG = cvp ? cvp->L.n_groups() : 0, cvD = cvp ? cvp->n_dev : 0, cvK = cvp ? cvp->kmax : 0;
  const size_t cRows = L.add<double>(size_t(cv_rows) * 8), cTruth = L.add<double>(size_t(cv_rows));
  const size_t cK = L.add<int>(size_t(cvD)), cMem = L.add<int>(size_t(cvD) * size_t(cvK));
  const size_t cER = L.add<int64_t>(size_t(cvD)), cEL = L.add<int>(size_t(cvD)), cEO = L.add<int64_t>(size_t(cvD));
  const size_t cFO = L.add<int64_t>(size_t(cvG)), cFL = L.add<int>(size_t(cvG));
  const size_t cFI = L.add<int>(cv_fold_items.size());
  const size_t cGO = L.add<int64_t>(size_t(cvG)), cGL = L.add<int>(size_t(cvG)), cGI = L.add<int>(cv_ens_items.size());
  const size_t up_bytes = L.bytes;
  // device-only outputs follow the uploaded part
  // the per-model results first, contiguous, so fetch is one D2H copy
  const size_t oF = L.add<double>(size_t(M));
  const size_t oMape = L.add<double>(size_t(M)), oThr = L.add<double>(size_t(M)), oRho = L.add<double>(size_t(M));
  const size_t oB = L.add<int>(size_t(M)), oK = L.add<int>(size_t(M)), oS = L.add<int>(size_t(M));
  pop.res_off = oF;
  pop.res_bytes = L.bytes - oF;
  pop.res_rel = {0, oMape - oF, oThr - oF, oRho - oF, oB - oF, oK - oF, oS - oF};
  const size_t oP = L.add<double>(size_t(t.total_params));
  const size_t oT = L.add<double>(size_t(pop.trace_total)), oPred = L.add<double>(size_t(n_eval_total));
  // cross-validation outputs: the fold-mean sets, then one contiguous result block (one D2H)
  const int64_t cv_out = cvp ? cvp->total_out : 0;
  const size_t cPred = L.add<double>(size_t(cv_out)), cTOut = L.add<double>(size_t(cv_out));
  const size_t cScr = L.add<double>(std::max(cv_fold_items.size(), cv_ens_items.size()));
  const size_t cRes = L.add<double>(size_t(cvD));  // ensemble MAPE (result block starts here)
  const size_t cThr = L.add<double>(size_t(cvD)), cRho = L.add<double>(size_t(cvD));
  const size_t cSF = L.add<double>(size_t(cvG) * 6), cSE = L.add<double>(size_t(cvG) * 6);
  const size_t cKept = L.add<int>(size_t(cvD)), cSt = L.add<int>(size_t(cvD)), cBad = L.add<int>(size_t(cvD));
  const size_t cNF = L.add<int>(size_t(cvG)), cNE = L.add<int>(size_t(cvG));
  if (cvp) {
    cvp->res_off = cRes;
    cvp->res_bytes = L.bytes - cRes;
    cvp->r_mape = 0;
    cvp->r_thr = cThr - cRes;
    cvp->r_rho = cRho - cRes;
    cvp->r_sf = cSF - cRes;
    cvp->r_se = cSE - cRes;
    cvp->r_kept = cKept - cRes;
    cvp->r_st = cSt - cRes;
    cvp->r_bad = cBad - cRes;
    cvp->r_nf = cNF - cRes;
    cvp->r_ne = cNE - cRes;
  }
  unsigned char* h = pinned_stage(e, up_bytes);
  auto H = [&](auto* type_tag, size_t off) { return reinterpret_cast<decltype(type_tag)>(h + off); };
  {
    double* X = H((double*)nullptr, oX);
    double* Y = H((double*)nullptr, oY);
    int64_t r0 = 0;
    for (size_t k = 0; k < tiles.size(); ++k) {
      t.tile_rows.push_back(std::max(1, tiles[k].n_train()));
      t.tile_inputs.push_back(std::max(1, tiles[k].n_inputs));
      t.tile_offset.push_back(r0);
      r0 += tiles[k].n_train();
    }
    double* norm = H((double*)nullptr, oN);
    double* ER = H((double*)nullptr, oER);
    double* ET = H((double*)nullptr, oET);
    int* EM = H((int*)nullptr, oEM);
    int* n_in = H((int*)nullptr, oI);
    int* logt = H((int*)nullptr, oLog);
    int* eval_len = H((int*)nullptr, oEL);
    int64_t* eval_off = H((int64_t*)nullptr, oEO);
    std::vector<int64_t> er_off(M);
    int64_t er = 0, et = 0;
    for (int m = 0; m < M; ++m) {
      const Tile& T = tiles[job_tile[pop.model_job[m]]];
      std::memcpy(norm + size_t(m) * 18, T.norm, sizeof T.norm);
      n_in[m] = T.n_inputs;
      logt[m] = T.log_target;
      eval_off[m] = et;
      eval_len[m] = T.n_eval();
      er_off[m] = er;
      er += int64_t(T.eval_rows.size());
      et += T.n_eval();
    }
    double* P0 = H((double*)nullptr, oP0);
    // the bulk copies (~1.5 MB for config 2) and the initial weights run on the pool: one thread is memory-latency bound
    const int nt = int(tiles.size());
    parallel_for(nt + M, [&](int j) {
      if (j < nt) {
        std::copy(tiles[j].Xn.begin(), tiles[j].Xn.end(), X + t.tile_offset[j] * 8);
        std::copy(tiles[j].yn.begin(), tiles[j].yn.end(), Y + t.tile_offset[j]);
        return;
      }
      const int m = j - nt;
      const Tile& T = tiles[job_tile[pop.model_job[m]]];
      std::copy(T.eval_rows.begin(), T.eval_rows.end(), ER + er_off[m]);
      std::copy(T.eval_truth.begin(), T.eval_truth.end(), ET + eval_off[m]);
      std::fill(EM + eval_off[m], EM + eval_off[m] + T.n_eval(), m);
      // glorot_init writes every weight and (zero) bias of the model
      glorot_init(n_in[m], t.h1[m], t.h2[m], jobs[pop.model_job[m]].init_seed, P0 + t.param_offset[m]);
    });
    std::copy(t.h1.begin(), t.h1.end(), H((int*)nullptr, oH1));
    std::copy(t.h2.begin(), t.h2.end(), H((int*)nullptr, oH2));
    std::copy(t.param_offset.begin(), t.param_offset.end(), H((int64_t*)nullptr, oPO));
    std::copy(pop.toff.begin(), pop.toff.end(), H((int64_t*)nullptr, oTO));
    if (cvp) {
      double* cr = H((double*)nullptr, cRows);
      double* ct = H((double*)nullptr, cTruth);
      for (size_t q = 0; q < cv_set_tile.size(); ++q) {
        const Tile& T = tiles[size_t(cv_set_tile[q])];
        std::copy(T.test_rows.begin(), T.test_rows.end(), cr + cv_set_row[q] * 8);
        std::copy(T.test_truth.begin(), T.test_truth.end(), ct + cv_set_row[q]);
      }
      int* ek = H((int*)nullptr, cK);
      int64_t* er_ = H((int64_t*)nullptr, cER);
      int* el = H((int*)nullptr, cEL);
      int64_t* eo = H((int64_t*)nullptr, cEO);
      std::copy(cvp->dev_members.begin(), cvp->dev_members.end(), H((int*)nullptr, cMem));
      int64_t out = 0;
      for (int en = 0, slot = 0; en < cvp->L.n_ens(); ++en) {
        if (cvp->dev_of[size_t(en)] < 0) continue;
        ek[slot] = cvp->L.group_folds[size_t(cvp->L.ens_group[size_t(en)])];
        er_[slot] = cv_set_row[size_t(cv_ens_set[size_t(slot)])];
        el[slot] = cvp->ens_test[size_t(en)];
        eo[slot] = out;
        out += el[slot];
        ++slot;
      }
      std::copy(cv_fold_off.begin(), cv_fold_off.end(), H((int64_t*)nullptr, cFO));
      std::copy(cv_fold_len.begin(), cv_fold_len.end(), H((int*)nullptr, cFL));
      std::copy(cv_fold_items.begin(), cv_fold_items.end(), H((int*)nullptr, cFI));
      std::copy(cv_ens_off.begin(), cv_ens_off.end(), H((int64_t*)nullptr, cGO));
      std::copy(cv_ens_len.begin(), cv_ens_len.end(), H((int*)nullptr, cGL));
      std::copy(cv_ens_items.begin(), cv_ens_items.end(), H((int*)nullptr, cGI));
    }
    hlog("pack", h2);
  }
  if (Status st = validate_train(t)) return set_err(e, st);
  hlog("pack+init", h2);
  const auto h3 = now();
  // one device blob, one upload
  cudaStream_t s = e->stream;
  pop.blob = DBuf<unsigned char>(L.bytes, s);
  pop.blob.up(h, up_bytes);
  unsigned char* d = pop.blob.p;
  auto V = [&](auto* type_tag, size_t off, size_t n) {
    using T = std::remove_pointer_t<decltype(type_tag)>;
    return DBuf<T>::view(reinterpret_cast<T*>(d + off), n, s);
  };
  const size_t Mz = size_t(M), Ez = size_t(n_eval_total), Pz = size_t(t.total_params);
  pop.dX = V((double*)nullptr, oX, size_t(pop.rows) * 8);
  pop.dY = V((double*)nullptr, oY, size_t(pop.rows));
  pop.dP0 = V((double*)nullptr, oP0, Pz);
  pop.dN = V((double*)nullptr, oN, Mz * 18);
  pop.dER = V((double*)nullptr, oER, size_t(eval_row_doubles));
  pop.dET = V((double*)nullptr, oET, Ez);
  pop.dEM = V((int*)nullptr, oEM, Ez);
  pop.dI = V((int*)nullptr, oI, Mz);
  pop.dh1 = V((int*)nullptr, oH1, Mz);
  pop.dh2 = V((int*)nullptr, oH2, Mz);
  pop.dlog = V((int*)nullptr, oLog, Mz);
  pop.dEL = V((int*)nullptr, oEL, Mz);
  pop.dpo = V((int64_t*)nullptr, oPO, Mz);
  pop.dEO = V((int64_t*)nullptr, oEO, Mz);
  pop.dTO = V((int64_t*)nullptr, oTO, Mz);
  pop.dP = V((double*)nullptr, oP, Pz);
  pop.dF = V((double*)nullptr, oF, Mz);
  pop.dT = V((double*)nullptr, oT, size_t(pop.trace_total));
  pop.dPred = V((double*)nullptr, oPred, Ez);
  pop.dMape = V((double*)nullptr, oMape, Mz);
  pop.dThr = V((double*)nullptr, oThr, Mz);
  pop.dRho = V((double*)nullptr, oRho, Mz);
  pop.dB = V((int*)nullptr, oB, Mz);
  pop.dK = V((int*)nullptr, oK, Mz);
  pop.dS = V((int*)nullptr, oS, Mz);
  // the per-model result block is fetched as one copy: zero it once so the alignment padding
  // between its arrays (M not a multiple of 4) is defined (compute-sanitizer initcheck)
  if (pop.res_bytes) ck(cudaMemsetAsync(d + pop.res_off, 0, pop.res_bytes, s), "memset");
  if (cvp) {
    // the result block is fetched as one copy: zero it once so its alignment padding is defined
    ck(cudaMemsetAsync(d + cvp->res_off, 0, cvp->res_bytes, s), "memset");
    auto P = [&](auto* type_tag, size_t off) { return reinterpret_cast<decltype(type_tag)>(d + off); };
    FoldMeanArgs& f = cvp->fm;
    f.n_ens = cvD;
    f.kmax = cvK;
    f.ens_k = P((const int*)nullptr, cK);
    f.ens_models = P((const int*)nullptr, cMem);
    f.ens_rows = P((const int64_t*)nullptr, cER);
    f.ens_len = P((const int*)nullptr, cEL);
    f.ens_out = P((const int64_t*)nullptr, cEO);
    f.rows = P((const double*)nullptr, cRows);
    f.truth = P((const double*)nullptr, cTruth);
    f.model_bad = pop.dB.p;
    f.model_status = pop.dS.p;
    f.pred = P((double*)nullptr, cPred);
    f.truth_out = P((double*)nullptr, cTOut);
    f.ens_bad = P((int*)nullptr, cBad);
    cvp->ev = EvalArgs{cvD, f.ens_out, f.ens_len, f.truth_out, f.pred, 0.3, P((double*)nullptr, cRes),
                       P((double*)nullptr, cThr), P((int*)nullptr, cKept), P((double*)nullptr, cRho),
                       P((int*)nullptr, cSt)};
    double* scr = P((double*)nullptr, cScr);
    cvp->sf = CvStatsArgs{cvG, P((const int64_t*)nullptr, cFO), P((const int*)nullptr, cFL),
                          P((const int*)nullptr, cFI), pop.dMape.p, pop.dThr.p, pop.dRho.p, pop.dS.p, pop.dB.p,
                          P((double*)nullptr, cSF), P((int*)nullptr, cNF), scr};
    cvp->se = CvStatsArgs{cvG, P((const int64_t*)nullptr, cGO), P((const int*)nullptr, cGL),
                          P((const int*)nullptr, cGI), cvp->ev.mape, cvp->ev.mape_thr, cvp->ev.rho, cvp->ev.status,
                          f.ens_bad, P((double*)nullptr, cSE), P((int*)nullptr, cNE), scr};
  }
  hlog("uploads", h3);
  const auto h4 = now();
  pop.plan = build_plan(e, t, precision, pop.dX.p, pop.dY.p, pop.rows);
  // a prepared population is resident when create returns; lann_run_population launches right
  // behind the uploads on the same stream instead (stream order suffices, nothing host-side
  // is reused before its own synchronisation)
  if (sync_uploads) ck(cudaStreamSynchronize(s), "prepare");
  hlog("plan", h4);
  return LANN_OK;
}

// One device-only pass: reset weights, train, predict every evaluation row, metrics.
void run_device(Population& pop) {
  lann_engine* e = pop.e;
  if (!pop.plan) throw CudaFail{"population has no launch plan"};
  cudaStream_t s = e->stream;
  ck(cudaMemcpyAsync(pop.dP.p, pop.dP0.p, pop.dP0.n * sizeof(double), cudaMemcpyDeviceToDevice, s), "D2D");
  execute_plan(e, *pop.plan, pop.dP.p, pop.dF.p, pop.dB.p, pop.trace_total ? pop.dT.p : nullptr, pop.dTO.p);
  PredictArgs pa{pop.n_eval_rows, pop.dER.p, pop.dEM.p, pop.dI.p, pop.dh1.p, pop.dh2.p, pop.dlog.p,
                 pop.dpo.p, pop.dP.p, pop.dN.p, pop.dPred.p};
  if (pop.precision == LANN_FP32) launch_predict_fp32(pa, pop.M, pop.t.total_params, s);
  else launch_predict_fp64(pa, s);
  e->launches += pop.n_eval_rows > 0 ? (pop.precision == LANN_FP32 ? 2 : 1) : 0;
  EvalArgs ea{pop.M, pop.dEO.p, pop.dEL.p, pop.dET.p, pop.dPred.p, 0.3, pop.dMape.p, pop.dThr.p,
              pop.dK.p, pop.dRho.p, pop.dS.p};
  launch_eval(ea, pop.max_eval, e->max_smem, pop.n_eval_rows, s);
  e->launches += eval_launch_count(pop.max_eval, e->max_smem);
  if (pop.cv) {  // cross-validation summary: fold-mean test scores, then the group statistics
    CvState& cv = *pop.cv;
    const bool exact = pop.precision != LANN_FP32;
    launch_fold_mean(pa, cv.fm, cv.max_test, exact, pop.M, pop.t.total_params, s);
    launch_eval(cv.ev, cv.max_test, e->max_smem, cv.total_out, s);
    launch_cv_stats(cv.sf, s);
    launch_cv_stats(cv.se, s);
    if (cv.n_dev > 0) e->launches += (exact ? 1 : 2) + eval_launch_count(cv.max_test, e->max_smem);
    if (cv.L.n_groups() > 0) e->launches += 2;
  }
  ck(cudaGetLastError(), "population launch");
}

int fetch_population(Population& pop, lann_job_result* results, double* params_out,
                     const int64_t* params_offset, double* trace_out, const int64_t* trace_offset) {
  const int M = pop.M;
  for (int j = 0; j < pop.n_jobs; ++j) results[j] = pop.base[j];
  if (M == 0) return pop.base[0].status;
  std::vector<double> params;
  // one D2H of the result block into the engine's pinned staging buffer (its upload finished
  // earlier on the same stream)
  unsigned char* hr = pinned_stage(pop.e, pop.res_bytes);
  ck(cudaMemcpyAsync(hr, pop.blob.p + pop.res_off, pop.res_bytes, cudaMemcpyDeviceToHost, pop.e->stream), "D2H");
  t_d2h += int64_t(pop.res_bytes);
  const double* fin = reinterpret_cast<const double*>(hr + pop.res_rel[0]);
  const double* mape = reinterpret_cast<const double*>(hr + pop.res_rel[1]);
  const double* thr = reinterpret_cast<const double*>(hr + pop.res_rel[2]);
  const double* rho = reinterpret_cast<const double*>(hr + pop.res_rel[3]);
  const int* bad = reinterpret_cast<const int*>(hr + pop.res_rel[4]);
  const int* kept = reinterpret_cast<const int*>(hr + pop.res_rel[5]);
  const int* est = reinterpret_cast<const int*>(hr + pop.res_rel[6]);
  if (params_out) {
    params.resize(pop.dP.n);
    pop.dP.down(params.data());
  }
  std::vector<double> trace(static_cast<size_t>(pop.trace_total));
  if (trace_out && pop.trace_total) pop.dT.down(trace.data());
  ck(cudaStreamSynchronize(pop.e->stream), "fetch");
  for (int m = 0; m < M; ++m) {
    const int j = pop.model_job[m];
    lann_job_result& r = results[j];
    r.final_loss = fin[m];
    r.nonfinite_epoch = bad[m];
    r.precision_run = pop.plan->model_precision[size_t(m)];
    if (bad[m] >= 0) {
      r.status = LANN_TRAINING_ERROR;
    } else {
      r.mape = mape[m];
      r.mape_thr = thr[m];
      r.rho = rho[m];
      r.n_kept = kept[m];
      if (est[m]) r.status = LANN_DOMAIN_ERROR;
    }
    if (params_out && params_offset)
      std::memcpy(params_out + params_offset[j], &params[size_t(pop.t.param_offset[m])],
                  sizeof(double) * size_t(r.n_params));
    if (trace_out && trace_offset && pop.trace_total)
      std::memcpy(trace_out + trace_offset[j], &trace[size_t(pop.toff[m])],
                  sizeof(double) * size_t(pop.t.epochs[m]));
  }
  for (int j = 0; j < pop.n_jobs; ++j)
    if (results[j].status != LANN_OK) {
      if (results[j].status == LANN_TRAINING_ERROR)
        pop.e->err = "training diverged (non-finite loss) at epoch " +
                     std::to_string(results[j].nonfinite_epoch);
      return results[j].status;
    }
  return LANN_OK;
}

}  // namespace
}  // namespace lann

using namespace lann;

struct lann_population {
  Population pop;
};

namespace {
// Live prepared populations: lann_population_destroy on a handle that is no longer live (already
// destroyed, or freed with its engine) is a no-op instead of a use-after-free.
std::mutex g_pop_mu;
std::vector<lann_population*> g_pops;
void pop_register(lann_population* p) {
  std::lock_guard<std::mutex> lk(g_pop_mu);
  g_pops.push_back(p);
  p->pop.e->pops.push_back(p);
}
bool pop_unregister(lann_population* p) {
  std::lock_guard<std::mutex> lk(g_pop_mu);
  auto it = std::find(g_pops.begin(), g_pops.end(), p);
  if (it == g_pops.end()) return false;
  g_pops.erase(it);
  auto& v = p->pop.e->pops;
  v.erase(std::remove(v.begin(), v.end(), p), v.end());
  return true;
}
void pop_free(lann_population* p) {
  cudaSetDevice(p->pop.e->device);
  cudaStreamSynchronize(p->pop.e->stream);
  delete p;  // device buffers are released on the engine's stream, which is still alive
}
}  // namespace

extern "C" {

int lann_engine_create(int device, lann_engine** out) {
  if (!out) return LANN_PARAM_ERROR;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return LANN_NO_DEVICE;
  }
  if (device < 0 || device >= n) return LANN_PARAM_ERROR;
  auto* e = new lann_engine;
  e->device = device;
  try {
    ck(cudaSetDevice(device), "cudaSetDevice");
    ck(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking), "stream");
    for (auto& a : e->aux) ck(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking), "stream");
    for (cudaEvent_t* ev : {&e->ev0, &e->ev1, &e->tr0, &e->tr1}) ck(cudaEventCreate(ev), "event");
    ck(cudaEventCreateWithFlags(&e->fork, cudaEventDisableTiming), "event");
    for (auto& j : e->join) ck(cudaEventCreateWithFlags(&j, cudaEventDisableTiming), "event");
    ck(cudaDeviceGetAttribute(&e->max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device), "attr");
    ck(cudaDeviceGetAttribute(&e->sms, cudaDevAttrMultiProcessorCount, device), "attr");
    // keep freed stream-ordered allocations in the device pool: repeated population calls
    // then reuse them instead of returning memory to the driver at every synchronisation
    if (std::getenv("LANN_POOL_RELEASE") == nullptr) {
      cudaMemPool_t pool;
      ck(cudaDeviceGetDefaultMemPool(&pool, device), "mempool");
      std::uint64_t keep = ~std::uint64_t(0);
      ck(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep), "mempool attr");
    }
  } catch (const CudaFail&) {
    delete e;
    return LANN_CUDA_ERROR;
  }
  *out = e;
  return LANN_OK;
}

void lann_engine_destroy(lann_engine* e) {
  if (!e) return;
  // populations still alive belong to this engine's stream and memory: free them first
  while (!e->pops.empty()) {
    lann_population* p = e->pops.back();
    if (pop_unregister(p)) pop_free(p);
    else e->pops.pop_back();
  }
  cudaSetDevice(e->device);
  if (e->stream) cudaStreamSynchronize(e->stream);
  for (cudaEvent_t ev : {e->ev0, e->ev1, e->tr0, e->tr1, e->fork})
    if (ev) cudaEventDestroy(ev);
  for (auto j : e->join)
    if (j) cudaEventDestroy(j);
  for (auto a : e->aux)
    if (a) cudaStreamDestroy(a);
  if (e->stream) cudaStreamDestroy(e->stream);
  if (e->pin) cudaFreeHost(e->pin);
  if (e->brcp) cudaFree(e->brcp);
  delete e;
}

const char* lann_last_error(const lann_engine* e) { return e ? e->err.c_str() : "no engine"; }
double lann_last_device_ms(const lann_engine* e) { return e ? e->last_ms : 0.0; }
double lann_last_train_ms(const lann_engine* e) { return e ? e->last_train_ms : 0.0; }
int64_t lann_last_launches(const lann_engine* e) { return e ? e->launches : 0; }

int lann_train(lann_engine* e, const lann_train_batch* b) {
  if (!e) return LANN_NO_DEVICE;
  if (!b) return set_err(e, {LANN_PARAM_ERROR, "null batch"});
  if (b->precision != LANN_FP64_EXACT && b->precision != LANN_FP32)
    return set_err(e, {LANN_PARAM_ERROR, "unknown precision"});
  if (b->n_models < 1 || b->n_tiles < 1)
    return set_err(e, {LANN_PARAM_ERROR, "population needs at least one model and tile"});
  DevTrain t;
  t.n_models = b->n_models;
  t.n_tiles = b->n_tiles;
  t.tile_rows.assign(b->tile_rows, b->tile_rows + b->n_tiles);
  t.tile_inputs.assign(b->tile_inputs, b->tile_inputs + b->n_tiles);
  t.tile_offset.assign(b->tile_offset, b->tile_offset + b->n_tiles);
  t.model_tile.assign(b->model_tile, b->model_tile + b->n_models);
  t.h1.assign(b->model_h1, b->model_h1 + b->n_models);
  t.h2.assign(b->model_h2, b->model_h2 + b->n_models);
  t.lr.assign(b->model_lr, b->model_lr + b->n_models);
  t.epochs.assign(b->model_epochs, b->model_epochs + b->n_models);
  t.param_offset.assign(b->model_param_offset, b->model_param_offset + b->n_models);
  t.total_params = b->total_params;
  t.trace_stride = b->trace_stride < 1 ? 1 : b->trace_stride;
  for (int k = 0; k < t.n_tiles; ++k)
    if (t.tile_offset[k] < 0 || t.tile_offset[k] + t.tile_rows[k] > b->total_rows)
      return set_err(e, {LANN_PARAM_ERROR, "tile exceeds the row buffer"});
  if (Status st = validate_train(t)) return set_err(e, st);
  try {
    ck(cudaSetDevice(e->device), "cudaSetDevice");
    cudaStream_t s = e->stream;
    Timer timer(e);
    DBuf<double> dX(b->X, size_t(b->total_rows) * LANN_ROW, s), dY(b->y, size_t(b->total_rows), s);
    DBuf<double> dP(b->params, size_t(b->total_params), s);
    DBuf<double> dF(size_t(b->n_models), s);
    DBuf<int> dB(size_t(b->n_models), s);
    int64_t trace_total = 0;
    std::vector<int64_t> toff(b->n_models, 0);
    if (b->loss_trace)
      for (int m = 0; m < b->n_models; ++m) {
        toff[m] = b->trace_offset[m];
        trace_total = std::max<int64_t>(trace_total, toff[m] + (t.epochs[m] + t.trace_stride - 1) / t.trace_stride);
      }
    DBuf<double> dT(size_t(trace_total), s);
    DBuf<int64_t> dTO(toff, s);
    auto plan = build_plan(e, t, b->precision, dX.p, dY.p, b->total_rows);
    execute_plan(e, *plan, dP.p, dF.p, dB.p, b->loss_trace ? dT.p : nullptr, dTO.p);
    dP.down(b->params);
    dF.down(b->final_loss);
    dB.down(b->nonfinite_epoch);
    if (b->loss_trace) dT.down(b->loss_trace);
    timer.stop();
    float tms = 0.f;
    ck(cudaEventElapsedTime(&tms, e->tr0, e->tr1), "elapsed");
    e->last_train_ms = tms;
    for (int m = 0; m < b->n_models; ++m)
      if (b->nonfinite_epoch[m] >= 0) {
        e->err = "training diverged (non-finite loss) at epoch " + std::to_string(b->nonfinite_epoch[m]);
        return LANN_TRAINING_ERROR;
      }
    e->err.clear();
    return LANN_OK;
  } catch (const CudaFail& f) {
    e->err = f.what;
    return LANN_CUDA_ERROR;
  }
}

int lann_predict(lann_engine* e, const lann_model_set* ms, int64_t n_rows, const double* rows,
                 const int32_t* row_model, double* out) {
  if (!e) return LANN_NO_DEVICE;
  if (!ms || ms->n_models < 1) return set_err(e, {LANN_PARAM_ERROR, "empty model set"});
  for (int m = 0; m < ms->n_models; ++m) {
    if (ms->n_inputs[m] < 1 || ms->n_inputs[m] > 7 || ms->h1[m] < 1 || ms->h2[m] < 0 ||
        ms->h1[m] > 64 || ms->h2[m] > 64)
      return set_err(e, {LANN_PARAM_ERROR, "bad model shape"});
    const int P = param_count(ms->n_inputs[m], ms->h1[m], ms->h2[m]);
    if (ms->param_offset[m] < 0 || ms->param_offset[m] + P > ms->total_params)
      return set_err(e, {LANN_PARAM_ERROR, "flat parameter size mismatch"});
  }
  for (int64_t r = 0; r < n_rows; ++r)
    if (row_model[r] < 0 || row_model[r] >= ms->n_models)
      return set_err(e, {LANN_SCHEMA_ERROR, "row references an unknown model"});
  try {
    ck(cudaSetDevice(e->device), "cudaSetDevice");
    cudaStream_t s = e->stream;
    Timer timer(e);
    const int M = ms->n_models;
    DBuf<double> drows(rows, size_t(n_rows) * LANN_ROW, s), dout(size_t(n_rows), s);
    DBuf<int> drm(row_model, size_t(n_rows), s), dI(ms->n_inputs, M, s), dh1(ms->h1, M, s),
        dh2(ms->h2, M, s), dlog(ms->log_target, M, s);
    DBuf<int64_t> dpo(ms->param_offset, M, s);
    DBuf<double> dp(ms->params, size_t(ms->total_params), s), dn(ms->norm, size_t(M) * 18, s);
    PredictArgs a{n_rows, drows.p, drm.p, dI.p, dh1.p, dh2.p, dlog.p, dpo.p, dp.p, dn.p, dout.p};
    ck(cudaEventRecord(e->tr0, s), "event");
    if (ms->precision == LANN_FP32) launch_predict_fp32(a, M, ms->total_params, s);
    else launch_predict_fp64(a, s);
    ck(cudaGetLastError(), "predict launch");
    ck(cudaEventRecord(e->tr1, s), "event");
    e->launches += n_rows > 0 ? (ms->precision == LANN_FP32 ? 2 : 1) : 0;
    dout.down(out);
    timer.stop();
    float kms = 0.f;
    ck(cudaEventElapsedTime(&kms, e->tr0, e->tr1), "elapsed");
    e->last_train_ms = kms;  // the predictor's own device time (inputs already resident)
    e->err.clear();
    return LANN_OK;
  } catch (const CudaFail& f) {
    e->err = f.what;
    return LANN_CUDA_ERROR;
  }
}

int lann_eval(lann_engine* e, int32_t n_sets, const int64_t* offset, const int32_t* len,
              const double* truth, const double* pred, double drop, double* mape,
              double* mape_thr, int32_t* n_kept, double* rho) {
  if (!e) return LANN_NO_DEVICE;
  if (n_sets < 1) return set_err(e, {LANN_DOMAIN_ERROR, "nothing to evaluate"});
  if (drop < 0.0 || drop > 1.0) return set_err(e, {LANN_DOMAIN_ERROR, "drop fraction must lie in [0,1]"});
  int64_t total = 0;
  int max_len = 1;
  for (int i = 0; i < n_sets; ++i) {
    if (len[i] < 1) return set_err(e, {LANN_DOMAIN_ERROR, "metric needs at least one sample"});
    total = std::max<int64_t>(total, offset[i] + len[i]);
    max_len = std::max(max_len, len[i]);
  }
  try {
    ck(cudaSetDevice(e->device), "cudaSetDevice");
    cudaStream_t s = e->stream;
    Timer timer(e);
    DBuf<int64_t> doff(offset, n_sets, s);
    DBuf<int> dlen(len, n_sets, s), dk(size_t(n_sets), s), dst(size_t(n_sets), s);
    DBuf<double> dt(truth, size_t(total), s), dp(pred, size_t(total), s), dm(size_t(n_sets), s),
        dmt(size_t(n_sets), s), dr(size_t(n_sets), s);
    EvalArgs a{n_sets, doff.p, dlen.p, dt.p, dp.p, drop, dm.p, dmt.p, dk.p, dr.p, dst.p};
    launch_eval(a, max_len, e->max_smem, total, s);
    ck(cudaGetLastError(), "eval launch");
    e->launches += eval_launch_count(max_len, e->max_smem);
    std::vector<int> status(n_sets);
    dm.down(mape);
    dmt.down(mape_thr);
    dk.down(n_kept);
    dr.down(rho);
    dst.down(status.data());
    timer.stop();
    for (int i = 0; i < n_sets; ++i)
      if (status[i]) return set_err(e, {LANN_DOMAIN_ERROR, "metric inputs outside their domain"});
    e->err.clear();
    return LANN_OK;
  } catch (const CudaFail& f) {
    e->err = f.what;
    return LANN_CUDA_ERROR;
  }
}

// ---- mlp.hpp building blocks (mlp_ops.cu) -------------------------------------------------------
extern "C++" {
namespace {
struct MlpHost {
  std::vector<int64_t> dims_off, param_off, row_off, x_off;
  std::vector<int> n_params, row_net;
  int64_t total_dims = 0, total_params = 0, total_rows = 0, total_x = 0;
};

Status plan_mlp(const lann_mlp_batch* b, bool need_y, bool single_output, MlpHost& h) {
  if (!b || b->n_nets < 1 || !b->n_dims || !b->dims || !b->params || !b->n_rows || !b->X)
    return {LANN_PARAM_ERROR, "bad training batch"};
  if (need_y && !b->y) return {LANN_PARAM_ERROR, "bad training batch"};
  for (int k = 0; k < b->n_nets; ++k) {
    const int nd = b->n_dims[k];
    if (nd < 2 || nd > kMaxLayers + 1) return {LANN_PARAM_ERROR, "network depth outside 1..8 layers"};
    const int32_t* d = b->dims + h.total_dims;
    int P = 0;
    for (int l = 0; l < nd; ++l)
      if (d[l] < 1 || d[l] > kMaxMlpWidth) return {LANN_PARAM_ERROR, "network widths must lie in 1..64"};
    for (int l = 0; l + 1 < nd; ++l) P += (d[l] + 1) * d[l + 1];
    if (single_output && d[nd - 1] != 1) return {LANN_PARAM_ERROR, "mse_gradient needs a single output"};
    if (b->n_rows[k] < 1) return {LANN_PARAM_ERROR, "bad training batch"};  // mlp.cpp:66,77
    h.dims_off.push_back(h.total_dims);
    h.param_off.push_back(h.total_params);
    h.n_params.push_back(P);
    h.row_off.push_back(h.total_rows);
    h.x_off.push_back(h.total_x);
    h.row_net.insert(h.row_net.end(), size_t(b->n_rows[k]), k);
    h.total_dims += nd;
    h.total_params += P;
    h.total_rows += b->n_rows[k];
    h.total_x += int64_t(b->n_rows[k]) * d[0];
  }
  return {};
}

// Uploads a batch and runs fn(args, stream) with device views; returns a status.
template <typename Fn>
int with_mlp_batch(lann_engine* e, const lann_mlp_batch* b, bool need_y, bool single_output, Fn&& fn) {
  if (!e) return LANN_NO_DEVICE;
  MlpHost h;
  if (Status st = plan_mlp(b, need_y, single_output, h)) return set_err(e, st);
  try {
    ck(cudaSetDevice(e->device), "cudaSetDevice");
    cudaStream_t s = e->stream;
    Timer timer(e);
    const int n = b->n_nets;
    DBuf<int> dnd(b->n_dims, size_t(n), s), ddims(b->dims, size_t(h.total_dims), s), dnp(h.n_params, s),
        dnr(b->n_rows, size_t(n), s), drn(h.row_net, s);
    DBuf<int64_t> ddo(h.dims_off, s), dpo(h.param_off, s), dro(h.row_off, s), dxo(h.x_off, s);
    DBuf<double> dp(b->params, size_t(h.total_params), s), dX(b->X, size_t(h.total_x), s);
    DBuf<double> dy;
    if (need_y) dy = DBuf<double>(b->y, size_t(h.total_rows), s);
    MlpArgs a{n, dnd.p, ddo.p, ddims.p, dpo.p, dnp.p, dp.p, dro.p, dnr.p, dxo.p, dX.p, dy.p, drn.p, h.total_rows};
    fn(a, h, s);
    ck(cudaGetLastError(), "mlp launch");
    timer.stop();
    e->err.clear();
    return LANN_OK;
  } catch (const CudaFail& f) {
    e->err = f.what;
    return LANN_CUDA_ERROR;
  }
}
}  // namespace
}  // extern "C++"

int lann_mlp_forward(lann_engine* e, const lann_mlp_batch* b, double* out) {
  if (!out) return set_err(e, {LANN_PARAM_ERROR, "null output"});
  return with_mlp_batch(e, b, false, false, [&](const MlpArgs& a, const MlpHost& h, cudaStream_t s) {
    DBuf<double> dout(size_t(h.total_rows), s);
    launch_mlp_forward(a, dout.p, s);
    e->launches += 1;
    dout.down(out);
  });
}

int lann_mse_loss(lann_engine* e, const lann_mlp_batch* b, double* loss) {
  if (!loss) return set_err(e, {LANN_PARAM_ERROR, "null output"});
  return with_mlp_batch(e, b, true, false, [&](const MlpArgs& a, const MlpHost& h, cudaStream_t s) {
    DBuf<double> dfwd(size_t(h.total_rows), s), dl(size_t(a.n_nets), s);
    launch_mlp_loss(a, dfwd.p, dl.p, s);
    e->launches += 2;
    dl.down(loss);
  });
}

int lann_mse_gradient(lann_engine* e, const lann_mlp_batch* b, double* loss, double* grad) {
  if (!loss || !grad) return set_err(e, {LANN_PARAM_ERROR, "null output"});
  return with_mlp_batch(e, b, true, true, [&](const MlpArgs& a, const MlpHost& h, cudaStream_t s) {
    std::vector<int64_t> soff(size_t(a.n_nets));
    int64_t total = 0;
    for (int k = 0; k < a.n_nets; ++k) {
      soff[size_t(k)] = total;
      total += int64_t(h.n_params[size_t(k)] + 1) * b->n_rows[k];
    }
    DBuf<int64_t> dso(soff, s);
    DBuf<double> scratch(size_t(total), s), dl(size_t(a.n_nets), s), dg(size_t(h.total_params), s);
    launch_mlp_grad(a, scratch.p, dso.p, dl.p, dg.p, s);
    e->launches += 1;
    dl.down(loss);
    dg.down(grad);
  });
}

int lann_adam_update(lann_engine* e, int64_t n, double* params, const double* grad, double* m, double* v,
                     int32_t step, double lr, double beta1, double beta2, double epsilon) {
  if (!e) return LANN_NO_DEVICE;
  if (n < 0 || (n > 0 && (!params || !grad || !m || !v))) return set_err(e, {LANN_PARAM_ERROR, "bad Adam buffers"});
  if (step < 1) return set_err(e, {LANN_PARAM_ERROR, "Adam step must be >= 1"});
  try {
    ck(cudaSetDevice(e->device), "cudaSetDevice");
    cudaStream_t s = e->stream;
    Timer timer(e);
    const size_t N = size_t(n);
    DBuf<double> dp(params, N, s), dg(grad, N, s), dm(m, N, s), dv(v, N, s);
    // mlp.cpp:145-146: the bias corrections through the host libm's pow, as the reference
    AdamArgs a{n, dp.p, dg.p, dm.p, dv.p, beta1, beta2, epsilon, lr,
               1.0 - std::pow(beta1, step), 1.0 - std::pow(beta2, step)};
    launch_adam(a, s);
    e->launches += n > 0;
    ck(cudaGetLastError(), "adam launch");
    dp.down(params);
    dm.down(m);
    dv.down(v);
    timer.stop();
    e->err.clear();
    return LANN_OK;
  } catch (const CudaFail& f) {
    e->err = f.what;
    return LANN_CUDA_ERROR;
  }
}

int lann_select_schedule(lann_engine* e, const lann_model_set* ms, uint32_t n_img, int64_t n_cands,
                         const uint32_t* cands, int64_t* chosen, double* chosen_score) {
  if (!e) return LANN_NO_DEVICE;
  if (n_cands < 1) return set_err(e, {LANN_PARAM_ERROR, "select needs at least one candidate"});
  if (!ms || ms->n_models < 1) return set_err(e, {LANN_PARAM_ERROR, "empty model set"});
  if (ms->n_inputs[0] != 6 && ms->n_inputs[0] != 5)
    return set_err(e, {LANN_SCHEMA_ERROR, "variant selection needs a model trained on the blur schema"});
  const int I = ms->n_inputs[0], H1 = ms->h1[0], H2 = ms->h2[0];
  if (H1 < 1 || H1 > 64 || H2 < 0 || H2 > 64) return set_err(e, {LANN_PARAM_ERROR, "bad model shape"});
  const int P = param_count(I, H1, H2);
  try {
    ck(cudaSetDevice(e->device), "cudaSetDevice");
    cudaStream_t s = e->stream;
    Timer timer(e);
    DBuf<uint32_t> dc(cands, size_t(n_cands) * 4, s);
    DBuf<double> dw(ms->params + ms->param_offset[0], size_t(P), s), dn(ms->norm, 18, s);
    const int64_t blocks = (n_cands + 255) / 256;
    DBuf<double> dbs(size_t(blocks), s);
    DBuf<int64_t> dbi(size_t(blocks), s);
    e->launches += select_schedule_launch(n_cands, dc.p, n_img, I, H1, H2, ms->log_target[0], dw.p,
                                          dn.p, dbs.p, dbi.p, s);
    ck(cudaGetLastError(), "select launch");
    ck(cudaMemcpyAsync(chosen, dbi.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaMemcpyAsync(chosen_score, dbs.p, sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
    timer.stop();
    e->err.clear();
    return LANN_OK;
  } catch (const CudaFail& f) {
    e->err = f.what;
    return LANN_CUDA_ERROR;
  }
}

namespace {
Status check_variant_models(const lann_model_set* ms, const int32_t* with_n_thd, int32_t kind, int32_t max_threads,
                            int64_t n_cands) {
  if (!ms || ms->n_models < 1) return {LANN_PARAM_ERROR, "empty model set"};
  if (kind < LANN_MM || kind > LANN_MP) return {LANN_PARAM_ERROR, "variant mapping covers the mm/mv/mc/mp kernels"};
  if (max_threads < 1) return {LANN_PARAM_ERROR, "max_threads must be >= 1"};
  if (n_cands < 1) return {LANN_PARAM_ERROR, "select needs at least one candidate"};
  if (!with_n_thd) return {LANN_PARAM_ERROR, "missing with_n_thd"};
  int max_p = 0;
  for (int m = 0; m < ms->n_models; ++m) {
    const int want = base_feature_count(kind, with_n_thd[m] != 0);
    if (ms->n_inputs[m] != want && ms->n_inputs[m] != want + 1)
      return {LANN_SCHEMA_ERROR, "model schema does not match the candidate kernel"};
    if (ms->h1[m] < 1 || ms->h1[m] > 64 || ms->h2[m] < 0 || ms->h2[m] > 64) return {LANN_PARAM_ERROR, "bad model shape"};
    max_p = std::max(max_p, param_count(ms->n_inputs[m], ms->h1[m], ms->h2[m]));
  }
  if (!select_variants_supported(ms->n_models, max_p))
    return {LANN_PARAM_ERROR, "variant scorer holds at most 32 lightweight models"};
  return {};
}
}  // namespace

int lann_select_variants(lann_engine* e, const lann_model_set* ms, const int32_t* with_n_thd,
                         int32_t kind, int32_t max_threads, uint64_t seed, int64_t first,
                         int64_t n_cands, int32_t* out_idx, double* out_score) {
  if (!e) return LANN_NO_DEVICE;
  if (Status st = check_variant_models(ms, with_n_thd, kind, max_threads, n_cands)) return set_err(e, st);
  try {
    ck(cudaSetDevice(e->device), "cudaSetDevice");
    cudaStream_t s = e->stream;
    const int M = ms->n_models;
    DBuf<int> dI(ms->n_inputs, M, s), dh1(ms->h1, M, s), dh2(ms->h2, M, s), dl(ms->log_target, M, s),
        dt(with_n_thd, M, s), didx(size_t(n_cands), s);
    DBuf<int64_t> dpo(ms->param_offset, M, s);
    DBuf<double> dp(ms->params, size_t(ms->total_params), s), dn(ms->norm, size_t(M) * 18, s),
        dsc(size_t(n_cands), s);
    Timer timer(e);
    ck(cudaEventRecord(e->tr0, s), "event");
    if (ms->precision == LANN_FP32 && !std::getenv("LANN_SELECT_GENERIC") &&
        select_variants_fast_launch(M, kind, max_threads, seed, first, n_cands, ms->n_inputs, ms->h1,
                                    ms->h2, ms->log_target, with_n_thd, ms->param_offset, ms->params,
                                    ms->norm, didx.p, dsc.p, false, nullptr, e->sms, s))
      e->launches += 1;
    else
      e->launches += select_variants_launch(M, ms->precision, kind, max_threads, seed, first, n_cands,
                                            dI.p, dh1.p, dh2.p, dl.p, dt.p, dpo.p, dp.p, dn.p, didx.p,
                                            dsc.p, false, nullptr, e->sms, s);
    ck(cudaGetLastError(), "select_variants launch");
    ck(cudaEventRecord(e->tr1, s), "event");
    didx.down(out_idx);
    dsc.down(out_score);
    timer.stop();
    float kms = 0.f;
    ck(cudaEventElapsedTime(&kms, e->tr0, e->tr1), "elapsed");
    e->last_train_ms = kms;  // the scoring kernel's own device time
    e->err.clear();
    return LANN_OK;
  } catch (const CudaFail& f) {
    e->err = f.what;
    return LANN_CUDA_ERROR;
  }
}

int lann_host_alloc(size_t bytes, void** out) {
  if (!out) return LANN_PARAM_ERROR;
  *out = nullptr;
  if (bytes == 0) return LANN_OK;
  return cudaMallocHost(out, bytes) == cudaSuccess ? LANN_OK : LANN_NO_DEVICE;
}

void lann_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

namespace {
bool is_pinned(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();  // clear the sticky-free error of an unregistered pointer
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}
}  // namespace

int lann_select_variants_compact(lann_engine* e, const lann_model_set* ms, const int32_t* with_n_thd, int32_t kind,
                                 int32_t max_threads, uint64_t seed, int64_t first, int64_t n_cands,
                                 uint8_t* out_idx, float* out_score, int64_t* hist) {
  if (!e) return LANN_NO_DEVICE;
  if (Status st = check_variant_models(ms, with_n_thd, kind, max_threads, n_cands)) return set_err(e, st);
  if (ms->n_models > 255) return set_err(e, {LANN_PARAM_ERROR, "compact indices hold at most 255 models"});
  if (!out_idx && !out_score && !hist) return set_err(e, {LANN_PARAM_ERROR, "no output requested"});
  try {
    ck(cudaSetDevice(e->device), "cudaSetDevice");
    cudaStream_t s = e->stream, cs = e->aux[0];
    const int M = ms->n_models;
    DBuf<int> dI(ms->n_inputs, M, s), dh1(ms->h1, M, s), dh2(ms->h2, M, s), dl(ms->log_target, M, s),
        dt(with_n_thd, M, s);
    DBuf<int64_t> dpo(ms->param_offset, M, s);
    DBuf<double> dp(ms->params, size_t(ms->total_params), s), dn(ms->norm, size_t(M) * 18, s);
    DBuf<unsigned char> didx(out_idx ? size_t(n_cands) : 0, s);
    DBuf<float> dsc(out_score ? size_t(n_cands) : 0, s);
    DBuf<unsigned long long> dh(hist ? size_t(M) : 0, s);
    if (hist) ck(cudaMemsetAsync(dh.p, 0, sizeof(unsigned long long) * size_t(M), s), "memset");
    // chunks: the scoring kernel of chunk k + 1 runs while chunk k is copied out
    // 4 chunks: measured e2e within 2% of 8 while each extra chunk's tail costs ~3% of kernel
    // time; without per-candidate outputs there is nothing to overlap
    int64_t max_chunks = out_idx || out_score ? 4 : 1;
    if (const char* env = std::getenv("LANN_SELECT_CHUNKS")) max_chunks = std::max(1, std::atoi(env));
    const int64_t n_chunks = std::min<int64_t>(max_chunks, std::max<int64_t>(1, n_cands / (1 << 20)));
    const int64_t chunk = (n_cands + n_chunks - 1) / n_chunks;
    const bool pin_idx = is_pinned(out_idx), pin_sc = is_pinned(out_score);
    const size_t row_bytes = (out_idx && !pin_idx ? 1 : 0) + (out_score && !pin_sc ? 4 : 0);
    unsigned char* stage = row_bytes ? pinned_stage(e, size_t(2 * chunk) * row_bytes) : nullptr;
    std::vector<cudaEvent_t> scored(static_cast<size_t>(n_chunks)), copied(static_cast<size_t>(n_chunks));
    for (int64_t k = 0; k < n_chunks; ++k) {
      ck(cudaEventCreateWithFlags(&scored[size_t(k)], cudaEventDisableTiming), "event");
      ck(cudaEventCreateWithFlags(&copied[size_t(k)], cudaEventDisableTiming), "event");
    }
    Timer timer(e);
    ck(cudaEventRecord(e->tr0, s), "event");
    for (int64_t k = 0; k < n_chunks; ++k) {
      const int64_t lo = k * chunk, n = std::min(chunk, n_cands - lo);
      if (n <= 0) break;
      void* pi = out_idx ? static_cast<void*>(didx.p + lo) : nullptr;
      void* ps = out_score ? static_cast<void*>(dsc.p + lo) : nullptr;
      if (ms->precision == LANN_FP32 && !std::getenv("LANN_SELECT_GENERIC") &&
          select_variants_fast_launch(M, kind, max_threads, seed, first + lo, n, ms->n_inputs, ms->h1, ms->h2,
                                      ms->log_target, with_n_thd, ms->param_offset, ms->params, ms->norm, pi, ps,
                                      true, hist ? dh.p : nullptr, e->sms, s))
        e->launches += 1;
      else
        e->launches += select_variants_launch(M, ms->precision, kind, max_threads, seed, first + lo, n, dI.p, dh1.p,
                                              dh2.p, dl.p, dt.p, dpo.p, dp.p, dn.p, pi, ps, true,
                                              hist ? dh.p : nullptr, e->sms, s);
      ck(cudaEventRecord(scored[size_t(k)], s), "event");
    }
    ck(cudaGetLastError(), "select_variants launch");
    ck(cudaEventRecord(e->tr1, s), "event");
    // copies on the side stream: pinned caller buffers directly, pageable ones through two
    // pinned staging slots whose host-side copy overlaps the next chunk's transfer
    unsigned char* slot[2] = {stage, stage ? stage + size_t(chunk) * row_bytes : nullptr};
    for (int64_t k = 0; k < n_chunks; ++k) {
      const int64_t lo = k * chunk, n = std::min(chunk, n_cands - lo);
      if (n <= 0) break;
      ck(cudaStreamWaitEvent(cs, scored[size_t(k)], 0), "wait");
      unsigned char* sl = slot[k & 1];
      if (out_idx) {
        void* dst = pin_idx ? static_cast<void*>(out_idx + lo) : static_cast<void*>(sl);
        ck(cudaMemcpyAsync(dst, didx.p + lo, size_t(n), cudaMemcpyDeviceToHost, cs), "D2H");
      }
      if (out_score) {
        void* dst = pin_sc ? static_cast<void*>(out_score + lo)
                           : static_cast<void*>(sl + (out_idx && !pin_idx ? size_t(n) : 0));
        ck(cudaMemcpyAsync(dst, dsc.p + lo, size_t(n) * 4, cudaMemcpyDeviceToHost, cs), "D2H");
      }
      t_d2h += int64_t(n) * ((out_idx ? 1 : 0) + (out_score ? 4 : 0));
      ck(cudaEventRecord(copied[size_t(k)], cs), "event");
      if (row_bytes && k >= 1) {  // drain chunk k - 1 from its slot while chunk k transfers
        const int64_t plo = (k - 1) * chunk, pn = std::min(chunk, n_cands - plo);
        ck(cudaEventSynchronize(copied[size_t(k - 1)]), "sync");
        unsigned char* ps = slot[(k - 1) & 1];
        if (out_idx && !pin_idx) std::memcpy(out_idx + plo, ps, size_t(pn));
        if (out_score && !pin_sc) std::memcpy(out_score + plo, ps + (out_idx && !pin_idx ? size_t(pn) : 0), size_t(pn) * 4);
      }
      if (row_bytes && k + 1 < n_chunks) ck(cudaEventSynchronize(copied[size_t(k)]), "sync");  // slot reuse
    }
    {  // the last chunk
      const int64_t k = n_chunks - 1, plo = k * chunk, pn = std::min(chunk, n_cands - plo);
      ck(cudaStreamSynchronize(cs), "sync");
      if (row_bytes && pn > 0) {
        unsigned char* ps = slot[k & 1];
        if (out_idx && !pin_idx) std::memcpy(out_idx + plo, ps, size_t(pn));
        if (out_score && !pin_sc) std::memcpy(out_score + plo, ps + (out_idx && !pin_idx ? size_t(pn) : 0), size_t(pn) * 4);
      }
    }
    if (hist) {
      std::vector<unsigned long long> h(static_cast<size_t>(M));
      dh.down(h.data());
      ck(cudaStreamSynchronize(s), "sync");
      for (int m = 0; m < M; ++m) hist[m] = int64_t(h[size_t(m)]);
    }
    timer.stop();
    float kms = 0.f;
    ck(cudaEventElapsedTime(&kms, e->tr0, e->tr1), "elapsed");
    e->last_train_ms = kms;  // the scoring kernels' own device time
    for (int64_t k = 0; k < n_chunks; ++k) {
      cudaEventDestroy(scored[size_t(k)]);
      cudaEventDestroy(copied[size_t(k)]);
    }
    e->err.clear();
    return LANN_OK;
  } catch (const CudaFail& f) {
    e->err = f.what;
    return LANN_CUDA_ERROR;
  }
}

int lann_build_dataset(const lann_world* w, uint64_t seed, int32_t count, double* feats,
                       uint64_t* c, double* runtime, int32_t* n_features) {
  if (!w) return LANN_PARAM_ERROR;
  Dataset ds;
  const Status st = build_dataset(*w, seed, count, ds);
  if (st) return st.code;
  std::memcpy(feats, ds.feats.data(), ds.feats.size() * sizeof(double));
  std::memcpy(c, ds.c.data(), ds.c.size() * sizeof(uint64_t));
  std::memcpy(runtime, ds.runtime.data(), ds.runtime.size() * sizeof(double));
  *n_features = ds.n_features;
  return LANN_OK;
}

int lann_measure(lann_engine* e, int32_t kind, const char* variant, int32_t n, const double* feats,
                 int32_t warmups, int32_t reps, uint64_t seed, double* runtime_s, double* checksum) {
  if (!e) return LANN_NO_DEVICE;
  if (n < 0 || (n > 0 && (!feats || !runtime_s))) return set_err(e, {LANN_PARAM_ERROR, "bad measurement request"});
  e->err.clear();
  try {
    ck(cudaSetDevice(e->device), "cudaSetDevice");
    Timer timer(e);
    const int st =
        measure_instances(kind, variant, n, feats, warmups, reps, seed, runtime_s, checksum, e->stream, e->err);
    timer.stop();
    return st;
  } catch (const CudaFail& f) {
    e->err = f.what;
    return LANN_CUDA_ERROR;
  }
}

int lann_measure_variant_count(int32_t kind) { return measure_variant_count(kind); }
const char* lann_measure_variant_name(int32_t kind, int32_t idx) { return measure_variant_name(kind, idx); }

int lann_build_measured_dataset(lann_engine* e, int32_t kind, const char* variant, int32_t blur_lattice,
                                int32_t blur_side, int32_t count, uint64_t seed, int32_t warmups, int32_t reps,
                                double* feats, uint64_t* c, double* runtime, int32_t* n_features) {
  if (!e) return LANN_NO_DEVICE;
  if (count < 2 || kind < LANN_MM || kind > LANN_BLUR || !feats || !c || !runtime || !n_features)
    return set_err(e, {LANN_PARAM_ERROR, "build_dataset needs count >= 2 and output buffers"});
  // sample_params draws of the GPU-class parameter space (datagen.cpp:60-110, n_thd pinned)
  SeqRng rng(derive_seed(seed, 0));
  std::vector<double> f(size_t(count) * LANN_ROW, 0.0);
  for (int i = 0; i < count; ++i) {
    Instance p = sample_instance(kind, 1, blur_lattice, rng);
    p.n_thd = 1;
    if (kind == LANN_BLUR && blur_side > 0) p.n = uint32_t(blur_side);
    base_features(p, false, &f[size_t(i) * LANN_ROW]);
    c[i] = complexity(p);
  }
  const int st = lann_measure(e, kind, variant, count, f.data(), warmups, reps, seed, runtime, nullptr);
  if (st) return st;
  std::memcpy(feats, f.data(), f.size() * sizeof(double));
  *n_features = base_feature_count(kind, false);
  return LANN_OK;
}

// ---- baseline families -------------------------------------------------------------------------
namespace {
Status check_design(const lann_design* d, int max_feats) {
  if (!d || d->n_models < 1 || !d->n_rows || !d->n_feats || !d->row_offset || !d->X || !d->y)
    return {LANN_PARAM_ERROR, "empty design"};
  for (int m = 0; m < d->n_models; ++m) {
    if (d->n_rows[m] < 2) return {LANN_PARAM_ERROR, "training needs at least 2 samples"};
    if (d->n_feats[m] < 1 || d->n_feats[m] > max_feats) return {LANN_PARAM_ERROR, "design columns out of range"};
    if (d->row_offset[m] < 0) return {LANN_PARAM_ERROR, "bad row offset"};
  }
  return {};
}
int64_t design_rows(const lann_design* d) {
  int64_t r = 0;
  for (int m = 0; m < d->n_models; ++m) r = std::max<int64_t>(r, d->row_offset[m] + d->n_rows[m]);
  return r;
}
}  // namespace

int lann_fit_linear(lann_engine* e, const lann_design* d, double ridge, double* weights, double* intercept,
                    int32_t* status) {
  if (!e) return LANN_NO_DEVICE;
  if (Status st = check_design(d, LANN_ROW)) return set_err(e, st);
  if (!weights || !intercept || !status) return set_err(e, {LANN_PARAM_ERROR, "missing output buffers"});
  try {
    ck(cudaSetDevice(e->device), "cudaSetDevice");
    Timer timer(e);
    cudaStream_t s = e->stream;
    const int M = d->n_models;
    const int64_t rows = design_rows(d);
    DBuf<int> dn(d->n_rows, size_t(M), s), df(d->n_feats, size_t(M), s), dst(size_t(M), s);
    DBuf<int64_t> doff(d->row_offset, size_t(M), s);
    DBuf<double> dX(d->X, size_t(rows) * LANN_ROW, s), dY(d->y, size_t(rows), s);
    DBuf<double> dW(size_t(M) * LANN_ROW, s), dI(size_t(M), s);
    launch_fit_linear({M, dn.p, df.p, doff.p, dX.p, dY.p, ridge, dW.p, dI.p, dst.p}, s);
    ck(cudaGetLastError(), "fit_linear launch");
    e->launches += 1;
    dW.down(weights);
    dI.down(intercept);
    dst.down(status);
    timer.stop();
    for (int m = 0; m < M; ++m) status[m] = status[m] ? LANN_DOMAIN_ERROR : LANN_OK;
    for (int m = 0; m < M; ++m)
      if (status[m]) return set_err(e, {LANN_DOMAIN_ERROR, "singular design matrix despite ridge"});
    return LANN_OK;
  } catch (const CudaFail& f) {
    e->err = f.what;
    return LANN_CUDA_ERROR;
  }
}

int lann_predict_linear(lann_engine* e, int32_t M, const int32_t* n_feats, const double* weights,
                        const double* intercept, int64_t n_rows, const double* rows, const int32_t* row_model,
                        double* out) {
  if (!e) return LANN_NO_DEVICE;
  if (M < 1 || !n_feats || !weights || !intercept || n_rows < 0 || (n_rows && (!rows || !row_model || !out)))
    return set_err(e, {LANN_PARAM_ERROR, "bad linear prediction request"});
  for (int64_t r = 0; r < n_rows; ++r)
    if (row_model[r] < 0 || row_model[r] >= M) return set_err(e, {LANN_PARAM_ERROR, "row model out of range"});
  try {
    ck(cudaSetDevice(e->device), "cudaSetDevice");
    Timer timer(e);
    cudaStream_t s = e->stream;
    DBuf<int> df(n_feats, size_t(M), s), dm(row_model, size_t(n_rows), s);
    DBuf<double> dW(weights, size_t(M) * LANN_ROW, s), dI(intercept, size_t(M), s);
    DBuf<double> dR(rows, size_t(n_rows) * LANN_ROW, s), dO(size_t(n_rows), s);
    launch_predict_linear({n_rows, dR.p, dm.p, df.p, dW.p, dI.p, dO.p}, s);
    ck(cudaGetLastError(), "predict_linear launch");
    e->launches += n_rows > 0;
    dO.down(out);
    timer.stop();
    return LANN_OK;
  } catch (const CudaFail& f) {
    e->err = f.what;
    return LANN_CUDA_ERROR;
  }
}

int lann_fit_forest(lann_engine* e, const lann_design* d, int32_t trees, int32_t max_depth,
                    int32_t min_samples_split, const uint64_t* seeds, int32_t* node_feature, double* node_threshold,
                    int32_t* node_left, int32_t* node_right, double* node_value, int32_t* node_count) {
  if (!e) return LANN_NO_DEVICE;
  if (Status st = check_design(d, LANN_ROW)) return set_err(e, st);
  if (trees < 1 || max_depth < 1) return set_err(e, {LANN_PARAM_ERROR, "forest needs trees >= 1 and max_depth >= 1"});
  if (!seeds || !node_feature || !node_threshold || !node_left || !node_right || !node_value || !node_count)
    return set_err(e, {LANN_PARAM_ERROR, "missing forest buffers"});
  const int M = d->n_models;
  int max_rows = 0;
  for (int m = 0; m < M; ++m) {
    if (d->n_rows[m] < 10) return set_err(e, {LANN_PARAM_ERROR, "forest needs at least 10 samples"});
    max_rows = std::max(max_rows, d->n_rows[m]);
  }
  if (max_rows > 65535)  // slot lists are 16-bit
    return set_err(e, {LANN_PARAM_ERROR, "forest training set above 65535 samples"});
  const bool ws_global = forest_smem_bytes(max_rows) > size_t(e->max_smem);
  // bootstraps (forest.cpp:132-136): Rng(derive_seed(seed, t)).bounded(n) x n, sorted
  std::vector<uint16_t> boot(size_t(M) * trees * max_rows, 0);
  parallel_for(M * trees, [&](int k) {
    const int m = k / trees, t = k % trees, n = d->n_rows[m];
    SeqRng rng(derive_seed(seeds[m], uint64_t(t)));
    uint16_t* b = &boot[size_t(k) * max_rows];
    for (int i = 0; i < n; ++i) b[i] = uint16_t(rng.bounded(uint64_t(n)));
    std::sort(b, b + n);
  });
  const size_t npt = size_t(2) * max_rows, total = size_t(M) * trees * npt;
  try {
    ck(cudaSetDevice(e->device), "cudaSetDevice");
    Timer timer(e);
    cudaStream_t s = e->stream;
    const int64_t rows = design_rows(d);
    DBuf<int> dn(d->n_rows, size_t(M), s), df(d->n_feats, size_t(M), s);
    DBuf<int64_t> doff(d->row_offset, size_t(M), s);
    DBuf<double> dX(d->X, size_t(rows) * LANN_ROW, s), dY(d->y, size_t(rows), s);
    DBuf<uint16_t> dB(boot, s);
    DBuf<int> nf(total, s), nl(total, s), nr(total, s), nc(size_t(M) * trees, s);
    DBuf<double> nt(total, s), nv(total, s);
    DBuf<double> ss(size_t(M) * trees * max_rows * LANN_ROW, s), sth(size_t(M) * trees * max_rows * LANN_ROW, s);
    ForestArgs fa{M, trees, max_depth, min_samples_split, max_rows, dn.p, df.p, doff.p, dX.p, dY.p, dB.p,
                  nf.p, nt.p, nl.p, nr.p, nv.p, nc.p, ss.p, sth.p};
    DBuf<unsigned char> ws;
    if (ws_global) {  // per-(model, tree) working set in HBM instead of shared memory
      fa.ws_stride = (forest_smem_bytes(max_rows) + 255) & ~size_t(255);
      ws = DBuf<unsigned char>(size_t(M) * trees * fa.ws_stride, s);
      fa.scratch_ws = ws.p;
    }
    launch_fit_forest(fa, s);
    ck(cudaGetLastError(), "fit_forest launch");
    e->launches += 1;
    std::vector<int> bf(total), bl(total), br(total), bc(size_t(M) * trees);
    std::vector<double> bt(total), bv(total);
    nf.down(bf.data());
    nl.down(bl.data());
    nr.down(br.data());
    nc.down(bc.data());
    nt.down(bt.data());
    nv.down(bv.data());
    timer.stop();
    // breadth-first -> the reference's depth-first preorder (Builder::build, forest.cpp:96-121)
    parallel_for(M * trees, [&](int k) {
      const size_t base = size_t(k) * npt;
      std::vector<int> stack = {0}, order;
      std::vector<int> newid(size_t(bc[size_t(k)]), -1);
      while (!stack.empty()) {
        const int v = stack.back();
        stack.pop_back();
        newid[size_t(v)] = int(order.size());
        order.push_back(v);
        if (bf[base + v] >= 0) {
          stack.push_back(br[base + v]);
          stack.push_back(bl[base + v]);
        }
      }
      for (size_t i = 0; i < npt; ++i) {
        const size_t o = base + i;
        if (i < order.size()) {
          const size_t src = base + size_t(order[i]);
          node_feature[o] = bf[src];
          node_threshold[o] = bt[src];
          node_left[o] = bf[src] >= 0 ? newid[size_t(bl[src])] : -1;
          node_right[o] = bf[src] >= 0 ? newid[size_t(br[src])] : -1;
          node_value[o] = bv[src];
        } else {
          node_feature[o] = node_left[o] = node_right[o] = -1;
          node_threshold[o] = node_value[o] = 0.0;
        }
      }
      node_count[k] = bc[size_t(k)];
    });
    return LANN_OK;
  } catch (const CudaFail& f) {
    e->err = f.what;
    return LANN_CUDA_ERROR;
  }
}

int lann_predict_forest(lann_engine* e, int32_t M, int32_t trees, int32_t npt, const int32_t* node_feature,
                        const double* node_threshold, const int32_t* node_left, const int32_t* node_right,
                        const double* node_value, int64_t n_rows, const double* rows, const int32_t* row_model,
                        double* out) {
  if (!e) return LANN_NO_DEVICE;
  if (M < 1 || trees < 1 || npt < 1 || !node_feature || !node_threshold || !node_left || !node_right ||
      !node_value || n_rows < 0 || (n_rows && (!rows || !row_model || !out)))
    return set_err(e, {LANN_PARAM_ERROR, "bad forest prediction request"});
  for (int64_t r = 0; r < n_rows; ++r)
    if (row_model[r] < 0 || row_model[r] >= M) return set_err(e, {LANN_PARAM_ERROR, "row model out of range"});
  const size_t total = size_t(M) * trees * npt;
  for (size_t i = 0; i < total; ++i)  // a malformed tree must not send the GPU walk off the arrays
    if (node_feature[i] >= LANN_ROW || (node_feature[i] >= 0 && (node_left[i] < 0 || node_left[i] >= npt ||
                                                                 node_right[i] < 0 || node_right[i] >= npt)))
      return set_err(e, {LANN_PARAM_ERROR, "malformed forest node"});
  try {
    ck(cudaSetDevice(e->device), "cudaSetDevice");
    Timer timer(e);
    cudaStream_t s = e->stream;
    DBuf<int> df(node_feature, total, s), dl(node_left, total, s), dr(node_right, total, s);
    DBuf<double> dt(node_threshold, total, s), dv(node_value, total, s);
    DBuf<int> dm(row_model, size_t(n_rows), s);
    DBuf<double> dR(rows, size_t(n_rows) * LANN_ROW, s), dO(size_t(n_rows), s);
    launch_predict_forest({n_rows, dR.p, dm.p, trees, npt, df.p, dt.p, dl.p, dr.p, dv.p, dO.p}, s);
    ck(cudaGetLastError(), "predict_forest launch");
    e->launches += n_rows > 0;
    dO.down(out);
    timer.stop();
    return LANN_OK;
  } catch (const CudaFail& f) {
    e->err = f.what;
    return LANN_CUDA_ERROR;
  }
}

int lann_build_mock_dataset(int32_t kind, int32_t single_threaded, int32_t max_threads, uint32_t dim_max,
                            int32_t n_sides, const uint32_t* sides, int32_t blur_lattice, int32_t count,
                            uint64_t seed, double* feats, uint64_t* c, double* runtime, int32_t* n_features) {
  if (!feats || !c || !runtime || !n_features || n_sides < 0 || (n_sides > 0 && !sides)) return LANN_PARAM_ERROR;
  SampleSpace sp;
  sp.kind = kind;
  sp.max_threads = max_threads;
  sp.gpu_lattice = blur_lattice;
  sp.dim_max = dim_max;
  if (n_sides > 0) sp.sides.assign(sides, sides + n_sides);
  Dataset ds;
  const Status st = build_mock_dataset(sp, single_threaded != 0, seed, count, ds);
  if (st) return st.code;
  std::memcpy(feats, ds.feats.data(), ds.feats.size() * sizeof(double));
  std::memcpy(c, ds.c.data(), ds.c.size() * sizeof(uint64_t));
  std::memcpy(runtime, ds.runtime.data(), ds.runtime.size() * sizeof(double));
  *n_features = ds.n_features;
  return LANN_OK;
}

int lann_mock_schedules(uint32_t image_n, int32_t n_thd, int32_t n, const uint32_t* sched, double* runtime) {
  if (n < 0 || (n > 0 && (!sched || !runtime)) || image_n == 0) return LANN_PARAM_ERROR;
  for (int i = 0; i < n; ++i) {
    Instance p;
    p.kind = LANN_BLUR;
    p.n = image_n;
    p.n_thd = n_thd;
    for (int j = 0; j < 4; ++j) p.sched[j] = sched[4 * i + j];
    runtime[i] = mock_runtime(p);
  }
  return LANN_OK;
}

int lann_probe_schedules(const lann_world* w, uint64_t seed, uint32_t image_n, int32_t n,
                         const uint32_t* sched, double* runtime) {
  if (!w || (n > 0 && (!sched || !runtime))) return LANN_PARAM_ERROR;
  return probe_schedules(*w, seed, image_n, n, sched, runtime).code;
}

int lann_split_order(int32_t n, uint64_t seed, int64_t* order) {
  std::vector<int64_t> o;
  int ntr = 0;
  const Status st = split_order(n, 0.5, seed, o, ntr);
  if (st) return st.code;
  std::memcpy(order, o.data(), o.size() * sizeof(int64_t));
  return LANN_OK;
}

int lann_init_params(int32_t n_dims, const int32_t* dims, uint64_t seed, double* params) {
  if (n_dims != 3 && n_dims != 4) return LANN_PARAM_ERROR;
  for (int i = 0; i < n_dims; ++i)
    if (dims[i] < 1) return LANN_PARAM_ERROR;
  if (dims[n_dims - 1] != 1) return LANN_PARAM_ERROR;
  glorot_init(dims[0], dims[1], n_dims == 4 ? dims[2] : 0, seed, params);
  return LANN_OK;
}

namespace {
int population_create(lann_engine* e, int32_t n_jobs, const lann_job* jobs, int32_t precision,
                      int32_t record_trace, lann_population** out, bool sync_uploads,
                      std::vector<lann_job_result>* base_out = nullptr);
// a device pass that failed (CUDA error): every job reports the failure (jobs that failed host
// preparation keep their own status)
void fail_results(const Population& pop, int rc, lann_job_result* results) {
  for (int j = 0; j < pop.n_jobs; ++j) {
    results[j] = pop.base[size_t(j)];
    if (results[j].status == LANN_OK) results[j].status = rc;
  }
}
}

int lann_population_create(lann_engine* e, int32_t n_jobs, const lann_job* jobs,
                           int32_t precision, int32_t record_trace, lann_population** out) {
  return population_create(e, n_jobs, jobs, precision, record_trace, out, true);
}

namespace {
int population_create(lann_engine* e, int32_t n_jobs, const lann_job* jobs, int32_t precision,
                      int32_t record_trace, lann_population** out, bool sync_uploads,
                      std::vector<lann_job_result>* base_out) {
  if (!e) return LANN_NO_DEVICE;
  if (!out || n_jobs < 1 || !jobs) return set_err(e, {LANN_PARAM_ERROR, "empty population"});
  if (precision != LANN_FP64_EXACT && precision != LANN_FP32)
    return set_err(e, {LANN_PARAM_ERROR, "unknown precision"});
  *out = nullptr;
  auto* p = new lann_population;
  try {
    ck(cudaSetDevice(e->device), "cudaSetDevice");
    const int st = prepare_population(e, n_jobs, jobs, precision, record_trace != 0, p->pop, sync_uploads);
    // any failure that left no launch plan is fatal for the whole population (M == 0: every job
    // failed host preparation; M > 0: a population-wide check after packing failed)
    if (st != LANN_OK && !p->pop.plan) {
      if (base_out && p->pop.M == 0) *base_out = p->pop.base;  // the per-job statuses
      delete p;
      return st;
    }
  } catch (const CudaFail& f) {
    delete p;
    e->err = f.what;
    return LANN_CUDA_ERROR;
  }
  pop_register(p);
  *out = p;
  return LANN_OK;
}
}  // namespace

int lann_population_run(lann_population* p, int32_t n_steps) {
  if (!p) return LANN_PARAM_ERROR;
  lann_engine* e = p->pop.e;
  try {
    ck(cudaSetDevice(e->device), "cudaSetDevice");
    Timer timer(e);
    double train_ms = 0.0;
    for (int i = 0; i < std::max(1, n_steps); ++i) {
      run_device(p->pop);
      float tms = 0.f;
      ck(cudaEventSynchronize(e->tr1), "sync");
      ck(cudaEventElapsedTime(&tms, e->tr0, e->tr1), "elapsed");
      train_ms += tms;
    }
    timer.stop();
    e->last_train_ms = train_ms;
    return LANN_OK;
  } catch (const CudaFail& f) {
    e->err = f.what;
    return LANN_CUDA_ERROR;
  }
}

int lann_population_fetch(lann_population* p, lann_job_result* results, double* params_out,
                          const int64_t* params_offset, double* trace_out,
                          const int64_t* trace_offset) {
  if (!p || !results) return LANN_PARAM_ERROR;
  try {
    ck(cudaSetDevice(p->pop.e->device), "cudaSetDevice");
    return fetch_population(p->pop, results, params_out, params_offset, trace_out, trace_offset);
  } catch (const CudaFail& f) {
    p->pop.e->err = f.what;
    return LANN_CUDA_ERROR;
  }
}

void lann_transfer_bytes(int64_t* h2d, int64_t* d2h, int32_t reset) {
  if (h2d) *h2d = t_h2d;
  if (d2h) *d2h = t_d2h;
  if (reset) t_h2d = t_d2h = 0;
}

int lann_population_norm(const lann_population* p, double* norm_out) {
  if (!p || !norm_out) return LANN_PARAM_ERROR;
  const Population& pop = p->pop;
  std::memset(norm_out, 0, sizeof(double) * 18 * size_t(pop.n_jobs));
  std::vector<double> norm(size_t(pop.M) * 18);
  if (pop.M) {
    pop.dN.down(norm.data());
    cudaStreamSynchronize(pop.e->stream);
  }
  for (int m = 0; m < pop.M; ++m)
    std::memcpy(norm_out + 18 * size_t(pop.model_job[m]), &norm[18 * size_t(m)], 18 * sizeof(double));
  return LANN_OK;
}

int lann_cv_layout(int32_t n_jobs, const lann_job* jobs, int32_t* n_groups, int32_t* n_ensembles) {
  if (n_jobs < 0 || (n_jobs > 0 && !jobs)) return LANN_PARAM_ERROR;
  const CvLayout L = cv_layout(n_jobs, jobs);
  if (n_groups) *n_groups = L.n_groups();
  if (n_ensembles) *n_ensembles = L.n_ens();
  return LANN_OK;
}

int lann_population_cv_count(const lann_population* p, int32_t* n_groups, int32_t* n_ensembles) {
  if (!p) return LANN_PARAM_ERROR;
  const CvState* cv = p->pop.cv.get();
  if (n_groups) *n_groups = cv ? cv->L.n_groups() : 0;
  if (n_ensembles) *n_ensembles = cv ? cv->L.n_ens() : 0;
  return LANN_OK;
}

int lann_population_cv(lann_population* p, lann_cv_group* groups, lann_cv_ensemble* ensembles) {
  if (!p) return LANN_PARAM_ERROR;
  Population& pop = p->pop;
  const CvState* cv = pop.cv.get();
  if (!cv) return LANN_OK;  // no k-fold jobs: nothing to summarise
  try {
    ck(cudaSetDevice(pop.e->device), "cudaSetDevice");
    std::vector<unsigned char> hr(cv->res_bytes);
    if (cv->res_bytes) {
      ck(cudaMemcpyAsync(hr.data(), pop.blob.p + cv->res_off, cv->res_bytes, cudaMemcpyDeviceToHost, pop.e->stream),
         "D2H");
      t_d2h += int64_t(cv->res_bytes);
    }
    ck(cudaStreamSynchronize(pop.e->stream), "cv fetch");
    auto D = [&](size_t off) { return reinterpret_cast<const double*>(hr.data() + off); };
    auto I = [&](size_t off) { return reinterpret_cast<const int*>(hr.data() + off); };
    const double *mape = D(cv->r_mape), *thr = D(cv->r_thr), *rho = D(cv->r_rho);
    const double *sf = D(cv->r_sf), *se = D(cv->r_se);
    const int *kept = I(cv->r_kept), *est = I(cv->r_st), *bad = I(cv->r_bad), *nf = I(cv->r_nf), *ne = I(cv->r_ne);
    const int G = cv->L.n_groups(), E = cv->L.n_ens();
    std::vector<int> group_test(size_t(G), 0);
    for (int en = 0; en < E; ++en) {
      const int slot = cv->dev_of[size_t(en)];
      lann_cv_ensemble r{};
      r.group = cv->L.ens_group[size_t(en)];
      r.init_seed = cv->L.ens_seed[size_t(en)];
      r.n_test = cv->ens_test[size_t(en)];
      if (slot < 0) {
        r.status = cv->host_status[size_t(en)];
      } else if (bad[slot] >= 0) {  // a member diverged or had no held-out metrics
        r.status = (bad[slot] & 1) ? LANN_DOMAIN_ERROR : LANN_TRAINING_ERROR;
      } else {
        r.status = est[slot] ? LANN_DOMAIN_ERROR : LANN_OK;
        r.mape = mape[slot];
        r.mape_thr = thr[slot];
        r.rho = rho[slot];
        r.n_kept = kept[slot];
      }
      if (slot >= 0) group_test[size_t(r.group)] = r.n_test;
      if (ensembles) ensembles[en] = r;
    }
    if (groups)
      for (int g = 0; g < G; ++g) {
        lann_cv_group& o = groups[g];
        o = lann_cv_group{};
        o.first_job = cv->L.group_first[size_t(g)];
        o.n_folds = cv->L.group_folds[size_t(g)];
        o.n_models = cv->L.group_models[size_t(g)];
        o.n_models_ok = nf[g];
        o.n_ensembles = cv->L.group_ens[size_t(g)];
        o.n_ensembles_ok = ne[g];
        o.n_test = group_test[size_t(g)];
        const double* a = sf + 6 * size_t(g);
        const double* b = se + 6 * size_t(g);
        o.fold_mape = {a[0], a[1]};
        o.fold_mape_thr = {a[2], a[3]};
        o.fold_rho = {a[4], a[5]};
        o.test_mape = {b[0], b[1]};
        o.test_mape_thr = {b[2], b[3]};
        o.test_rho = {b[4], b[5]};
      }
    return LANN_OK;
  } catch (const CudaFail& f) {
    pop.e->err = f.what;
    return LANN_CUDA_ERROR;
  }
}

double lann_population_flop(const lann_population* p) { return p ? p->pop.train_flop : 0.0; }
int64_t lann_population_models(const lann_population* p) { return p ? p->pop.M : 0; }

void lann_population_destroy(lann_population* p) {
  if (!p || !pop_unregister(p)) return;  // not live: destroyed already, or with its engine
  pop_free(p);
}

// One-shot pipeline = create + one device pass + fetch, timed as a whole.
int lann_run_population(lann_engine* e, int32_t n_jobs, const lann_job* jobs, int32_t precision,
                        lann_job_result* results, double* params_out,
                        const int64_t* params_offset, double* trace_out,
                        const int64_t* trace_offset) {
  if (!e) return LANN_NO_DEVICE;
  if (!results) return set_err(e, {LANN_PARAM_ERROR, "null results"});
  lann_population* p = nullptr;
  std::vector<lann_job_result> base;
  const int st = population_create(e, n_jobs, jobs, precision, trace_out != nullptr, &p, false, &base);
  if (!p) {
    for (int j = 0; j < n_jobs && jobs; ++j) {
      if (size_t(j) < base.size()) {  // every job failed host preparation: its own status
        results[j] = base[j];
        continue;
      }
      std::memset(&results[j], 0, sizeof(lann_job_result));
      results[j].status = st;
      results[j].nonfinite_epoch = -1;
      results[j].precision_run = -1;
    }
    return st;
  }
  int rc = lann_population_run(p, 1);
  if (rc == LANN_OK) rc = lann_population_fetch(p, results, params_out, params_offset, trace_out, trace_offset);
  else fail_results(p->pop, rc, results);
  lann_population_destroy(p);
  return rc;
}

int lann_default_combos(lann_world* out, int32_t cap) {
  const auto combos = default_combos();
  const int n = int(combos.size());
  for (int i = 0; i < n && i < cap; ++i) out[i] = combos[i];
  return n;
}

}  // extern "C"

// ---- multi-GPU populations: one engine and one host thread per device ---------------------------
struct lann_group {
  std::vector<lann_engine*> engines;
  std::string err;
  double last_device_ms = 0.0, last_wall_ms = 0.0;
};

namespace {
// the sharding cost of a job: epochs x train rows x parameters (paper_2003_07497_b200/sharding.py)
double job_cost(const lann_job& j) {
  int n_train = int(std::llround(double(j.count) * j.train_fraction));
  if (j.n_folds >= 2) n_train -= n_train / j.n_folds;
  static const int base[5] = {5, 3, 4, 5, 5};  // features per kind without n_thd and c
  const int k = j.world.kind >= 0 && j.world.kind < 5 ? j.world.kind : 0;
  const int I = base[k] + (j.world.hw_class == LANN_HW_CPU && j.world.kind != LANN_BLUR ? 1 : 0) +
                (j.family == LANN_NNC ? 1 : 0);
  const int h1 = std::max(1, j.hidden[0]), h2 = j.n_hidden > 1 ? std::max(1, j.hidden[1]) : 0;
  const double p = h2 ? double((I + 1) * h1 + (h1 + 1) * h2 + h2 + 1) : double((I + 1) * h1 + h1 + 1);
  return double(j.epochs) * double(std::max(0, n_train)) * p;
}

// adjacent jobs of one cross-validation ensemble (same group, same init seed) are never cut apart
bool same_ensemble(const lann_job& a, const lann_job& b) {
  return a.n_folds >= 2 && b.n_folds >= 2 && a.init_seed == b.init_seed && cv_group_key(a) == cv_group_key(b);
}

void shard_bounds(int n_jobs, const lann_job* jobs, int world, int32_t* b) {
  double total = 0.0;
  for (int i = 0; i < n_jobs; ++i) total += job_cost(jobs[i]);
  int r = 1, nb = 1;
  b[0] = 0;
  double acc = 0.0;
  for (int i = 0; i < n_jobs; ++i) {
    acc += job_cost(jobs[i]);
    while (r < world && acc >= total * r / world) {
      b[nb++] = i + 1;
      ++r;
    }
  }
  while (nb < world) b[nb++] = n_jobs;
  b[world] = n_jobs;
  for (int w = 1; w < world; ++w) {  // snap each cut forward to the end of the ensemble it splits
    int c = std::max(b[w], b[w - 1]);
    while (c > 0 && c < n_jobs && same_ensemble(jobs[c - 1], jobs[c])) ++c;
    b[w] = c;
  }
}
}  // namespace

int lann_group_create(int32_t n_devices, const int32_t* devices, lann_group** out) {
  if (!out || n_devices < 1 || !devices) return LANN_PARAM_ERROR;
  *out = nullptr;
  auto* g = new lann_group;
  for (int i = 0; i < n_devices; ++i) {
    lann_engine* e = nullptr;
    const int st = lann_engine_create(devices[i], &e);
    if (st) {
      for (lann_engine* x : g->engines) lann_engine_destroy(x);
      delete g;
      return st;
    }
    g->engines.push_back(e);
  }
  *out = g;
  return LANN_OK;
}

void lann_group_destroy(lann_group* g) {
  if (!g) return;
  for (lann_engine* e : g->engines) lann_engine_destroy(e);
  delete g;
}

const char* lann_group_last_error(const lann_group* g) { return g ? g->err.c_str() : "no group"; }
int32_t lann_group_size(const lann_group* g) { return g ? int32_t(g->engines.size()) : 0; }
double lann_group_last_device_ms(const lann_group* g) { return g ? g->last_device_ms : 0.0; }
double lann_group_last_wall_ms(const lann_group* g) { return g ? g->last_wall_ms : 0.0; }

int lann_shard_bounds(int32_t n_shards, int32_t n_jobs, const lann_job* jobs, int32_t* bounds) {
  if (n_shards < 1 || !bounds || n_jobs < 0 || (n_jobs > 0 && !jobs)) return LANN_PARAM_ERROR;
  shard_bounds(n_jobs, jobs, n_shards, bounds);
  return LANN_OK;
}

int lann_group_shard_bounds(const lann_group* g, int32_t n_jobs, const lann_job* jobs, int32_t* bounds) {
  if (!g || !bounds || n_jobs < 0 || (n_jobs > 0 && !jobs)) return LANN_PARAM_ERROR;
  shard_bounds(n_jobs, jobs, int(g->engines.size()), bounds);
  return LANN_OK;
}

int lann_group_run_population(lann_group* g, int32_t n_jobs, const lann_job* jobs, int32_t precision,
                              lann_job_result* results, double* params_out, const int64_t* params_offset,
                              double* trace_out, const int64_t* trace_offset) {
  if (!g) return LANN_NO_DEVICE;
  if (!results || !jobs || n_jobs < 1) {
    g->err = "empty population";
    return LANN_PARAM_ERROR;
  }
  const int W = int(g->engines.size());
  std::vector<int32_t> b(size_t(W) + 1);
  shard_bounds(n_jobs, jobs, W, b.data());
  std::vector<int> st(size_t(W), LANN_OK);
  std::vector<double> dev_ms(size_t(W), 0.0);
  std::vector<int64_t> h2d(size_t(W), 0), d2h(size_t(W), 0);
  const auto t0 = std::chrono::steady_clock::now();
  auto work = [&](int w) {
    const int lo = b[size_t(w)], n = b[size_t(w) + 1] - lo;
    if (n <= 0) return;
    lann_transfer_bytes(nullptr, nullptr, 1);
    // offsets are absolute indices into the caller's arrays: pass them shifted, the bases as is
    st[size_t(w)] = lann_run_population(g->engines[size_t(w)], n, jobs + lo, precision, results + lo, params_out,
                                        params_offset ? params_offset + lo : nullptr, trace_out,
                                        trace_offset ? trace_offset + lo : nullptr);
    dev_ms[size_t(w)] = lann_last_device_ms(g->engines[size_t(w)]);
    lann_transfer_bytes(&h2d[size_t(w)], &d2h[size_t(w)], 1);
  };
  std::vector<std::thread> threads;
  for (int w = 1; w < W; ++w) threads.emplace_back(work, w);
  work(0);
  for (auto& t : threads) t.join();
  g->last_wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  g->last_device_ms = *std::max_element(dev_ms.begin(), dev_ms.end());
  for (int w = 0; w < W; ++w) {  // the caller's thread accounts for every shard's copies
    t_h2d += h2d[size_t(w)];
    t_d2h += d2h[size_t(w)];
  }
  g->err.clear();
  int rc = LANN_OK;
  for (int w = 0; w < W; ++w)
    if (st[size_t(w)] != LANN_OK && rc == LANN_OK) {
      rc = st[size_t(w)];
      g->err = std::string("device ") + std::to_string(g->engines[size_t(w)]->device) + ": " +
               lann_last_error(g->engines[size_t(w)]);
    }
  return rc;
}

// ---- cross-validation statistics from host results (multi-device / multi-process merges) ------
namespace {
Status cv_group_stats(lann_engine* e, int n_jobs, const lann_job* jobs, const lann_job_result* results,
                      const lann_cv_ensemble* ensembles, lann_cv_group* groups) {
  const CvLayout L = cv_layout(n_jobs, jobs);
  const int G = L.n_groups(), E = L.n_ens();
  if (G == 0) return {};
  // items: fold models (job order) and ensembles (ensemble order) of every group; their metrics
  // and statuses packed beside them (bad = -1: the statuses carry every failure)
  std::vector<int64_t> fo(static_cast<size_t>(G)), eo(static_cast<size_t>(G));
  std::vector<int> fl(size_t(G), 0), el(size_t(G), 0), fi, ei;
  std::vector<std::vector<int>> fg(static_cast<size_t>(G)), eg(static_cast<size_t>(G));
  for (int j = 0; j < n_jobs; ++j)
    if (L.job_group[size_t(j)] >= 0) fg[size_t(L.job_group[size_t(j)])].push_back(j);
  for (int en = 0; en < E; ++en) eg[size_t(L.ens_group[size_t(en)])].push_back(en);
  for (int g = 0; g < G; ++g) {
    fo[size_t(g)] = int64_t(fi.size());
    fl[size_t(g)] = int(fg[size_t(g)].size());
    fi.insert(fi.end(), fg[size_t(g)].begin(), fg[size_t(g)].end());
    eo[size_t(g)] = int64_t(ei.size());
    el[size_t(g)] = int(eg[size_t(g)].size());
    ei.insert(ei.end(), eg[size_t(g)].begin(), eg[size_t(g)].end());
  }
  const int N = std::max(n_jobs, E);
  BlobLayout B;
  const size_t oFO = B.add<int64_t>(size_t(G)), oFL = B.add<int>(size_t(G)), oFI = B.add<int>(fi.size());
  const size_t oEO = B.add<int64_t>(size_t(G)), oEL = B.add<int>(size_t(G)), oEI = B.add<int>(ei.size());
  const size_t oM = B.add<double>(size_t(N) * 6);      // job mape/thr/rho, then ensemble mape/thr/rho
  const size_t oS = B.add<int>(size_t(N) * 2), oBad = B.add<int>(size_t(N));
  const size_t up = B.bytes;
  const size_t oOut = B.add<double>(size_t(G) * 12), oNok = B.add<int>(size_t(G) * 2);
  const size_t oScr = B.add<double>(std::max(fi.size(), ei.size()));
  std::vector<unsigned char> h(B.bytes, 0);
  auto H = [&](auto* tag, size_t off) { return reinterpret_cast<decltype(tag)>(h.data() + off); };
  std::copy(fo.begin(), fo.end(), H((int64_t*)nullptr, oFO));
  std::copy(fl.begin(), fl.end(), H((int*)nullptr, oFL));
  std::copy(fi.begin(), fi.end(), H((int*)nullptr, oFI));
  std::copy(eo.begin(), eo.end(), H((int64_t*)nullptr, oEO));
  std::copy(el.begin(), el.end(), H((int*)nullptr, oEL));
  std::copy(ei.begin(), ei.end(), H((int*)nullptr, oEI));
  double* m = H((double*)nullptr, oM);
  int* st = H((int*)nullptr, oS);
  for (int j = 0; j < n_jobs; ++j) {
    m[size_t(j)] = results[j].mape;
    m[size_t(N) + size_t(j)] = results[j].mape_thr;
    m[2 * size_t(N) + size_t(j)] = results[j].rho;
    st[j] = results[j].status;
  }
  for (int en = 0; en < E; ++en) {
    m[3 * size_t(N) + size_t(en)] = ensembles[en].mape;
    m[4 * size_t(N) + size_t(en)] = ensembles[en].mape_thr;
    m[5 * size_t(N) + size_t(en)] = ensembles[en].rho;
    st[size_t(N) + size_t(en)] = ensembles[en].status;
  }
  std::fill(H((int*)nullptr, oBad), H((int*)nullptr, oBad) + N, -1);
  ck(cudaSetDevice(e->device), "cudaSetDevice");
  DBuf<unsigned char> d(B.bytes, e->stream);
  d.up(h.data(), up);
  auto D = [&](auto* tag, size_t off) { return reinterpret_cast<decltype(tag)>(d.p + off); };
  const double* dm = D((const double*)nullptr, oM);
  const int* ds = D((const int*)nullptr, oS);
  const int* dbad = D((const int*)nullptr, oBad);
  double* out = D((double*)nullptr, oOut);
  int* nok = D((int*)nullptr, oNok);
  double* scr = D((double*)nullptr, oScr);
  const size_t n = size_t(N);
  launch_cv_stats(CvStatsArgs{G, D((const int64_t*)nullptr, oFO), D((const int*)nullptr, oFL),
                              D((const int*)nullptr, oFI), dm, dm + n, dm + 2 * n, ds, dbad, out, nok, scr},
                  e->stream);
  launch_cv_stats(CvStatsArgs{G, D((const int64_t*)nullptr, oEO), D((const int*)nullptr, oEL),
                              D((const int*)nullptr, oEI), dm + 3 * n, dm + 4 * n, dm + 5 * n, ds + n, dbad,
                              out + size_t(G) * 6, nok + G, scr},
                  e->stream);
  ck(cudaGetLastError(), "cv stats launch");
  ck(cudaMemcpyAsync(h.data() + oOut, d.p + oOut, B.bytes - oOut, cudaMemcpyDeviceToHost, e->stream), "D2H");
  t_d2h += int64_t(B.bytes - oOut);
  ck(cudaStreamSynchronize(e->stream), "cv stats");
  const double* so = H((const double*)nullptr, oOut);
  const int* no = H((const int*)nullptr, oNok);
  for (int g = 0; g < G; ++g) {
    lann_cv_group& o = groups[g];
    o = lann_cv_group{};
    o.first_job = L.group_first[size_t(g)];
    o.n_folds = L.group_folds[size_t(g)];
    o.n_models = L.group_models[size_t(g)];
    o.n_models_ok = no[g];
    o.n_ensembles = L.group_ens[size_t(g)];
    o.n_ensembles_ok = no[G + g];
    for (int en : eg[size_t(g)])
      if (ensembles[en].n_test > 0) o.n_test = ensembles[en].n_test;
    const double* a = so + 6 * size_t(g);
    const double* b = so + 6 * size_t(G) + 6 * size_t(g);
    o.fold_mape = {a[0], a[1]};
    o.fold_mape_thr = {a[2], a[3]};
    o.fold_rho = {a[4], a[5]};
    o.test_mape = {b[0], b[1]};
    o.test_mape_thr = {b[2], b[3]};
    o.test_rho = {b[4], b[5]};
  }
  return {};
}
}  // namespace

extern "C" {

int lann_cv_summarize(lann_engine* e, int32_t n_jobs, const lann_job* jobs, const lann_job_result* results,
                      const lann_cv_ensemble* ensembles, lann_cv_group* groups) {
  if (!e) return LANN_NO_DEVICE;
  if (n_jobs < 0 || (n_jobs > 0 && (!jobs || !results)) || !groups)
    return set_err(e, {LANN_PARAM_ERROR, "null arguments"});
  try {
    return set_err(e, cv_group_stats(e, n_jobs, jobs, results, ensembles, groups));
  } catch (const CudaFail& f) {
    e->err = f.what;
    return LANN_CUDA_ERROR;
  }
}

int lann_group_run_cv(lann_group* g, int32_t n_jobs, const lann_job* jobs, int32_t precision,
                      lann_job_result* results, lann_cv_group* groups, lann_cv_ensemble* ensembles) {
  if (!g) return LANN_NO_DEVICE;
  if (!results || !jobs || n_jobs < 1 || !groups || !ensembles) {
    g->err = "empty population or null outputs";
    return LANN_PARAM_ERROR;
  }
  const CvLayout L = cv_layout(n_jobs, jobs);
  // every ensemble's jobs adjacent (ensembles in order of first appearance, members in job
  // order), so the snapped shard cut keeps each ensemble on one device
  std::vector<int> perm;
  perm.reserve(static_cast<size_t>(n_jobs));
  {
    std::vector<std::vector<int>> members(static_cast<size_t>(L.n_ens()));
    for (int j = 0; j < n_jobs; ++j)
      if (L.job_ens[size_t(j)] >= 0) members[size_t(L.job_ens[size_t(j)])].push_back(j);
    std::vector<char> done(static_cast<size_t>(L.n_ens()), 0);
    for (int j = 0; j < n_jobs; ++j) {
      const int en = L.job_ens[size_t(j)];
      if (en < 0) {
        perm.push_back(j);
      } else if (!done[size_t(en)]) {
        done[size_t(en)] = 1;
        perm.insert(perm.end(), members[size_t(en)].begin(), members[size_t(en)].end());
      }
    }
  }
  std::vector<lann_job> pj(static_cast<size_t>(n_jobs));
  for (int i = 0; i < n_jobs; ++i) pj[size_t(i)] = jobs[perm[size_t(i)]];
  const int W = int(g->engines.size());
  std::vector<int32_t> b(size_t(W) + 1);
  shard_bounds(n_jobs, pj.data(), W, b.data());
  std::vector<lann_job_result> pres(static_cast<size_t>(n_jobs));
  std::vector<int> st(static_cast<size_t>(W), LANN_OK);
  std::vector<double> dev_ms(static_cast<size_t>(W), 0.0);
  std::vector<int64_t> h2d(static_cast<size_t>(W), 0), d2h(static_cast<size_t>(W), 0);
  std::vector<std::vector<lann_cv_ensemble>> sh_ens(static_cast<size_t>(W));
  std::vector<std::vector<int>> sh_first(static_cast<size_t>(W));  // first member (permuted index) of each local ensemble
  const auto t0 = std::chrono::steady_clock::now();
  auto work = [&](int w) {
    const int lo = b[size_t(w)], n = b[size_t(w) + 1] - lo;
    if (n <= 0) return;
    lann_engine* e = g->engines[size_t(w)];
    lann_transfer_bytes(nullptr, nullptr, 1);
    lann_population* p = nullptr;
    std::vector<lann_job_result> base;
    int rc = population_create(e, n, pj.data() + lo, precision, 0, &p, false, &base);
    if (!p) {
      for (int j = 0; j < n; ++j) {
        if (size_t(j) < base.size()) {
          pres[size_t(lo + j)] = base[size_t(j)];
        } else {
          pres[size_t(lo + j)] = lann_job_result{};
          pres[size_t(lo + j)].status = rc;
          pres[size_t(lo + j)].nonfinite_epoch = -1;
          pres[size_t(lo + j)].precision_run = -1;
        }
      }
    } else {
      rc = lann_population_run(p, 1);
      if (rc == LANN_OK) rc = lann_population_fetch(p, pres.data() + lo, nullptr, nullptr, nullptr, nullptr);
      else fail_results(p->pop, rc, pres.data() + lo);
      const CvState* cv = p->pop.cv.get();
      if (cv && (rc == LANN_OK || rc == LANN_TRAINING_ERROR || rc == LANN_DOMAIN_ERROR)) {
        sh_ens[size_t(w)].resize(size_t(cv->L.n_ens()));
        const int rc2 = lann_population_cv(p, nullptr, sh_ens[size_t(w)].data());
        if (rc2 != LANN_OK) rc = rc2;
        for (int en = 0; en < cv->L.n_ens(); ++en) sh_first[size_t(w)].push_back(lo + cv->L.ens_first[size_t(en)]);
      }
      lann_population_destroy(p);
    }
    st[size_t(w)] = rc;
    dev_ms[size_t(w)] = lann_last_device_ms(e);
    lann_transfer_bytes(&h2d[size_t(w)], &d2h[size_t(w)], 1);
  };
  std::vector<std::thread> threads;
  for (int w = 1; w < W; ++w) threads.emplace_back(work, w);
  work(0);
  for (auto& t : threads) t.join();
  g->last_device_ms = *std::max_element(dev_ms.begin(), dev_ms.end());
  for (int w = 0; w < W; ++w) {
    t_h2d += h2d[size_t(w)];
    t_d2h += d2h[size_t(w)];
  }
  for (int i = 0; i < n_jobs; ++i) results[perm[size_t(i)]] = pres[size_t(i)];
  // ensembles in the global layout's order; an ensemble not scored on any shard (every one of its
  // jobs failed before a population formed) reports its missing / failed members from the results
  for (int en = 0; en < L.n_ens(); ++en) {
    lann_cv_ensemble& o = ensembles[en];
    o = lann_cv_ensemble{};
    o.group = L.ens_group[size_t(en)];
    o.init_seed = L.ens_seed[size_t(en)];
    o.status = LANN_PARAM_ERROR;
    for (int j : L.ens_member[size_t(en)])
      if (j >= 0 && results[j].status != LANN_OK) {
        o.status = results[j].status;
        break;
      }
  }
  for (int w = 0; w < W; ++w)
    for (size_t q = 0; q < sh_ens[size_t(w)].size(); ++q) {
      const int global_job = perm[size_t(sh_first[size_t(w)][q])];
      const int en = L.job_ens[size_t(global_job)];
      lann_cv_ensemble r = sh_ens[size_t(w)][q];
      r.group = L.ens_group[size_t(en)];
      ensembles[en] = r;
    }
  g->err.clear();
  int rc = LANN_OK;
  for (int w = 0; w < W; ++w)
    if (st[size_t(w)] != LANN_OK && rc == LANN_OK) {
      rc = st[size_t(w)];
      g->err = std::string("device ") + std::to_string(g->engines[size_t(w)]->device) + ": " +
               lann_last_error(g->engines[size_t(w)]);
    }
  // the group statistics over every shard's models and ensembles, on the first device
  const int rs = lann_cv_summarize(g->engines[0], n_jobs, jobs, results, ensembles, groups);
  if (rs != LANN_OK && rc == LANN_OK) {
    rc = rs;
    g->err = lann_last_error(g->engines[0]);
  }
  g->last_wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return rc;
}

}  // extern "C"
