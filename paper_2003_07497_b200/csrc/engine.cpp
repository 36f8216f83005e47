// engine.cpp — the C ABI of include/lann_engine.h: argument validation with the
// reference's error contract, device buffers, kernel launches, and the
// whole-population pipeline. There is no CPU fallback: without a CUDA device
// every compute entry point returns LANN_NO_DEVICE.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/lann_engine.h"
#include "domain.hpp"
#include "kernels.cuh"

struct lann_engine {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::string err;
  double last_ms = 0.0;
  int64_t launches = 0;
  int max_smem = 0;
};

namespace lann {
namespace {

struct CudaFail {
  std::string what;
};

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaFail{std::string(what) + ": " + cudaGetErrorString(e)};
}

// Stream-ordered device buffer.
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
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
    return *this;
  }
  ~DBuf() {
    if (p) cudaFreeAsync(p, s);
  }
  void up(const T* host) {
    if (n) ck(cudaMemcpyAsync(p, host, n * sizeof(T), cudaMemcpyHostToDevice, s), "H2D");
  }
  void down(T* host) const {
    if (n) ck(cudaMemcpyAsync(host, p, n * sizeof(T), cudaMemcpyDeviceToHost, s), "D2H");
  }
  void zero() {
    if (n) ck(cudaMemsetAsync(p, 0, n * sizeof(T), s), "memset");
  }
};

int set_err(lann_engine* e, const Status& st) {
  if (e) e->err = st.msg;
  return st.code;
}

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

// ---- device-resident training input, shared by lann_train and lann_run_population ----
struct DevTrain {
  int n_models = 0, n_tiles = 0;
  std::vector<int> tile_rows, tile_inputs, model_tile, h1, h2, epochs;
  std::vector<int64_t> tile_offset, param_offset, trace_offset;
  std::vector<double> lr;
  int64_t total_params = 0;
  int trace_stride = 1;
  bool want_trace = false;
  int64_t trace_len = 0;
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
    const int P = param_count(t.tile_inputs[t.model_tile[m]], t.h1[m], t.h2[m]);
    if (t.param_offset[m] < 0 || t.param_offset[m] + P > t.total_params)
      return {LANN_PARAM_ERROR, "flat parameter size mismatch"};
  }
  return {};
}

// Runs the trainer on device buffers (X, y, params already resident).
void run_train(lann_engine* e, const DevTrain& t, int precision, const double* dX,
               const double* dY, int64_t total_rows, double* dparams, double* dfinal,
               int* dbad, double* dtrace, const DBuf<int64_t>& dtrace_off) {
  cudaStream_t s = e->stream;
  DBuf<int> d_tile_rows(t.tile_rows, s), d_tile_inputs(t.tile_inputs, s), d_model_tile(t.model_tile, s),
      d_h1(t.h1, s), d_h2(t.h2, s), d_epochs(t.epochs, s);
  DBuf<int64_t> d_tile_off(t.tile_offset, s), d_poff(t.param_offset, s);
  DBuf<double> d_lr(t.lr, s);
  const int max_e = *std::max_element(t.epochs.begin(), t.epochs.end());

  // FP32 mode: models of a supported compiled shape go to the FP32 kernels; any
  // other shape is trained by the (generic, exact) FP64 kernel below.
  std::vector<int> fp64_models;
  if (precision == LANN_FP32) {
    DBuf<float> rows_f(size_t(total_rows) * 8, s);
    launch_pack_rows(dX, dY, total_rows, rows_f.p, s);
    e->launches += 1;
    using Shape = std::tuple<int, int, int>;
    std::map<Shape, std::vector<int>> buckets;
    for (int m = 0; m < t.n_models; ++m) {
      const int tile = t.model_tile[m];
      const int I = t.tile_inputs[tile];
      if (fp32_shape_supported(I, t.h1[m], t.h2[m]) && t.tile_rows[tile] * 32 <= 96 * 1024)
        buckets[{I, t.h1[m], t.h2[m]}].push_back(m);
      else
        fp64_models.push_back(m);
    }
    int lanes = 0;
    if (const char* env = std::getenv("LANN_FP32_LANES")) lanes = std::atoi(env);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, e->device);
    if (lanes != 1 && lanes != 2 && lanes != 4 && lanes != 8 && lanes != 32) {
      // smallest lanes-per-model that still gives >= 16 warps per SM
      const int total = t.n_models - int(fp64_models.size());
      lanes = 32;
      for (int k : {1, 2, 4, 8, 32})
        if ((total + 32 / k - 1) / (32 / k) >= 16 * sms) {
          lanes = k;
          break;
        }
    }
    const int G = 32 / lanes;
    std::vector<DBuf<int>> keep;
    for (auto& [shape, ms] : buckets) {
      // group: same tile and epoch count, up to G models; longest groups first
      std::stable_sort(ms.begin(), ms.end(), [&](int a, int b) {
        const double ca = double(t.epochs[a]) * t.tile_rows[t.model_tile[a]];
        const double cb = double(t.epochs[b]) * t.tile_rows[t.model_tile[b]];
        if (ca != cb) return ca > cb;
        if (t.model_tile[a] != t.model_tile[b]) return t.model_tile[a] < t.model_tile[b];
        return t.epochs[a] < t.epochs[b];
      });
      std::vector<int> gfirst, gcount;
      int max_rows = 1;
      for (size_t i = 0; i < ms.size();) {
        size_t j = i + 1;
        while (j < ms.size() && int(j - i) < G && t.model_tile[ms[j]] == t.model_tile[ms[i]] &&
               t.epochs[ms[j]] == t.epochs[ms[i]])
          ++j;
        gfirst.push_back(int(i));
        gcount.push_back(int(j - i));
        max_rows = std::max(max_rows, t.tile_rows[t.model_tile[ms[i]]]);
        i = j;
      }
      keep.emplace_back(gfirst, s);
      const int* d_gf = keep.back().p;
      keep.emplace_back(gcount, s);
      const int* d_gc = keep.back().p;
      keep.emplace_back(ms, s);
      const int* d_sm = keep.back().p;
      TrainF32Args a{};
      a.n_groups = int(gfirst.size());
      a.group_first = d_gf;
      a.group_count = d_gc;
      a.sorted_model = d_sm;
      a.rows = rows_f.p;
      a.tile_rows = d_tile_rows.p;
      a.tile_offset = d_tile_off.p;
      a.model_tile = d_model_tile.p;
      a.lr = d_lr.p;
      a.epochs = d_epochs.p;
      a.param_offset = d_poff.p;
      a.params = dparams;
      a.final_loss = dfinal;
      a.nonfinite_epoch = dbad;
      a.loss_trace = dtrace;
      a.trace_offset = dtrace_off.p;
      a.trace_stride = t.trace_stride;
      if (!launch_train_fp32(a, std::get<0>(shape), std::get<1>(shape), std::get<2>(shape), lanes,
                             max_rows * 32, s))
        throw CudaFail{"no FP32 kernel for this shape"};
      ck(cudaGetLastError(), "train_fp32 launch");
      e->launches += 1;
    }
    if (fp64_models.empty()) return;
  } else {
    fp64_models.resize(t.n_models);
    std::iota(fp64_models.begin(), fp64_models.end(), 0);
  }
  {
    // longest models first so the block scheduler packs the tail
    std::vector<int> order = fp64_models;
    auto cost = [&](int m) {
      const int tile = t.model_tile[m];
      return double(t.epochs[m]) * t.tile_rows[tile] *
             param_count(t.tile_inputs[tile], t.h1[m], t.h2[m]);
    };
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost(a) > cost(b); });
    const auto& bc = adam_bias_table(max_e);
    DBuf<double2> d_bc(reinterpret_cast<const double2*>(bc.data()), size_t(max_e), s);
    // shared-memory plan: records in smem when every model's records fit
    int max_p = 0;
    size_t max_bytes_smem = 0, max_state = 0;
    std::vector<int64_t> soff(t.n_models);
    int64_t scratch = 0;
    for (int m : order) {
      const int tile = t.model_tile[m];
      const int P = param_count(t.tile_inputs[tile], t.h1[m], t.h2[m]);
      max_p = std::max(max_p, P);
      const size_t rec = size_t(fp64_record_doubles(t.tile_inputs[tile], t.h1[m], t.h2[m])) *
                         t.tile_rows[tile] * 8;
      const size_t state = size_t(3 * P + 2) * 8;
      max_state = std::max(max_state, state);
      max_bytes_smem = std::max(max_bytes_smem, state + rec);
      soff[m] = scratch;
      scratch += int64_t(rec / 8);
    }
    const bool in_smem = max_bytes_smem <= size_t(e->max_smem);
    DBuf<double> d_scratch(in_smem ? 0 : size_t(scratch), s);
    DBuf<int64_t> d_soff(soff, s);
    DBuf<int> d_order(order, s);
    TrainArgs a{};
    a.n_models = int(order.size());
    a.order = d_order.p;
    a.tile_rows = d_tile_rows.p;
    a.tile_inputs = d_tile_inputs.p;
    a.tile_offset = d_tile_off.p;
    a.X = dX;
    a.y = dY;
    a.model_tile = d_model_tile.p;
    a.h1 = d_h1.p;
    a.h2 = d_h2.p;
    a.lr = d_lr.p;
    a.epochs = d_epochs.p;
    a.param_offset = d_poff.p;
    a.params = dparams;
    a.final_loss = dfinal;
    a.nonfinite_epoch = dbad;
    a.loss_trace = dtrace;
    a.trace_offset = dtrace_off.p;
    a.trace_stride = t.trace_stride;
    a.bias_corr = d_bc.p;
    a.scratch = d_scratch.p;
    a.scratch_offset = d_soff.p;
    a.smem_records = in_smem ? 1 : 0;
    launch_train_fp64(a, max_p, int(in_smem ? max_bytes_smem : max_state), s);
    ck(cudaGetLastError(), "train_fp64 launch");
    e->launches += 1;
  }
}

}  // namespace
}  // namespace lann

using namespace lann;

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
    ck(cudaEventCreate(&e->ev0), "event");
    ck(cudaEventCreate(&e->ev1), "event");
    ck(cudaDeviceGetAttribute(&e->max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device), "attr");
  } catch (const CudaFail& f) {
    delete e;
    return LANN_CUDA_ERROR;
  }
  *out = e;
  return LANN_OK;
}

void lann_engine_destroy(lann_engine* e) {
  if (!e) return;
  cudaSetDevice(e->device);
  if (e->stream) cudaStreamSynchronize(e->stream);
  if (e->ev0) cudaEventDestroy(e->ev0);
  if (e->ev1) cudaEventDestroy(e->ev1);
  if (e->stream) cudaStreamDestroy(e->stream);
  delete e;
}

const char* lann_last_error(const lann_engine* e) { return e ? e->err.c_str() : "no engine"; }
double lann_last_device_ms(const lann_engine* e) { return e ? e->last_ms : 0.0; }
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
    if (b->loss_trace) {
      for (int m = 0; m < b->n_models; ++m) {
        toff[m] = b->trace_offset[m];
        trace_total = std::max<int64_t>(trace_total, toff[m] + (t.epochs[m] + t.trace_stride - 1) / t.trace_stride);
      }
    }
    DBuf<double> dT(size_t(trace_total), s);
    DBuf<int64_t> dTO(toff, s);
    run_train(e, t, b->precision, dX.p, dY.p, b->total_rows, dP.p, dF.p, dB.p,
              b->loss_trace ? dT.p : nullptr, dTO);
    dP.down(b->params);
    dF.down(b->final_loss);
    dB.down(b->nonfinite_epoch);
    if (b->loss_trace) dT.down(b->loss_trace);
    timer.stop();
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
    const int P = param_count(ms->n_inputs[m], ms->h1[m], ms->h2[m]);
    if (ms->n_inputs[m] < 1 || ms->n_inputs[m] > 7 || ms->h1[m] < 1 || ms->h2[m] < 0 ||
        ms->h1[m] > 64 || ms->h2[m] > 64)
      return set_err(e, {LANN_PARAM_ERROR, "bad model shape"});
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
    if (ms->precision == LANN_FP32) launch_predict_fp32(a, s);
    else launch_predict_fp64(a, s);
    ck(cudaGetLastError(), "predict launch");
    e->launches += n_rows > 0;
    dout.down(out);
    timer.stop();
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
  if (size_t(max_len) * 36 + 16 > size_t(e->max_smem))
    return set_err(e, {LANN_PARAM_ERROR, "evaluation set too large for one CTA"});
  try {
    ck(cudaSetDevice(e->device), "cudaSetDevice");
    cudaStream_t s = e->stream;
    Timer timer(e);
    DBuf<int64_t> doff(offset, n_sets, s);
    DBuf<int> dlen(len, n_sets, s), dk(size_t(n_sets), s), dst(size_t(n_sets), s);
    DBuf<double> dt(truth, size_t(total), s), dp(pred, size_t(total), s), dm(size_t(n_sets), s),
        dmt(size_t(n_sets), s), dr(size_t(n_sets), s);
    EvalArgs a{n_sets, doff.p, dlen.p, dt.p, dp.p, drop, dm.p, dmt.p, dk.p, dr.p, dst.p};
    launch_eval(a, max_len, s);
    ck(cudaGetLastError(), "eval launch");
    e->launches += 1;
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

int lann_select_variants(lann_engine* e, const lann_model_set* ms, const int32_t* with_n_thd,
                         int32_t kind, int32_t max_threads, uint64_t seed, int64_t first,
                         int64_t n_cands, int32_t* out_idx, double* out_score) {
  if (!e) return LANN_NO_DEVICE;
  if (!ms || ms->n_models < 1) return set_err(e, {LANN_PARAM_ERROR, "empty model set"});
  if (kind < LANN_MM || kind > LANN_MP)
    return set_err(e, {LANN_PARAM_ERROR, "variant mapping covers the mm/mv/mc/mp kernels"});
  if (max_threads < 1) return set_err(e, {LANN_PARAM_ERROR, "max_threads must be >= 1"});
  if (n_cands < 1) return set_err(e, {LANN_PARAM_ERROR, "select needs at least one candidate"});
  int max_p = 0;
  for (int m = 0; m < ms->n_models; ++m) {
    const int want = base_feature_count(kind, with_n_thd[m] != 0);
    if (ms->n_inputs[m] != want && ms->n_inputs[m] != want + 1)
      return set_err(e, {LANN_SCHEMA_ERROR, "model schema does not match the candidate kernel"});
    if (ms->h1[m] < 1 || ms->h1[m] > 64 || ms->h2[m] < 0 || ms->h2[m] > 64)
      return set_err(e, {LANN_PARAM_ERROR, "bad model shape"});
    max_p = std::max(max_p, param_count(ms->n_inputs[m], ms->h1[m], ms->h2[m]));
  }
  if (!select_variants_supported(ms->n_models, max_p))
    return set_err(e, {LANN_PARAM_ERROR, "variant scorer holds at most 32 lightweight models"});
  try {
    ck(cudaSetDevice(e->device), "cudaSetDevice");
    cudaStream_t s = e->stream;
    const int M = ms->n_models;
    DBuf<int> dI(ms->n_inputs, M, s), dh1(ms->h1, M, s), dh2(ms->h2, M, s), dl(ms->log_target, M, s),
        dt(with_n_thd, M, s), didx(size_t(n_cands), s);
    DBuf<int64_t> dpo(ms->param_offset, M, s);
    DBuf<double> dp(ms->params, size_t(ms->total_params), s), dn(ms->norm, size_t(M) * 18, s),
        dsc(size_t(n_cands), s);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, e->device);
    Timer timer(e);
    e->launches += select_variants_launch(M, ms->precision, kind, max_threads, seed, first, n_cands,
                                          dI.p, dh1.p, dh2.p, dl.p, dt.p, dpo.p, dp.p, dn.p, didx.p,
                                          dsc.p, sms, s);
    ck(cudaGetLastError(), "select_variants launch");
    didx.down(out_idx);
    dsc.down(out_score);
    timer.stop();
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

// Whole-population pipeline: host builds datasets / tiles / initial weights (each
// distinct dataset and tile once), then ONE device pass trains every model,
// predicts every evaluation row and computes every model's metrics.
int lann_run_population(lann_engine* e, int32_t n_jobs, const lann_job* jobs, int32_t precision,
                        lann_job_result* results, double* params_out,
                        const int64_t* params_offset, double* trace_out,
                        const int64_t* trace_offset) {
  if (!e) return LANN_NO_DEVICE;
  if (n_jobs < 1 || !jobs || !results) return set_err(e, {LANN_PARAM_ERROR, "empty population"});
  if (precision != LANN_FP64_EXACT && precision != LANN_FP32)
    return set_err(e, {LANN_PARAM_ERROR, "unknown precision"});
  for (int j = 0; j < n_jobs; ++j) {
    std::memset(&results[j], 0, sizeof(lann_job_result));
    results[j].nonfinite_epoch = -1;
  }
  // ---- distinct datasets, splits and tiles ----
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
  const int nthreads = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  auto parallel_for = [&](int n, auto&& fn) {
    std::atomic<int> next{0};
    std::vector<std::thread> pool;
    auto worker = [&] {
      for (int i; (i = next.fetch_add(1)) < n;) fn(i);
    };
    for (int t = 1; t < std::min(nthreads, n); ++t) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
  };
  std::vector<Dataset> dsets(dsrc.size());
  std::vector<Status> dstat(dsrc.size());
  parallel_for(int(dsrc.size()), [&](int d) {
    dstat[d] = build_dataset(dsrc[d]->world, dsrc[d]->data_seed, dsrc[d]->count, dsets[d]);
  });
  std::vector<Tile> tiles(tsrc.size());
  std::vector<Status> tstat(tsrc.size());
  parallel_for(int(tsrc.size()), [&](int k) {
    const auto& [d, frac, folds, fold, family, logt] = tsrc[k];
    if (dstat[d]) {
      tstat[k] = dstat[d];
      return;
    }
    std::vector<int64_t> order;
    int ntr = 0;
    tstat[k] = split_order(dsets[d].size(), frac, dsrc[d]->data_seed, order, ntr);
    if (!tstat[k]) tstat[k] = make_tile(dsets[d], order, ntr, folds, fold, family, logt != 0, tiles[k]);
  });
  // ---- per-job validation and initial weights ----
  std::vector<int> model_job;  // trained model -> job
  std::vector<int> job_model(n_jobs, -1);
  for (int j = 0; j < n_jobs; ++j) {
    const int k = job_tile[j];
    Status st = tstat[k];
    if (!st) st = validate_config(jobs[j], tiles[k].n_inputs);
    results[j].status = st.code;
    if (st) {
      if (e->err.empty()) e->err = st.msg;
      continue;
    }
    results[j].n_inputs = tiles[k].n_inputs;
    results[j].n_params = param_count(tiles[k].n_inputs, jobs[j].hidden[0],
                                      jobs[j].n_hidden > 1 ? jobs[j].hidden[1] : 0);
    results[j].n_train = tiles[k].n_train();
    results[j].n_eval = tiles[k].n_eval();
    job_model[j] = int(model_job.size());
    model_job.push_back(j);
  }
  const int M = int(model_job.size());
  if (M == 0) return set_err(e, {results[0].status, e->err});
  DevTrain t;
  t.n_models = M;
  t.n_tiles = int(tiles.size());
  std::vector<double> X, Y, eval_rows, eval_truth;
  std::vector<int> eval_model;
  std::vector<int64_t> eval_off(M), tile_eval_off(tiles.size());
  int64_t rows = 0;
  for (size_t k = 0; k < tiles.size(); ++k) {
    t.tile_rows.push_back(tiles[k].n_train());
    t.tile_inputs.push_back(std::max(1, tiles[k].n_inputs));
    t.tile_offset.push_back(rows);
    X.insert(X.end(), tiles[k].Xn.begin(), tiles[k].Xn.end());
    Y.insert(Y.end(), tiles[k].yn.begin(), tiles[k].yn.end());
    rows += tiles[k].n_train();
  }
  std::vector<double> norm(size_t(M) * 18);
  std::vector<int> n_in(M), logt(M), eval_len(M);
  int max_eval = 1;
  for (int m = 0; m < M; ++m) {
    const lann_job& J = jobs[model_job[m]];
    const Tile& T = tiles[job_tile[model_job[m]]];
    t.model_tile.push_back(job_tile[model_job[m]]);
    t.h1.push_back(J.hidden[0]);
    t.h2.push_back(J.n_hidden > 1 ? J.hidden[1] : 0);
    t.lr.push_back(J.learning_rate);
    t.epochs.push_back(J.epochs);
    t.param_offset.push_back(t.total_params);
    t.total_params += param_count(T.n_inputs, t.h1.back(), t.h2.back());
    std::memcpy(&norm[size_t(m) * 18], T.norm, sizeof T.norm);
    n_in[m] = T.n_inputs;
    logt[m] = T.log_target;
    eval_off[m] = int64_t(eval_truth.size());
    eval_len[m] = T.n_eval();
    max_eval = std::max(max_eval, T.n_eval());
    eval_rows.insert(eval_rows.end(), T.eval_rows.begin(), T.eval_rows.end());
    eval_truth.insert(eval_truth.end(), T.eval_truth.begin(), T.eval_truth.end());
    for (int r = 0; r < T.n_eval(); ++r) eval_model.push_back(m);
  }
  std::vector<double> params(size_t(t.total_params));
  parallel_for(M, [&](int m) {
    const lann_job& J = jobs[model_job[m]];
    glorot_init(n_in[m], t.h1[m], t.h2[m], J.init_seed, &params[size_t(t.param_offset[m])]);
  });
  if (Status st = validate_train(t)) return set_err(e, st);
  const bool want_trace = trace_out && trace_offset;
  std::vector<int64_t> toff(M, 0);
  int64_t trace_total = 0;
  if (want_trace)
    for (int m = 0; m < M; ++m) {
      toff[m] = trace_total;
      trace_total += t.epochs[m];
    }
  for (int m = 0; m < M; ++m)
    if (eval_len[m] < 2) {
      results[model_job[m]].status = LANN_DOMAIN_ERROR;  // spearman needs two samples
    }
  if (size_t(max_eval) * 36 + 16 > size_t(e->max_smem))
    return set_err(e, {LANN_PARAM_ERROR, "evaluation set too large for one CTA"});
  try {
    ck(cudaSetDevice(e->device), "cudaSetDevice");
    cudaStream_t s = e->stream;
    Timer timer(e);
    DBuf<double> dX(X, s), dY(Y, s), dP(params, s), dF(size_t(M), s), dT(size_t(trace_total), s);
    DBuf<int> dB(size_t(M), s);
    DBuf<int64_t> dTO(toff, s);
    run_train(e, t, precision, dX.p, dY.p, rows, dP.p, dF.p, dB.p, want_trace ? dT.p : nullptr, dTO);
    // predictions on every evaluation row, straight from the device-resident weights
    const int64_t n_eval_rows = int64_t(eval_truth.size());
    DBuf<double> dER(eval_rows, s), dPred(size_t(n_eval_rows), s), dN(norm, s), dET(eval_truth, s);
    DBuf<int> dEM(eval_model, s), dI(n_in, s), dh1(t.h1, s), dh2(t.h2, s), dlog(logt, s);
    DBuf<int64_t> dpo(t.param_offset, s);
    PredictArgs pa{n_eval_rows, dER.p, dEM.p, dI.p, dh1.p, dh2.p, dlog.p, dpo.p, dP.p, dN.p, dPred.p};
    if (precision == LANN_FP32) launch_predict_fp32(pa, s);
    else launch_predict_fp64(pa, s);
    e->launches += n_eval_rows > 0;
    DBuf<int64_t> dEO(eval_off, s);
    DBuf<int> dEL(eval_len, s), dK(size_t(M), s), dS(size_t(M), s);
    DBuf<double> dMape(size_t(M), s), dThr(size_t(M), s), dRho(size_t(M), s);
    EvalArgs ea{M, dEO.p, dEL.p, dET.p, dPred.p, 0.3, dMape.p, dThr.p, dK.p, dRho.p, dS.p};
    launch_eval(ea, max_eval, s);
    e->launches += 1;
    ck(cudaGetLastError(), "population launch");
    std::vector<double> fin(M), mape(M), thr(M), rho(M);
    std::vector<int> bad(M), kept(M), est(M);
    dF.down(fin.data());
    dB.down(bad.data());
    dMape.down(mape.data());
    dThr.down(thr.data());
    dRho.down(rho.data());
    dK.down(kept.data());
    dS.down(est.data());
    if (params_out) dP.down(params.data());
    std::vector<double> trace(static_cast<size_t>(trace_total));
    if (want_trace) dT.down(trace.data());
    timer.stop();
    int first_err = LANN_OK;
    for (int m = 0; m < M; ++m) {
      const int j = model_job[m];
      lann_job_result& r = results[j];
      r.final_loss = fin[m];
      r.nonfinite_epoch = bad[m];
      if (bad[m] >= 0) {
        r.status = LANN_TRAINING_ERROR;
      } else if (r.status == LANN_OK) {
        r.mape = mape[m];
        r.mape_thr = thr[m];
        r.rho = rho[m];
        r.n_kept = kept[m];
        if (est[m]) r.status = LANN_DOMAIN_ERROR;
      }
      if (params_out && params_offset)
        std::memcpy(params_out + params_offset[j], &params[size_t(t.param_offset[m])],
                    sizeof(double) * size_t(r.n_params));
      if (want_trace)
        std::memcpy(trace_out + trace_offset[j], &trace[size_t(toff[m])],
                    sizeof(double) * size_t(t.epochs[m]));
    }
    for (int j = 0; j < n_jobs; ++j)
      if (results[j].status != LANN_OK && first_err == LANN_OK) first_err = results[j].status;
    return first_err;
  } catch (const CudaFail& f) {
    e->err = f.what;
    return LANN_CUDA_ERROR;
  }
}

int lann_default_combos(lann_world* out, int32_t cap) {
  const auto combos = default_combos();
  const int n = int(combos.size());
  for (int i = 0; i < n && i < cap; ++i) out[i] = combos[i];
  return n;
}

}  // extern "C"
