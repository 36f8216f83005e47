// domain.hpp — host-side domain logic of the engine (C++20): seeded sampling of
// kernel instances, the synthetic runtime worlds, dataset split / k-fold,
// min-max normalisation and Glorot init. Everything here is the engine's own
// code (not linked to the reference); each function names the reference
// behaviour it must reproduce bit for bit (paths relative to
// /root/reference/proj/core/).
#pragma once

#include <cstdint>
#include <random>
#include <span>
#include <string>
#include <vector>

#include "../../include/lann_engine.h"

namespace lann {

// ---- errors carried as status codes through the C ABI ------------------------------
struct Status {
  int code = LANN_OK;
  std::string msg;
  int epoch = -1;
  explicit operator bool() const { return code != LANN_OK; }
};

// ---- rng.hpp:10-63 -------------------------------------------------------------------
inline std::uint64_t splitmix64(std::uint64_t& s) {
  std::uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
inline std::uint64_t derive_seed(std::uint64_t root, std::uint64_t stream) {
  std::uint64_t s = root ^ (0x9e3779b97f4a7c15ULL * (stream + 1));
  splitmix64(s);
  return splitmix64(s);
}

// Sequential stream (mt19937_64) with the reference's hand-rolled draws.
class SeqRng {
 public:
  explicit SeqRng(std::uint64_t seed) : e_(seed) {}
  std::uint64_t next() { return e_(); }
  // Rng::bounded (rng.hpp): reject r < 2^64 mod n, return r mod n. Powers of two take a mask
  // and small n a cached exact remainder (floor((2^64-1)/n) multiplier, mulhi, <= 2
  // corrections) instead of two 64-bit divisions per draw; the results are identical.
  std::uint64_t bounded(std::uint64_t n) {
    if ((n & (n - 1)) == 0) return e_() & (n - 1);  // 2^64 mod 2^k = 0: nothing to reject
    if (n <= kSmallN) {
      const SmallMod& t = small_mod(n);
      for (;;) {
        const std::uint64_t r = e_();
        if (r >= t.thr) {
          std::uint64_t rem = r - std::uint64_t((unsigned __int128)r * t.mul >> 64) * n;
          if (rem >= n) rem -= n;
          if (rem >= n) rem -= n;
          return rem;
        }
      }
    }
    const std::uint64_t thr = (0 - n) % n;
    for (;;) {
      const std::uint64_t r = e_();
      if (r >= thr) return r % n;
    }
  }
  double uniform() { return double(e_() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }

 private:
  static constexpr std::uint64_t kSmallN = 4096;
  struct SmallMod {
    std::uint64_t mul, thr;
  };
  static const SmallMod& small_mod(std::uint64_t n) {
    static const std::vector<SmallMod> table = [] {
      std::vector<SmallMod> t(kSmallN + 1, SmallMod{0, 0});
      for (std::uint64_t k = 1; k <= kSmallN; ++k) t[k] = SmallMod{~std::uint64_t(0) / k, (0 - k) % k};
      return t;
    }();
    return table[n];
  }
  std::mt19937_64 e_;
};

// ---- kernel instances (kernels.hpp:84-116) -----------------------------------------------
struct Instance {
  int kind = LANN_MM;
  std::uint32_t m = 0, n = 0, k = 0, r = 0, s = 0;
  double d1 = 1.0, d2 = 1.0, d = 1.0;
  int n_thd = 1;
  std::uint32_t sched[4] = {0, 0, 0, 0};
};

std::uint64_t complexity(const Instance& p);                          // kernels.cpp:184-206
int base_features(const Instance& p, bool with_n_thd, double* out);   // features.cpp:23-54
int base_feature_count(int kind, bool with_n_thd);                    // features.cpp:10-21
const std::vector<std::uint32_t>& schedule_lattice(int gpu_style);    // kernels.cpp:77-87
// ParamSpace (datagen.hpp:19-40): dims U{dim_min..dim_max}, blur sides, schedule lattice
struct SampleSpace {
  int kind = LANN_MM;
  int max_threads = 1;
  int gpu_lattice = 0;
  std::uint32_t dim_min = 1, dim_max = 1024;
  std::vector<std::uint32_t> sides = {1024, 2048, 4096, 8192, 16384, 32768};
};
Instance sample_instance(const SampleSpace& space, SeqRng& rng);                     // datagen.cpp:60-110
Instance sample_instance(int kind, int max_threads, int gpu_lattice, SeqRng& rng);  // default space
double mock_runtime(const Instance& p);                                               // perfsage.cpp:71-84

// ---- datasets ------------------------------------------------------------------------------
struct Dataset {
  int kind = LANN_MM;
  int n_features = 0;               // base features (no c)
  std::vector<double> feats;        // [n][LANN_ROW]
  std::vector<std::uint64_t> c;
  std::vector<double> runtime;
  int size() const { return int(runtime.size()); }
};

Status build_dataset(const lann_world& w, std::uint64_t seed, int count, Dataset& out);  // datagen.cpp:177-223
// build_dataset of a native (CPU-class) variant with the CLI's --mock-timer probe
Status build_mock_dataset(const SampleSpace& space, bool single_threaded, std::uint64_t seed, int count,
                          Dataset& out);
Status split_order(int n, double frac, std::uint64_t seed, std::vector<std::int64_t>& order,
                   int& n_train);                                                      // datagen.cpp:225-248

// Training tile of one model: model-input rows (features [+ c]) normalised with the
// tile's own NormStats (models.cpp:89-133), plus the raw evaluation rows.
struct Tile {
  int n_inputs = 0;
  bool log_target = false;
  double norm[18] = {0};                 // f_min[8], f_max[8], t_min, t_max
  std::vector<double> Xn, yn;            // [n_train][LANN_ROW], [n_train]
  std::vector<double> eval_rows;         // raw model inputs [n_eval][LANN_ROW]
  std::vector<double> eval_truth;        // [n_eval]
  std::vector<double> test_rows;         // k-fold tiles: the split's test part, raw [n_test][LANN_ROW]
  std::vector<double> test_truth;        // [n_test]
  int n_train() const { return int(yn.size()); }
  int n_eval() const { return int(eval_truth.size()); }
  int n_test() const { return int(test_truth.size()); }
};

Status make_tile(const Dataset& ds, const std::vector<std::int64_t>& order, int n_train,
                 int n_folds, int fold, int family, bool log_target, Tile& out);

// ---- models ---------------------------------------------------------------------------------
int param_count(int n_inputs, int h1, int h2);                            // models.cpp:37-46
Status validate_config(const lann_job& j, int n_inputs);                  // models.cpp:48-64
void glorot_init(int n_inputs, int h1, int h2, std::uint64_t seed, double* params);  // mlp.cpp:9-25

// Adam bias-correction table: bc[2t] = 1 - 0.9^(t+1), bc[2t+1] = 1 - 0.999^(t+1)
// evaluated with the host libm's pow exactly as AdamState::update does (mlp.cpp:144-146).
const std::vector<double>& adam_bias_table(int epochs);

// The 48 kernel-variant-hardware combinations (config 2); see DESIGN.md.
std::vector<lann_world> default_combos();
Status probe_schedules(const lann_world& w, std::uint64_t seed, std::uint32_t image_n, int n,
                       const std::uint32_t* sched, double* runtime);

}  // namespace lann
