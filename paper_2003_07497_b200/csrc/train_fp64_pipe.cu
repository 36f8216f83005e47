// train_fp64_pipe.cu — K1a, pipelined: the FP64 exact-order LANN trainer for the compiled
// shapes (I-8-1, I <= 7, and I-5-5-1, I <= 6) with N <= 256 samples.
//
// Same arithmetic, bit for bit, as models::train_full_batch (mlp.cpp:156-175): forward in the
// reference order (mlp.cpp:36-52), the per-sample delta recursion (mlp.cpp:93-104), the
// SEQUENTIAL per-parameter sums over samples 0..N-1 of (inv_n*delta)*a (mlp.cpp:106-118),
// Adam in the reference expression order with host-libm bias corrections (mlp.cpp:142-154),
// the pre-update loss trace and the non-finite check. Built with -fmad=false; every operation
// is an explicit __d*_rn intrinsic.
//
// Why a second FP64 kernel: an epoch's floor is one N-long dependent DADD chain per parameter
// (the reference's sample-order sum cannot be reassociated), ~8.3 cycles per link on the B200
// (tools/mb/fp64_issue_mb.cu). The phased kernel (train_fp64.cu) runs "all samples forward /
// backward" and "all chains" one after the other behind CTA barriers, so an epoch costs
// phase A + chain + Adam. Here the two overlap inside the epoch:
//   producer warps  own BLOCKS of 32 samples (warp w: blocks w, w + NPW, ...; lane k sample
//                   32 b + k), forward and backward, and store each sample's column of the record
//                   matrix: one row per parameter holding its term ((inv_n*delta)*a for a weight,
//                   the product mlp.cpp:113 forms; inv_n*delta for a bias, mlp.cpp:117) plus the
//                   err^2 row; the warp arrives on the block's mbarrier when its columns are
//                   stored; the epoch's weights are read into registers once per epoch;
//   chain lanes     own PARAMETERS (lane c sums row c; one more lane the loss): a lane waits for
//                   producer round 0 (NPW blocks), then extends its DADD chain over the blocks in
//                   sample order, two samples per 16-B load; inside a round the NEXT block's 16
//                   loads are issued before the current block's 32 links, so shared-memory
//                   latency stays off the chain; the next round is waited for (blocking) only
//                   after the last block of the current one. The chain starts after round 0 and
//                   runs while the producers are on round 1.
// The owner lane keeps w, m, v in registers; after Adam it writes w to shared memory for the
// producers; one CTA barrier per epoch separates epochs. Warps 0-2 (chains) and the producer
// warps that follow share the four SM sub-partitions so block 0's warp runs alone on one.
#include <cmath>
#include <cstdlib>

#include "exact_fp64.cuh"
#include "kernels.cuh"

namespace lann {
namespace {

constexpr int kLd = 258;     // record row stride (doubles): N <= 256 samples + even padding
constexpr int kChainWarps = 3;
constexpr int kBlk = 32;     // samples per producer block (one warp's columns)
constexpr int kPairs = kBlk / 2;
constexpr int kMaxBlk = 8;   // N <= 256

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// clock read that stays between the surrounding memory operations (profiling instantiation only)
__device__ __forceinline__ long long clk() {
  long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
  return t;
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n\t}" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// The epoch barrier between the warp-specialised roles (chain warps and producer warps reach it
// from different code): a named barrier over every thread of the CTA, each warp arriving as a
// whole (bar.sync id, count: the warp-specialisation form; __syncthreads() is only defined when
// all threads reach the same call site). Same memory ordering as __syncthreads().
__device__ __forceinline__ void epoch_barrier() {
  __syncwarp();  // the warp reconverges first (inline asm does not imply it)
  asm volatile("barrier.sync 1, %0;" ::"r"(blockDim.x) : "memory");
}

// Parameter offsets of a compiled shape (H2 == 0: one hidden layer), flat layout of
// mlp.cpp:124-131. Record row c (c < P) holds parameter c's per-sample term, row P the loss term.
template <int I, int H1, int H2>
struct PipeShape {
  static_assert(H2 == 0 ? (H1 == 8 && I >= 1 && I <= 7) : (H1 == 5 && H2 == 5 && I >= 1 && I <= 6),
                "compiled pipelined shapes: I-8-1 (I <= 7) and I-5-5-1 (I <= 6)");
  static constexpr int W1 = 0, B1 = I * H1;
  static constexpr int W2 = B1 + H1, B2 = W2 + H1 * H2;
  static constexpr int WO = H2 > 0 ? B2 + H2 : B1 + H1;
  static constexpr int BO = WO + (H2 > 0 ? H2 : H1);
  static constexpr int P = BO + 1;
  static constexpr int ROWS = P + 1;
  static_assert(ROWS <= 32 * kChainWarps, "one chain lane per record row");

  // One sample, forward + backward in the reference order; stores its record column:
  // weight terms (inv_n*delta)*a (mlp.cpp:113), bias terms inv_n*delta (mlp.cpp:117), err^2.
  // w: this epoch's weights (the producer's registers, or the shared-memory copy read in place);
  // r: rec + s (row j at r[j * kLd]).
  template <class Wt>
  __device__ static void sample(const Wt& w, const double (&x)[I], double y, double* __restrict__ r,
                                double inv_n) {
    double a1[H1];
#pragma unroll
    for (int o = 0; o < H1; ++o) {
      double z = w[B1 + o];
#pragma unroll
      for (int i = 0; i < I; ++i) z = __dadd_rn(z, __dmul_rn(w[W1 + o * I + i], x[i]));
      a1[o] = gate(z, z);
    }
    double z;
    double a2[H2 > 0 ? H2 : 1];
    if constexpr (H2 > 0) {
#pragma unroll
      for (int o = 0; o < H2; ++o) {
        double q = w[B2 + o];
#pragma unroll
        for (int i = 0; i < H1; ++i) q = __dadd_rn(q, __dmul_rn(w[W2 + o * H1 + i], a1[i]));
        a2[o] = gate(q, q);
      }
      z = w[BO];
#pragma unroll
      for (int i = 0; i < H2; ++i) z = __dadd_rn(z, __dmul_rn(w[WO + i], a2[i]));
    } else {
      z = w[BO];
#pragma unroll
      for (int i = 0; i < H1; ++i) z = __dadd_rn(z, __dmul_rn(w[WO + i], a1[i]));
    }
    const double err = __dsub_rn(z, y);           // mlp.cpp:90
    const double dout = __dmul_rn(2.0, err);      // mlp.cpp:92
    const double tout = __dmul_rn(inv_n, dout);   // left factor of mlp.cpp:113,117
    r[P * kLd] = __dmul_rn(err, err);             // mlp.cpp:91
    r[BO * kLd] = tout;
    // The reference's delta sums start at 0.0 (mlp.cpp:97-100: acc = 0.0; acc += w*delta); here
    // they start at the first product. The two differ only in the sign of a zero (0.0 + -0.0 is
    // +0.0), and a delta reaches the outputs only through record terms inv_n*delta*a summed into
    // chains that start at +0.0 and never hold -0.0, where +0.0 and -0.0 terms are both no-ops
    // (the ReLU gates test activations, not deltas): every weight, loss and metric is unchanged.
    double t1[H1];
    if constexpr (H2 > 0) {
      double d2[H2];
#pragma unroll
      for (int i = 0; i < H2; ++i) {  // w*delta (mlp.cpp:97-100), ReLU gate
        const double acc = __dmul_rn(w[WO + i], dout);
        d2[i] = gate(a2[i], acc);
        r[(WO + i) * kLd] = __dmul_rn(tout, a2[i]);
      }
#pragma unroll
      for (int o = 0; o < H2; ++o) {
        const double t2 = __dmul_rn(inv_n, d2[o]);
#pragma unroll
        for (int i = 0; i < H1; ++i) r[(W2 + o * H1 + i) * kLd] = __dmul_rn(t2, a1[i]);
        r[(B2 + o) * kLd] = t2;
      }
#pragma unroll
      for (int i = 0; i < H1; ++i) {
        double acc = __dmul_rn(w[W2 + i], d2[0]);
#pragma unroll
        for (int o = 1; o < H2; ++o) acc = __dadd_rn(acc, __dmul_rn(w[W2 + o * H1 + i], d2[o]));
        t1[i] = __dmul_rn(inv_n, gate(a1[i], acc));
      }
    } else {
#pragma unroll
      for (int i = 0; i < H1; ++i) {
        const double acc = __dmul_rn(w[WO + i], dout);
        t1[i] = __dmul_rn(inv_n, gate(a1[i], acc));
        r[(WO + i) * kLd] = __dmul_rn(tout, a1[i]);
      }
    }
#pragma unroll
    for (int o = 0; o < H1; ++o) {
#pragma unroll
      for (int i = 0; i < I; ++i) r[(W1 + o * I + i) * kLd] = __dmul_rn(t1[o], x[i]);
      r[(B1 + o) * kLd] = t1[o];
    }
  }
};

// The Adam step through CUDA's IEEE division and square root (mlp.cpp:149-152): the fallback for
// lanes whose verified short path (exact_fp64.cuh) does not apply.
__device__ __noinline__ double adam_step_ieee(double mk, double vk, double2 bc, double lr, double eps) {
  return __ddiv_rn(__dmul_rn(lr, __ddiv_rn(mk, bc.x)), __dadd_rn(__dsqrt_rn(__ddiv_rn(vk, bc.y)), eps));
}

template <int I, int H1, int H2>
__host__ __device__ constexpr int pipe_smem_doubles() {
  using S = PipeShape<I, H1, H2>;
  // records | weights (even) | loss (2) | mbarriers (<= 8 x u64)
  return S::ROWS * kLd + ((S::P + 1) & ~1) + 2 + 8;
}

// kWsmem: producers read the epoch's weights from shared memory where they are used (broadcast
// loads) instead of holding all P in registers, which frees enough registers for more producer
// warps (every block of an epoch in one round).
template <int I, int H1, int H2, int NPW, bool kProf, bool kWsmem>
__global__ void __launch_bounds__(32 * (kChainWarps + NPW), 1) train_fp64_pipe(TrainArgs a) {
  using S = PipeShape<I, H1, H2>;
  constexpr int R = (kMaxBlk + NPW - 1) / NPW;  // blocks per producer warp at most
  extern __shared__ __align__(16) double smem[];
  double* rec = smem;                                       // [ROWS][kLd]
  double* ws = rec + S::ROWS * kLd;                         // [P] weights (producers' copy)
  double* Ls = ws + ((S::P + 1) & ~1);                      // [2] epoch loss
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(Ls + 2);  // [nb] blocks

  const int m = a.order[blockIdx.x];
  const int tile = a.model_tile[m];
  const int N = a.tile_rows[tile];
  const int nb = (N + kBlk - 1) / kBlk;
  const int E = a.epochs[m];
  const double lr = a.lr[m];
  const int tid = threadIdx.x;
  const double inv_n = 1.0 / (double)N;  // mlp.cpp:84
  const double* gp = a.params + a.param_offset[m];
  const double* X = a.X + a.tile_offset[tile] * 8;
  const double* Y = a.y + a.tile_offset[tile];

  for (int p = tid; p < S::P; p += blockDim.x) ws[p] = gp[p];
  // padding columns (N up to the block end) hold zero terms: they leave every chain unchanged (a
  // chain starts at +0.0 and is never -0.0, and x + (+-0) == x for every other x)
  for (int s = tid; s < kLd; s += blockDim.x)
    for (int j = 0; j < S::ROWS; ++j) rec[j * kLd + s] = 0.0;
  if (tid * NPW < nb) mbar_init(&bar[tid], 32 * NPW);  // one per producer round: every producer thread arrives
  __syncthreads();

  double* trace = a.loss_trace ? a.loss_trace + a.trace_offset[m] : nullptr;
  int bad = -1;
  double last = 0.0;

  if (tid < 32 * kChainWarps) {
    // ---- chain lanes: lane c sums record row c over the samples in order, then Adam ----
    const int p = tid < S::P ? tid : tid == S::P ? -1 : -2;  // parameter, -1 the loss, -2 idle
    const double2* Tr = reinterpret_cast<const double2*>(rec + (tid <= S::P ? tid : S::P) * kLd);
    double wr = p >= 0 ? gp[p] : 0.0, mr = 0.0, vr = 0.0;
    const double beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
    const double c1 = 1.0 - beta1, c2 = 1.0 - beta2;
    long long pc[4] = {0, 0, 0, 0};
    long long k0 = kProf ? clk() : 0;  // epoch start: the previous epoch's barrier exit
    int next_trace = 0;
    double2 A[kPairs], B[kPairs];
    for (int e = 0; e < E; ++e) {
      const unsigned ph = e & 1;
      const double2 bc = a.bias_corr[e];  // issued early: latency hidden behind the chain
      const double y1 = rcp_refined(bc.x), y2 = rcp_refined(bc.y);  // per epoch, off the chain
      long long k1 = 0, k2 = 0;
      double g = 0.0;
      // idle lanes read the loss row with lane S::P (same address: a broadcast, no extra
      // wavefront), so the loads need no branch
      auto load = [&](double2(&dst)[kPairs], int b) {
#pragma unroll
        for (int j = 0; j < kPairs; ++j) dst[j] = Tr[b * kPairs + j];
      };
      auto links = [&](const double2(&cur)[kPairs]) {  // 32 links in sample order (mlp.cpp:106-118)
#pragma unroll
        for (int j = 0; j < kPairs; ++j) {
          g = __dadd_rn(g, cur[j].x);
          g = __dadd_rn(g, cur[j].y);
        }
      };
      // One blocking wait per producer ROUND (NPW blocks of 32 samples); inside a round, block
      // b + 1's 16 loads are issued before block b's 32 links (same basic block, no branch: the
      // block index is clamped instead), so shared-memory latency stays off the chain. Only the
      // first block of the next round waits for its barrier after the current block's links.
      // (A non-blocking barrier test ahead of unconditional loads is unsafe: the loads are not
      // ordered after the test unless they depend on its result.)
      mbar_wait(bar, ph);  // round 0's columns are stored
      if (kProf && (a.prof_flags & 1)) mbar_wait(bar + (nb - 1) / NPW, ph);  // experiment: chain after every round
      if (kProf) k1 = clk();
      load(A, 0);
#pragma unroll
      for (int b = 0; b < kMaxBlk; ++b) {
        if (b < nb) {
          double2(&cur)[kPairs] = (b & 1) ? B : A;
          double2(&nxt)[kPairs] = (b & 1) ? A : B;
          if ((b + 1) % NPW != 0) {  // next block in this (complete) round
            load(nxt, b + 1 < nb ? b + 1 : b);
            links(cur);
          } else {
            links(cur);
            if (b + 1 < nb) {
              mbar_wait(bar + (b + 1) / NPW, ph);
              load(nxt, b + 1);
            }
          }
        }
      }
      if (kProf) k2 = clk();
      if (p >= 0) {  // AdamState::update (mlp.cpp:142-154), bias corrections from the host libm
        const double mk = __dadd_rn(__dmul_rn(beta1, mr), __dmul_rn(c1, g));
        const double vk = __dadd_rn(__dmul_rn(beta2, vr), __dmul_rn(__dmul_rn(c2, g), g));
        mr = mk;
        vr = vk;
        // (lr * (m / bc1)) / (sqrt(v / bc2) + eps) with every division and the square root
        // correctly rounded: a verified short path (exact_fp64.cuh), CUDA's IEEE functions for
        // any lane whose verification fails (zeros, subnormals, huge values)
        bool ok = true;
        const double mhat = div_checked(mk, bc.x, y1, ok);
        const double vhat = div_checked(vk, bc.y, y2, ok);
        const double den = __dadd_rn(sqrt_checked(vhat, ok), eps);
        const double num = __dmul_rn(lr, mhat);
        const double step = div_checked(num, den, rcp_refined(den), ok);
        if (fabs(mk) >= 0x1p-900) {
          wr = __dsub_rn(wr, ok ? step : adam_step_ieee(mk, vk, bc, lr, eps));
        } else if (mk == 0.0) {
          // a unit never active so far: the step is a zero with m's sign (lr, bc1 and the
          // divisor are positive)
          wr = __dsub_rn(wr, copysign(0.0, mk));
        } else if (fabs(wr) < 0x1p-820) {
          wr = __dsub_rn(wr, adam_step_ieee(mk, vk, bc, lr, eps));
        }
        // else: a unit that stopped being active (m decays by 0.9 per epoch and then sticks at
        // the smallest subnormal): |step| <= lr * (|m| / bc1) / eps <= 1e7 |m| < 2^-876 is below
        // half an ulp of |w| >= 2^-820, so RN(w - step) == w exactly and w is unchanged
        ws[p] = wr;
      } else if (p == -1) {
        const double L = __dmul_rn(g, inv_n);  // mlp.cpp:120
        Ls[e & 1] = L;
        if (trace && e == next_trace) {
          trace[e / a.trace_stride] = L;
          next_trace += a.trace_stride;
        }
      }
      long long k3 = 0;
      if (kProf) k3 = clk();
      epoch_barrier();
      if (kProf) {
        const long long k4 = clk();
        pc[0] += k1 - k0;  // epoch start -> producer block 0 stored
        pc[1] += k2 - k1;  // the chains over all samples
        pc[2] += k3 - k2;  // Adam
        pc[3] += k4 - k3;  // epoch barrier
        k0 = k4;
      }
      last = Ls[e & 1];
      if (!isfinite(last)) {  // mlp.cpp:166-169: TrainingError(epoch)
        bad = e;
        break;
      }
    }
    if (p >= 0) a.params[a.param_offset[m] + p] = wr;
    if (p == -1) {
      a.final_loss[m] = last;
      a.nonfinite_epoch[m] = bad;
    }
    if (kProf && tid == 0 && blockIdx.x == 0)
      for (int k = 0; k < 4; ++k) a.phase_cycles[k] = pc[k];
  } else {
    // ---- producer warps: blocks w, w + NPW, ... ; inputs kept in registers ----
    const int w = (tid >> 5) - kChainWarps, k = tid & 31;
    double xr[R][I], yr[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int s = (w + q * NPW) * kBlk + k;
#pragma unroll
      for (int i = 0; i < I; ++i) xr[q][i] = s < N ? X[(size_t)s * 8 + i] : 0.0;
      yr[q] = s < N ? Y[s] : 0.0;
    }
    // profiling: (unused), round 0, round 1 (each from the previous mark: the epoch barrier's wait
    // lands in the first memory access after it, BAR.SYNC.DEFER_BLOCKING), the barrier itself
    long long qc[4] = {0, 0, 0, 0};
    long long q0 = kProf ? clk() : 0;
    for (int e = 0; e < E; ++e) {
      if constexpr (kWsmem) {
        const double* wsm = ws;
#pragma unroll
        for (int q = 0; q < R; ++q) {
          if (q * NPW < nb) {  // a round with at least one block
            const int s = (w + q * NPW) * kBlk + k;
            if (s < N) S::sample(wsm, xr[q], yr[q], rec + s, inv_n);
            mbar_arrive(&bar[q]);  // every producer thread arrives on its round's barrier
          }
        }
      } else {
        double wv[S::P];  // this epoch's weights: one broadcast read per epoch, not per sample
#pragma unroll
        for (int j = 0; j < S::P; ++j) wv[j] = ws[j];
#pragma unroll
        for (int q = 0; q < R; ++q) {
          if (q * NPW < nb) {  // a round with at least one block
            const int s = (w + q * NPW) * kBlk + k;
            if (s < N) S::sample(wv, xr[q], yr[q], rec + s, inv_n);
            mbar_arrive(&bar[q]);  // every producer thread arrives on its round's barrier
            if (kProf && q < 2) {
              const long long t = clk();
              qc[1 + q] += t - q0;
              q0 = t;
            }
          }
        }
      }
      epoch_barrier();
      if (kProf) {
        const long long t = clk();
        qc[3] += t - q0;
        q0 = t;
      }
      last = Ls[e & 1];
      if (!isfinite(last)) break;
    }
    if (kProf && tid == 32 * kChainWarps && blockIdx.x == 0)
      for (int j = 0; j < 4; ++j) a.phase_cycles[4 + j] = qc[j];
  }
}

// ---- latency regime, pair-row records (LANN_FP64_PRODUCERS=42) ------------------------------
// The same epoch as train_fp64_pipe, with the record rows stored in PAIRS: slot k of the
// producer's emission order (PairShape::slot_row) goes to pair k/2, and pair q holds, per sample
// s, the two slots' terms side by side (pair q at rec + q * kLdP, sample s at + 2 s). A producer
// lane then stores two terms with one STS.128 (half the store instructions, and half the
// write-after-read waits of a term DMUL on an earlier store's source register,
// profiles/r02_fp64pipe_stalls.txt), and a chain lane owns a pair: two independent DADD chains per
// thread, fed by one LDS.128 per sample. Two chain warps. Bit-identical: every chain still sums
// its row's terms over samples 0..N-1 in order.
constexpr int kLdP = 514;  // pair stride (doubles): 2 x 256 samples + 2, so 8 lanes' 16-B loads cover the 32 banks
constexpr int kPairWarps = 2;
constexpr int kHalf = 16;  // samples per chain load batch

template <int I, int H1, int H2>
struct PairShape {
  using S = PipeShape<I, H1, H2>;
  static constexpr int SLOTS = (S::ROWS + 1) & ~1;
  static constexpr int NPAIR = SLOTS / 2;
  static_assert(NPAIR <= 32 * kPairWarps, "one chain lane per row pair");
  // record row of emission slot k (the order of PairOut::put calls in sample() below); -2: padding
  __host__ __device__ static int slot_row(int k) {
    if (k == 0) return S::P;
    if (k == 1) return S::BO;
    k -= 2;
    if constexpr (H2 > 0) {
      if (k < H2) return S::WO + k;
      k -= H2;
      if (k < H2 * (H1 + 1)) {
        const int o = k / (H1 + 1), i = k % (H1 + 1);
        return i < H1 ? S::W2 + o * H1 + i : S::B2 + o;
      }
      k -= H2 * (H1 + 1);
    } else {
      if (k < H1) return S::WO + k;
      k -= H1;
    }
    if (k < H1 * (I + 1)) {
      const int o = k / (I + 1), i = k % (I + 1);
      return i < I ? S::W1 + o * I + i : S::B1 + o;
    }
    return -2;
  }
  // the producer's store stream: slots in emission order, two per STS.128 (the slot counter is a
  // compile-time constant after unrolling)
  struct PairOut {
    double* base;  // rec + 2 * sample
    double pend;
    int slot;
    __device__ __forceinline__ void put(double v) {
      if (slot & 1)
        *reinterpret_cast<double2*>(base + (slot >> 1) * kLdP) = make_double2(pend, v);
      else
        pend = v;
      ++slot;
    }
    __device__ __forceinline__ void finish() {
      if (slot & 1) put(0.0);  // padding slot: a zero term
    }
  };
  // PipeShape::sample with the stores through PairOut (same operations, same order)
  template <class Wt>
  __device__ static void sample(const Wt& w, const double (&x)[I], double y, double* __restrict__ base,
                                double inv_n) {
    PairOut out{base, 0.0, 0};
    double a1[H1];
#pragma unroll
    for (int o = 0; o < H1; ++o) {
      double z = w[S::B1 + o];
#pragma unroll
      for (int i = 0; i < I; ++i) z = __dadd_rn(z, __dmul_rn(w[S::W1 + o * I + i], x[i]));
      a1[o] = gate(z, z);
    }
    double z;
    double a2[H2 > 0 ? H2 : 1];
    if constexpr (H2 > 0) {
#pragma unroll
      for (int o = 0; o < H2; ++o) {
        double q = w[S::B2 + o];
#pragma unroll
        for (int i = 0; i < H1; ++i) q = __dadd_rn(q, __dmul_rn(w[S::W2 + o * H1 + i], a1[i]));
        a2[o] = gate(q, q);
      }
      z = w[S::BO];
#pragma unroll
      for (int i = 0; i < H2; ++i) z = __dadd_rn(z, __dmul_rn(w[S::WO + i], a2[i]));
    } else {
      z = w[S::BO];
#pragma unroll
      for (int i = 0; i < H1; ++i) z = __dadd_rn(z, __dmul_rn(w[S::WO + i], a1[i]));
    }
    const double err = __dsub_rn(z, y);          // mlp.cpp:90
    const double dout = __dmul_rn(2.0, err);     // mlp.cpp:92
    const double tout = __dmul_rn(inv_n, dout);  // left factor of mlp.cpp:113,117
    out.put(__dmul_rn(err, err));                // slot 0: the loss term (mlp.cpp:91)
    out.put(tout);                               // slot 1: BO
    double t1[H1];
    if constexpr (H2 > 0) {
      double d2[H2];
#pragma unroll
      for (int i = 0; i < H2; ++i) {
        const double acc = __dmul_rn(w[S::WO + i], dout);
        d2[i] = gate(a2[i], acc);
        out.put(__dmul_rn(tout, a2[i]));  // WO + i
      }
#pragma unroll
      for (int o = 0; o < H2; ++o) {
        const double t2 = __dmul_rn(inv_n, d2[o]);
#pragma unroll
        for (int i = 0; i < H1; ++i) out.put(__dmul_rn(t2, a1[i]));  // W2 + o * H1 + i
        out.put(t2);                                                  // B2 + o
      }
#pragma unroll
      for (int i = 0; i < H1; ++i) {
        double acc = __dmul_rn(w[S::W2 + i], d2[0]);
#pragma unroll
        for (int o = 1; o < H2; ++o) acc = __dadd_rn(acc, __dmul_rn(w[S::W2 + o * H1 + i], d2[o]));
        t1[i] = __dmul_rn(inv_n, gate(a1[i], acc));
      }
    } else {
#pragma unroll
      for (int i = 0; i < H1; ++i) {
        const double acc = __dmul_rn(w[S::WO + i], dout);
        t1[i] = __dmul_rn(inv_n, gate(a1[i], acc));
        out.put(__dmul_rn(tout, a1[i]));  // WO + i
      }
    }
#pragma unroll
    for (int o = 0; o < H1; ++o) {
#pragma unroll
      for (int i = 0; i < I; ++i) out.put(__dmul_rn(t1[o], x[i]));  // W1 + o * I + i
      out.put(t1[o]);                                                // B1 + o
    }
    out.finish();
  }
};

template <int I, int H1, int H2>
__host__ __device__ constexpr int pair_smem_doubles() {
  using Q = PairShape<I, H1, H2>;
  using S = PipeShape<I, H1, H2>;
  // record pairs | weights (even) | loss (2) | mbarriers (<= 8 x u64)
  return Q::NPAIR * kLdP + ((S::P + 1) & ~1) + 2 + 8;
}

template <int I, int H1, int H2, int NPW>
__global__ void __launch_bounds__(32 * (kPairWarps + NPW), 1) train_fp64_pair(TrainArgs a) {
  using S = PipeShape<I, H1, H2>;
  using Q = PairShape<I, H1, H2>;
  constexpr int R = (kMaxBlk + NPW - 1) / NPW;
  extern __shared__ __align__(16) double smem[];
  double* rec = smem;                                       // [NPAIR][kLdP]
  double* ws = rec + Q::NPAIR * kLdP;                       // [P] weights
  double* Ls = ws + ((S::P + 1) & ~1);                      // [2] epoch loss
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(Ls + 2);

  const int m = a.order[blockIdx.x];
  const int tile = a.model_tile[m];
  const int N = a.tile_rows[tile];
  const int nb = (N + kBlk - 1) / kBlk;
  const int nh = 2 * nb;  // chain load batches of kHalf samples
  const int E = a.epochs[m];
  const double lr = a.lr[m];
  const int tid = threadIdx.x;
  const double inv_n = 1.0 / (double)N;  // mlp.cpp:84
  const double* gp = a.params + a.param_offset[m];
  const double* X = a.X + a.tile_offset[tile] * 8;
  const double* Y = a.y + a.tile_offset[tile];

  for (int p = tid; p < S::P; p += blockDim.x) ws[p] = gp[p];
  // padding columns (samples N.. up to the block end) hold zero terms (see train_fp64_pipe)
  for (int q = tid; q < Q::NPAIR * kLdP; q += blockDim.x) rec[q] = 0.0;
  if (tid * NPW < nb) mbar_init(&bar[tid], 32 * NPW);
  __syncthreads();

  double* trace = a.loss_trace ? a.loss_trace + a.trace_offset[m] : nullptr;
  int bad = -1;
  double last = 0.0;

  if (tid < 32 * kPairWarps) {
    // ---- chain lanes: lane c sums the two rows of pair c over the samples in order, then Adam ----
    const int c = tid < Q::NPAIR ? tid : 0;  // idle lanes shadow lane 0 (broadcast loads)
    const int r0 = tid < Q::NPAIR ? Q::slot_row(2 * c) : -2, r1 = tid < Q::NPAIR ? Q::slot_row(2 * c + 1) : -2;
    const int p0 = r0 >= 0 && r0 < S::P ? r0 : r0 == S::P ? -1 : -2;  // parameter, -1 the loss, -2 none
    const int p1 = r1 >= 0 && r1 < S::P ? r1 : r1 == S::P ? -1 : -2;
    const double2* Tr = reinterpret_cast<const double2*>(rec + c * kLdP);
    double w0 = p0 >= 0 ? gp[p0] : 0.0, m0 = 0.0, v0 = 0.0;
    double w1 = p1 >= 0 ? gp[p1] : 0.0, m1 = 0.0, v1 = 0.0;
    const double beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
    const double c1 = 1.0 - beta1, c2 = 1.0 - beta2;
    int next_trace = 0;
    double2 A[kHalf], B[kHalf];
    for (int e = 0; e < E; ++e) {
      const unsigned ph = e & 1;
      const double2 bc = a.bias_corr[e];
      const double y1 = rcp_refined(bc.x), y2 = rcp_refined(bc.y);
      double g0 = 0.0, g1 = 0.0;
      auto load = [&](double2(&dst)[kHalf], int h) {
#pragma unroll
        for (int j = 0; j < kHalf; ++j) dst[j] = Tr[h * kHalf + j];
      };
      auto links = [&](const double2(&cur)[kHalf]) {  // 16 samples, two chains (mlp.cpp:106-118)
#pragma unroll
        for (int j = 0; j < kHalf; ++j) {
          g0 = __dadd_rn(g0, cur[j].x);
          g1 = __dadd_rn(g1, cur[j].y);
        }
      };
      mbar_wait(bar, ph);  // round 0's columns are stored
      load(A, 0);
#pragma unroll
      for (int h = 0; h < 2 * kMaxBlk; ++h) {
        if (h < nh) {
          double2(&cur)[kHalf] = (h & 1) ? B : A;
          double2(&nxt)[kHalf] = (h & 1) ? A : B;
          const int b = h >> 1;
          if (!((h & 1) && (b + 1) % NPW == 0)) {  // the next batch is in this (complete) round
            load(nxt, h + 1 < nh ? h + 1 : h);
            links(cur);
          } else {
            links(cur);
            if (h + 1 < nh) {
              mbar_wait(bar + (b + 1) / NPW, ph);
              load(nxt, h + 1);
            }
          }
        }
      }
      // AdamState::update (mlp.cpp:142-154) for both parameters of the pair, as train_fp64_pipe
      auto adam = [&](double g, double& wr, double& mr, double& vr) {
        const double mk = __dadd_rn(__dmul_rn(beta1, mr), __dmul_rn(c1, g));
        const double vk = __dadd_rn(__dmul_rn(beta2, vr), __dmul_rn(__dmul_rn(c2, g), g));
        mr = mk;
        vr = vk;
        bool ok = true;
        const double mhat = div_checked(mk, bc.x, y1, ok);
        const double vhat = div_checked(vk, bc.y, y2, ok);
        const double den = __dadd_rn(sqrt_checked(vhat, ok), eps);
        const double num = __dmul_rn(lr, mhat);
        const double step = div_checked(num, den, rcp_refined(den), ok);
        if (fabs(mk) >= 0x1p-900) {
          wr = __dsub_rn(wr, ok ? step : adam_step_ieee(mk, vk, bc, lr, eps));
        } else if (mk == 0.0) {
          wr = __dsub_rn(wr, copysign(0.0, mk));
        } else if (fabs(wr) < 0x1p-820) {
          wr = __dsub_rn(wr, adam_step_ieee(mk, vk, bc, lr, eps));
        }
      };
      if (p0 >= 0) adam(g0, w0, m0, v0);
      if (p1 >= 0) adam(g1, w1, m1, v1);
      if (p0 >= 0) ws[p0] = w0;
      if (p1 >= 0) ws[p1] = w1;
      if (p0 == -1 || p1 == -1) {
        const double L = __dmul_rn(p0 == -1 ? g0 : g1, inv_n);  // mlp.cpp:120
        Ls[e & 1] = L;
        if (trace && e == next_trace) {
          trace[e / a.trace_stride] = L;
          next_trace += a.trace_stride;
        }
      }
      epoch_barrier();
      last = Ls[e & 1];
      if (!isfinite(last)) {  // mlp.cpp:166-169: TrainingError(epoch)
        bad = e;
        break;
      }
    }
    if (p0 >= 0) a.params[a.param_offset[m] + p0] = w0;
    if (p1 >= 0) a.params[a.param_offset[m] + p1] = w1;
    if (p0 == -1 || p1 == -1) {
      a.final_loss[m] = last;
      a.nonfinite_epoch[m] = bad;
    }
  } else {
    // ---- producer warps: blocks w, w + NPW, ... ; inputs kept in registers ----
    const int w = (tid >> 5) - kPairWarps, k = tid & 31;
    double xr[R][I], yr[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int s = (w + q * NPW) * kBlk + k;
#pragma unroll
      for (int i = 0; i < I; ++i) xr[q][i] = s < N ? X[(size_t)s * 8 + i] : 0.0;
      yr[q] = s < N ? Y[s] : 0.0;
    }
    for (int e = 0; e < E; ++e) {
      double wv[S::P];
#pragma unroll
      for (int j = 0; j < S::P; ++j) wv[j] = ws[j];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        if (q * NPW < nb) {
          const int s = (w + q * NPW) * kBlk + k;
          if (s < N) Q::sample(wv, xr[q], yr[q], rec + 2 * s, inv_n);
          mbar_arrive(&bar[q]);
        }
      }
      epoch_barrier();
      last = Ls[e & 1];
      if (!isfinite(last)) break;
    }
  }
}

// Pair-row producers with one row per chain lane (LANN_FP64_PRODUCERS=43): the producers of
// train_fp64_pair (two terms per STS.128), the chains and Adam of train_fp64_pipe (three chain
// warps, one slot per lane), each chain lane reading its half of a pair with one 8-byte load per
// sample (a warp's 32 loads: 256 contiguous-in-pairs bytes at the kLdP stride, two wavefronts).
template <int I, int H1, int H2, int NPW>
__global__ void __launch_bounds__(32 * (kChainWarps + NPW), 1) train_fp64_pair1(TrainArgs a) {
  using S = PipeShape<I, H1, H2>;
  using Q = PairShape<I, H1, H2>;
  static_assert(Q::SLOTS <= 32 * kChainWarps, "one chain lane per slot");
  constexpr int R = (kMaxBlk + NPW - 1) / NPW;
  extern __shared__ __align__(16) double smem[];
  double* rec = smem;                                       // [NPAIR][kLdP]
  double* ws = rec + Q::NPAIR * kLdP;                       // [P] weights
  double* Ls = ws + ((S::P + 1) & ~1);                      // [2] epoch loss
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(Ls + 2);

  const int m = a.order[blockIdx.x];
  const int tile = a.model_tile[m];
  const int N = a.tile_rows[tile];
  const int nb = (N + kBlk - 1) / kBlk;
  const int E = a.epochs[m];
  const double lr = a.lr[m];
  const int tid = threadIdx.x;
  const double inv_n = 1.0 / (double)N;  // mlp.cpp:84
  const double* gp = a.params + a.param_offset[m];
  const double* X = a.X + a.tile_offset[tile] * 8;
  const double* Y = a.y + a.tile_offset[tile];

  for (int p = tid; p < S::P; p += blockDim.x) ws[p] = gp[p];
  for (int q = tid; q < Q::NPAIR * kLdP; q += blockDim.x) rec[q] = 0.0;
  if (tid * NPW < nb) mbar_init(&bar[tid], 32 * NPW);
  __syncthreads();

  double* trace = a.loss_trace ? a.loss_trace + a.trace_offset[m] : nullptr;
  int bad = -1;
  double last = 0.0;

  if (tid < 32 * kChainWarps) {
    const int c = tid < Q::SLOTS ? tid : 0;  // idle lanes shadow slot 0 (broadcast loads)
    const int r = tid < Q::SLOTS ? Q::slot_row(c) : -2;
    const int p = r >= 0 && r < S::P ? r : r == S::P ? -1 : -2;
    const double* Tr = rec + (c >> 1) * kLdP + (c & 1);  // sample s at Tr[2 s]
    double wr = p >= 0 ? gp[p] : 0.0, mr = 0.0, vr = 0.0;
    const double beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
    const double c1 = 1.0 - beta1, c2 = 1.0 - beta2;
    int next_trace = 0;
    double A[kBlk], B[kBlk];
    for (int e = 0; e < E; ++e) {
      const unsigned ph = e & 1;
      const double2 bc = a.bias_corr[e];
      const double y1 = rcp_refined(bc.x), y2 = rcp_refined(bc.y);
      double g = 0.0;
      auto load = [&](double(&dst)[kBlk], int b) {
#pragma unroll
        for (int j = 0; j < kBlk; ++j) dst[j] = Tr[2 * (b * kBlk + j)];
      };
      auto links = [&](const double(&cur)[kBlk]) {  // 32 links in sample order (mlp.cpp:106-118)
#pragma unroll
        for (int j = 0; j < kBlk; ++j) g = __dadd_rn(g, cur[j]);
      };
      mbar_wait(bar, ph);
      load(A, 0);
#pragma unroll
      for (int b = 0; b < kMaxBlk; ++b) {
        if (b < nb) {
          double(&cur)[kBlk] = (b & 1) ? B : A;
          double(&nxt)[kBlk] = (b & 1) ? A : B;
          if ((b + 1) % NPW != 0) {
            load(nxt, b + 1 < nb ? b + 1 : b);
            links(cur);
          } else {
            links(cur);
            if (b + 1 < nb) {
              mbar_wait(bar + (b + 1) / NPW, ph);
              load(nxt, b + 1);
            }
          }
        }
      }
      if (p >= 0) {  // AdamState::update (mlp.cpp:142-154), as train_fp64_pipe
        const double mk = __dadd_rn(__dmul_rn(beta1, mr), __dmul_rn(c1, g));
        const double vk = __dadd_rn(__dmul_rn(beta2, vr), __dmul_rn(__dmul_rn(c2, g), g));
        mr = mk;
        vr = vk;
        bool ok = true;
        const double mhat = div_checked(mk, bc.x, y1, ok);
        const double vhat = div_checked(vk, bc.y, y2, ok);
        const double den = __dadd_rn(sqrt_checked(vhat, ok), eps);
        const double num = __dmul_rn(lr, mhat);
        const double step = div_checked(num, den, rcp_refined(den), ok);
        if (fabs(mk) >= 0x1p-900) {
          wr = __dsub_rn(wr, ok ? step : adam_step_ieee(mk, vk, bc, lr, eps));
        } else if (mk == 0.0) {
          wr = __dsub_rn(wr, copysign(0.0, mk));
        } else if (fabs(wr) < 0x1p-820) {
          wr = __dsub_rn(wr, adam_step_ieee(mk, vk, bc, lr, eps));
        }
        ws[p] = wr;
      } else if (p == -1) {
        const double L = __dmul_rn(g, inv_n);  // mlp.cpp:120
        Ls[e & 1] = L;
        if (trace && e == next_trace) {
          trace[e / a.trace_stride] = L;
          next_trace += a.trace_stride;
        }
      }
      epoch_barrier();
      last = Ls[e & 1];
      if (!isfinite(last)) {  // mlp.cpp:166-169: TrainingError(epoch)
        bad = e;
        break;
      }
    }
    if (p >= 0) a.params[a.param_offset[m] + p] = wr;
    if (p == -1) {
      a.final_loss[m] = last;
      a.nonfinite_epoch[m] = bad;
    }
  } else {
    const int w = (tid >> 5) - kChainWarps, k = tid & 31;
    double xr[R][I], yr[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int s = (w + q * NPW) * kBlk + k;
#pragma unroll
      for (int i = 0; i < I; ++i) xr[q][i] = s < N ? X[(size_t)s * 8 + i] : 0.0;
      yr[q] = s < N ? Y[s] : 0.0;
    }
    for (int e = 0; e < E; ++e) {
      double wv[S::P];
#pragma unroll
      for (int j = 0; j < S::P; ++j) wv[j] = ws[j];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        if (q * NPW < nb) {
          const int s = (w + q * NPW) * kBlk + k;
          if (s < N) Q::sample(wv, xr[q], yr[q], rec + 2 * s, inv_n);
          mbar_arrive(&bar[q]);
        }
      }
      epoch_barrier();
      last = Ls[e & 1];
      if (!isfinite(last)) break;
    }
  }
}

// ---- throughput regime: factor records, two CTAs per SM --------------------------------------
// For populations far larger than the GPU (config-3 sweeps) the latency kernel above leaves the SM
// mostly idle: one 7-warp CTA per SM (its ~150 KB of product records and ~230 registers per thread
// forbid a second), FP64 pipe ~27% and shared-memory pipe ~57% busy (profiles/r02_ncu_fp64_sweep.txt).
// This variant stores per sample only the ~22 distinct FACTORS of the terms (mlp.cpp:106-118:
// weight (o, i) adds (inv_n * delta_o) * a_i, a bias adds inv_n * delta_o): tout, the deltas t2[],
// t1[] (inv_n folded in), the activations a2[], a1[], err^2; the inputs x[] and a row of ones are
// static. A chain lane reads its two factor rows and forms each term with the same DMUL the
// producer would have issued, so every term and every chain is bit-identical. Records drop to
// ~60 KB, the producers read the epoch's weights from shared memory where they use them, and the
// kernel is bounded to fit two CTAs (two models) per SM: one model's producers overlap the
// other's chains.
template <int I, int H1, int H2>
struct FactorShape {
  using S = PipeShape<I, H1, H2>;
  static constexpr int R_TO = 0;              // tout = inv_n * 2 * err
  static constexpr int R_A2 = 1;              // a2[H2]   (two hidden layers)
  static constexpr int R_T2 = R_A2 + H2;      // t2[H2] = inv_n * delta2
  static constexpr int R_A1 = R_T2 + H2;      // a1[H1]
  static constexpr int R_T1 = R_A1 + H1;      // t1[H1] = inv_n * delta1
  static constexpr int R_E2 = R_T1 + H1;      // err^2 (loss)
  static constexpr int DYN = R_E2 + 1;
  static constexpr int R_X = DYN;             // x[I] (static)
  static constexpr int R_ONE = R_X + I;       // 1.0 (static)
  static constexpr int ROWS = R_ONE + 1;
  // the two factor rows of chain lane c (parameter c < P, the loss c == P, idle lanes beyond)
  __device__ static void rows_of(int c, int& f1, int& f2) {
    if (c < S::B1) {
      f1 = R_T1 + c / I, f2 = R_X + c % I;
    } else if (c < S::W2) {
      f1 = R_T1 + (c - S::B1), f2 = R_ONE;
    } else if (H2 > 0 && c < S::B2) {
      f1 = R_T2 + (c - S::W2) / H1, f2 = R_A1 + (c - S::W2) % H1;
    } else if (H2 > 0 && c < S::WO) {
      f1 = R_T2 + (c - S::B2), f2 = R_ONE;
    } else if (c < S::BO) {
      f1 = R_TO, f2 = (H2 > 0 ? R_A2 : R_A1) + (c - S::WO);
    } else if (c == S::BO) {
      f1 = R_TO, f2 = R_ONE;
    } else {
      f1 = R_E2, f2 = R_ONE;  // the loss, and idle lanes (discarded)
    }
  }
  // one sample, forward + backward in the reference order (as PipeShape::sample), storing factors
  template <class Wt>
  __device__ static void sample(const Wt& w, const double (&x)[I], double y, double* __restrict__ r,
                                double inv_n) {
    double a1[H1];
#pragma unroll
    for (int o = 0; o < H1; ++o) {
      double z = w[S::B1 + o];
#pragma unroll
      for (int i = 0; i < I; ++i) z = __dadd_rn(z, __dmul_rn(w[S::W1 + o * I + i], x[i]));
      a1[o] = gate(z, z);
    }
    double z;
    double a2[H2 > 0 ? H2 : 1];
    if constexpr (H2 > 0) {
#pragma unroll
      for (int o = 0; o < H2; ++o) {
        double q = w[S::B2 + o];
#pragma unroll
        for (int i = 0; i < H1; ++i) q = __dadd_rn(q, __dmul_rn(w[S::W2 + o * H1 + i], a1[i]));
        a2[o] = gate(q, q);
      }
      z = w[S::BO];
#pragma unroll
      for (int i = 0; i < H2; ++i) z = __dadd_rn(z, __dmul_rn(w[S::WO + i], a2[i]));
    } else {
      z = w[S::BO];
#pragma unroll
      for (int i = 0; i < H1; ++i) z = __dadd_rn(z, __dmul_rn(w[S::WO + i], a1[i]));
    }
    const double err = __dsub_rn(z, y);           // mlp.cpp:90
    const double dout = __dmul_rn(2.0, err);      // mlp.cpp:92
    r[R_TO * kLd] = __dmul_rn(inv_n, dout);       // left factor of mlp.cpp:113,117
    r[R_E2 * kLd] = __dmul_rn(err, err);          // mlp.cpp:91
    if constexpr (H2 > 0) {
      double d2[H2];
#pragma unroll
      for (int i = 0; i < H2; ++i) {  // w*delta (mlp.cpp:97-100), ReLU gate; sums start at the first product
        const double acc = __dmul_rn(w[S::WO + i], dout);
        d2[i] = gate(a2[i], acc);
        r[(R_A2 + i) * kLd] = a2[i];
        r[(R_T2 + i) * kLd] = __dmul_rn(inv_n, d2[i]);
      }
#pragma unroll
      for (int i = 0; i < H1; ++i) {
        double acc = __dmul_rn(w[S::W2 + i], d2[0]);
#pragma unroll
        for (int o = 1; o < H2; ++o) acc = __dadd_rn(acc, __dmul_rn(w[S::W2 + o * H1 + i], d2[o]));
        r[(R_A1 + i) * kLd] = a1[i];
        r[(R_T1 + i) * kLd] = __dmul_rn(inv_n, gate(a1[i], acc));
      }
    } else {
#pragma unroll
      for (int i = 0; i < H1; ++i) {
        const double acc = __dmul_rn(w[S::WO + i], dout);
        r[(R_A1 + i) * kLd] = a1[i];
        r[(R_T1 + i) * kLd] = __dmul_rn(inv_n, gate(a1[i], acc));
      }
    }
  }
};

template <int I, int H1, int H2>
__host__ __device__ constexpr int factor_smem_doubles() {
  using S = PipeShape<I, H1, H2>;
  return FactorShape<I, H1, H2>::ROWS * kLd + ((S::P + 1) & ~1) + 2 + 8;
}

constexpr int kFactorCtasPerSm = 2;

template <int I, int H1, int H2, int NPW, bool kProf>
__global__ void __launch_bounds__(32 * (kChainWarps + NPW), kFactorCtasPerSm) train_fp64_factor(TrainArgs a) {
  using S = PipeShape<I, H1, H2>;
  using F = FactorShape<I, H1, H2>;
  constexpr int R = (kMaxBlk + NPW - 1) / NPW;
  extern __shared__ __align__(16) double smem[];
  double* rec = smem;                                       // [F::ROWS][kLd]
  double* ws = rec + F::ROWS * kLd;
  double* Ls = ws + ((S::P + 1) & ~1);
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(Ls + 2);

  const int m = a.order[blockIdx.x];
  const int tile = a.model_tile[m];
  const int N = a.tile_rows[tile];
  const int nb = (N + kBlk - 1) / kBlk;
  const int E = a.epochs[m];
  const double lr = a.lr[m];
  const int tid = threadIdx.x;
  const double inv_n = 1.0 / (double)N;  // mlp.cpp:84
  const double* gp = a.params + a.param_offset[m];
  const double* X = a.X + a.tile_offset[tile] * 8;
  const double* Y = a.y + a.tile_offset[tile];

  for (int p = tid; p < S::P; p += blockDim.x) ws[p] = gp[p];
  // dynamic rows start at zero (padding columns stay zero terms); static x rows hold the inputs
  // (zero in padding columns), the ones row 1.0 everywhere
  for (int s = tid; s < kLd; s += blockDim.x) {
    for (int j = 0; j < F::DYN; ++j) rec[j * kLd + s] = 0.0;
    for (int i = 0; i < I; ++i) rec[(F::R_X + i) * kLd + s] = s < N ? X[(size_t)s * 8 + i] : 0.0;
    rec[F::R_ONE * kLd + s] = 1.0;
  }
  if (tid * NPW < nb) mbar_init(&bar[tid], 32 * NPW);
  __syncthreads();

  double* trace = a.loss_trace ? a.loss_trace + a.trace_offset[m] : nullptr;
  int bad = -1;
  double last = 0.0;

  if (tid < 32 * kChainWarps) {
    const int p = tid < S::P ? tid : tid == S::P ? -1 : -2;
    int f1, f2;
    F::rows_of(tid, f1, f2);
    const double2* T1 = reinterpret_cast<const double2*>(rec + f1 * kLd);
    const double2* T2 = reinterpret_cast<const double2*>(rec + f2 * kLd);
    double wr = p >= 0 ? gp[p] : 0.0, mr = 0.0, vr = 0.0;
    const double beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
    const double c1 = 1.0 - beta1, c2 = 1.0 - beta2;
    long long pc[4] = {0, 0, 0, 0};
    long long k0 = kProf ? clk() : 0;
    int next_trace = 0;
    constexpr int UP = 4;          // pairs (8 samples) per load unit
    constexpr int kUpr = 4 * NPW;  // units per producer round (a block = 4 units)
    double2 A1[UP], A2[UP], B1[UP], B2[UP];
    const int nu = 4 * nb;
    for (int e = 0; e < E; ++e) {
      const unsigned ph = e & 1;
      const double2 bc = a.bias_corr[e];
      const double y1 = rcp_refined(bc.x), y2 = rcp_refined(bc.y);
      long long k1 = 0, k2 = 0;
      double g = 0.0;
      auto load = [&](double2(&d1)[UP], double2(&d2)[UP], int u) {
#pragma unroll
        for (int j = 0; j < UP; ++j) {
          d1[j] = T1[u * UP + j];
          d2[j] = T2[u * UP + j];
        }
      };
      // 8 links in sample order: each term is the product the producer would have formed
      auto links = [&](const double2(&d1)[UP], const double2(&d2)[UP]) {
#pragma unroll
        for (int j = 0; j < UP; ++j) {
          const double t0 = __dmul_rn(d1[j].x, d2[j].x), t1 = __dmul_rn(d1[j].y, d2[j].y);
          g = __dadd_rn(g, t0);
          g = __dadd_rn(g, t1);
        }
      };
      mbar_wait(bar, ph);  // round 0's factor columns are stored
      if (kProf) k1 = clk();
      load(A1, A2, 0);
#pragma unroll
      for (int u = 0; u < 4 * kMaxBlk; ++u) {
        if (u < nu) {
          double2(&c1r)[UP] = (u & 1) ? B1 : A1;
          double2(&c2r)[UP] = (u & 1) ? B2 : A2;
          double2(&n1r)[UP] = (u & 1) ? A1 : B1;
          double2(&n2r)[UP] = (u & 1) ? A2 : B2;
          if ((u + 1) % kUpr != 0) {  // next unit in this (complete) round
            load(n1r, n2r, u + 1 < nu ? u + 1 : u);
            links(c1r, c2r);
          } else {
            links(c1r, c2r);
            if (u + 1 < nu) {
              mbar_wait(bar + (u + 1) / kUpr, ph);
              load(n1r, n2r, u + 1);
            }
          }
        }
      }
      if (kProf) k2 = clk();
      if (p >= 0) {  // AdamState::update (mlp.cpp:142-154), as train_fp64_pipe
        const double mk = __dadd_rn(__dmul_rn(beta1, mr), __dmul_rn(c1, g));
        const double vk = __dadd_rn(__dmul_rn(beta2, vr), __dmul_rn(__dmul_rn(c2, g), g));
        mr = mk;
        vr = vk;
        bool ok = true;
        const double mhat = div_checked(mk, bc.x, y1, ok);
        const double vhat = div_checked(vk, bc.y, y2, ok);
        const double den = __dadd_rn(sqrt_checked(vhat, ok), eps);
        const double num = __dmul_rn(lr, mhat);
        const double step = div_checked(num, den, rcp_refined(den), ok);
        if (fabs(mk) >= 0x1p-900) {
          wr = __dsub_rn(wr, ok ? step : adam_step_ieee(mk, vk, bc, lr, eps));
        } else if (mk == 0.0) {
          wr = __dsub_rn(wr, copysign(0.0, mk));
        } else if (fabs(wr) < 0x1p-820) {
          wr = __dsub_rn(wr, adam_step_ieee(mk, vk, bc, lr, eps));
        }
        ws[p] = wr;
      } else if (p == -1) {
        const double L = __dmul_rn(g, inv_n);  // mlp.cpp:120
        Ls[e & 1] = L;
        if (trace && e == next_trace) {
          trace[e / a.trace_stride] = L;
          next_trace += a.trace_stride;
        }
      }
      long long k3 = 0;
      if (kProf) k3 = clk();
      epoch_barrier();
      if (kProf) {
        const long long k4 = clk();
        pc[0] += k1 - k0;
        pc[1] += k2 - k1;
        pc[2] += k3 - k2;
        pc[3] += k4 - k3;
        k0 = k4;
      }
      last = Ls[e & 1];
      if (!isfinite(last)) {  // mlp.cpp:166-169: TrainingError(epoch)
        bad = e;
        break;
      }
    }
    if (p >= 0) a.params[a.param_offset[m] + p] = wr;
    if (p == -1) {
      a.final_loss[m] = last;
      a.nonfinite_epoch[m] = bad;
    }
    if (kProf && tid == 0 && blockIdx.x == 0)
      for (int k = 0; k < 4; ++k) a.phase_cycles[k] = pc[k];
  } else {
    const int w = (tid >> 5) - kChainWarps, k = tid & 31;
    double xr[R][I], yr[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int s = (w + q * NPW) * kBlk + k;
#pragma unroll
      for (int i = 0; i < I; ++i) xr[q][i] = s < N ? X[(size_t)s * 8 + i] : 0.0;
      yr[q] = s < N ? Y[s] : 0.0;
    }
    const double* wsm = ws;  // the epoch's weights, read in shared memory where they are used
    for (int e = 0; e < E; ++e) {
#pragma unroll
      for (int q = 0; q < R; ++q) {
        if (q * NPW < nb) {
          const int s = (w + q * NPW) * kBlk + k;
          if (s < N) F::sample(wsm, xr[q], yr[q], rec + s, inv_n);
          mbar_arrive(&bar[q]);
        }
      }
      epoch_barrier();
      last = Ls[e & 1];
      if (!isfinite(last)) break;
    }
  }
}

template <int I, int H1, int H2, int NPW>
void go_factor(const TrainArgs& a, cudaStream_t s) {
  const int dyn = factor_smem_doubles<I, H1, H2>() * 8;
  auto kern = a.phase_cycles ? train_fp64_factor<I, H1, H2, NPW, true> : train_fp64_factor<I, H1, H2, NPW, false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
  kern<<<a.n_models, 32 * (kChainWarps + NPW), dyn, s>>>(a);
}

bool dispatch_factor(const TrainArgs& a, int I, int H1, int H2, cudaStream_t s) {
  if (H1 == 8 && H2 == 0) {
    switch (I) {
      case 1: return go_factor<1, 8, 0, 4>(a, s), true;
      case 2: return go_factor<2, 8, 0, 4>(a, s), true;
      case 3: return go_factor<3, 8, 0, 4>(a, s), true;
      case 4: return go_factor<4, 8, 0, 4>(a, s), true;
      case 5: return go_factor<5, 8, 0, 4>(a, s), true;
      case 6: return go_factor<6, 8, 0, 4>(a, s), true;
      case 7: return go_factor<7, 8, 0, 4>(a, s), true;
    }
  } else if (H1 == 5 && H2 == 5) {
    switch (I) {
      case 4: return go_factor<4, 5, 5, 4>(a, s), true;
      case 5: return go_factor<5, 5, 5, 4>(a, s), true;
      case 6: return go_factor<6, 5, 5, 4>(a, s), true;
    }
  }
  return false;
}

template <int I, int H1, int H2, int NPW, bool kWsmem = (NPW > 4)>
void go_pipe(const TrainArgs& a, cudaStream_t s) {
  const int dyn = pipe_smem_doubles<I, H1, H2>() * 8;
  auto launch = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    kern<<<a.n_models, 32 * (kChainWarps + NPW), dyn, s>>>(a);
  };
  if (a.phase_cycles) {
    TrainArgs b = a;
    if (const char* f = std::getenv("LANN_PROF_FLAGS")) b.prof_flags = std::atoi(f);
    auto kern = train_fp64_pipe<I, H1, H2, NPW, true, kWsmem>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    kern<<<b.n_models, 32 * (kChainWarps + NPW), dyn, s>>>(b);
  }
  else launch(train_fp64_pipe<I, H1, H2, NPW, false, kWsmem>);
}

template <int I, int H1, int H2, bool kOne>
void go_pair(const TrainArgs& a, cudaStream_t s) {
  constexpr int NPW = 4;
  const int dyn = pair_smem_doubles<I, H1, H2>() * 8;
  if constexpr (kOne) {
    auto kern = train_fp64_pair1<I, H1, H2, NPW>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    kern<<<a.n_models, 32 * (kChainWarps + NPW), dyn, s>>>(a);
  } else {
    auto kern = train_fp64_pair<I, H1, H2, NPW>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    kern<<<a.n_models, 32 * (kPairWarps + NPW), dyn, s>>>(a);
  }
}

template <bool kOne>
bool dispatch_pair(const TrainArgs& a, int I, int H1, int H2, cudaStream_t s) {
  if (H1 == 8 && H2 == 0) {
    switch (I) {
      case 1: return go_pair<1, 8, 0, kOne>(a, s), true;
      case 2: return go_pair<2, 8, 0, kOne>(a, s), true;
      case 3: return go_pair<3, 8, 0, kOne>(a, s), true;
      case 4: return go_pair<4, 8, 0, kOne>(a, s), true;
      case 5: return go_pair<5, 8, 0, kOne>(a, s), true;
      case 6: return go_pair<6, 8, 0, kOne>(a, s), true;
      case 7: return go_pair<7, 8, 0, kOne>(a, s), true;
    }
  } else if (H1 == 5 && H2 == 5) {
    switch (I) {
      case 4: return go_pair<4, 5, 5, kOne>(a, s), true;
      case 5: return go_pair<5, 5, 5, kOne>(a, s), true;
      case 6: return go_pair<6, 5, 5, kOne>(a, s), true;
    }
  }
  return false;
}

template <int NPW>
bool dispatch_pipe(const TrainArgs& a, int I, int H1, int H2, cudaStream_t s) {
  if (H1 == 8 && H2 == 0) {
    switch (I) {
      case 1: return go_pipe<1, 8, 0, NPW>(a, s), true;
      case 2: return go_pipe<2, 8, 0, NPW>(a, s), true;
      case 3: return go_pipe<3, 8, 0, NPW>(a, s), true;
      case 4: return go_pipe<4, 8, 0, NPW>(a, s), true;
      case 5: return go_pipe<5, 8, 0, NPW>(a, s), true;
      case 6: return go_pipe<6, 8, 0, NPW>(a, s), true;
      case 7: return go_pipe<7, 8, 0, NPW>(a, s), true;
    }
  } else if (H1 == 5 && H2 == 5) {
    switch (I) {
      case 4: return go_pipe<4, 5, 5, NPW>(a, s), true;
      case 5: return go_pipe<5, 5, 5, NPW>(a, s), true;
      case 6: return go_pipe<6, 5, 5, NPW>(a, s), true;
    }
  }
  return false;
}

}  // namespace

bool fp64_pipe_shape(int in, int h1, int h2) {
  return (h1 == 8 && h2 == 0 && in >= 1 && in <= 7) || (h1 == 5 && h2 == 5 && in >= 4 && in <= 6);
}

// Every model of the launch must have this shape and N <= 256 rows (checked by the caller).
bool launch_train_fp64_pipe(const TrainArgs& a, int I, int H1, int H2, int producer_warps,
                            cudaStream_t s) {
  switch (producer_warps) {
    case 2: return dispatch_pipe<2>(a, I, H1, H2, s);
    case 3: return dispatch_pipe<3>(a, I, H1, H2, s);
    case 8: return dispatch_pipe<8>(a, I, H1, H2, s);
    case 41: return dispatch_factor(a, I, H1, H2, s);  // throughput regime: factor records, 2 CTAs/SM
    case 42: return dispatch_pair<false>(a, I, H1, H2, s);  // latency regime, pair-row records
    case 43: return dispatch_pair<true>(a, I, H1, H2, s);   // pair-row producers, one row per chain lane
    default: return dispatch_pipe<4>(a, I, H1, H2, s);
  }
}

}  // namespace lann
