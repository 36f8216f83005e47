// train_fp64.cu — K1a: the FP64 exact-order LANN trainer ("parity mode").
//
// Reproduces models::train_full_batch (mlp.cpp:156-175) bit for bit: the same
// forward order (mlp.cpp:36-52), the same per-sample delta recursion
// (mlp.cpp:93-104), the same SEQUENTIAL per-parameter gradient accumulation
// over samples (mlp.cpp:106-118), the same Adam expression order
// (mlp.cpp:142-154) and the pre-update loss trace / non-finite check.
// Built with -fmad=false and written with explicit __d*_rn intrinsics so no
// multiply-add is ever contracted (the reference object code has no FMA).
//
// Mapping (one CTA per model, models ordered longest-first):
//   phase A  threads own SAMPLES: forward + backward for their samples, writing the
//            sample's column of the record matrix {x, y, hidden activations,
//            inv_n*delta, err^2};
//   phase B  threads own PARAMETERS: each sums its N per-sample terms in sample
//            order (the only order-sensitive reduction), then applies Adam;
//            one thread sums the loss terms in sample order.
// Product rows (compiled shapes, N <= 256, the default): phase A also forms every weight's
// term t*a for its sample (the same rounded product mlp.cpp:113 forms) and stores it as a
// row, so a phase-B chain is a pure DADD chain over one row (~10.6 cycles per link against
// ~18.7 with the DMUL inside the chain: one warp's FP64 issue, not shared memory, bounded
// those); the single owner keeps w, m, v in registers.
// Two __syncthreads per epoch. The record matrix is stored structure-of-arrays
// (one row per quantity, samples contiguous): phase-A stores are contiguous across
// lanes, and a phase-B chain fetches two samples per 128-bit shared-memory load, so
// the N-long dependent DADD chain (8 cycles per link) — not shared-memory
// wavefronts — bounds the epoch latency. Phase A is compiled per network shape for
// the default topologies (unrolled, immediate offsets); other shapes use a generic path.
#include <cmath>
#include <cstdlib>

#include "exact_fp64.cuh"
#include "kernels.cuh"

namespace lann {
namespace {

constexpr int kMaxKB = 8;  // parameters owned per thread in phase B (P <= 8 * blockDim)

// Record rows: [0,7) inputs x0..x6 | 7 target y | [8, 8+H1) a1 | [.., +H2) a2 |
// t1[H1] | t2[H2] | tout | e2 | ones. Row r of sample s lives at r * ld + s.
__host__ __device__ constexpr int rec_rows(int H1, int H2) {
  return 8 + 2 * (H1 + (H2 > 0 ? H2 : 0)) + 3;
}
__host__ __device__ constexpr int rec_ld(int N) { return (N + 1) & ~1; }  // even: 16-B aligned pairs
// chunked records: a row stride = 2 (mod 16) doubles, so the 16-B loads of lanes reading different
// rows at one sample column fall in distinct bank quads (conflict-free phase-B loads)
__host__ __device__ constexpr int chunk_ld(int ch) { return ((ch + 15) & ~15) + 2; }
// Product-row kernels (N <= 256) use one compile-time row stride: every phase-A record access
// is then an immediate offset from the thread's sample column (no address arithmetic), and
// 258 doubles = 516 words = 4 (mod 32) banks keeps a quarter-warp's 16-B loads of eight
// consecutive rows at one sample conflict-free in phase B.
constexpr int kProdMaxRows = 256;
constexpr int kProdLd = 258;

struct Shape {
  int I, H1, H2, nl, P, R;
  int dims[4];
  int woff[3], boff[3];
  int inoff[3];  // record row of each layer's input vector
  int toff[3];   // record row of each layer's (scaled) deltas
  int e2, ones;  // record rows of err^2 and of the constant 1.0
};

__device__ Shape make_shape(int I, int H1, int H2) {
  Shape s;
  s.I = I;
  s.H1 = H1;
  s.H2 = H2;
  s.nl = H2 > 0 ? 3 : 2;
  s.dims[0] = I;
  s.dims[1] = H1;
  s.dims[2] = H2 > 0 ? H2 : 1;
  s.dims[3] = 1;
  int off = 0;
  for (int l = 0; l < s.nl; ++l) {
    s.woff[l] = off;
    off += s.dims[l] * s.dims[l + 1];
    s.boff[l] = off;
    off += s.dims[l + 1];
  }
  s.P = off;
  const int hidden = H1 + (H2 > 0 ? H2 : 0);
  s.inoff[0] = 0;
  s.inoff[1] = 8;
  s.inoff[2] = 8 + H1;
  const int t0 = 8 + hidden;
  s.toff[0] = t0;
  s.toff[1] = t0 + s.dims[1];
  s.toff[2] = t0 + s.dims[1] + s.dims[2];
  s.e2 = t0 + hidden + 1;
  s.ones = s.e2 + 1;
  s.R = rec_rows(H1, H2);
  return s;
}

// ---- phase A, compiled shape ------------------------------------------------------
template <int I, int H1, int H2>
struct Fixed {
  static constexpr int HS = H1 + H2;
  static constexpr int A1 = 8, A2 = 8 + H1;
  static constexpr int T1 = 8 + HS, T2 = T1 + H1, TO = T1 + HS, E2 = TO + 1;
  static constexpr int W1 = 0, B1 = I * H1;
  static constexpr int W2 = B1 + H1, B2 = W2 + H1 * H2;  // 2 hidden layers
  static constexpr int WO = H2 > 0 ? B2 + H2 : B1 + H1;  // output weights
  static constexpr int BO = WO + (H2 > 0 ? H2 : H1);
  static constexpr int P = BO + 1;
  // product rows (kProd): one per weight, in parameter order without the biases, after the
  // record rows: W1 (o,i) -> PR + o*I + i, W2 (o,i) -> PR + I*H1 + o*H1 + i, output i -> PO + i
  static constexpr int PR = rec_rows(H1, H2);
  static constexpr int P2 = PR + I * H1, PO = P2 + H1 * H2;

  // r = column s of the record matrix (r[row * ld])
  template <bool kProd>
  __device__ static void sample(const double* __restrict__ w, double* __restrict__ r, int ld,
                                double inv_n) {
    double x[I];
#pragma unroll
    for (int i = 0; i < I; ++i) x[i] = r[i * ld];
    const double y = r[7 * ld];
    // layer 1 in groups of 4 neurons (4 DADD chains in flight); the group loop is not
    // unrolled so the weights are not all hoisted into registers at once
    constexpr int G1 = (H1 + 3) / 4;
#pragma unroll 1
    for (int gi = 0; gi < G1; ++gi) {
      double z[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) z[k] = (gi * 4 + k < H1) ? w[B1 + gi * 4 + k] : 0.0;
#pragma unroll
      for (int i = 0; i < I; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (gi * 4 + k < H1) z[k] = __dadd_rn(z[k], __dmul_rn(w[W1 + (gi * 4 + k) * I + i], x[i]));
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (gi * 4 + k < H1) r[(A1 + gi * 4 + k) * ld] = gate(z[k], z[k]);
    }
    if constexpr (H2 == 0 && H1 > 16 && !kProd) {
      // wide one-hidden-layer nets (the unconstrained I-64-1): the activations stay in the record
      // rows just stored instead of a register array, same operation order (no spills)
      double z = w[BO];
      for (int i = 0; i < H1; ++i) z = __dadd_rn(z, __dmul_rn(w[WO + i], r[(A1 + i) * ld]));
      const double err = __dsub_rn(z, y);
      r[E2 * ld] = __dmul_rn(err, err);
      const double dout = __dmul_rn(2.0, err);
      r[TO * ld] = __dmul_rn(inv_n, dout);
#pragma unroll 8
      for (int i = 0; i < H1; ++i) {
        const double acc = __dadd_rn(0.0, __dmul_rn(w[WO + i], dout));
        r[(T1 + i) * ld] = __dmul_rn(inv_n, gate(r[(A1 + i) * ld], acc));
      }
      return;
    }
    double a1[H1];
#pragma unroll
    for (int o = 0; o < H1; ++o) a1[o] = r[(A1 + o) * ld];
    double a2[H2 > 0 ? H2 : 1];
    double z;
    if constexpr (H2 > 0) {
#pragma unroll
      for (int o = 0; o < H2; ++o) a2[o] = w[B2 + o];
#pragma unroll
      for (int i = 0; i < H1; ++i)
#pragma unroll
        for (int o = 0; o < H2; ++o) a2[o] = __dadd_rn(a2[o], __dmul_rn(w[W2 + o * H1 + i], a1[i]));
#pragma unroll
      for (int o = 0; o < H2; ++o) {
        a2[o] = gate(a2[o], a2[o]);
        if constexpr (!kProd) r[(A2 + o) * ld] = a2[o];  // kProd: only phase A reads a2
      }
      z = w[BO];
#pragma unroll
      for (int i = 0; i < H2; ++i) z = __dadd_rn(z, __dmul_rn(w[WO + i], a2[i]));
    } else {
      z = w[BO];
#pragma unroll
      for (int i = 0; i < H1; ++i) z = __dadd_rn(z, __dmul_rn(w[WO + i], a1[i]));
    }
    const double err = __dsub_rn(z, y);
    r[E2 * ld] = __dmul_rn(err, err);
    const double dout = __dmul_rn(2.0, err);
    const double tout = __dmul_rn(inv_n, dout);
    r[TO * ld] = tout;
    double t1[H1];
    if constexpr (H2 > 0) {
      double d2[H2], t2[H2];
#pragma unroll
      for (int i = 0; i < H2; ++i) {
        const double acc = __dadd_rn(0.0, __dmul_rn(w[WO + i], dout));
        d2[i] = gate(a2[i], acc);
        t2[i] = __dmul_rn(inv_n, d2[i]);
        r[(T2 + i) * ld] = t2[i];
      }
      double acc[H1];
#pragma unroll
      for (int i = 0; i < H1; ++i) acc[i] = 0.0;
#pragma unroll
      for (int o = 0; o < H2; ++o)
#pragma unroll
        for (int i = 0; i < H1; ++i) acc[i] = __dadd_rn(acc[i], __dmul_rn(w[W2 + o * H1 + i], d2[o]));
#pragma unroll
      for (int i = 0; i < H1; ++i) {
        t1[i] = __dmul_rn(inv_n, gate(a1[i], acc[i]));
        r[(T1 + i) * ld] = t1[i];
      }
      if constexpr (kProd) {  // the terms t * a of mlp.cpp:113 (same product, formed once here)
#pragma unroll
        for (int i = 0; i < H2; ++i) r[(PO + i) * ld] = __dmul_rn(tout, a2[i]);
#pragma unroll
        for (int o = 0; o < H2; ++o)
#pragma unroll
          for (int i = 0; i < H1; ++i) r[(P2 + o * H1 + i) * ld] = __dmul_rn(t2[o], a1[i]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < H1; ++i) {
        const double acc = __dadd_rn(0.0, __dmul_rn(w[WO + i], dout));
        t1[i] = __dmul_rn(inv_n, gate(a1[i], acc));
        r[(T1 + i) * ld] = t1[i];
      }
      if constexpr (kProd) {
#pragma unroll
        for (int i = 0; i < H1; ++i) r[(PO + i) * ld] = __dmul_rn(tout, a1[i]);
      }
    }
    if constexpr (kProd) {
#pragma unroll
      for (int o = 0; o < H1; ++o)
#pragma unroll
        for (int i = 0; i < I; ++i) r[(PR + o * I + i) * ld] = __dmul_rn(t1[o], x[i]);
    }
  }
};

// ---- phase A, generic shape (runtime loops) ------------------------------------------
__device__ void sample_generic(const Shape& sh, const double* __restrict__ w, double* __restrict__ r,
                               int ld, double inv_n) {
  const double y = r[7 * ld];
  for (int l = 0; l < sh.nl; ++l) {
    const int in = sh.dims[l], out = sh.dims[l + 1];
    const double* wl = w + sh.woff[l];
    const double* bl = w + sh.boff[l];
    const double* ain = r + sh.inoff[l] * ld;
    if (l + 1 < sh.nl) {
      double* aout = r + sh.inoff[l + 1] * ld;
      for (int o = 0; o < out; o += 4) {  // four independent DADD chains in flight
        const int n4 = out - o < 4 ? out - o : 4;
        double z[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) z[k] = k < n4 ? bl[o + k] : 0.0;
        for (int i = 0; i < in; ++i) {
          const double ai = ain[i * ld];
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (k < n4) z[k] = __dadd_rn(z[k], __dmul_rn(wl[(o + k) * in + i], ai));
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (k < n4) aout[(o + k) * ld] = gate(z[k], z[k]);
      }
    } else {
      double z = bl[0];
      for (int i = 0; i < in; ++i) z = __dadd_rn(z, __dmul_rn(wl[i], ain[i * ld]));
      const double err = __dsub_rn(z, y);
      r[sh.e2 * ld] = __dmul_rn(err, err);
      r[sh.toff[l] * ld] = __dmul_rn(2.0, err);  // unscaled output delta (mlp.cpp:92)
    }
  }
  for (int l = sh.nl - 2; l >= 0; --l) {  // hidden deltas from the next layer's, unscaled
    const int nin = sh.dims[l + 1], nout = sh.dims[l + 2];
    const double* wn = w + sh.woff[l + 1];
    const double* dn = r + sh.toff[l + 1] * ld;
    const double* act = r + sh.inoff[l + 1] * ld;
    double* d = r + sh.toff[l] * ld;
    for (int i = 0; i < nin; i += 4) {
      const int n4 = nin - i < 4 ? nin - i : 4;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int o = 0; o < nout; ++o) {
        const double dno = dn[o * ld];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (k < n4) acc[k] = __dadd_rn(acc[k], __dmul_rn(wn[o * nin + i + k], dno));
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < n4) d[(i + k) * ld] = gate(act[(i + k) * ld], acc[k]);
    }
  }
  // scale in place: t = inv_n * delta (the left factor of mlp.cpp:113,117)
  for (int j = sh.toff[0]; j < sh.e2; ++j) r[j * ld] = __dmul_rn(inv_n, r[j * ld]);
}

// Sequential sum over samples 0..N-1 of t[s] * a[s] (or t[s] alone), in sample order.
// Rows are contiguous and 16-B aligned: each 128-bit load brings two samples; two
// alternating register buffers of U pairs keep the loads of the next batch in flight
// while the DADD chain of the current one runs.
template <int U, bool kMul>
__device__ __forceinline__ double chain_sum_impl(const double* __restrict__ tp,
                                                 const double* __restrict__ ap, int N, double g = 0.0) {
  const double2* t2 = reinterpret_cast<const double2*>(tp);
  const double2* a2 = reinterpret_cast<const double2*>(ap);
  const int npairs = N / 2;
  double2 ta[U], xa[U], tb[U], xb[U];
  auto load = [&](int j0, double2* t, double2* x) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      t[u] = t2[j0 + u];
      if (kMul) x[u] = a2[j0 + u];
    }
  };
  auto consume = [&](const double2* t, const double2* x) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      g = __dadd_rn(g, kMul ? __dmul_rn(t[u].x, x[u].x) : t[u].x);
      g = __dadd_rn(g, kMul ? __dmul_rn(t[u].y, x[u].y) : t[u].y);
    }
  };
  int j = 0;
  if (npairs >= U) load(0, ta, xa);
  for (; j + 2 * U <= npairs; j += 2 * U) {
    load(j + U, tb, xb);
    consume(ta, xa);
    if (j + 3 * U <= npairs) load(j + 2 * U, ta, xa);
    consume(tb, xb);
  }
  if (j + U <= npairs) {
    consume(ta, xa);
    j += U;
  }
  for (int s = 2 * j; s < N; ++s) g = __dadd_rn(g, kMul ? __dmul_rn(tp[s], ap[s]) : tp[s]);
  return g;
}

template <int KB, int I, int H1, int H2, bool SMEM, bool PROD = false>
__global__ void __launch_bounds__(256) train_fp64_exact(TrainArgs a) {
  constexpr bool kFixed = I > 0;
  static_assert(!PROD || (kFixed && SMEM && KB == 1), "product rows: compiled shapes in shared memory");
  using F = Fixed<(I > 0 ? I : 1), (H1 > 0 ? H1 : 1), H2>;
  extern __shared__ double smem[];
  const int m = a.order[blockIdx.x];
  const int tile = a.model_tile[m];
  const int N = a.tile_rows[tile];
  const int E = a.epochs[m];
  const double lr = a.lr[m];
  const Shape sh = make_shape(a.tile_inputs[tile], a.h1[m], a.h2[m]);
  const int P = sh.P;
  // SMEM with a.rec_chunk: the records hold CH samples at a time; the sample range is processed
  // in chunks, in order, and every chain carries its partial sum from one chunk to the next
  const int CH = (SMEM && a.rec_chunk > 0 && a.rec_chunk < N) ? a.rec_chunk : N;
  const bool chunked = CH < N;
  const int ld = PROD ? kProdLd : chunked ? chunk_ld(CH) : rec_ld(CH);
  const int tid = threadIdx.x, nt = blockDim.x;

  double* w = smem;           // [P]
  double* mom = w + P;        // [P] Adam m
  double* vel = mom + P;      // [P] Adam v
  double* Ls = vel + P;       // [1] epoch loss
  // SMEM: the record matrix follows the model state in shared memory, 16-B aligned (a
  // pointer the compiler can prove is shared: every access is an LDS/STS); else global scratch
  double* rec;
  if constexpr (SMEM) rec = smem + ((3 * P + 2 + 1) & ~1);
  else rec = a.scratch + a.scratch_offset[m];

  const double* gp = a.params + a.param_offset[m];
  for (int p = tid; p < P; p += nt) {
    w[p] = gp[p];
    mom[p] = 0.0;
    vel[p] = 0.0;
  }
  // KB == 1: the owner keeps w, m, v of its parameter in registers (smem w is phase A's copy)
  double wr = (KB == 1 && tid < P) ? gp[tid] : 0.0, mr = 0.0, vr = 0.0;
  const double* X = a.X + a.tile_offset[tile] * 8;
  const double* Y = a.y + a.tile_offset[tile];
  // inputs use rows 0..I-1 (I <= 7), row 7 holds the target, bias terms are t * 1.0 (exact)
  auto stage_inputs = [&](int c0, int nc) {
    for (int s = tid; s < nc; s += nt) {
      for (int i = 0; i < 7; ++i) rec[i * ld + s] = X[(size_t)(c0 + s) * 8 + i];
      rec[7 * ld + s] = Y[c0 + s];
      rec[sh.ones * ld + s] = 1.0;
    }
  };
  if (!chunked) stage_inputs(0, N);


  // phase-B ownership: parameter p -> (record row of its delta, of its input or of 1.0)
  int tix[KB], aix[KB];
#pragma unroll
  for (int k = 0; k < KB; ++k) {
    const int p = tid + k * nt;
    tix[k] = -1;
    aix[k] = -1;
    if (p < P) {
      for (int l = 0; l < sh.nl; ++l) {
        const int in = sh.dims[l], out = sh.dims[l + 1];
        if (p >= sh.woff[l] && p < sh.boff[l]) {
          const int q = p - sh.woff[l];
          tix[k] = sh.toff[l] + q / in;
          aix[k] = sh.inoff[l] + q % in;
          if (PROD) {  // the product row phase A stored: a pure DADD chain
            tix[k] = F::PR + (l == 0 ? 0 : l == 1 && sh.nl == 3 ? F::P2 - F::PR : F::PO - F::PR) + q;
            aix[k] = -2;
          }
        } else if (p >= sh.boff[l] && p < sh.boff[l] + out) {
          tix[k] = sh.toff[l] + (p - sh.boff[l]);
          aix[k] = PROD ? -2 : sh.ones;  // x 1.0 is exact: PROD sums the delta row itself
        }
      }
    }
  }
  const int e2row = sh.e2;
  const int loss_tid = nt - 1;
  const double inv_n = 1.0 / (double)N;  // mlp.cpp:84
  const double beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
  const double c1 = 1.0 - beta1, c2 = 1.0 - beta2;
  double* trace = a.loss_trace ? a.loss_trace + a.trace_offset[m] : nullptr;
  int bad = -1;
  double last = 0.0;
  __syncthreads();

  const bool prof = a.phase_cycles && blockIdx.x == 0 && tid == 0;
  long long pc[4] = {0, 0, 0, 0};
  for (int e = 0; e < E; ++e) {
    const long long clk0 = prof ? clock64() : 0;
    const double2 bc = a.bias_corr[e];  // issued early: its latency hides behind phase A
    double g[KB];
#pragma unroll
    for (int k = 0; k < KB; ++k) g[k] = 0.0;
    double Lacc = 0.0;
    long long clk1 = 0, clk2 = 0, tA = 0, tB = 0;
    for (int c0 = 0; c0 < N; c0 += CH) {
      const int nc = N - c0 < CH ? N - c0 : CH;
      if (chunked) {
        if (c0 > 0) __syncthreads();  // the previous chunk's chains are done with the records
        stage_inputs(c0, nc);
        __syncthreads();
      }
      const long long ca = prof ? clock64() : 0;
      // ---- phase A: per-sample forward / backward (mlp.cpp:86-104) ----
      for (int s = tid; s < nc; s += nt) {
        if constexpr (kFixed) F::template sample<PROD>(w, rec + s, ld, inv_n);
        else sample_generic(sh, w, rec + s, ld, inv_n);
      }
      __syncthreads();
      if (prof) {
        clk1 = clock64();
        tA += clk1 - ca;
      }
      // ---- phase B: sequential per-parameter sums, continued over this chunk (mlp.cpp:106-118) ----
      if (tix[0] >= 0) {
        if (PROD) {
          g[0] = chain_sum_impl<4, false>(rec + tix[0] * ld, nullptr, nc, g[0]);
        } else if (KB == 1) {
          g[0] = chain_sum_impl<4, true>(rec + tix[0] * ld, rec + aix[0] * ld, nc, g[0]);
        } else {
          // the KB chains of a thread advance together (independent DADD chains interleave), two
          // samples per 16-B load, the next pair's loads in flight while the current pair's links
          // run; unowned slots read row 0 and are discarded
          const double2* r2 = reinterpret_cast<const double2*>(rec);
          int tr[KB], ar[KB];
#pragma unroll
          for (int k = 0; k < KB; ++k) {
            tr[k] = (tix[k] >= 0 ? tix[k] : 0) * (ld / 2);
            ar[k] = (tix[k] >= 0 ? aix[k] : 0) * (ld / 2);
          }
          const int npairs = nc / 2;
          double2 ct[KB], ca[KB];
#pragma unroll
          for (int k = 0; k < KB; ++k) ct[k] = r2[tr[k]], ca[k] = r2[ar[k]];
          for (int j = 0; j < npairs; ++j) {
            const int jn = j + 1 < npairs ? j + 1 : j;
            double p0[KB], p1[KB];
#pragma unroll
            for (int k = 0; k < KB; ++k) {
              p0[k] = __dmul_rn(ct[k].x, ca[k].x);
              p1[k] = __dmul_rn(ct[k].y, ca[k].y);
              ct[k] = r2[tr[k] + jn];
              ca[k] = r2[ar[k] + jn];
            }
#pragma unroll
            for (int k = 0; k < KB; ++k)
              if (tix[k] >= 0) g[k] = __dadd_rn(__dadd_rn(g[k], p0[k]), p1[k]);
          }
          if (nc & 1) {
            const int sl = nc - 1;
#pragma unroll
            for (int k = 0; k < KB; ++k)
              if (tix[k] >= 0) g[k] = __dadd_rn(g[k], __dmul_rn(rec[tix[k] * ld + sl], rec[aix[k] * ld + sl]));
          }
        }
      }
      if (tid == loss_tid) Lacc = chain_sum_impl<4, false>(rec + e2row * ld, nullptr, nc, Lacc);
      if (prof) {
        clk2 = clock64();
        tB += clk2 - clk1;
      }
    }
    if (tix[0] >= 0) {
      if (KB == 1) {
        const double mk = __dadd_rn(__dmul_rn(beta1, mr), __dmul_rn(c1, g[0]));
        const double vk = __dadd_rn(__dmul_rn(beta2, vr), __dmul_rn(__dmul_rn(c2, g[0]), g[0]));
        mr = mk;
        vr = vk;
        const double mhat = __ddiv_rn(mk, bc.x);
        const double vhat = __ddiv_rn(vk, bc.y);
        wr = __dsub_rn(wr, __ddiv_rn(__dmul_rn(lr, mhat), __dadd_rn(__dsqrt_rn(vhat), eps)));
        w[tid] = wr;
      } else
#pragma unroll
      for (int k = 0; k < KB; ++k) {
        const int p = tid + k * nt;
        if (tix[k] >= 0) {
          const double mk = __dadd_rn(__dmul_rn(beta1, mom[p]), __dmul_rn(c1, g[k]));
          const double vk = __dadd_rn(__dmul_rn(beta2, vel[p]), __dmul_rn(__dmul_rn(c2, g[k]), g[k]));
          mom[p] = mk;
          vel[p] = vk;
          const double mhat = __ddiv_rn(mk, bc.x);
          const double vhat = __ddiv_rn(vk, bc.y);
          w[p] = __dsub_rn(w[p], __ddiv_rn(__dmul_rn(lr, mhat), __dadd_rn(__dsqrt_rn(vhat), eps)));
        }
      }
    }
    if (tid == loss_tid) {
      const double L = __dmul_rn(Lacc, inv_n);  // mlp.cpp:120
      Ls[0] = L;
      if (trace && (e % a.trace_stride) == 0) trace[e / a.trace_stride] = L;
    }
    const long long clk3 = prof ? clock64() : 0;
    __syncthreads();
    if (prof) {
      const long long clk4 = clock64();
      pc[0] += tA;           // phase A + barrier (all chunks)
      pc[1] += tB;           // parameter-0 chains (all chunks)
      pc[2] += clk3 - clk2;  // its Adam step
      pc[3] += clk4 - clk3 + (clk1 - clk0) - tA - tB;  // waits + chunk staging
    }
    last = Ls[0];
    if (!isfinite(last)) {  // mlp.cpp:166-169: TrainingError(epoch) before the update
      bad = e;
      break;
    }
  }
  if (prof)
    for (int k = 0; k < 4; ++k) a.phase_cycles[k] = pc[k];

  double* outp = a.params + a.param_offset[m];
  for (int p = tid; p < P; p += nt) outp[p] = w[p];
  if (tid == 0) {
    a.final_loss[m] = last;
    a.nonfinite_epoch[m] = bad;
  }
}

}  // namespace

// doubles of record matrix per model (rows x padded samples) and of model state
size_t fp64_record_bytes(int in, int h1, int h2, int n) {
  (void)in;
  return size_t(rec_rows(h1, h2)) * size_t(rec_ld(n)) * 8;
}
size_t fp64_product_record_bytes(int in, int h1, int h2, int n) {
  const int nw = in * h1 + h1 * h2 + (h2 > 0 ? h2 : h1);
  if (n > kProdMaxRows) return ~size_t(0) >> 1;  // never fits: products need N <= 256
  return size_t(rec_rows(h1, h2) + nw) * size_t(kProdLd) * 8;
}
size_t fp64_state_bytes(int p) { return size_t((3 * p + 2 + 1) & ~1) * 8; }
int fp64_record_rows(int h1, int h2) { return rec_rows(h1, h2); }
int fp64_chunk_ld(int ch) { return chunk_ld(ch); }

bool fp64_shape_compiled(int in, int h1, int h2) {
  if (h1 == 8 && h2 == 0) return in >= 1 && in <= 7;
  if (h1 == 5 && h2 == 5) return in >= 4 && in <= 6;
  if (h1 == 64 && h2 == 0) return in >= 1 && in <= 7;  // the unconstrained prediction nets (x8 widths)
  return false;
}

// Dynamic shared memory = model state (3P + 2 doubles, padded even), plus the record
// matrix when a.smem_records is set; the host sizes dyn_bytes for the largest model.
// shape = {I, H1, H2} when every model of the launch has that compiled shape, else null.
void launch_train_fp64(const TrainArgs& a, int max_p, int dyn_bytes, const int* shape,
                       cudaStream_t s) {
  const int block = 256;
  const int kb = (max_p + block - 1) / block;
  // product-row buckets (compiled shape, every model N <= 256) run the pipelined trainer
  // (train_fp64_pipe.cu) unless LANN_FP64_PHASED asks for this phased one
  if (shape && shape[0] > 0 && a.smem_records && a.rec_products && !std::getenv("LANN_FP64_PHASED") &&
      fp64_pipe_shape(shape[0], shape[1], shape[2])) {
    // latency regime (fewer models than ~2 per SM: config 2): the product-record kernel, one CTA
    // per SM; throughput regime (sweeps): factor records, two CTAs (models) per SM
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int npw = a.n_models >= 2 * sms ? 41 : 4;
    if (const char* env = std::getenv("LANN_FP64_PRODUCERS")) npw = std::atoi(env);
    if (launch_train_fp64_pipe(a, shape[0], shape[1], shape[2], npw, s)) return;
  }
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_bytes);
    kern<<<a.n_models, block, dyn_bytes, s>>>(a);
  };

  if (shape && shape[0] > 0 && kb <= 1 && a.smem_records && a.rec_products) {
    const int I = shape[0], H1 = shape[1], H2 = shape[2];
    if (H1 == 8 && H2 == 0) {
      switch (I) {
        case 1: return go(train_fp64_exact<1, 1, 8, 0, true, true>);
        case 2: return go(train_fp64_exact<1, 2, 8, 0, true, true>);
        case 3: return go(train_fp64_exact<1, 3, 8, 0, true, true>);
        case 4: return go(train_fp64_exact<1, 4, 8, 0, true, true>);
        case 5: return go(train_fp64_exact<1, 5, 8, 0, true, true>);
        case 6: return go(train_fp64_exact<1, 6, 8, 0, true, true>);
        case 7: return go(train_fp64_exact<1, 7, 8, 0, true, true>);
      }
    } else if (H1 == 5 && H2 == 5) {
      switch (I) {
        case 4: return go(train_fp64_exact<1, 4, 5, 5, true, true>);
        case 5: return go(train_fp64_exact<1, 5, 5, 5, true, true>);
        case 6: return go(train_fp64_exact<1, 6, 5, 5, true, true>);
      }
    }
  }
  if (shape && shape[0] > 0 && kb <= 1 && a.smem_records) {
    const int I = shape[0], H1 = shape[1], H2 = shape[2];
    if (H1 == 8 && H2 == 0) {
      switch (I) {
        case 1: return go(train_fp64_exact<1, 1, 8, 0, true>);
        case 2: return go(train_fp64_exact<1, 2, 8, 0, true>);
        case 3: return go(train_fp64_exact<1, 3, 8, 0, true>);
        case 4: return go(train_fp64_exact<1, 4, 8, 0, true>);
        case 5: return go(train_fp64_exact<1, 5, 8, 0, true>);
        case 6: return go(train_fp64_exact<1, 6, 8, 0, true>);
        case 7: return go(train_fp64_exact<1, 7, 8, 0, true>);
      }
    } else if (H1 == 5 && H2 == 5) {
      switch (I) {
        case 4: return go(train_fp64_exact<1, 4, 5, 5, true>);
        case 5: return go(train_fp64_exact<1, 5, 5, 5, true>);
        case 6: return go(train_fp64_exact<1, 6, 5, 5, true>);
      }
    }
  }
  if (shape && shape[0] > 0 && shape[1] == 64 && shape[2] == 0 && kb <= 3 && a.smem_records) {
    switch (shape[0]) {  // unconstrained I-64-1 nets: phase A unrolled, activations in registers
      case 1: return go(train_fp64_exact<3, 1, 64, 0, true>);
      case 2: return go(train_fp64_exact<3, 2, 64, 0, true>);
      case 3: return go(train_fp64_exact<3, 3, 64, 0, true>);
      case 4: return go(train_fp64_exact<3, 4, 64, 0, true>);
      case 5: return go(train_fp64_exact<3, 5, 64, 0, true>);
      case 6: return go(train_fp64_exact<3, 6, 64, 0, true>);
      case 7: return go(train_fp64_exact<3, 7, 64, 0, true>);
    }
  }
  if (a.smem_records) {
    if (kb <= 1) go(train_fp64_exact<1, 0, 0, 0, true>);
    else if (kb <= 2) go(train_fp64_exact<2, 0, 0, 0, true>);
    else if (kb <= 4) go(train_fp64_exact<4, 0, 0, 0, true>);
    else go(train_fp64_exact<kMaxKB, 0, 0, 0, true>);
  } else {
    if (kb <= 1) go(train_fp64_exact<1, 0, 0, 0, false>);
    else if (kb <= 2) go(train_fp64_exact<2, 0, 0, 0, false>);
    else if (kb <= 4) go(train_fp64_exact<4, 0, 0, 0, false>);
    else go(train_fp64_exact<kMaxKB, 0, 0, 0, false>);
  }
}

}  // namespace lann
