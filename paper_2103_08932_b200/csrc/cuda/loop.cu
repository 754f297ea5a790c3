// Device-resident time loop (reference: proj/src/tlsph/runner.cpp:341-391).
//
// Per step the GPU runs, with no host synchronisation:
//   step_begin (one reduction kernel; its last block does the scalar work:
//               accounting of the previous step, t += dt, ++steps, NaN check,
//               probe sample at output marks, end/KE stop test,
//               stable_dt -> dt)
//   verlet passes A, B, C                      (elastic, captured as a graph)
//   folds + colour phases of the damping sweep (damped steps only, a graph)
// The eta~ sequence is state independent (one RandomSource draw per step,
// runner.cpp:358-360), so the host draws it up front and launches the
// damped or undamped graph per step; every kernel reads dt from device
// memory and returns immediately once the loop has halted.
#include <algorithm>
#include <cmath>
#include <random>
#include <vector>

#include "system.cuh"

namespace tlsph_cuda {

void enqueue_verlet(DevSystem& s, const DMaterial& mat, double dt, int loop);
void enqueue_explicit(DevSystem& s, double eta, double* acc);

namespace {

unsigned grid_for(long long n, int block) { return static_cast<unsigned>((n + block - 1) / block); }

enum Param { P_H = 0, P_C = 1, P_VISC = 2, P_FIXED_DT = 3, P_END = 4 };

template <int D>
__global__ void k_step_begin(DFields f, DScalars* sc, double* __restrict__ partials, int finalize) {
  if (sc->halt) return;
  __shared__ double s_v[256], s_a[256], s_k[256];
  __shared__ bool last;
  const int want_ke = sc->ke_stop;
  // check_finite runs after a completed step only (runner.cpp:379), never on
  // the initial state.
  const bool check = sc->pending != 0;
  double vmax = 0.0, amax = 0.0, ke = 0.0;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < f.n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (!is_owned(f, i)) continue;
    double sv = f.v[0][i] * f.v[0][i], sa = f.a[0][i] * f.a[0][i];
    bool fin = isfinite(f.v[0][i]) && isfinite(f.r[0][i]);
#pragma unroll
    for (int d = 1; d < D; ++d) {
      sv = sv + f.v[d][i] * f.v[d][i];
      sa = sa + f.a[d][i] * f.a[d][i];
      fin = fin && isfinite(f.v[d][i]) && isfinite(f.r[d][i]);
    }
    vmax = fmax(vmax, sqrt(sv));
    amax = fmax(amax, sqrt(sa));
    if (want_ke) ke += 0.5 * f.m[i] * sv;
    if (check && !fin) record_error(sc, ERR_NAN, static_cast<unsigned long long>(f.perm[i]));
  }
  s_v[threadIdx.x] = vmax;
  s_a[threadIdx.x] = amax;
  s_k[threadIdx.x] = ke;
  __syncthreads();
  for (int off = 128; off > 0; off >>= 1) {
    if (threadIdx.x < off) {
      s_v[threadIdx.x] = fmax(s_v[threadIdx.x], s_v[threadIdx.x + off]);
      s_a[threadIdx.x] = fmax(s_a[threadIdx.x], s_a[threadIdx.x + off]);
      s_k[threadIdx.x] += s_k[threadIdx.x + off];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    atomicMax(&sc->vmax_bits, ordered_bits(s_v[0]));
    atomicMax(&sc->amax_bits, ordered_bits(s_a[0]));
    partials[blockIdx.x] = s_k[0];
    __threadfence();
    last = atomicAdd(&sc->block_counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // the last block sums the per-block KE partials in parallel (fixed order: strided per thread,
  // then the shared-memory tree), so the serial tail does not walk them one by one
  if (want_ke) {
    const volatile double* pv = partials;
    double e = 0.0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) e += pv[b];
    s_k[threadIdx.x] = e;
    __syncthreads();
    for (int off = 128; off > 0; off >>= 1) {
      if (threadIdx.x < off) s_k[threadIdx.x] += s_k[threadIdx.x + off];
      __syncthreads();
    }
  }
  if (threadIdx.x != 0) return;
  // ---- serial tail (one thread)
  sc->block_counter = 0;
  const double vm = from_ordered_bits(atomicExch(&sc->vmax_bits, 0ull));
  const double am = from_ordered_bits(atomicExch(&sc->amax_bits, 0ull));
  const double end_time = sc->params[P_END];
  bool mark = false;
  if (sc->pending) {  // accounting of the step that just finished (runner.cpp:376-379)
    sc->t = sc->t + sc->dt;
    sc->steps += 1;
    sc->last_dt = sc->dt;
    sc->pending = 0;
    // probe output (runner.cpp:381-383); after check_finite, which is
    // resolved below through `failed`
    const double eps = 1e-12 * end_time;
    if (sc->probe >= 0 && sc->interval > 0.0 && sc->t >= sc->next_mark - eps) {
      if (sc->probe_count < sc->probe_cap) {
        double* out = sc->probe_buf + 4 * sc->probe_count;
        out[0] = sc->t;
        for (int d = 0; d < 3; ++d)
          out[1 + d] = d < D ? f.r[d][sc->probe] - f.r0[d][sc->probe] : 0.0;
      }
      sc->probe_count += 1;
      while (sc->next_mark <= sc->t + eps) sc->next_mark += sc->interval;
      mark = true;
    }
  }
  if (*reinterpret_cast<volatile int*>(&sc->failed)) {
    sc->err_step = sc->steps;
    sc->halt = 1;
    return;
  }
  if (want_ke) {
    const double e = s_k[0];
    sc->ke = e;
    if (e > sc->ke_peak) sc->ke_peak = e;
    if (sc->steps > 0 && e < sc->ke_peak && e < sc->ke_ratio * sc->ke_peak) {
      sc->stopped_on_ke = 1;
      sc->done = 1;
      sc->halt = 1;
      return;
    }
  }
  if (mark && sc->pause_on_mark) {  // the host writes a snapshot, then resumes
    sc->paused = 1;
    sc->halt = 1;
    return;
  }
  if (finalize) {
    sc->halt = 1;
    return;
  }
  if (end_time > 0.0 && !(sc->t < end_time)) {  // while (t < end_time)
    sc->done = 1;
    sc->halt = 1;
    return;
  }
  double dt;
  if (sc->params[P_FIXED_DT] > 0.0) {
    dt = sc->params[P_FIXED_DT];
  } else {
    // stable_dt (integrator.cpp:154-169) then the viscous bound (runner.cpp:343-351)
    const double h = sc->params[P_H];
    double bound = h / (sc->params[P_C] + vm);
    if (am > 0.0) {
      const double b2 = sqrt(h / am);
      bound = b2 < bound ? b2 : bound;
    }
    dt = 0.6 * bound;
    const double vb = sc->params[P_VISC];
    if (vb > 0.0) dt = vb < dt ? vb : dt;
  }
  if (end_time > 0.0) {
    const double rest = end_time - sc->t;
    dt = rest < dt ? rest : dt;  // runner.cpp:352
  }
  sc->dt = dt;
  sc->pending = 1;
}

struct Graph {
  cudaGraph_t g = nullptr;
  cudaGraphExec_t e = nullptr;
  ~Graph() {
    if (e) cudaGraphExecDestroy(e);
    if (g) cudaGraphDestroy(g);
  }
};

template <typename Fn>
void capture(cudaStream_t st, Graph& out, Fn&& fn) {
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  fn();
  CK(cudaStreamEndCapture(st, &out.g));
  CK(cudaGraphInstantiate(&out.e, out.g, 0));
}

// kernel nodes of a captured graph (the launches one replay issues)
uint64_t kernel_nodes(const Graph& g) {
  if (!g.g) return 0;
  size_t count = 0;
  CK(cudaGraphGetNodes(g.g, nullptr, &count));
  std::vector<cudaGraphNode_t> nodes(count);
  if (count) CK(cudaGraphGetNodes(g.g, nodes.data(), &count));
  uint64_t k = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType t;
    CK(cudaGraphNodeGetType(nd, &t));
    if (t == cudaGraphNodeTypeKernel) ++k;
  }
  return k;
}

}  // namespace

void DevSystem::run(const tlsph_dev_loop_params& p, tlsph_dev_loop_result& res) {
  res = tlsph_dev_loop_result{};
  if (p.end_time <= 0.0 && p.max_steps == 0)
    throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "loop needs end_time > 0 or max_steps > 0");
  const bool damping_active = p.eta > 0.0;
  if (damping_active && !(p.alpha > 0.0 && p.alpha <= 1.0))
    throw DevError(TLSPH_ERR_INVALID_ARGUMENT,
                   "random-choice probability must lie in (0, 1], got " + std::to_string(p.alpha));
  if (p.resume && !loop_paused) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "no paused or completed loop to resume");
  const DMaterial mat = to_dmat(p.material);
  const bool want_probe = p.probe_index >= 0 && p.output_interval > 0.0;
  if (want_probe && (p.probe_index >= n || (p.probe_capacity > 0 && !p.probe_out)))
    throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "probe index or buffer invalid");

  if (!p.resume) {
    DScalars init{};
    for (int k = 0; k < ERR_SITES; ++k) init.err_key[k] = ~0ull;
    init.ke_stop = p.ke_stop;
    init.ke_ratio = p.ke_ratio;
    init.params[P_H] = p.h;
    init.params[P_C] = p.material.c;
    init.params[P_FIXED_DT] = p.fixed_dt;
    init.params[P_END] = p.end_time;
    if (damping_active) {
      // viscous_dt_bounds(h, eta/(alpha rho0), D) (damping.cpp:12-27, runner.cpp:317-320)
      const double nu = p.eta / (p.alpha * p.material.rho0);
      const double expl = 0.5 * p.h * p.h / (nu * D);
      const double impl = 50.0 * p.h * p.h / (nu * D);
      if (p.scheme == TLSPH_SCHEME_EXPLICIT) init.params[P_VISC] = expl;
      else if (p.scheme == TLSPH_SCHEME_PARTICLE_SPLIT) init.params[P_VISC] = impl;
    }
    init.interval = p.output_interval;
    init.next_mark = p.output_interval;  // runner.cpp:337
    init.probe = -1;
    if (want_probe) {
      int sp = 0;
      CK(cudaMemcpy(&sp, rank.p + p.probe_index, sizeof(int), cudaMemcpyDeviceToHost));
      init.probe = sp;
      probe_dev.alloc(std::max<size_t>(p.probe_capacity, 1) * 4);
      init.probe_buf = probe_dev.p;
      init.probe_cap = static_cast<long long>(p.probe_capacity);
    }
    init.pause_on_mark = p.pause_on_mark;
    CK(cudaMemcpyAsync(scal.p, &init, sizeof(DScalars), cudaMemcpyHostToDevice, stream));
    loop_flags.clear();
    loop_consumed = 0;
    loop_el = loop_dm = loop_tot = 0.0;
  } else {
    // clear the pause; the accounting of the paused step is already done
    DScalars hs;
    CK(cudaMemcpyAsync(&hs, scal.p, sizeof(DScalars), cudaMemcpyDeviceToHost, stream));
    sync();
    hs.paused = 0;
    hs.halt = 0;  // a loop that reached max_steps continues like an uninterrupted one: its last
                  // step is accounted for (pending 0), the next step_begin only forms dt
    hs.pause_on_mark = p.pause_on_mark;
    CK(cudaMemcpyAsync(scal.p, &hs, sizeof(DScalars), cudaMemcpyHostToDevice, stream));
  }
  loop_paused = false;

  const unsigned nb = std::min<unsigned>(592, grid_for(n, 256));
  red.alloc(nb);
  DBuf<double> visc;
  if (damping_active && p.scheme == TLSPH_SCHEME_EXPLICIT) visc.alloc(static_cast<size_t>(n) * D);
  const double eta_tilde = damping_active ? p.eta / p.alpha : 0.0;

  // graphs
  Graph g_begin, g_elastic, g_damp;
  DFields f = fields();
  auto begin_launch = [&](int finalize) {
    if (D == 2) k_step_begin<2><<<nb, 256, 0, stream>>>(f, scal.p, red.p, finalize);
    else k_step_begin<3><<<nb, 256, 0, stream>>>(f, scal.p, red.p, finalize);
  };
  capture(stream, g_begin, [&] {
    begin_launch(0);
    enqueue_resort();  // BASELINE cfg4's per-step re-sort (no-op unless set_resort)
  });
  if (p.elastic) capture(stream, g_elastic, [&] { enqueue_verlet(*this, mat, 0.0, 1); });
  if (damping_active) {
    if (p.scheme != TLSPH_SCHEME_EXPLICIT) prepare_sweep_schedule(p.scheme);  // no allocation under capture
    capture(stream, g_damp, [&] {
      if (p.scheme == TLSPH_SCHEME_EXPLICIT) enqueue_explicit(*this, eta_tilde, visc.p);
      else enqueue_sweep(p.scheme, eta_tilde, 0.0, true);
    });
  }

  // RandomSource (damping.hpp:41-50): outcomes are regenerated from the seed
  // so a resumed loop continues the same stream.
  std::mt19937_64 rng(p.seed);
  for (size_t k = 0; k < loop_flags.size(); ++k) rng();
  auto outcome = [&](uint64_t step) -> bool {
    while (loop_flags.size() <= step) {
      const double phi = static_cast<double>(rng() >> 11) * 0x1.0p-53;
      loop_flags.push_back(phi < p.alpha ? 1 : 0);  // random_choice_eta (damping.cpp:29-34)
    }
    return loop_flags[step] != 0;
  };

  const uint64_t per_begin = kernel_nodes(g_begin), per_elastic = p.elastic ? kernel_nodes(g_elastic) : 0;
  const uint64_t per_damp = damping_active ? kernel_nodes(g_damp) : 0;
  uint64_t launches = 0;
  const uint64_t chunk = 64;
  std::vector<cudaEvent_t> ev(3 * chunk + 2);
  for (auto& e : ev) CK(cudaEventCreate(&e));
  DScalars hs{};
  CK(cudaMemcpyAsync(&hs, scal.p, sizeof(DScalars), cudaMemcpyDeviceToHost, stream));
  sync();
  uint64_t enq = static_cast<uint64_t>(hs.steps);  // next step index to enqueue
  bool finished = false;
  while (!finished) {
    const uint64_t todo = p.max_steps ? std::min<uint64_t>(chunk, p.max_steps - std::min(p.max_steps, enq)) : chunk;
    CK(cudaEventRecord(ev[3 * chunk], stream));
    for (uint64_t k = 0; k < todo; ++k) {
      CK(cudaEventRecord(ev[3 * k], stream));
      CK(cudaGraphLaunch(g_begin.e, stream));  // the elastic window includes step_begin (stable_dt, checks)
      if (p.elastic) CK(cudaGraphLaunch(g_elastic.e, stream));
      launches += per_begin + per_elastic;
      CK(cudaEventRecord(ev[3 * k + 1], stream));
      if (damping_active && outcome(enq + k)) {
        CK(cudaGraphLaunch(g_damp.e, stream));
        launches += per_damp;
      }
      CK(cudaEventRecord(ev[3 * k + 2], stream));
    }
    enq += todo;
    const bool last_chunk = p.max_steps && enq >= p.max_steps;
    if (last_chunk) {
      begin_launch(1);  // accounting of the final step
      launches += 1;
    }
    CK_LAUNCH("k_step_begin");
    CK(cudaEventRecord(ev[3 * chunk + 1], stream));
    CK(cudaMemcpyAsync(&hs, scal.p, sizeof(DScalars), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    float ms = 0.f;
    for (uint64_t k = 0; k < todo; ++k) {
      CK(cudaEventElapsedTime(&ms, ev[3 * k], ev[3 * k + 1]));
      loop_el += ms * 1e-3;
      CK(cudaEventElapsedTime(&ms, ev[3 * k + 1], ev[3 * k + 2]));
      loop_dm += ms * 1e-3;
    }
    CK(cudaEventElapsedTime(&ms, ev[3 * chunk], ev[3 * chunk + 1]));
    loop_tot += ms * 1e-3;
    finished = hs.halt || last_chunk;
    if (!finished && static_cast<uint64_t>(hs.steps) + todo < enq)
      throw DevError(TLSPH_ERR_INTERNAL, "device time loop stopped advancing");
  }
  for (auto& e : ev) cudaEventDestroy(e);
  res.steps = static_cast<uint64_t>(hs.steps);
  uint64_t damped = 0;
  for (uint64_t k = 0; k < res.steps && k < loop_flags.size(); ++k) damped += loop_flags[k];
  res.damped_steps = damping_active ? damped : 0;
  res.t = hs.t;
  res.last_dt = hs.last_dt;
  res.elastic_seconds = loop_el;
  res.damping_seconds = loop_dm;
  res.total_seconds = loop_tot;
  res.peak_ke = hs.ke_peak;
  res.final_ke = hs.ke;
  res.stopped_on_ke = hs.stopped_on_ke;
  res.paused = hs.paused;
  res.probe_samples = static_cast<size_t>(hs.probe_count);
  res.kernel_launches = launches;
  if (want_probe && hs.probe_count > 0 && p.probe_out) {
    const size_t ncopy = std::min<size_t>(static_cast<size_t>(hs.probe_count), p.probe_capacity);
    CK(cudaMemcpy(p.probe_out, probe_dev.p, ncopy * 4 * sizeof(double), cudaMemcpyDeviceToHost));
  }
  last_elapsed = loop_tot;
  last_run_steps = static_cast<long long>(hs.steps);  // also when the loop stopped on an error
  last_run_t = hs.t;
  // resumable: paused at a mark, or stopped at max_steps (not failed, not done by end time / KE)
  loop_paused = !hs.failed && (hs.paused != 0 || (!hs.done && p.max_steps && hs.steps >= static_cast<long long>(p.max_steps)));
  if (hs.failed) raise_if_failed("run");
}

}  // namespace tlsph_cuda
