// tafv_gpu.hpp — header-only C++ shim over the C ABI (tafv_gpu.h) with the
// reference's solver signatures and exception classes, so reference-style
// callers (proj/core/include/tafv/reference.hpp) switch by changing the
// namespace and passing a Solver instead of (Mesh, SolverState):
//
//   reference                                   this shim
//   plan_iteration(mesh, st, opt)               tafv::gpu::plan_iteration(solver, opt)
//   run_iteration(mesh, st, opt, plan)          tafv::gpu::run_iteration(solver)  (current plan)
//   build_iteration_plan(mesh, make_level_map)  tafv::gpu::inject_levels(solver, tau, dt)
//   reference_iteration(mesh, st, opt)          tafv::gpu::reference_iteration(solver, opt)
//   reference_integrate(mesh, st, opt, n)       tafv::gpu::reference_integrate(solver, opt, n)
//
// Status codes map back to std::invalid_argument (1), std::logic_error (2)
// and std::runtime_error (3: divergence; 4/5: CUDA/NCCL failures).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "tafv_gpu.h"

namespace tafv::gpu {

struct SolverOptions {  // reference.hpp:13-18 (the model lives in Physics)
  int theta_max = 3;
  double cfl = 0.9;
  double dt_cap = 1.0;
  tafv_options c() const { return tafv_options{theta_max, cfl, dt_cap}; }
};

struct IterationRecord {  // reference.hpp:20-29
  int iteration = 0;
  double t_start = 0.0;
  double dt = 0.0;
  int theta = 0;
  double advance = 0.0;
  std::vector<double> total_extensive;  // one sum per conserved component
  double cost_ratio = 1.0;
  std::vector<double> boundary_flux;    // new: outflow through transmissive faces (ledger)
  std::vector<int64_t> level_cells;
};

inline void throw_status(int rc, const char* what) {
  switch (rc) {
    case TAFV_OK: return;
    case TAFV_EINVAL: throw std::invalid_argument(what);
    case TAFV_ELOGIC: throw std::logic_error(what);
    default: throw std::runtime_error(what);
  }
}

inline IterationRecord to_record(const tafv_record& r) {
  IterationRecord o;
  o.iteration = r.iteration;
  o.t_start = r.t_start;
  o.dt = r.dt;
  o.theta = r.theta;
  o.advance = r.advance;
  o.total_extensive.assign(r.total_extensive, r.total_extensive + r.nv);
  o.boundary_flux.assign(r.boundary_flux, r.boundary_flux + r.nv);
  o.cost_ratio = r.cost_ratio;
  o.level_cells.assign(r.level_cells, r.level_cells + r.n_levels);
  return o;
}

// Mesh + SolverState resident on one GPU (one handle per GPU / host thread).
class Solver {
 public:
  Solver(const tafv_mesh_view& mesh, const tafv_physics& physics, int device = 0) {
    const int rc = tafv_gpu_create(&mesh, &physics, device, &h_);
    if (rc != TAFV_OK) throw_status(rc, tafv_gpu_last_error(nullptr));
  }
  ~Solver() { tafv_gpu_destroy(h_); }
  Solver(const Solver&) = delete;
  Solver& operator=(const Solver&) = delete;
  Solver(Solver&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}

  // SolverState w, W (row-major [cells][nv]), t0, iteration. W == nullptr:
  // W = w * V (init_* + sync_extensive, state.cpp:46-68).
  void set_state(const double* w, const double* W = nullptr, double t0 = 0.0, int iteration = 0) {
    check(tafv_gpu_set_state(h_, w, W, t0, iteration));
  }
  void get_state(double* w, double* W, double* t0 = nullptr, int* iteration = nullptr) {
    int32_t it = 0;
    check(tafv_gpu_get_state(h_, w, W, t0, &it));
    if (iteration) *iteration = it;
  }
  tafv_gpu* handle() { return h_; }
  void check(int rc) const {
    if (rc != TAFV_OK) throw_status(rc, tafv_gpu_last_error(h_));
  }

 private:
  tafv_gpu* h_ = nullptr;
};

inline tafv_plan_info plan_iteration(Solver& s, const SolverOptions& opt) {  // reference.hpp:35
  tafv_plan_info info{};
  const tafv_options o = opt.c();
  s.check(tafv_gpu_plan(s.handle(), &o, &info));
  return info;
}

inline tafv_plan_info inject_levels(Solver& s, const std::vector<int32_t>& tau, double dt) {
  tafv_plan_info info{};
  s.check(tafv_gpu_inject_levels(s.handle(), tau.data(), dt, nullptr, &info));
  return info;
}

inline IterationRecord run_iteration(Solver& s) {  // reference.hpp:37-40
  tafv_record r{};
  s.check(tafv_gpu_run_iteration(s.handle(), &r));
  return to_record(r);
}

inline IterationRecord reference_iteration(Solver& s, const SolverOptions& opt) {
  plan_iteration(s, opt);
  return run_iteration(s);
}

inline std::vector<IterationRecord> reference_integrate(Solver& s, const SolverOptions& opt,
                                                        int iterations) {  // reference.hpp:49-52
  if (iterations < 0) throw std::invalid_argument("integrate: negative iteration count");
  std::vector<tafv_record> raw(iterations > 0 ? iterations : 1);
  const tafv_options o = opt.c();
  s.check(tafv_gpu_iterate(s.handle(), &o, iterations, raw.data()));
  std::vector<IterationRecord> out;
  out.reserve(iterations);
  for (int i = 0; i < iterations; ++i) out.push_back(to_record(raw[i]));
  return out;
}

// DistOptions (exchange.hpp:136-144): the options the GPU shards honour.
struct DistOptions {
  int repartition_every = 0;  // 0 = keep the initial partition (exchange.hpp:140-142)
  int axis = 0;               // slab axis of the level-cost re-cuts
};

// One rank of the distributed integrator (DistDriver, exchange.hpp:149-170,
// exchange.cpp:541-660): the rank's shard (owned cells + 2-ring halo) of the
// GLOBAL mesh resident on `device`, the communicator for the collectives and
// the halo exchange. The caller keeps `mesh` alive (DistDriver keeps its
// `const Mesh&`). State arrays are GLOBAL: set_state takes the whole state,
// get_state writes this rank's owned rows. Every call is collective.
class DistDriver {
 public:
  DistDriver(const tafv_mesh_view& mesh, const tafv_physics& physics, std::vector<int32_t> rank_of_cell,
             int rank, tafv_comm* comm, DistOptions opt = {}, int device = 0)
      : mesh_(mesh), part_(std::move(rank_of_cell)) {
    const int rc = tafv_gpu_create_shard(&mesh_, &physics, device, part_.data(), rank, comm, &h_);
    if (rc != TAFV_OK) throw_status(rc, tafv_gpu_last_error(nullptr));
    check(tafv_gpu_set_repartition(h_, &mesh_, opt.repartition_every, opt.axis));
  }
  ~DistDriver() { tafv_gpu_destroy(h_); }
  DistDriver(const DistDriver&) = delete;
  DistDriver& operator=(const DistDriver&) = delete;

  void set_state(const double* w, const double* W = nullptr, double t0 = 0.0, int iteration = 0) {
    check(tafv_gpu_set_state(h_, w, W, t0, iteration));
  }
  void get_state(double* w, double* W, double* t0 = nullptr, int* iteration = nullptr) {
    int32_t it = 0;
    check(tafv_gpu_get_state(h_, w, W, t0, &it));
    if (iteration) *iteration = it;
  }
  // DistDriver::integrate (exchange.cpp:611-631), repartition_every included.
  std::vector<IterationRecord> integrate(const SolverOptions& opt, int iterations) {
    if (iterations < 0) throw std::invalid_argument("integrate: negative iteration count");
    std::vector<tafv_record> raw(iterations > 0 ? iterations : 1);
    const tafv_options o = opt.c();
    check(tafv_gpu_iterate(h_, &o, iterations, raw.data()));
    std::vector<IterationRecord> out;
    for (int i = 0; i < iterations; ++i) out.push_back(to_record(raw[i]));
    return out;
  }
  // DistDriver::repartition (exchange.cpp:595-609): level-cost slabs along
  // `axis` from the last plan, or the given partition.
  const std::vector<int32_t>& repartition(int axis = 0, const std::vector<int32_t>* rank_of_cell = nullptr) {
    check(tafv_gpu_repartition(h_, &mesh_, rank_of_cell ? rank_of_cell->data() : nullptr, axis, part_.data()));
    return part_;
  }
  const std::vector<int32_t>& partition() const { return part_; }
  tafv_gpu* handle() { return h_; }
  void check(int rc) const {
    if (rc != TAFV_OK) throw_status(rc, tafv_gpu_last_error(h_));
  }

 private:
  tafv_mesh_view mesh_;
  std::vector<int32_t> part_;
  tafv_gpu* h_ = nullptr;
};

}  // namespace tafv::gpu
