/*
 * tafv_gpu.h — C-ABI drop-in boundary of the B200-native LTS finite-volume
 * hot path (arXiv 1704.01144; reference library `tafv`, proj/core).
 *
 * Plain pointers and sizes only; no torch, no C++ types. Every entry point
 * cites the reference interface it replaces (paths relative to the
 * reference root, proj/core/...). Status codes mirror the reference's
 * exception classes so the C++ shim (include/tafv_gpu.hpp) can rethrow them:
 *   0 ok
 *   1 std::invalid_argument   (tafv::require, common.hpp:9-11)
 *   2 std::logic_error        (TAFV_ASSERT,   common.hpp:15-19)
 *   3 std::runtime_error      (divergence,    reference.cpp:123-124)
 *   4 CUDA error              (new: device failure)
 *   5 NCCL error              (new: multi-GPU transport; replaces transport.cpp:39-41)
 * A handle is not thread-safe; use one handle per GPU (one host thread each).
 *
 * Conventions:
 *   - ids are the caller's ORIGINAL cell / face ids; the library renumbers
 *     internally and maps every array in and out.
 *   - per-cell state arrays are row-major [n_cells][nv] (nv = 1 scalar,
 *     5 Euler: rho, rho*u, rho*v, rho*w, E).
 *   - geometry is Vec3; 2D meshes pass z = 0 (the reference's Vec2,
 *     geometry.hpp:7-17).
 */
#ifndef TAFV_GPU_H
#define TAFV_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  TAFV_OK = 0,
  TAFV_EINVAL = 1,
  TAFV_ELOGIC = 2,
  TAFV_EDIVERGED = 3,
  TAFV_ECUDA = 4,
  TAFV_ENCCL = 5
};

/* Physics: FluxModel (physics.hpp:14-28) extended with compressible Euler. */
enum { TAFV_ADVECTION = 0, TAFV_BURGERS = 1, TAFV_EULER = 2 };

#define TAFV_MAX_LEVELS 16

/* Mesh view: the reference Mesh/Cell/Face layout (mesh.hpp:26-65) as SoA
 * arrays. The CSR adjacency (mesh.cpp:241-271) is rebuilt inside
 * tafv_gpu_create in ascending original face id, exactly as the reference
 * builds it, and geometric closure is checked (mesh.cpp:273-284). */
typedef struct tafv_mesh_view {
  int32_t dim;                      /* 1 or 2 (scalar reference meshes) or 3 */
  int32_t n_cells;
  int32_t n_faces;
  const double* cell_volume;        /* [n_cells]    Cell::volume */
  const double* cell_centroid;      /* [n_cells][3] Cell::centroid */
  const double* cell_char_length;   /* [n_cells]    Cell::char_length */
  const int32_t* face_left;         /* [n_faces]    Face::left */
  const int32_t* face_right;        /* [n_faces]    Face::right (-1 boundary) */
  const int32_t* face_partner;      /* [n_faces]    Face::periodic_partner (-1 none) */
  const double* face_normal;        /* [n_faces][3] Face::normal (unit, left->right) */
  const double* face_area;          /* [n_faces]    Face::area */
  const double* face_centroid;      /* [n_faces][3] Face::centroid */
} tafv_mesh_view;

/* FluxModel (physics.hpp:14-28; parse_flux_model physics.cpp:7-21):
 * advection a=(ax,ay); Burgers direction a (normalised here, as
 * parse_flux_model does); Euler gamma. */
typedef struct tafv_physics {
  int32_t model;
  double a[3];
  double gamma;
} tafv_physics;

/* SolverOptions (reference.hpp:13-18) minus the model. */
typedef struct tafv_options {
  int32_t theta_max;
  double cfl;
  double dt_cap;
} tafv_options;

/* IterationRecord (reference.hpp:20-29); total_extensive per component.
 * boundary_flux (new, the conservation ledger): per component, what the
 * iteration's correctors took out of the domain through transmissive
 * boundary faces (the sum of those faces' int_substep integrals, each the
 * +sign*phi term of its left cell's flux_sum_correct, kernels.cpp:204-216),
 * so that total_extensive(n) = total_extensive(n-1) - boundary_flux(n) up to
 * rounding. Compensated sums; 0 on closed / periodic meshes. */
typedef struct tafv_record {
  int32_t iteration;
  int32_t theta;
  double t_start;
  double dt;
  double advance;
  double cost_ratio;
  double total_extensive[8];
  int64_t level_cells[TAFV_MAX_LEVELS];
  int32_t n_levels;
  int32_t nv;
  double boundary_flux[8];
} tafv_record;

/* Summary of an IterationPlan (levels.hpp:46-61) held on the device.
 * c_eff = sum_tau 2^(theta-tau)|Omega(tau)| (LevelMap::level_cost,
 * levels.cpp:68-79); f_eff = sum_f 2^(theta-cadence_f);
 * r_eff = sum_{l<theta} 2^(theta-l)|fringe[l]|. */
typedef struct tafv_plan_info {
  int32_t theta;
  int32_t n_levels;
  double dt;
  double cost_ratio;
  int64_t cells_per_level[TAFV_MAX_LEVELS];
  int64_t faces_per_cadence[TAFV_MAX_LEVELS];
  int64_t fringe_per_level[TAFV_MAX_LEVELS];
  int64_t c_eff;
  int64_t f_eff;
  int64_t r_eff;
} tafv_plan_info;

typedef struct tafv_gpu tafv_gpu;

/* Upload an immutable mesh (replaces the caller-owned `const Mesh&` that every
 * reference entry takes, mesh.hpp:41) and allocate the SolverState
 * (state.hpp:17-50, SolverState::init state.cpp:14-38) on `device`. */
int tafv_gpu_create(const tafv_mesh_view* mesh, const tafv_physics* physics, int device,
                    tafv_gpu** out);
void tafv_gpu_destroy(tafv_gpu* h);

/* Message of the last failure on this handle (or of the last failed create
 * on this thread when h == NULL). */
const char* tafv_gpu_last_error(const tafv_gpu* h);

/* State in/out (SolverState::w, ::W, ::t0, ::iteration). W == NULL means
 * W = w * V, i.e. init_* + sync_extensive (state.cpp:46-68); w == NULL means
 * w = W / V, the relation every corrector leaves (intensive_correct,
 * kernels.cpp:237-241), so a state saved as W alone after an iteration is
 * restored bitwise. get_state skips a NULL output. */
int tafv_gpu_set_state(tafv_gpu* h, const double* w, const double* W, double t0,
                       int32_t iteration);
int tafv_gpu_get_state(tafv_gpu* h, double* w, double* W, double* t0, int32_t* iteration);

/* plan_iteration (reference.hpp:35, reference.cpp:89-98): dt_max, global min,
 * ilogb classification, smoothing to the |dtau|<=1 fixpoint, level map,
 * face cadences and the per-level compacted index lists, all on device. */
int tafv_gpu_plan(tafv_gpu* h, const tafv_options* opt, tafv_plan_info* out);

/* build_iteration_plan(mesh, make_level_map(tau, dt)) (levels.cpp:53-66,
 * 123-155): inject a hand-made level map, as the reference tests do through
 * run_iteration's plan argument (reference.hpp:37-40). tau in original ids.
 * dt <= 0 selects dt = min_c dt_max_c / 2^tau_c (computed on device with
 * `opt`'s cfl/dt_cap) for synthetic level maps. */
int tafv_gpu_inject_levels(tafv_gpu* h, const int32_t* tau, double dt, const tafv_options* opt,
                           tafv_plan_info* out);

/* Export the current plan in original ids for bit-exact list checks:
 * tau[n_cells], face_cadence[n_faces], cells_of_level flattened level by
 * level (ascending ids), faces_of_cadence likewise, fringe[l] likewise
 * (sizes from tafv_plan_info). Any pointer may be NULL. */
int tafv_gpu_get_plan_lists(tafv_gpu* h, int32_t* tau, int32_t* face_cadence,
                            int32_t* cells_flat, int32_t* faces_flat, int32_t* fringe_flat);

/* run_iteration (reference.hpp:37-40, reference.cpp:100-129) under the
 * current plan: 2^theta subiterations of {corrector, predictor} over the
 * active prefix sets, the trailing corrector, divergence check, record. */
int tafv_gpu_run_iteration(tafv_gpu* h, tafv_record* out);

/* reference_integrate (reference.hpp:49-52, reference.cpp:135-142):
 * n x {plan_iteration, run_iteration}; out has room for n records. */
int tafv_gpu_iterate(tafv_gpu* h, const tafv_options* opt, int32_t n, tafv_record* out);

/* Same as tafv_gpu_iterate but keeps only the record of the LAST iteration.
 * The host still synchronises once per iteration (one pinned read-back
 * carries the next plan -- its theta picks the next sweep graph -- and the
 * divergence flag), exactly as tafv_gpu_iterate does; the state never
 * leaves the device. */
int tafv_gpu_advance(tafv_gpu* h, const tafv_options* opt, int32_t n, tafv_record* last);

/* A batch of independent inputs (ensemble members, restarts): for each
 * j < n_inputs, the state becomes W_in[j] (extensive, original cell order;
 * w = W / V, t0 = 0, iteration = 0), `iterations` iterations run
 * (reference_integrate), and the resulting W is written to W_out[j]. Input
 * j+1 uploads and output j-1 downloads on separate copy streams while input
 * j computes; pass pinned host buffers for the overlap. `last` (optional)
 * receives the record of the last iteration of the last input. Shards: the
 * arrays hold the rank's local cells in the order of its shard cell list. */
int tafv_gpu_run_batch(tafv_gpu* h, const tafv_options* opt, int32_t n_inputs, int32_t iterations,
                       const double* const* W_in, double* const* W_out, tafv_record* last);

/* reference_integrate (reference.cpp:135-142) on a HOST-resident state:
 * the caller's SolverState (state.hpp:17-50) stays in host memory and every
 * iteration crosses the link both ways -- W uploaded from W_host (w = W / V
 * on the device, the relation every corrector leaves, kernels.cpp:237-241),
 * plan_iteration + run_iteration, the new W written back into W_host before
 * the next upload (chunked, so the two directions overlap). W_host: extensive
 * rows in original cell order (shards: local cells in shard order); pass
 * pinned memory. out has room for n records. Bitwise equal to
 * tafv_gpu_iterate from set_state(NULL, W). */
int tafv_gpu_iterate_host(tafv_gpu* h, const tafv_options* opt, int32_t n, double* W_host, tafv_record* out);

/* Debug/parity access to intermediate SolverState arrays in original ids:
 * "w_pred" [nc][nv], "grad" [nc][nv][3], "phi_pred" / "int_substep" /
 * "int_window" [nf][nv], "dt_max" [nc] (double); "raw_level" [nc] (int32);
 * "mesh_digest" [20] (uint64: FNV-1a of every internal mesh array, slot
 * count, boundary count, flags -- compares the device and host builds);
 * "repartition_ms" [1] (double: wall time of the last repartition);
 * "brick_info" [4] (double: bricks of the brick K1, ragged bricks, cells
 * left to the general K1, structures built). */
int tafv_gpu_get_array(tafv_gpu* h, const char* name, void* out);

/* Launch configuration knobs (bench/profiling; every setting leaves the
 * results bitwise unchanged -- each has a parity test -- and drops the
 * captured graphs):
 *   "grid_cap"       max blocks per grid-stride launch;
 *   "kernel_timing"  1: time every hot kernel with CUDA events on the
 *                    library stream (resets the per-kind totals);
 *   "use_graph", "plan_graph"  0: direct launches instead of the captured
 *                    sweep / plan graphs;
 *   "k1_tile"        identity-phase K1 with Morton-brick staging (-1 auto);
 *   "k1_brick"       identity-phase K1 with bulk-copied brick streams (off);
 *   "slot_geo", "slot_n", "slot_dx", "face_dx"  0: per-face geometry /
 *                    centroid gathers instead of the per-slot / per-face
 *                    offset streams;
 *   "iwin_alias"     0: materialise int_window of equal-level faces;
 *   "alt_dir"        0: every kernel walks its items forwards;
 *   "sweep_marks"    0: every Jacobi sweep re-evaluates every tile;
 *   "skip_top_lists" 0: write the top level's entries of the level-sorted
 *                    lists too;
 *   "batch_lanes", "dl_stream"  run_batch lanes / download stream. */
int tafv_gpu_set_flag(tafv_gpu* h, const char* name, int64_t value);

/* Kernel launches issued by the last run/iterate/advance call (own kernels
 * only), and device timings of the last call in milliseconds: [0] whole
 * call, [1] plan, [2] sweep (subiterations + trailing corrector). */
int tafv_gpu_stats(tafv_gpu* h, int64_t* launches, double* ms3);

/* Per-kind device time (ms), launch counts and processed items since
 * kernel_timing was set: [0] K1 stage+gradient+limiter, [1] K2 face flux
 * (predictor), [2] K2 face flux (corrector), [3] K3 gather+update
 * (predictor), [4] K3 gather+update (corrector), [5] whole plan.
 * items6x3[3k..3k+2] = active cells, active faces, fringe cells summed over
 * kind k's launches (the inputs of the bench's algorithmic-byte model). */
int tafv_gpu_kernel_times(tafv_gpu* h, double* ms6, int64_t* counts6, int64_t* items6x3);

/* n_cells, n_faces, adjacency slots, nv of the uploaded mesh/physics. */
int tafv_gpu_mesh_info(tafv_gpu* h, int64_t* info4);

/* ---- multi-GPU decomposition (host only) -----------------
 * Contiguous slab partition along `axis` balancing `weight` (NULL = cell
 * count; level cost 2^(theta-tau) as DistDriver::repartition weighs,
 * exchange.cpp:598-603). */
int tafv_partition_slabs(const tafv_mesh_view* mesh, int32_t nranks, int32_t axis,
                         const double* weight, int32_t* rank_of_cell);

/* The shard of `rank`: owned cells + 2-ring halo, faces touching owned or
 * ring-1 cells, and per-peer exchange lists (the reference's ghost
 * components, ce.cpp:66-90, widened to two rings). counts[8] = n_own, n_r1,
 * n_r2, n_faces, n_faces_touching_owned, n_peers, send total, recv total;
 * cells/faces = local -> global ids (ascending); send/recv lists are local
 * cell ids, peer by peer, ascending global id. Any output may be NULL. */
int tafv_shard_describe(const tafv_mesh_view* mesh, const int32_t* rank_of_cell, int32_t rank,
                        int32_t nranks, int32_t* counts, int32_t* cells, int32_t* faces,
                        int32_t* peers, int32_t* send_counts, int32_t* recv_counts,
                        int32_t* send_flat, int32_t* recv_flat);
const char* tafv_shard_last_error(void);

/* smooth_to_fixpoint (levels.cpp:33-51) on the host, in place: the slab cut
 * weights of a decomposed run come from the initial plan's levels before
 * any device is set up (DistDriver::repartition, exchange.cpp:598-603). */
int tafv_level_smooth(const tafv_mesh_view* mesh, int32_t* tau);

/* ---- multi-GPU ranks -------------------------------------------------------
 * A communicator replaces the reference's Transport + RankComm
 * (transport.hpp, exchange.cpp:126-322): NCCL (one process per GPU; get the
 * 128-byte unique id on rank 0 and broadcast it) or an in-process loopback
 * for `nranks` host threads (one handle each, possibly on one GPU). */
typedef struct tafv_comm tafv_comm;
int tafv_comm_nccl_unique_id(uint8_t* out128);
int tafv_comm_create_nccl(const uint8_t* id128, int32_t rank, int32_t nranks, int device,
                          tafv_comm** out);
int tafv_comm_create_loopback(int32_t nranks, tafv_comm** out);
void tafv_comm_destroy(tafv_comm* comm);

/* One rank of a decomposed run (DistDriver, exchange.cpp:541-660): the
 * GLOBAL mesh and partition in, the rank's shard (owned cells + 2-ring halo)
 * resident on `device`. Afterwards every call is collective over the
 * communicator's ranks; set_state / inject_levels take GLOBAL arrays,
 * get_state writes the rank's OWNED rows into the global arrays, records are
 * global. Periodic meshes are not supported in this mode. */
int tafv_gpu_create_shard(const tafv_mesh_view* global_mesh, const tafv_physics* physics, int device,
                          const int32_t* rank_of_cell, int32_t rank, tafv_comm* comm,
                          tafv_gpu** out);

/* DistDriver::repartition (exchange.cpp:595-609), collective over the
 * shard's communicator, in place (the handle pointer stays valid): the
 * ranks all-reduce their owned rows of the committed state and the last
 * plan's level map, cut a new partition -- `rank_of_cell` if given, else
 * contiguous slabs along `axis` balancing the level cost 2^(theta - tau)
 * (exchange.cpp:598-603) -- and rebuild the shard on the device from
 * `global_mesh` (the mesh the shard was created from; the caller keeps it,
 * as DistDriver keeps its `const Mesh&`). State, t0 and iteration carry over
 * bitwise. rank_of_cell_out (optional, [n_cells]) receives the partition.
 * logic_error (TAFV_ELOGIC) before any plan, as the reference. On a failure
 * after the rebuild started the handle must be destroyed. */
int tafv_gpu_repartition(tafv_gpu* h, const tafv_mesh_view* global_mesh, const int32_t* rank_of_cell,
                         int32_t axis, int32_t* rank_of_cell_out);

/* DistOptions::repartition_every (exchange.hpp:140-143): tafv_gpu_iterate
 * repartitions the shard (level-cost slabs along `axis`) before iteration i
 * whenever i > 0 and i % every == 0, as DistDriver::integrate does
 * (exchange.cpp:611-618). every = 0 switches it off. `global_mesh` must
 * outlive the setting. */
int tafv_gpu_set_repartition(tafv_gpu* h, const tafv_mesh_view* global_mesh, int32_t every, int32_t axis);

/* ---- formats (host only) ----------------------------
 * TFVM mesh files: version 1 = the reference's 2D format (Mesh::save,
 * mesh.cpp:345-382), read here; version 2 = Vec3 geometry + connectivity,
 * written here. Two-call load: NULL arrays -> counts only. */
int tafv_mesh_save(const char* path, const tafv_mesh_view* mesh);
int tafv_mesh_load(const char* path, int32_t* dim, int32_t* n_cells, int32_t* n_faces,
                   double* cell_volume, double* cell_centroid, double* cell_char_length,
                   int32_t* face_left, int32_t* face_right, int32_t* face_partner, double* face_normal,
                   double* face_area, double* face_centroid);
/* Mesh::hash (mesh.cpp:326-343, FNV-1a): identical for dim <= 2; + z in 3D. */
uint64_t tafv_mesh_hash(const tafv_mesh_view* mesh);
/* Snapshots (save_snapshot / Snapshot::load, state.cpp:77-116): text
 * "tafv-snapshot 1" byte-identical to the reference for nv == 1, "... 2" with
 * a component count for nv > 1, or binary TFVS (binary != 0). Rows [n][nv]. */
int tafv_snapshot_save(const char* path, int32_t binary, uint64_t mesh_hash, int32_t n_cells, int32_t nv,
                       double time, int32_t iteration, const double* w, const double* W);
int tafv_snapshot_load(const char* path, uint64_t* mesh_hash, int32_t* n_cells, int32_t* nv, double* time,
                       int32_t* iteration, double* w, double* W);
/* compare_snapshots (state.cpp:118-132): max relative difference over w, W. */
int tafv_snapshot_compare(const char* path_a, const char* path_b, double* worst);
const char* tafv_io_last_error(void);

/* 3D hexahedral mesh generator (new: the reference generator is 1D/2D only,
 * mesh.cpp:302-317). Tensor-product node lattice x[nx+1], y[ny+1], z[nz+1],
 * interior nodes jittered uniformly by +-jitter of the local spacing
 * (SplitMix64, seeded), optional random cell/face permutation from `seed`.
 * Two-call protocol: with out arrays NULL, writes the counts. */
int tafv_mesh_hex(int32_t nx, int32_t ny, int32_t nz, const double* x, const double* y,
                  const double* z, double jitter, uint64_t seed, int32_t permute,
                  int32_t* n_cells, int32_t* n_faces, double* cell_volume, double* cell_centroid,
                  double* cell_char_length, int32_t* face_left, int32_t* face_right,
                  int32_t* face_partner, double* face_normal, double* face_area,
                  double* face_centroid);

/* The cells [box6[0], box6[1]) x [box6[2], box6[3]) x [box6[4], box6[5]) of
 * the tafv_mesh_hex lattice (nx, ny, nz, xs, ys, zs, jitter, seed; no
 * permutation): every node -- jitter included -- sits exactly where the full
 * mesh puts it, so the window's cells are bitwise the full mesh's cells
 * there; faces on the window's sides become transmissive boundary faces.
 * Bounded samples of a config (CPU baselines) and per-rank slabs. Same
 * two-call protocol. */
int tafv_mesh_hex_window(int32_t nx, int32_t ny, int32_t nz, const double* xs, const double* ys,
                         const double* zs, const int32_t* box6, double jitter, uint64_t seed,
                         int32_t* n_cells, int32_t* n_faces, double* cell_volume, double* cell_centroid,
                         double* cell_char_length, int32_t* face_left, int32_t* face_right,
                         int32_t* face_partner, double* face_normal, double* face_area,
                         double* face_centroid);

#ifdef __cplusplus
}
#endif

#endif /* TAFV_GPU_H */
