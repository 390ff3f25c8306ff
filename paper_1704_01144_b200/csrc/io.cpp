// Mesh and state formats (host C++): hand configs
// between the GPU solver, the oracle and CPU baselines without regeneration.
//
//   * TFVM mesh files. Version 1 is the reference's 2D format
//     (Mesh::save/load, proj/core/src/mesh.cpp:345-428) and is READ here, so
//     reference-written meshes load unchanged. Version 2 is the Vec3
//     generalisation (no generator spec; geometry + connectivity only),
//     little-endian like binio.hpp.
//   * Mesh hash: FNV-1a exactly as Mesh::hash (mesh.cpp:326-343) for dim <= 2
//     meshes (z ignored), extended with the z components for 3D.
//   * Snapshots: the reference's text format "tafv-snapshot 1"
//     (save_snapshot / Snapshot::load, state.cpp:77-116) for nv = 1, written
//     byte-identically; "tafv-snapshot 2" text with a component count for
//     nv > 1; and a binary "TFVS" v1 for large states.
//   * compare_snapshots: max relative per-entry difference over w and W with
//     the 1e-300 floor, invalid_argument on different meshes
//     (state.cpp:118-132).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "tafv_gpu.h"

namespace {

thread_local std::string g_io_err;

constexpr uint32_t kMeshMagic = 0x4d564654u;  // "TFVM"
constexpr uint32_t kSnapMagic = 0x53564654u;  // "TFVS"

void put_u32(std::ostream& os, uint32_t v) { os.write(reinterpret_cast<const char*>(&v), 4); }
void put_i32(std::ostream& os, int32_t v) { put_u32(os, static_cast<uint32_t>(v)); }
void put_u64(std::ostream& os, uint64_t v) { os.write(reinterpret_cast<const char*>(&v), 8); }
uint64_t bits_of(double v) {
  uint64_t b;
  std::memcpy(&b, &v, 8);
  return b;
}
double double_of(uint64_t b) {
  double v;
  std::memcpy(&v, &b, 8);
  return v;
}
void put_f64(std::ostream& os, double v) { put_u64(os, bits_of(v)); }
uint32_t get_u32(std::istream& is) {
  uint32_t v = 0;
  is.read(reinterpret_cast<char*>(&v), 4);
  if (!is) throw std::runtime_error("binary read failed (truncated input)");
  return v;
}
int32_t get_i32(std::istream& is) { return static_cast<int32_t>(get_u32(is)); }
uint64_t get_u64(std::istream& is) {
  uint64_t v = 0;
  is.read(reinterpret_cast<char*>(&v), 8);
  if (!is) throw std::runtime_error("binary read failed (truncated input)");
  return v;
}
double get_f64(std::istream& is) { return double_of(get_u64(is)); }

void require(bool c, const char* what) {
  if (!c) throw std::invalid_argument(what);
}

uint64_t fnv(uint64_t h, const void* p, size_t n) {
  const auto* b = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 1099511628211ull;
  }
  return h;
}
uint64_t fnv_f64(uint64_t h, double v) {
  const uint64_t bits = bits_of(v);
  return fnv(h, &bits, 8);
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return TAFV_OK;
  } catch (const std::invalid_argument& e) {
    g_io_err = e.what();
    return TAFV_EINVAL;
  } catch (const std::exception& e) {
    g_io_err = e.what();
    return TAFV_EDIVERGED;  // runtime_error class (I/O failure)
  }
}

struct MeshArrays {
  int32_t dim = 3, nc = 0, nf = 0;
  std::vector<double> vol, cen, chl, fn, fa, fc;
  std::vector<int32_t> fl, fr, fp;
};

MeshArrays read_mesh(const char* path) {
  std::ifstream is(path, std::ios::binary);
  require(is.good(), "mesh file: cannot open");
  require(get_u32(is) == kMeshMagic, "mesh file: bad magic");
  const uint32_t version = get_u32(is);
  MeshArrays m;
  if (version == 1) {  // the reference's 2D layout (mesh.cpp:384-428)
    m.dim = (int32_t)get_u32(is);
    get_u32(is);  // nx
    get_u32(is);  // ny
    get_u32(is);  // periodic flags
    for (int i = 0; i < 4; ++i) get_f64(is);  // domain
    const uint32_t nreg = get_u32(is);
    for (uint32_t r = 0; r < nreg; ++r) {
      for (int i = 0; i < 4; ++i) get_f64(is);
      get_u32(is);
    }
    m.nc = (int32_t)get_u32(is);
    m.nf = (int32_t)get_u32(is);
    m.vol.resize(m.nc);
    m.cen.assign(3 * (size_t)m.nc, 0.0);
    m.chl.resize(m.nc);
    for (int c = 0; c < m.nc; ++c) {
      m.cen[3 * (size_t)c] = get_f64(is);
      m.cen[3 * (size_t)c + 1] = get_f64(is);
      m.vol[c] = get_f64(is);
      m.chl[c] = get_f64(is);
    }
    m.fl.resize(m.nf);
    m.fr.resize(m.nf);
    m.fp.resize(m.nf);
    m.fn.assign(3 * (size_t)m.nf, 0.0);
    m.fa.resize(m.nf);
    m.fc.assign(3 * (size_t)m.nf, 0.0);
    for (int f = 0; f < m.nf; ++f) {
      m.fl[f] = get_i32(is);
      m.fr[f] = get_i32(is);
      m.fn[3 * (size_t)f] = get_f64(is);
      m.fn[3 * (size_t)f + 1] = get_f64(is);
      m.fa[f] = get_f64(is);
      m.fc[3 * (size_t)f] = get_f64(is);
      m.fc[3 * (size_t)f + 1] = get_f64(is);
      m.fp[f] = get_i32(is);
    }
    return m;
  }
  require(version == 2, "mesh file: unsupported version");
  m.dim = (int32_t)get_u32(is);
  m.nc = (int32_t)get_u32(is);
  m.nf = (int32_t)get_u32(is);
  m.vol.resize(m.nc);
  m.cen.resize(3 * (size_t)m.nc);
  m.chl.resize(m.nc);
  for (int c = 0; c < m.nc; ++c) {
    for (int d = 0; d < 3; ++d) m.cen[3 * (size_t)c + d] = get_f64(is);
    m.vol[c] = get_f64(is);
    m.chl[c] = get_f64(is);
  }
  m.fl.resize(m.nf);
  m.fr.resize(m.nf);
  m.fp.resize(m.nf);
  m.fn.resize(3 * (size_t)m.nf);
  m.fa.resize(m.nf);
  m.fc.resize(3 * (size_t)m.nf);
  for (int f = 0; f < m.nf; ++f) {
    m.fl[f] = get_i32(is);
    m.fr[f] = get_i32(is);
    m.fp[f] = get_i32(is);
    for (int d = 0; d < 3; ++d) m.fn[3 * (size_t)f + d] = get_f64(is);
    m.fa[f] = get_f64(is);
    for (int d = 0; d < 3; ++d) m.fc[3 * (size_t)f + d] = get_f64(is);
  }
  return m;
}

uint64_t mesh_hash(const tafv_mesh_view& m) {  // mesh.cpp:326-343 (+ z in 3D)
  uint64_t h = 1469598103934665603ull;
  const int32_t header[3] = {m.dim, m.n_cells, m.n_faces};
  h = fnv(h, header, sizeof header);
  for (int c = 0; c < m.n_cells; ++c) {
    h = fnv_f64(h, m.cell_centroid[3 * (size_t)c]);
    h = fnv_f64(h, m.cell_centroid[3 * (size_t)c + 1]);
    if (m.dim == 3) h = fnv_f64(h, m.cell_centroid[3 * (size_t)c + 2]);
    h = fnv_f64(h, m.cell_volume[c]);
  }
  for (int f = 0; f < m.n_faces; ++f) {
    const int32_t ids[3] = {m.face_left[f], m.face_right[f], m.face_partner[f]};
    h = fnv(h, ids, sizeof ids);
    h = fnv_f64(h, m.face_normal[3 * (size_t)f]);
    h = fnv_f64(h, m.face_normal[3 * (size_t)f + 1]);
    if (m.dim == 3) h = fnv_f64(h, m.face_normal[3 * (size_t)f + 2]);
    h = fnv_f64(h, m.face_area[f]);
  }
  return h;
}

struct Snap {
  uint64_t hash = 0;
  int32_t nc = 0, nv = 1, iteration = 0;
  double time = 0.0;
  std::vector<double> w, W;
};

Snap read_snapshot(const char* path) {
  std::ifstream is(path, std::ios::binary);
  require(is.good(), "snapshot: cannot open");
  Snap s;
  char head[4] = {0, 0, 0, 0};
  is.read(head, 4);
  uint32_t magic = 0;
  std::memcpy(&magic, head, 4);
  if (is && magic == kSnapMagic) {  // binary TFVS v1
    require(get_u32(is) == 1, "snapshot: unsupported binary version");
    s.hash = get_u64(is);
    s.nc = (int32_t)get_u32(is);
    s.nv = (int32_t)get_u32(is);
    s.time = get_f64(is);
    s.iteration = get_i32(is);
    const size_t n = (size_t)s.nc * s.nv;
    s.w.resize(n);
    s.W.resize(n);
    is.read(reinterpret_cast<char*>(s.w.data()), n * 8);
    is.read(reinterpret_cast<char*>(s.W.data()), n * 8);
    require((bool)is, "snapshot: truncated");
    return s;
  }
  // text: "tafv-snapshot 1" (state.cpp:93-116) or 2 (with components)
  is.clear();
  is.seekg(0);
  std::string word;
  int version = 0;
  is >> word >> version;
  require(is.good() && word == "tafv-snapshot" && (version == 1 || version == 2), "snapshot: bad header");
  is >> word >> std::hex >> s.hash >> std::dec;
  require(is.good() && word == "mesh_hash", "snapshot: missing mesh_hash");
  is >> word >> s.nc;
  require(is.good() && word == "cells" && s.nc >= 0, "snapshot: missing cell count");
  if (version == 2) {
    is >> word >> s.nv;
    require(is.good() && word == "components" && s.nv >= 1, "snapshot: missing component count");
  }
  is >> word >> s.time;
  require(is.good() && word == "time", "snapshot: missing time");
  is >> word >> s.iteration;
  require(is.good() && word == "iteration", "snapshot: missing iteration");
  s.w.resize((size_t)s.nc * s.nv);
  s.W.resize((size_t)s.nc * s.nv);
  for (int c = 0; c < s.nc; ++c) {
    int id = -1;
    is >> id;
    for (int k = 0; k < s.nv; ++k) is >> s.w[(size_t)c * s.nv + k];
    for (int k = 0; k < s.nv; ++k) is >> s.W[(size_t)c * s.nv + k];
    require(is.good() && id == c, "snapshot: truncated or misordered cell rows");
  }
  return s;
}

}  // namespace

extern "C" {

const char* tafv_io_last_error(void) { return g_io_err.c_str(); }

uint64_t tafv_mesh_hash(const tafv_mesh_view* m) { return m ? mesh_hash(*m) : 0; }

int tafv_mesh_save(const char* path, const tafv_mesh_view* m) {
  return guard([&] {
    require(path && m, "mesh save: null argument");
    std::ofstream os(path, std::ios::binary);
    require(os.good(), "mesh save: cannot open");
    put_u32(os, kMeshMagic);
    put_u32(os, 2);
    put_u32(os, (uint32_t)m->dim);
    put_u32(os, (uint32_t)m->n_cells);
    put_u32(os, (uint32_t)m->n_faces);
    for (int c = 0; c < m->n_cells; ++c) {
      for (int d = 0; d < 3; ++d) put_f64(os, m->cell_centroid[3 * (size_t)c + d]);
      put_f64(os, m->cell_volume[c]);
      put_f64(os, m->cell_char_length[c]);
    }
    for (int f = 0; f < m->n_faces; ++f) {
      put_i32(os, m->face_left[f]);
      put_i32(os, m->face_right[f]);
      put_i32(os, m->face_partner[f]);
      for (int d = 0; d < 3; ++d) put_f64(os, m->face_normal[3 * (size_t)f + d]);
      put_f64(os, m->face_area[f]);
      for (int d = 0; d < 3; ++d) put_f64(os, m->face_centroid[3 * (size_t)f + d]);
    }
    require(os.good(), "mesh save: write failed");
  });
}

int tafv_mesh_load(const char* path, int32_t* dim, int32_t* n_cells, int32_t* n_faces,
                   double* cell_volume, double* cell_centroid, double* cell_char_length,
                   int32_t* face_left, int32_t* face_right, int32_t* face_partner, double* face_normal,
                   double* face_area, double* face_centroid) {
  return guard([&] {
    require(path != nullptr, "mesh load: null path");
    const MeshArrays m = read_mesh(path);
    if (dim) *dim = m.dim;
    if (n_cells) *n_cells = m.nc;
    if (n_faces) *n_faces = m.nf;
    auto cp = [](auto* dst, const auto& src) {
      if (dst) std::memcpy(dst, src.data(), src.size() * sizeof(src[0]));
    };
    cp(cell_volume, m.vol);
    cp(cell_centroid, m.cen);
    cp(cell_char_length, m.chl);
    cp(face_left, m.fl);
    cp(face_right, m.fr);
    cp(face_partner, m.fp);
    cp(face_normal, m.fn);
    cp(face_area, m.fa);
    cp(face_centroid, m.fc);
  });
}

int tafv_snapshot_save(const char* path, int32_t binary, uint64_t mesh_hash_v, int32_t n_cells,
                       int32_t nv, double time, int32_t iteration, const double* w, const double* W) {
  return guard([&] {
    require(path && w && W && n_cells >= 0 && nv >= 1, "snapshot save: bad arguments");
    if (binary) {
      std::ofstream os(path, std::ios::binary);
      require(os.good(), "snapshot save: cannot open");
      put_u32(os, kSnapMagic);
      put_u32(os, 1);
      put_u64(os, mesh_hash_v);
      put_u32(os, (uint32_t)n_cells);
      put_u32(os, (uint32_t)nv);
      put_f64(os, time);
      put_i32(os, iteration);
      os.write(reinterpret_cast<const char*>(w), (size_t)n_cells * nv * 8);
      os.write(reinterpret_cast<const char*>(W), (size_t)n_cells * nv * 8);
      require(os.good(), "snapshot save: write failed");
      return;
    }
    // text, byte-identical to save_snapshot (state.cpp:77-91) for nv == 1
    std::FILE* fp = std::fopen(path, "w");
    require(fp != nullptr, "snapshot save: cannot open");
    std::fprintf(fp, "tafv-snapshot %d\n", nv == 1 ? 1 : 2);
    std::fprintf(fp, "mesh_hash %016llx\n", (unsigned long long)mesh_hash_v);
    std::fprintf(fp, "cells %d\n", n_cells);
    if (nv != 1) std::fprintf(fp, "components %d\n", nv);
    std::fprintf(fp, "time %.17g\n", time);
    std::fprintf(fp, "iteration %d\n", iteration);
    for (int c = 0; c < n_cells; ++c) {
      std::fprintf(fp, "%d", c);
      for (int k = 0; k < nv; ++k) std::fprintf(fp, " %.17g", w[(size_t)c * nv + k]);
      for (int k = 0; k < nv; ++k) std::fprintf(fp, " %.17g", W[(size_t)c * nv + k]);
      std::fputc('\n', fp);
    }
    const bool ok = std::ferror(fp) == 0;
    std::fclose(fp);
    require(ok, "snapshot save: write failed");
  });
}

int tafv_snapshot_load(const char* path, uint64_t* mesh_hash_v, int32_t* n_cells, int32_t* nv,
                       double* time, int32_t* iteration, double* w, double* W) {
  return guard([&] {
    const Snap s = read_snapshot(path);
    if (mesh_hash_v) *mesh_hash_v = s.hash;
    if (n_cells) *n_cells = s.nc;
    if (nv) *nv = s.nv;
    if (time) *time = s.time;
    if (iteration) *iteration = s.iteration;
    if (w) std::memcpy(w, s.w.data(), s.w.size() * 8);
    if (W) std::memcpy(W, s.W.data(), s.W.size() * 8);
  });
}

// compare_snapshots (state.cpp:118-132): max relative difference over w and
// W, relative to max(|x|, |y|, 1e-300); different meshes -> invalid_argument.
int tafv_snapshot_compare(const char* path_a, const char* path_b, double* worst) {
  return guard([&] {
    const Snap a = read_snapshot(path_a), b = read_snapshot(path_b);
    require(a.hash == b.hash && a.w.size() == b.w.size(), "compare: snapshots come from different meshes");
    double m = 0.0;
    auto rel = [](double x, double y) {
      const double diff = std::abs(x - y);
      if (diff == 0.0) return 0.0;
      return diff / std::max({std::abs(x), std::abs(y), 1e-300});
    };
    for (size_t i = 0; i < a.w.size(); ++i) {
      m = std::max(m, rel(a.w[i], b.w[i]));
      m = std::max(m, rel(a.W[i], b.W[i]));
    }
    if (worst) *worst = m;
  });
}

}  // extern "C"
