// Gmsh ASCII v2.2 mesh files: the reference's load_mesh / write_mesh
// (mesh_io.cpp:68-210) restated host-side, so a user of the drop-in can feed
// the same .msh files (e.g. written by the reference's tube generator) to the
// GPU path. Grammar, canonical tag map (TagMap::canonical, mesh_io.cpp:14-26),
// orientation canonicalisation (Mesh::canonicalize_orientation, mesh.cpp:50-61)
// and validation (validate, mesh.cpp:185-265: conformity, boundary labels equal
// to classify_boundary) follow the reference; errors carry "path:line: what".
#include "mesh_io.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <map>
#include <sstream>
#include <unordered_map>

#include "ect_internal.h"

namespace ect {
namespace {

constexpr int kTube = 0, kTsp = 1, kDefect = 2;
constexpr int kLateral = 0, kTop = 1, kBottom = 2, kGamma = 3, kGammaP = 4;

// TagMap::canonical (mesh_io.cpp:14-26)
int region_of_tag(int tag) { return tag >= 1 && tag <= 6 ? tag - 1 : -1; }
int label_of_tag(int tag) { return tag >= 11 && tag <= 15 ? tag - 11 : -1; }
int tag_of_region(int r) { return r + 1; }
int tag_of_label(int l) { return l + 11; }

bool is_conductor(int r) { return r == kTube || r == kTsp || r == kDefect; }

const char* label_name(int l) {
  static const char* names[] = {"OUTER_LATERAL", "OUTER_TOP", "OUTER_BOTTOM", "GAMMA", "GAMMA_P"};
  return l >= 0 && l < 5 ? names[l] : "?";
}

// signed_tet_volume (mesh.cpp:36-38), the shim's cross/dot order
double signed_volume(const double* a, const double* b, const double* c, const double* d) {
  const double u0 = b[0] - a[0], u1 = b[1] - a[1], u2 = b[2] - a[2];
  const double v0 = c[0] - a[0], v1 = c[1] - a[1], v2 = c[2] - a[2];
  const double w0 = d[0] - a[0], w1 = d[1] - a[1], w2 = d[2] - a[2];
  const double cx = u1 * v2 - u2 * v1, cy = u2 * v0 - u0 * v2, cz = u0 * v1 - u1 * v0;
  return ((cx * w0 + cy * w1) + cz * w2) / 6.0;
}

struct Reader {
  std::istream& in;
  std::string path;
  int line_no = 0;
  std::string line;
  bool next() {
    if (!std::getline(in, line)) return false;
    ++line_no;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    return true;
  }
  [[noreturn]] void fail(const std::string& what) const {
    ect::fail(ECT_ERR_MESH, path + ":" + std::to_string(line_no) + ": " + what);
  }
  std::string expect(const char* what) {
    if (!next()) fail(std::string("unexpected end of file, expected ") + what);
    return line;
  }
};

using Face = std::array<int, 3>;
Face sorted_face(int a, int b, int c) {
  Face f{a, b, c};
  std::sort(f.begin(), f.end());
  return f;
}

// classify_boundary (mesh.cpp:145-182): exterior faces by z-extremes, interior
// conductor/insulator interfaces as GAMMA (GAMMA_P next to TSP)
std::map<Face, int> classify(const GmshMesh& m) {
  const int64_t nn = (int64_t)m.xyz.size() / 3, nt = (int64_t)m.region.size();
  double z_lo = 0.0, z_hi = 0.0;
  if (nn) {
    z_lo = z_hi = m.xyz[2];
    for (int64_t i = 0; i < nn; ++i) {
      z_lo = std::min(z_lo, m.xyz[3 * i + 2]);
      z_hi = std::max(z_hi, m.xyz[3 * i + 2]);
    }
  }
  const double tol = 1e-9 * std::max(1.0, z_hi - z_lo);
  struct Rec {
    Face f;
    int tet;
  };
  std::vector<Rec> recs;
  recs.reserve(4 * nt);
  static const int fl[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
  for (int64_t t = 0; t < nt; ++t) {
    const int* k = &m.tets[4 * t];
    for (const auto& q : fl) recs.push_back({sorted_face(k[q[0]], k[q[1]], k[q[2]]), (int)t});
  }
  std::stable_sort(recs.begin(), recs.end(), [](const Rec& a, const Rec& b) { return a.f < b.f; });
  std::map<Face, int> out;
  for (size_t i = 0; i < recs.size();) {
    size_t j = i;
    while (j < recs.size() && recs[j].f == recs[i].f) ++j;
    if (j - i > 2) {
      ect::fail(ECT_ERR_MESH, "non-conforming face (" + std::to_string(recs[i].f[0]) + "," +
                                  std::to_string(recs[i].f[1]) + "," +
                                  std::to_string(recs[i].f[2]) + ") shared by " +
                                  std::to_string(j - i) + " tets");
    }
    const Face& f = recs[i].f;
    if (j - i == 1) {
      bool top = true, bottom = true;
      for (int n : f) {
        top = top && std::abs(m.xyz[3 * n + 2] - z_hi) <= tol;
        bottom = bottom && std::abs(m.xyz[3 * n + 2] - z_lo) <= tol;
      }
      out[f] = top ? kTop : bottom ? kBottom : kLateral;
    } else {
      const int r0 = m.region[recs[i].tet], r1 = m.region[recs[i + 1].tet];
      const bool c0 = is_conductor(r0), c1 = is_conductor(r1);
      if (c0 != c1) out[f] = (c0 ? r0 : r1) == kTsp ? kGammaP : kGamma;
    }
    i = j;
  }
  return out;
}

}  // namespace

GmshMesh read_gmsh(const std::string& path) {
  std::ifstream in(path);
  if (!in) fail(ECT_ERR_IO, "cannot open mesh file: " + path);
  Reader rd{in, path};
  GmshMesh m;
  std::unordered_map<long long, int> node_index;
  bool saw_nodes = false, saw_elements = false;
  while (rd.next()) {
    const std::string section = rd.line;
    if (section.empty()) continue;
    if (section == "$MeshFormat") {
      std::istringstream fs(rd.expect("format line"));
      double version = 0.0;
      int file_type = 0, data_size = 0;
      if (!(fs >> version >> file_type >> data_size)) rd.fail("malformed $MeshFormat line");
      if (version < 2.0 || version >= 3.0 || file_type != 0)
        rd.fail("unsupported mesh format (need ASCII v2.x)");
      if (rd.expect("$EndMeshFormat") != "$EndMeshFormat") rd.fail("missing $EndMeshFormat");
    } else if (section == "$PhysicalNames") {
      while (rd.expect("$EndPhysicalNames") != "$EndPhysicalNames") {
      }
    } else if (section == "$Nodes") {
      std::istringstream hs(rd.expect("node count"));
      long long count = 0;
      if (!(hs >> count) || count < 0) rd.fail("malformed node count");
      m.xyz.reserve(3 * (size_t)count);
      for (long long i = 0; i < count; ++i) {
        std::istringstream ns(rd.expect("node line"));
        long long id = 0;
        double x = 0, y = 0, z = 0;
        if (!(ns >> id >> x >> y >> z)) rd.fail("malformed node line");
        if (node_index.count(id)) rd.fail("duplicate node id " + std::to_string(id));
        node_index[id] = (int)(m.xyz.size() / 3);
        m.xyz.insert(m.xyz.end(), {x, y, z});
      }
      if (rd.expect("$EndNodes") != "$EndNodes") rd.fail("missing $EndNodes");
      saw_nodes = true;
    } else if (section == "$Elements") {
      if (!saw_nodes) rd.fail("$Elements before $Nodes");
      std::istringstream hs(rd.expect("element count"));
      long long count = 0;
      if (!(hs >> count) || count < 0) rd.fail("malformed element count");
      for (long long e = 0; e < count; ++e) {
        std::istringstream es(rd.expect("element line"));
        long long id = 0;
        int type = 0, ntags = 0;
        if (!(es >> id >> type >> ntags)) rd.fail("malformed element line");
        int physical = 0;
        for (int t = 0; t < ntags; ++t) {
          int tag = 0;
          if (!(es >> tag)) rd.fail("malformed element tags");
          if (t == 0) physical = tag;
        }
        if (ntags < 1) rd.fail("element without physical tag");
        auto node = [&]() {
          long long nid = 0;
          if (!(es >> nid)) rd.fail("malformed element connectivity");
          auto it = node_index.find(nid);
          if (it == node_index.end()) rd.fail("element references unknown node " + std::to_string(nid));
          return it->second;
        };
        if (type == 2) {
          const int a = node(), b = node(), c = node();
          const int l = label_of_tag(physical);
          if (l < 0) rd.fail("unknown boundary physical tag " + std::to_string(physical));
          m.faces.insert(m.faces.end(), {a, b, c});
          m.labels.push_back(l);
        } else if (type == 4) {
          const int a = node(), b = node(), c = node(), d = node();
          const int r = region_of_tag(physical);
          if (r < 0) rd.fail("unknown region physical tag " + std::to_string(physical));
          m.tets.insert(m.tets.end(), {a, b, c, d});
          m.region.push_back((uint8_t)r);
        } else {
          rd.fail("unsupported element type " + std::to_string(type) +
                  " (supported: 2 triangle, 4 tet)");
        }
      }
      if (rd.expect("$EndElements") != "$EndElements") rd.fail("missing $EndElements");
      saw_elements = true;
    } else if (section[0] == '$') {
      const std::string end = "$End" + section.substr(1);
      while (rd.expect(end.c_str()) != end) {
      }
    } else {
      rd.fail("unexpected content outside any section: '" + section + "'");
    }
  }
  if (!saw_nodes || !saw_elements) fail(ECT_ERR_MESH, path + ": missing $Nodes or $Elements section");
  if (m.region.empty()) fail(ECT_ERR_MESH, path + ": mesh contains no tetrahedra");

  // Mesh::canonicalize_orientation (mesh.cpp:50-61)
  for (size_t t = 0; t < m.region.size(); ++t) {
    int* k = &m.tets[4 * t];
    double vol = signed_volume(&m.xyz[3 * k[0]], &m.xyz[3 * k[1]], &m.xyz[3 * k[2]], &m.xyz[3 * k[3]]);
    if (vol < 0.0) {
      std::swap(k[2], k[3]);
      vol = -vol;
    }
    if (!(vol > 0.0)) fail(ECT_ERR_MESH, "degenerate tet " + std::to_string(t) + " (zero volume)");
  }
  // validate (mesh.cpp:185-265): labels must equal the recomputed classification
  const std::map<Face, int> expected = classify(m);
  std::map<Face, int> seen;
  std::string issues;
  for (size_t f = 0; f < m.labels.size(); ++f) {
    const Face key = sorted_face(m.faces[3 * f], m.faces[3 * f + 1], m.faces[3 * f + 2]);
    if (++seen[key] > 1) {
      issues += "boundary face " + std::to_string(f) + " duplicates another entry\n";
      continue;
    }
    auto it = expected.find(key);
    if (it == expected.end()) {
      issues += "boundary face " + std::to_string(f) + " labeled " + label_name(m.labels[f]) +
                " lies on no classified surface (misclassified)\n";
    } else if (it->second != m.labels[f]) {
      issues += "boundary face " + std::to_string(f) + " labeled " + label_name(m.labels[f]) +
                " but classification says " + label_name(it->second) + "\n";
    }
  }
  for (const auto& [key, label] : expected) {
    if (!seen.count(key)) {
      issues += "surface face (" + std::to_string(key[0]) + "," + std::to_string(key[1]) + "," +
                std::to_string(key[2]) + ") should be labeled " + label_name(label) +
                " but is missing\n";
    }
  }
  if (!issues.empty()) fail(ECT_ERR_MESH, path + ": invalid mesh:\n" + issues);
  return m;
}

void write_gmsh(const std::string& path, const GmshMesh& m) {
  std::ofstream out(path);
  if (!out) fail(ECT_ERR_IO, "cannot open mesh file for writing: " + path);
  out << "$MeshFormat\n2.2 0 8\n$EndMeshFormat\n";
  const size_t nn = m.xyz.size() / 3;
  out << "$Nodes\n" << nn << "\n";
  char buf[128];
  for (size_t i = 0; i < nn; ++i) {
    std::snprintf(buf, sizeof(buf), "%zu %.17g %.17g %.17g\n", i + 1, m.xyz[3 * i],
                  m.xyz[3 * i + 1], m.xyz[3 * i + 2]);
    out << buf;
  }
  out << "$EndNodes\n";
  out << "$Elements\n" << (m.labels.size() + m.region.size()) << "\n";
  long long id = 1;
  for (size_t f = 0; f < m.labels.size(); ++f) {
    const int tag = tag_of_label(m.labels[f]);
    out << id++ << " 2 2 " << tag << ' ' << tag << ' ' << m.faces[3 * f] + 1 << ' '
        << m.faces[3 * f + 1] + 1 << ' ' << m.faces[3 * f + 2] + 1 << "\n";
  }
  for (size_t t = 0; t < m.region.size(); ++t) {
    const int tag = tag_of_region(m.region[t]);
    out << id++ << " 4 2 " << tag << ' ' << tag << ' ' << m.tets[4 * t] + 1 << ' '
        << m.tets[4 * t + 1] + 1 << ' ' << m.tets[4 * t + 2] + 1 << ' ' << m.tets[4 * t + 3] + 1
        << "\n";
  }
  out << "$EndElements\n";
  if (!out) fail(ECT_ERR_IO, "failed writing mesh file: " + path);
}

}  // namespace ect
