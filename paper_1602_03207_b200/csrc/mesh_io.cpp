// Gmsh ASCII v2.2 files for the drop-in (host only): read a
// .msh as the reference's load_mesh accepts it and write one that its
// write_mesh would produce byte for byte, so meshes from the reference's tube
// generator reach the GPU path.
//
// Behaviour contract (not structure) taken from the reference:
//  * file grammar and the canonical tag map (regions 1..6, boundary labels
//    11..15; TagMap::canonical, mesh_io.cpp:14-26), unknown sections skipped;
//  * tets reoriented to positive volume by swapping nodes 2 and 3
//    (canonicalize_orientation, mesh.cpp:50-61), zero volume rejected;
//  * the labelled boundary faces must equal the geometric classification
//    (validate + classify_boundary, mesh.cpp:145-265);
//  * errors: ECT_ERR_IO for files that cannot be opened, ECT_ERR_MESH with
//    "path:line: what" for malformed content.
//
// Design: the file is read in one piece and cut into lines once; a cursor
// hands out lines, numbers are parsed with from_chars/strtod, each section
// has its own handler, node ids map through a dense table when they are
// compact (the usual 1..n) and a hash table otherwise, and the boundary check
// runs on sorted node-triple face keys.
#include "mesh_io.h"

#include <algorithm>
#include <array>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iterator>
#include <string_view>
#include <unordered_map>

#include "ect_internal.h"

namespace ect {
namespace {

enum : int { kTube = 0, kTsp = 1, kDefect = 2 };
enum : int { kLateral = 0, kTop = 1, kBottom = 2, kGamma = 3, kGammaP = 4 };
constexpr int kRegionTagBase = 1, kLabelTagBase = 11;

const char* label_name(int l) {
  switch (l) {
    case kLateral: return "OUTER_LATERAL";
    case kTop: return "OUTER_TOP";
    case kBottom: return "OUTER_BOTTOM";
    case kGamma: return "GAMMA";
    case kGammaP: return "GAMMA_P";
    default: return "?";
  }
}

// ---- lines ----------------------------------------------------------------------
class Lines {
 public:
  Lines(std::string text, std::string path) : text_(std::move(text)), path_(std::move(path)) {
    size_t pos = 0;
    while (pos < text_.size()) {
      size_t end = text_.find('\n', pos);
      if (end == std::string::npos) end = text_.size();
      size_t len = end - pos;
      if (len && text_[pos + len - 1] == '\r') --len;
      views_.emplace_back(text_.data() + pos, len);
      pos = end + 1;
    }
  }
  bool done() const { return at_ >= views_.size(); }
  std::string_view take() { return views_[at_++]; }
  // next line, failing at end of file
  std::string_view need(const char* what) {
    if (done()) error(std::string("unexpected end of file, expected ") + what);
    return take();
  }
  // the line number of the last line taken (1-based)
  size_t line() const { return at_; }
  [[noreturn]] void error(const std::string& what) const {
    fail(ECT_ERR_MESH, path_ + ":" + std::to_string(line()) + ": " + what);
  }
  const std::string& path() const { return path_; }

 private:
  std::string text_, path_;
  std::vector<std::string_view> views_;
  size_t at_ = 0;
};

// whitespace-separated fields of a line
class Fields {
 public:
  explicit Fields(std::string_view s) : s_(s) {}
  template <typename I>
  bool integer(I& v) {
    if (!skip()) return false;
    auto r = std::from_chars(s_.data() + p_, s_.data() + s_.size(), v);
    if (r.ec != std::errc()) return false;
    p_ = (size_t)(r.ptr - s_.data());
    return true;
  }
  bool real(double& v) {
    if (!skip()) return false;
    const size_t e = s_.find_first_of(" \t", p_);
    std::string tok(s_.substr(p_, e == std::string_view::npos ? std::string_view::npos : e - p_));
    char* end = nullptr;
    v = std::strtod(tok.c_str(), &end);
    if (end == tok.c_str()) return false;
    p_ += (size_t)(end - tok.c_str());
    return true;
  }

 private:
  bool skip() {
    while (p_ < s_.size() && (s_[p_] == ' ' || s_[p_] == '\t')) ++p_;
    return p_ < s_.size();
  }
  std::string_view s_;
  size_t p_ = 0;
};

// ---- node ids ------------------------------------------------------------------
class NodeIds {
 public:
  void add(long long id, int index, Lines& in) {
    if (id >= 0 && id < (1ll << 26)) {
      if ((size_t)id >= dense_.size()) dense_.resize((size_t)id + 1, -1);
      if (dense_[id] >= 0) in.error("duplicate node id " + std::to_string(id));
      dense_[id] = index;
    } else if (!sparse_.emplace(id, index).second) {
      in.error("duplicate node id " + std::to_string(id));
    }
  }
  int find(long long id) const {
    if (id >= 0 && (size_t)id < dense_.size()) return dense_[id];
    auto it = sparse_.find(id);
    return it == sparse_.end() ? -1 : it->second;
  }

 private:
  std::vector<int> dense_;
  std::unordered_map<long long, int> sparse_;
};

// ---- sections --------------------------------------------------------------------
struct Parse {
  Lines& in;
  GmshMesh& m;
  NodeIds ids;
  bool nodes = false, elements = false;
};

void expect_end(Parse& P, const char* end) {
  if (P.in.need(end) != end) P.in.error(std::string("missing ") + end);
}

void section_format(Parse& P) {
  Fields f(P.in.need("format line"));
  double version = 0.0;
  int file_type = -1, data_size = 0;
  if (!f.real(version) || !f.integer(file_type) || !f.integer(data_size))
    P.in.error("malformed $MeshFormat line");
  if (!(version >= 2.0 && version < 3.0) || file_type != 0)
    P.in.error("unsupported mesh format (need ASCII v2.x)");
  expect_end(P, "$EndMeshFormat");
}

void section_nodes(Parse& P) {
  long long count = -1;
  Fields h(P.in.need("node count"));
  if (!h.integer(count) || count < 0) P.in.error("malformed node count");
  P.m.xyz.reserve(P.m.xyz.size() + 3 * (size_t)count);
  for (long long q = 0; q < count; ++q) {
    Fields f(P.in.need("node line"));
    long long id = 0;
    double c[3];
    if (!f.integer(id) || !f.real(c[0]) || !f.real(c[1]) || !f.real(c[2]))
      P.in.error("malformed node line");
    P.ids.add(id, (int)(P.m.xyz.size() / 3), P.in);
    P.m.xyz.insert(P.m.xyz.end(), c, c + 3);
  }
  expect_end(P, "$EndNodes");
  P.nodes = true;
}

void section_elements(Parse& P) {
  if (!P.nodes) P.in.error("$Elements before $Nodes");
  long long count = -1;
  Fields h(P.in.need("element count"));
  if (!h.integer(count) || count < 0) P.in.error("malformed element count");
  for (long long q = 0; q < count; ++q) {
    Fields f(P.in.need("element line"));
    long long id = 0;
    int type = 0, ntags = 0;
    if (!f.integer(id) || !f.integer(type) || !f.integer(ntags)) P.in.error("malformed element line");
    int physical = 0;
    for (int t = 0; t < ntags; ++t) {
      int tag = 0;
      if (!f.integer(tag)) P.in.error("malformed element tags");
      if (t == 0) physical = tag;
    }
    if (ntags < 1) P.in.error("element without physical tag");
    const int nv = type == 2 ? 3 : type == 4 ? 4 : 0;
    if (!nv) {
      P.in.error("unsupported element type " + std::to_string(type) +
                 " (supported: 2 triangle, 4 tet)");
    }
    int v[4];
    for (int a = 0; a < nv; ++a) {
      long long nid = 0;
      if (!f.integer(nid)) P.in.error("malformed element connectivity");
      v[a] = P.ids.find(nid);
      if (v[a] < 0) P.in.error("element references unknown node " + std::to_string(nid));
    }
    if (nv == 3) {
      const int label = physical - kLabelTagBase;
      if (label < kLateral || label > kGammaP)
        P.in.error("unknown boundary physical tag " + std::to_string(physical));
      P.m.faces.insert(P.m.faces.end(), v, v + 3);
      P.m.labels.push_back(label);
    } else {
      const int region = physical - kRegionTagBase;
      if (region < 0 || region >= ECT_REGION_COUNT)
        P.in.error("unknown region physical tag " + std::to_string(physical));
      P.m.tets.insert(P.m.tets.end(), v, v + 4);
      P.m.region.push_back((uint8_t)region);
    }
  }
  expect_end(P, "$EndElements");
  P.elements = true;
}

void section_skip(Parse& P, std::string_view name) {
  const std::string end = "$End" + std::string(name.substr(1));
  while (P.in.need(end.c_str()) != end) {
  }
}

// ---- geometry checks ---------------------------------------------------------------
double volume6(const double* a, const double* b, const double* c, const double* d) {
  // signed_tet_volume (mesh.cpp:36-38) x 6, same operation order
  const double u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
  const double v[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
  const double w[3] = {d[0] - a[0], d[1] - a[1], d[2] - a[2]};
  const double x = u[1] * v[2] - u[2] * v[1];
  const double y = u[2] * v[0] - u[0] * v[2];
  const double z = u[0] * v[1] - u[1] * v[0];
  return (x * w[0] + y * w[1]) + z * w[2];
}

// a face as its sorted node triple (lexicographic order)
using FaceKey = std::array<int, 3>;
FaceKey face_key(int a, int b, int c) {
  FaceKey k{a, b, c};
  std::sort(k.begin(), k.end());
  return k;
}
std::string face_str(const FaceKey& k) {
  return "(" + std::to_string(k[0]) + "," + std::to_string(k[1]) + "," + std::to_string(k[2]) + ")";
}

bool conductor(int r) { return r == kTube || r == kTsp || r == kDefect; }

// expected (face, label) pairs sorted by face: exterior faces by the z
// extremes, conductor/insulator interfaces GAMMA (GAMMA_P next to TSP)
std::vector<std::pair<FaceKey, int>> classified_faces(const GmshMesh& m) {
  const size_t nn = m.xyz.size() / 3, nt = m.region.size();
  double lo = nn ? m.xyz[2] : 0.0, hi = lo;
  for (size_t i = 0; i < nn; ++i) {
    lo = std::min(lo, m.xyz[3 * i + 2]);
    hi = std::max(hi, m.xyz[3 * i + 2]);
  }
  const double tol = 1e-9 * std::max(1.0, hi - lo);
  std::vector<std::pair<FaceKey, int>> sides;  // (face, tet) for all 4 sides
  sides.reserve(4 * nt);
  for (size_t t = 0; t < nt; ++t) {
    const int* k = &m.tets[4 * t];
    for (int skip = 0; skip < 4; ++skip) {
      int f[3], n = 0;
      for (int a = 0; a < 4; ++a)
        if (a != skip) f[n++] = k[a];
      sides.emplace_back(face_key(f[0], f[1], f[2]), (int)t);
    }
  }
  std::stable_sort(sides.begin(), sides.end(),
                   [](const auto& x, const auto& y) { return x.first < y.first; });
  std::vector<std::pair<FaceKey, int>> out;
  auto node_z = [&](int n) { return m.xyz[3 * n + 2]; };
  for (size_t i = 0; i < sides.size();) {
    size_t j = i + 1;
    while (j < sides.size() && sides[j].first == sides[i].first) ++j;
    const FaceKey& key = sides[i].first;
    if (j - i > 2)
      fail(ECT_ERR_MESH, "non-conforming face " + face_str(key) + " shared by " +
                             std::to_string(j - i) + " tets");
    if (j - i == 1) {
      bool top = true, bottom = true;
      for (int n : key) {
        top = top && std::fabs(node_z(n) - hi) <= tol;
        bottom = bottom && std::fabs(node_z(n) - lo) <= tol;
      }
      out.emplace_back(key, top ? kTop : bottom ? kBottom : kLateral);
    } else {
      const int r0 = m.region[sides[i].second], r1 = m.region[sides[i + 1].second];
      if (conductor(r0) != conductor(r1))
        out.emplace_back(key, (conductor(r0) ? r0 : r1) == kTsp ? kGammaP : kGamma);
    }
    i = j;
  }
  return out;  // sorted by key (sides were)
}

void check_mesh(GmshMesh& m, const std::string& path) {
  if (m.region.empty()) fail(ECT_ERR_MESH, path + ": mesh contains no tetrahedra");
  for (size_t t = 0; t < m.region.size(); ++t) {
    int* k = &m.tets[4 * t];
    const double* x = m.xyz.data();
    double v = volume6(x + 3 * k[0], x + 3 * k[1], x + 3 * k[2], x + 3 * k[3]);
    if (v < 0.0) {
      std::swap(k[2], k[3]);
      v = -v;
    }
    if (!(v > 0.0)) fail(ECT_ERR_MESH, "degenerate tet " + std::to_string(t) + " (zero volume)");
  }
  const auto expected = classified_faces(m);
  std::vector<std::pair<FaceKey, size_t>> given;  // (face, entry)
  for (size_t f = 0; f < m.labels.size(); ++f)
    given.emplace_back(face_key(m.faces[3 * f], m.faces[3 * f + 1], m.faces[3 * f + 2]), f);
  std::stable_sort(given.begin(), given.end(),
                   [](const auto& x, const auto& y) { return x.first < y.first; });
  std::vector<std::string> issue_by_entry(m.labels.size());
  std::vector<bool> covered(expected.size(), false);
  for (size_t q = 0; q < given.size(); ++q) {
    const auto [key, f] = given[q];
    if (q && given[q - 1].first == key) {
      issue_by_entry[f] = "boundary face " + std::to_string(f) + " duplicates another entry\n";
      continue;
    }
    auto it = std::lower_bound(expected.begin(), expected.end(), key,
                               [](const auto& e, const FaceKey& k) { return e.first < k; });
    if (it == expected.end() || it->first != key) {
      issue_by_entry[f] = "boundary face " + std::to_string(f) + " labeled " +
                          label_name(m.labels[f]) + " lies on no classified surface (misclassified)\n";
      continue;
    }
    covered[(size_t)(it - expected.begin())] = true;
    if (it->second != m.labels[f]) {
      issue_by_entry[f] = "boundary face " + std::to_string(f) + " labeled " +
                          label_name(m.labels[f]) + " but classification says " +
                          label_name(it->second) + "\n";
    }
  }
  std::string issues;
  for (const auto& s : issue_by_entry) issues += s;
  for (size_t e = 0; e < expected.size(); ++e)
    if (!covered[e])
      issues += "surface face " + face_str(expected[e].first) + " should be labeled " +
                label_name(expected[e].second) + " but is missing\n";
  if (!issues.empty()) fail(ECT_ERR_MESH, path + ": invalid mesh:\n" + issues);
}

}  // namespace

GmshMesh read_gmsh(const std::string& path) {
  std::ifstream file(path, std::ios::binary);
  if (!file) fail(ECT_ERR_IO, "cannot open mesh file: " + path);
  std::string text((std::istreambuf_iterator<char>(file)), std::istreambuf_iterator<char>());
  Lines in(std::move(text), path);
  GmshMesh m;
  Parse P{in, m, {}};
  while (!in.done()) {
    const std::string_view head = in.take();
    if (head.empty()) continue;
    if (head == "$MeshFormat") section_format(P);
    else if (head == "$Nodes") section_nodes(P);
    else if (head == "$Elements") section_elements(P);
    else if (head.front() == '$') section_skip(P, head);  // $PhysicalNames and the like
    else in.error("unexpected content outside any section: '" + std::string(head) + "'");
  }
  if (!P.nodes || !P.elements) fail(ECT_ERR_MESH, path + ": missing $Nodes or $Elements section");
  check_mesh(m, path);
  return m;
}

void write_gmsh(const std::string& path, const GmshMesh& m) {
  // the layout write_mesh produces (mesh_io.cpp:192-213): %.17g coordinates,
  // boundary triangles then tets, physical == elementary tag, 1-based ids
  std::string s = "$MeshFormat\n2.2 0 8\n$EndMeshFormat\n$Nodes\n";
  const size_t nn = m.xyz.size() / 3;
  char b[160];
  s += std::to_string(nn) + "\n";
  for (size_t i = 0; i < nn; ++i) {
    std::snprintf(b, sizeof b, "%zu %.17g %.17g %.17g\n", i + 1, m.xyz[3 * i], m.xyz[3 * i + 1],
                  m.xyz[3 * i + 2]);
    s += b;
  }
  s += "$EndNodes\n$Elements\n" + std::to_string(m.labels.size() + m.region.size()) + "\n";
  size_t id = 1;
  for (size_t f = 0; f < m.labels.size(); ++f, ++id) {
    const int tag = m.labels[f] + kLabelTagBase;
    std::snprintf(b, sizeof b, "%zu 2 2 %d %d %d %d %d\n", id, tag, tag, m.faces[3 * f] + 1,
                  m.faces[3 * f + 1] + 1, m.faces[3 * f + 2] + 1);
    s += b;
  }
  for (size_t t = 0; t < m.region.size(); ++t, ++id) {
    const int tag = m.region[t] + kRegionTagBase;
    std::snprintf(b, sizeof b, "%zu 4 2 %d %d %d %d %d %d\n", id, tag, tag, m.tets[4 * t] + 1,
                  m.tets[4 * t + 1] + 1, m.tets[4 * t + 2] + 1, m.tets[4 * t + 3] + 1);
    s += b;
  }
  s += "$EndElements\n";
  std::ofstream out(path, std::ios::binary);
  if (!out) fail(ECT_ERR_IO, "cannot open mesh file for writing: " + path);
  out.write(s.data(), (std::streamsize)s.size());
  if (!out) fail(ECT_ERR_IO, "failed writing mesh file: " + path);
}

}  // namespace ect
