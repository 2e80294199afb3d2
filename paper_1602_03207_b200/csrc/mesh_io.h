// Gmsh ASCII v2.2 I/O (host only): see mesh_io.cpp.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace ect {

struct GmshMesh {
  std::vector<double> xyz;      // [n_nodes][3]
  std::vector<int32_t> tets;    // [n_tets][4], canonical orientation
  std::vector<uint8_t> region;  // RegionTag per tet
  std::vector<int32_t> faces;   // [n_faces][3] labelled boundary faces, file order
  std::vector<int32_t> labels;  // BoundaryLabel per face
};

GmshMesh read_gmsh(const std::string& path);             // load_mesh (mesh_io.cpp:68-190)
void write_gmsh(const std::string& path, const GmshMesh& m);  // write_mesh (mesh_io.cpp:192-213)

}  // namespace ect
