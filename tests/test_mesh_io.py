"""Gmsh ASCII v2.2 files: the host-side reader/writer of
the drop-in against the reference's own load_mesh / write_mesh
(mesh_io.cpp:68-213) on the reference's tube geometry (tube_mesh.cpp)."""
import numpy as np
import pytest

from oracle import ref
from paper_1602_03207_b200 import ect
from tests.helpers import golden

TUBE = dict(domain_radius=0.03, z_min=-0.02, z_max=0.02, tube_r_inner=0.0085,
            tube_r_outer=0.0097, defect=(0.0085, 0.0097, -0.001, 0.001),
            coil=(0.006, 0.0075, 0.001, 0.0005), coil_ref_z=0.0, scan_z=[0.0], resolution=4)


@pytest.fixture(scope="module")
def ref_tube(tmp_path_factory):
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    m = ref.RefMesh.tube(TUBE)
    path = tmp_path_factory.mktemp("msh") / "tube.msh"
    m.write(path)
    return m, path


def test_reader_matches_reference_loader(ref_tube):
    m, path = ref_tube
    g = ect.read_gmsh(path)
    back = ref.RefMesh.load(path)
    xyz, region = back.geometry()
    ex = back.export()
    assert g["xyz"].tobytes() == xyz.tobytes()                 # %.17g round trip, exact
    assert np.array_equal(g["tets"], ex["tets"])               # canonical orientation
    assert np.array_equal(g["region"], region)
    assert np.array_equal(g["faces"], ex["faces"]) and np.array_equal(g["labels"], ex["face_labels"])
    assert set(np.unique(g["labels"])) >= {0, 1, 2, 3}         # lateral, top, bottom, gamma


def test_writer_is_byte_identical(ref_tube, tmp_path):
    m, path = ref_tube
    xyz, region = m.geometry()
    ex = m.export()
    ours = tmp_path / "ours.msh"
    ect.write_gmsh(ours, xyz, ex["tets"], region, ex["faces"], ex["face_labels"])
    assert ours.read_bytes() == path.read_bytes()


def test_reader_reorients_and_accepts_golden_box(tmp_path):
    g = golden("small_4x4x8")
    tets = g["tets"].copy()
    tets[::3, [2, 3]] = tets[::3, [3, 2]]                       # flip every third tet
    p = tmp_path / "box.msh"
    rm = ref.RefMesh(g["xyz"], g["tets"], g["region"])
    ex = rm.export()
    ect.write_gmsh(p, g["xyz"], tets, g["region"], ex["faces"], ex["face_labels"])
    back = ect.read_gmsh(p)
    assert np.array_equal(back["tets"], g["tets"])              # canonicalize_orientation


@pytest.mark.parametrize("edit, err", [
    (lambda s: s.replace("2.2 0 8", "4.1 0 8"), "unsupported mesh format"),
    (lambda s: s.replace(" 4 2 1 1 ", " 4 2 9 9 ", 1), "unknown region physical tag"),
    (lambda s: s.replace(" 2 2 12 12 ", " 2 2 13 13 ", 1), "classification says"),
    (lambda s: s.replace("$EndNodes", "$EndNodez"), "missing $EndNodes"),
])
def test_reader_errors(ref_tube, tmp_path, edit, err):
    _, path = ref_tube
    bad = tmp_path / "bad.msh"
    bad.write_text(edit(path.read_text()))
    with pytest.raises(ect.MeshError, match=err.replace("$", r"\$")):
        ect.read_gmsh(bad)


def test_missing_file_is_io_error(tmp_path):
    with pytest.raises(ect.IoError):
        ect.read_gmsh(tmp_path / "nope.msh")
