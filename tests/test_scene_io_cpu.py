"""Scene file and output formats against the reference:
the YAML loader (scene.py:292-354), the snapshot binary (scene.py:771-866) and
the metrics.csv schema (scene.py:541-547).  Fixtures in tests/golden/scene_io*
were written by the reference itself (make_golden.py scene_io).  CPU only."""

import csv
import json
import os
import shutil

import numpy as np
import pytest

from conftest import GOLDEN


@pytest.fixture(scope="module")
def sc():
    from paper_2306_06946_b200 import scene

    return scene


def test_load_scene_matches_reference(sc, golden, tmp_path):
    path = tmp_path / "io.scn"
    shutil.copy(os.path.join(GOLDEN, "scene_io.scn"), path)
    cfg = sc.load_scene(str(path))
    ref = json.load(open(os.path.join(GOLDEN, "scene_io.json")))
    arr = golden("scene_io.npz")
    assert cfg.h == ref["h"] and cfg.threshold == ref["threshold"]
    assert list(cfg.gravity) == ref["gravity"]
    assert [cfg.pgs.max_iterations, cfg.pgs.tolerance, cfg.pgs.friction] == ref["pgs"]
    assert [cfg.newton.scheme, cfg.newton.max_iterations, cfg.newton.penetration_tol,
            cfg.newton.relinearize] == ref["newton"]
    assert [cfg.output.snapshots, cfg.output.metrics, cfg.output.every] == ref["output"]
    assert len(cfg.objects) == len(ref["objects"])
    for k, (o, r) in enumerate(zip(cfg.objects, ref["objects"])):
        assert o.name == r["name"]
        if r["type"] == "SoftSpec":
            assert [o.young, o.poisson, o.density, o.rayleigh_mass, o.rayleigh_stiffness] == \
                [r["young"], r["poisson"], r["density"], r["rayleigh_mass"], r["rayleigh_stiffness"]]
            assert list(o.velocity) == r["velocity"]
            assert np.array_equal(o.mesh.nodes, arr[f"nodes{k}"])  # procedural box mesh, bit-exact
            assert np.array_equal(o.mesh.tets, arr[f"tets{k}"])
        elif r["type"] == "KinematicMeshSpec":
            assert np.array_equal(o.points, arr[f"points{k}"]) and np.array_equal(o.triangles, arr[f"triangles{k}"])
            m = o.motion
            assert [list(m.axis), list(m.center), m.angular_velocity, list(m.velocity)] == \
                [r["axis"], r["center"], r["angular_velocity"], r["velocity"]]
        else:
            assert list(o.normal) == r["normal"] and o.offset == r["offset"]


@pytest.mark.parametrize("step", [0, 2])
def test_snapshot_roundtrip_bytes(sc, tmp_path, step):
    """Reading the reference's snapshot and writing it again gives the same bytes."""
    src = os.path.join(GOLDEN, f"scene_io_step_{step:06d}.bin")
    snap = sc.load_snapshot(src)
    assert snap.step == step + 1
    out = tmp_path / "again.bin"
    sc.save_snapshot(snap, str(out))
    assert open(src, "rb").read() == open(out, "rb").read()


def test_snapshot_rejects_other_files(sc, tmp_path):
    from paper_2306_06946_b200.errors import ParseError

    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"not a snapshot\nend\n")
    with pytest.raises(ParseError):
        sc.load_snapshot(str(bad))


def test_metrics_schema(sc):
    with open(os.path.join(GOLDEN, "scene_io_metrics.csv")) as fh:
        header = next(csv.reader(fh))
    assert tuple(header) == tuple(sc.StepReport.CSV_FIELDS)


def test_rigid_sphere_entry(tmp_path):
    """rigid_sphere scene entries (reference scene.py:268-290): default solid-sphere
    inertia, 3- or 6-component velocities, validation."""
    import numpy as np
    import pytest

    from paper_2306_06946_b200.errors import ValidationError
    from paper_2306_06946_b200.scene import RigidSphereSpec, load_scene

    path = tmp_path / "r.scn"
    path.write_text("objects:\n  - {name: b, type: rigid_sphere, mass: 2.0, radius: 0.1, position: [0, 1, 0],"
                    " velocity: [1, 0, 0]}\n  - {name: c, type: rigid_sphere, mass: 1.0, radius: 0.2,"
                    " inertia: [1, 2, 3], velocity: [0, 0, 0, 0, 0, 5]}\n  - {name: g, type: plane}\n")
    cfg = load_scene(path)
    b, c = cfg.objects[0], cfg.objects[1]
    assert isinstance(b, RigidSphereSpec) and b.mass == 2.0 and b.position == (0.0, 1.0, 0.0)
    assert np.allclose(b.inertia, 0.4 * 2.0 * 0.01 * np.eye(3), rtol=1e-15, atol=0)
    assert b.velocity == (1.0, 0.0, 0.0, 0.0, 0.0, 0.0)
    assert np.array_equal(c.inertia, np.diag([1.0, 2.0, 3.0])) and c.velocity[5] == 5.0
    path.write_text("objects:\n  - {name: b, type: rigid_sphere, mass: 1, radius: 1, velocity: [1, 2]}\n")
    with pytest.raises(ValidationError):
        load_scene(path)
