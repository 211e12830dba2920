"""C-ABI library tests that run without a GPU: libmrv.so loads, exports every
symbol include/mrv.h declares, and argument validation is synchronous and
happens before any device work (include/mrv.h conventions)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2604_23960_b200 import build, gen, mrv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    build.build()
    return mrv.lib()


def header_functions():
    src = open(os.path.join(ROOT, "include", "mrv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mrv_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    names = header_functions()
    assert len(names) >= 10
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(mrv.EXPORTS)


def test_status_strings_and_version(L):
    assert mrv.status_string(0) == "MRV_OK"
    assert mrv.status_string(4) == "MRV_ERANGE"
    assert L.mrv_abi_version() == 5


def _descs(scene):
    keep = []
    rbs = (mrv.RobotDesc * len(scene.robots))()
    for i, r in enumerate(scene.robots):
        arrs = [None if a is None else np.ascontiguousarray(a) for a in (r.joint_origin, r.joint_type, r.base,
                                                                          r.sphere_link, r.sphere)]
        keep += arrs
        ptr = [None if a is None else a.ctypes.data for a in arrs]
        rbs[i] = mrv.RobotDesc(r.kind, r.dof, ptr[0], ptr[1], ptr[2], r.sphere.shape[0], ptr[3], ptr[4])
    osph = np.ascontiguousarray(scene.obs_spheres, np.float32)
    box = np.ascontiguousarray(scene.obs_boxes, np.float32)
    keep += [osph, box]
    env = mrv.EnvDesc(osph.shape[0], osph.ctypes.data if osph.size else None, box.shape[0],
                      box.ctypes.data if box.size else None)
    return rbs, env, keep


def _create(L, scene, n=None):
    rbs, env, keep = _descs(scene)
    h = C.c_void_p()
    st = L.mrv_create_scene(rbs, len(scene.robots) if n is None else n, C.byref(env), 0, C.byref(h))
    return st


def test_validation_rejects_bad_scenes_before_device(L):
    sc = gen.scene_cfg2()
    bad = gen.scene_cfg2()
    bad.robots[1].sphere[3, 3] = 0.0                       # radius <= 0
    assert _create(L, bad) == mrv.MRV_EINVAL
    bad = gen.scene_cfg2()
    bad.robots[0].sphere[0, 3] = -0.1
    assert _create(L, bad) == mrv.MRV_EINVAL
    bad = gen.scene_cfg2()
    bad.obs_boxes[5, 0] = bad.obs_boxes[5, 3] + 0.1        # lo >= hi
    assert _create(L, bad) == mrv.MRV_EINVAL
    bad = gen.scene_cfg2()
    bad.robots[2].sphere_link[0] = 7                      # link out of range
    assert _create(L, bad) == mrv.MRV_EINVAL
    bad = gen.scene_cfg2()
    bad.robots[0].joint_type[2] = 3
    assert _create(L, bad) == mrv.MRV_EINVAL
    bad = gen.scene_cfg1()
    bad.robots[0].dof = 4                                 # SE2 must be 3-DOF
    assert _create(L, bad) == mrv.MRV_EINVAL
    bad = gen.scene_cfg1()
    bad.obs_spheres[0, 3] = 0.0
    assert _create(L, bad) == mrv.MRV_EINVAL
    bad = gen.scene_cfg2()
    bad.robots[0].sphere[0, 0] = np.nan
    assert _create(L, bad) == mrv.MRV_EINVAL
    assert _create(L, sc, n=0) == mrv.MRV_EINVAL
    h = C.c_void_p()
    assert L.mrv_create_scene(None, 1, None, 0, C.byref(h)) == mrv.MRV_EINVAL


def test_obstacle_count_above_limit_is_unsupported(L):
    """Obstacle ids are u16 in the grid's cell lists: more than 65535 obstacles in total
    is refused before any device work (rather than silently dropping obstacles)."""
    bad = gen.scene_cfg1()
    rng = np.random.default_rng(0)
    c = rng.uniform(0, 4, (40000, 3))
    bad.obs_spheres = np.concatenate([c, np.full((40000, 1), 0.1)], axis=1).astype(np.float32)
    bad.obs_boxes = np.concatenate([c - 0.05, c + 0.05], axis=1).astype(np.float32)[:30000]
    assert _create(L, bad) == mrv.MRV_EUNSUPPORTED


def test_dof_above_limit_is_unsupported(L):
    rb = gen.Robot(kind=gen.CHAIN, dof=17, sphere_link=np.zeros(1, np.int32),
                   sphere=np.array([[0, 0, 0, 0.1]], np.float32),
                   joint_origin=np.tile(np.eye(3, 4).reshape(12), (17, 1)).astype(np.float32),
                   joint_type=np.zeros(17, np.int32), base=None)
    assert _create(L, gen.Scene([rb], np.zeros((0, 4), np.float32), np.zeros((0, 6), np.float32))) == \
        mrv.MRV_EUNSUPPORTED


def test_valid_scene_without_gpu_reports_ecuda(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    assert _create(L, gen.scene_cfg2()) == mrv.MRV_ECUDA


def test_batch_calls_reject_null_scene(L):
    b = mrv.MotionBatch(0, 2, 7, None, None, 10)
    assert L.mrv_motval_batch(None, C.byref(b), 0, None, None) == mrv.MRV_EINVAL
    assert L.mrv_ffc_batch(None, C.byref(b), 0, None, None) == mrv.MRV_EINVAL
    assert L.mrv_fk_states(None, C.byref(b), 0, None, None, None, None) == mrv.MRV_EINVAL
    assert L.mrv_run_host_batch(None, C.byref(b), 0, None, 0, None, 0, None) == mrv.MRV_EINVAL
    t, i, j = C.c_int32(), C.c_int32(), C.c_int32()
    assert L.mrv_decode_conflict(None, 5, C.byref(t), C.byref(i), C.byref(j)) == mrv.MRV_EINVAL


def test_no_cpu_fallback_in_product_path():
    """The product package never imports the oracle and has no CPU compute path."""
    pkg = os.path.join(ROOT, "paper_2604_23960_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            src = open(os.path.join(pkg, f)).read()
            assert "import oracle" not in src and "from oracle" not in src, f


def test_self_pair_validation(L):
    bad = gen.scene_cfg2()
    bad.robots[0].self_pairs = np.array([[0, 7]], np.int32)      # link out of range
    assert _create_sp(L, bad) == mrv.MRV_EINVAL
    bad = gen.scene_cfg2()
    bad.robots[0].self_pairs = np.array([[3, 3]], np.int32)      # a == b
    assert _create_sp(L, bad) == mrv.MRV_EINVAL
    bad = gen.scene_cfg3()
    bad.robots[0].self_pairs = np.array([[0, 0]], np.int32)      # bodies have no links to pair
    assert _create_sp(L, bad) == mrv.MRV_EINVAL


def _create_sp(L, scene):
    """mrv_create_scene through the binding's descriptor marshalling (self pairs included)."""
    try:
        mrv.Scene(scene)
    except mrv.MrvError as e:
        return e.status
    return mrv.MRV_OK


def test_c_example_builds_against_the_header():
    """include/mrv.h is plain C11: examples/mrv_example.c (the ABI used from C, no Python
    or torch) compiles with -pedantic and links against libmrv.so and the CUDA runtime."""
    from paper_2604_23960_b200 import build
    build.build()
    exe = build.build_example(force=True)
    assert os.path.exists(exe) and os.access(exe, os.X_OK)
