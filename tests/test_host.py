"""Host-side checks that need no GPU: the C-ABI library loads and exports
every symbol include/hrt.h declares, the ctypes mirror matches the C struct
layout, scene packing/config shapes follow SURVEY Appendix B, image codecs
and error behaviour follow the reference."""

import math
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2309_04581_b200 import _lib, configs
from paper_2309_04581_b200.core import Transform, tone_map
from paper_2309_04581_b200.field import NeuralField, level_resolutions
from paper_2309_04581_b200.images import HdrImage, decode_pfm, decode_ppm, encode_pfm, encode_ppm
from paper_2309_04581_b200.pack import pack_scene
from paper_2309_04581_b200.scene import Camera, EmitterSet, make_scene, scene_diagonal
from paper_2309_04581_b200.surface import Lambertian, Mirror, TriangleMesh

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hrt.h")


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(hrt_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libhrt.so not built (run __graft_entry__.build())")
    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(_lib.SIGNATURES) == names
    assert lib.hrt_version() == 1


def test_ctypes_structs_match_c_layout(tmp_path):
    src = tmp_path / "sizes.c"
    src.write_text('#include "hrt.h"\n#include <stdio.h>\n#include <stddef.h>\n'
                   "int main(void){printf(\"%zu %zu %zu %zu %zu %zu\\n\", sizeof(hrt_field_desc),"
                   " sizeof(hrt_scene_desc), sizeof(hrt_camera), sizeof(hrt_stats),"
                   " offsetof(hrt_scene_desc, field), offsetof(hrt_field_desc, occ_bits));return 0;}\n")
    exe = tmp_path / "sizes"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    import ctypes
    want = [ctypes.sizeof(_lib.FieldDesc), ctypes.sizeof(_lib.SceneDesc),
            ctypes.sizeof(_lib.CameraDesc), ctypes.sizeof(_lib.Stats),
            _lib.SceneDesc.field.offset, _lib.FieldDesc.occ_bits.offset]
    assert got == want


@pytest.mark.parametrize("cfg,entries,dense,top", [(0, 32768, 0, 128), (1, 6098925, 5, 2048),
                                                   (4, 22566329, 6, 4095)])
def test_hash_grid_tables_match_survey(cfg, entries, dense, top):
    field = configs.network(cfg)
    assert field.n_entries == entries
    assert int(field.level_dense.sum()) == dense
    assert int(field.level_n[-1]) == top
    assert field.table.dtype == np.float32 and field.w_density1.dtype == np.float16


def test_level_resolutions_cfg1():
    assert list(level_resolutions(16, 16, 2048)) == [16, 22, 30, 42, 58, 80, 111, 153, 212, 294,
                                                     406, 561, 776, 1072, 1482, 2048]


def test_neural_init_is_seeded_and_xavier():
    a, b = NeuralField.random(3), NeuralField.random(3)
    assert np.array_equal(a.table, b.table) and np.array_equal(a.w_color2, b.w_color2)
    lim = math.sqrt(6.0 / (16 + 64))
    assert np.abs(a.w_density1.astype(np.float64)).max() <= lim * (1 + 1e-3)
    assert np.all(a.w_color1[31] == 0)        # zero pad row of the 31-wide colour input
    assert abs(a.table.std() - 0.1) < 0.01


def test_config_geometry_counts():
    assert sum(len(m.indices) for m in configs.cfg0().meshes) == 320
    assert sum(len(m.indices) for m in configs.cfg1().meshes) == 20480
    assert [len(m.indices) for m in configs.cfg2().meshes] == [2, 50000]
    s3 = configs.cfg3(res=(64, 36))
    assert len(s3.meshes) == 200 and sum(len(m.indices) for m in s3.meshes) == 1024000
    s4 = configs.cfg4(res=(64, 36))
    assert [len(m.indices) for m in s4.meshes] == [2, 300000]
    pk = pack_scene(s4)
    assert len(pk["bv0"]) == 300000               # emissive quad excluded from blockers
    assert len(pk["emitters"]["cdf"]) == 2 and pk["emitters"]["r_src"].tolist() == [1.0, 1.0]


def test_cfg1_cameras_on_radius_four():
    cams = configs.cfg1_cameras()
    assert len(cams) == 100
    for c in cams[:10]:
        assert abs(np.linalg.norm(c.pose.m[:3, 3]) - 4.0) < 1e-12
        fwd = -c.pose.m[:3, 2]
        assert np.allclose(fwd, -c.pose.m[:3, 3] / 4.0)


def test_pack_scene_face_order_and_spawn_eps():
    v, f = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0.0]]), np.array([[0, 1, 2]])
    a = TriangleMesh(v, f, Mirror(np.ones(3)))
    b = TriangleMesh(v + 2, f, Lambertian(np.zeros(3)), emission=np.ones(3))
    c = TriangleMesh(v - 2, f, Lambertian(np.full(3, 0.5)))
    sc = make_scene(meshes=[a, b, c])
    pk = pack_scene(sc)
    assert pk["mesh_of"].tolist() == [0, 1, 2]
    assert np.array_equal(pk["bv0"], np.stack([a.vertices[0], c.vertices[0]]))
    assert sc.spawn_eps == 1e-4 * scene_diagonal(None, [a, b, c])
    assert pk["mat_kind"].tolist() == [1, 0, 0]


def test_emitter_cdf_and_clip():
    em = EmitterSet([[[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 0, 0], [2, 0, 0], [0, 2, 0]]], [1.5, -1])
    assert em.r_src.tolist() == [1.0, 0.0]
    assert np.allclose(em.cdf, [0.2, 1.0])


def test_images_round_trip_and_ppm_codes(rng):
    img = HdrImage(rng.uniform(0, 3, (5, 7, 3)))
    back = decode_pfm(encode_pfm(img))
    assert np.array_equal(back.pixels, img.pixels.astype(np.float32))
    codes = decode_ppm(encode_ppm(HdrImage(np.array([[[0.0] * 3, [1.0] * 3, [0.5] * 3]]))))
    assert codes[0].tolist() == [[0, 0, 0], [255, 255, 255], [188, 188, 188]]
    assert tone_map(np.array([2.0]))[0] == 1.0


def test_camera_and_transform_validation():
    with pytest.raises(ValueError):
        Camera(Transform.identity(), 0.0, (4, 4))
    with pytest.raises(ValueError):
        Camera(Transform.identity(), 1.0, (0, 4))
    with pytest.raises(ValueError):
        Transform(np.zeros((4, 4)))


def test_render_rejects_bad_spp_before_touching_the_gpu():
    from paper_2309_04581_b200 import render
    with pytest.raises(ValueError):
        render(configs.cfg0(), spp=0)


def test_renderer_cache_tracks_bvh_object_and_field_placement(hybridrt):
    """renderer_for's cache key: a reference Scene's Bvh OBJECT
    (held and compared with `is`, so a freed-and-reused id() cannot hide a
    rebuild) and the field placement bytes (a dynamic field moves without a
    BVH rebuild, sim.py:673-698)."""
    import importlib
    from paper_2309_04581_b200.renderer import _Cached, _field_key
    rs = importlib.import_module("hybridrt.scene")
    rf = importlib.import_module("hybridrt.field")
    sf = importlib.import_module("hybridrt.surface")
    rr = importlib.import_module("hybridrt.render")
    core = importlib.import_module("hybridrt.core")
    v = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float)
    mesh = sf.TriangleMesh(v, [[0, 1, 2]], sf.Lambertian((0.5, 0.5, 0.5)))
    field = rf.RadianceGrid.constant((0, 0, 0), (1, 1, 1), 1.0, (1, 1, 1))
    bvh = sf.Bvh([mesh])
    cam = rr.Camera(core.Transform.look_at((0, 0, 3), (0, 0, 0)), 0.5, (4, 4))
    scene = rs.Scene(config=None, camera=cam, render=rs.RenderConfig(), field=field, meshes=[mesh],
                     bvh=bvh, blocker_bvh=bvh, emitters=None, collider_sdfs=[], spawn_eps=1e-4)
    c = _Cached(scene, None, 0)
    assert not c.geometry_changed(scene) and _field_key(scene) == c.field
    scene.rebuild_bvh()
    assert c.geometry_changed(scene)
    c.stamp(scene)
    assert not c.geometry_changed(scene)
    scene.field.world_from_field = core.Transform.translate((0.1, 0.0, 0.0))
    assert _field_key(scene) != c.field and not c.geometry_changed(scene)


def test_nerf_file_round_trip(tmp_path):
    """.hrtnerf: hyper-parameters in the header, arrays bit-exact."""
    from paper_2309_04581_b200.nerffile import is_nerf_file, load_nerf, save_nerf
    f = NeuralField.random(5, n_levels=8, n_features=2, log2_table=12, n_min=16, n_max=128,
                           out_activation="softplus", occupancy_res=32)
    f.world_from_field = Transform.translate((0.25, -0.5, 0.0))
    p = tmp_path / "f.hrtnerf"
    save_nerf(p, f)
    assert is_nerf_file(p) and not is_nerf_file(__file__)
    g = load_nerf(p)
    for name in ("table", "w_density1", "w_density2", "w_color1", "w_color2", "w_color3"):
        a, b = getattr(f, name), getattr(g, name)
        assert a.dtype == b.dtype and np.array_equal(a, b), name
    assert (g.n_levels, g.n_features, g.log2_table, g.n_min, g.n_max) == (8, 2, 12, 16, 128)
    assert g.out_activation == "softplus" and g.occupancy_res == 32
    assert np.array_equal(g.world_from_field.m, f.world_from_field.m)
    assert np.array_equal(g.bbox_lo, f.bbox_lo) and np.array_equal(g.bbox_hi, f.bbox_hi)


def test_load_scene_with_a_nerf_field_file(hybridrt, tmp_path):
    """A reference scene JSON whose field.path is a .hrtnerf file loads
    through the reference's own parser / builder with the NeuralField
    attached (the hyper-parameters live in the field file)."""
    import json as _json
    import importlib
    from paper_2309_04581_b200 import assets
    from paper_2309_04581_b200.nerffile import load_scene, save_nerf
    f = NeuralField.random(3, n_levels=8, n_features=2, log2_table=12, n_min=16, n_max=128)
    save_nerf(tmp_path / "fog.hrtnerf", f)
    v, fc = assets.icosphere(0.4, 2)
    importlib.import_module("hybridrt.surface").save_obj(str(tmp_path / "ball.obj"), v, fc)
    doc = {"field": {"path": "fog.hrtnerf", "transform": {"translate": [0.0, 0.1, 0.0]}},
           "meshes": [{"path": "ball.obj", "bsdf": {"type": "mirror", "reflectance": [1.0, 1.0, 1.0]}}],
           "camera": {"position": [0.0, 0.0, 3.0], "look_at": [0.0, 0.0, 0.0], "up": [0.0, 1.0, 0.0],
                      "fov_deg": 40.0, "resolution": [16, 16]},
           "render": {"spp": 1, "n_bounces": 2, "march_step": 0.0203, "seed": 0}}
    (tmp_path / "s.json").write_text(_json.dumps(doc))
    scene = load_scene(str(tmp_path / "s.json"))
    assert type(scene).__module__.startswith("hybridrt")
    assert scene.field.kind == "neural" and np.array_equal(scene.field.table, f.table)
    assert scene.field.world_from_field.m[1, 3] == 0.1
    assert len(scene.meshes) == 1 and scene.spawn_eps > 0
    pk = pack_scene(scene)
    assert pk["field"]["kind"] == 2 and not pk["field"]["identity"]
