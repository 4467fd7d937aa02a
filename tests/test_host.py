"""Host-side logic and the C-ABI library, CPU only (no compute calls).

Known-answer values from the reference suite: patch sizes 15/133/37/69
(tests/test_netspec.py:118-166), 256->388 padding, the example-net size chain
19->18->17->15->11->5 and dilation schedules [1,1,2,2,6] / extents 3,5,7
(tests/test_acceptance.py:223-248), the s^2 m^2/(s+m)^2 model
(test_acceptance.py:301-320), mask parsing (tests/test_backward.py:444-470).
"""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_1412_4526_b200 as dp
from golden_io import manifest, net_names
from paper_1412_4526_b200 import _lib, backend, fmap, trainer
from paper_1412_4526_b200.netspec import SpecError, layer_input_sizes

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "denseprop_b200.h")


def _fixture_text(kind, **kw):
    # the reference fixtures (fixtures.py:33-79), restated for the host tests
    seed = kw.get("seed", 0)
    tok = lambda k: f"seed:{seed * 10000 + k}"  # noqa: E731
    if kind == "example":
        return ("input channels=1\n"
                f"conv out=1 in=1 k=2 stride=1 weights={tok(0)}\n"
                "pool kind=max k=2 stride=2\n"
                f"conv out=1 in=1 k=2 stride=1 weights={tok(2)}\n"
                "pool kind=max k=3 stride=3\n"
                f"conv out=1 in=1 k=2 stride=1 weights={tok(4)}\n")
    c1, c2, c3 = kw.get("channels", (50, 50, 32))
    pk, ps = kw.get("pool1", (8, 8))
    return ("input channels=3\n"
            f"conv out={c1} in=3 k=6 stride=1 weights={tok(0)}\n"
            f"pool kind=max k={pk} stride={ps}\nnonlin kind=tanh\n"
            f"conv out={c2} in={c1} k=3 stride=1 weights={tok(3)}\n"
            "pool kind=max k=2 stride=2\nnonlin kind=tanh\n"
            f"conv out={c3} in={c2} k=7 stride=1 weights={tok(6)}\n")


def test_patch_sizes_and_padding():
    assert dp.patch_size(dp.parse_spec(_fixture_text("example"))) == 15
    plain = dp.parse_spec(_fixture_text("plain"))
    assert dp.patch_size(plain) == 133
    assert dp.patch_size(dp.parse_spec(_fixture_text("plain", pool1=(2, 2)))) == 37
    assert dp.patch_size(dp.parse_spec(_fixture_text("plain", pool1=(4, 4)))) == 69
    assert 256 + 2 * dp.padding_margin(plain) == 388


def test_dilation_schedule_and_shapes():
    plan = dp.compile_plan(dp.parse_spec(_fixture_text("example")))
    assert plan.dilations == [1, 1, 2, 2, 6]
    assert [l.extent for l in plan.layers[2:]] == [3, 5, 7]
    chain = [s[1] for s in plan.layer_shapes(5, 5)]
    assert chain == [19, 18, 17, 15, 11, 5]
    full = dp.compile_plan(dp.parse_spec(_fixture_text("plain")))
    assert full.layer_shapes(256, 256)[0] == (3, 388, 388)
    assert full.layer_shapes(256, 256)[-1] == (32, 256, 256)


@pytest.mark.parametrize("name", net_names())
def test_plan_metadata_matches_reference(name):
    meta = manifest()["nets"][name]
    plan = dp.compile_plan(dp.parse_spec(meta["spec"]))
    assert plan.patch_size == meta["patch_size"]
    assert [plan.lead_margin, plan.trail_margin] == meta["margins"]
    assert plan.dilations == meta["dilations"]
    assert [getattr(l, "extent", None) for l in plan.layers] == meta["extents"]
    shapes = plan.layer_shapes(meta["side"], meta["side"])
    assert shapes[-1][1:] == (meta["side"], meta["side"])


def test_fusion_groups_cover_every_layer_once():
    for name in net_names():
        plan = dp.compile_plan(dp.parse_spec(manifest()["nets"][name]["spec"]))
        flat = [k for g in plan.fusion_groups() for k in g]
        assert flat == list(range(len(plan.layers)))


def test_theoretical_speedup_model():
    spec = dp.parse_spec(_fixture_text("plain"))
    assert layer_input_sizes(spec)[0] == 133
    for s in (64, 256):
        r = dp.theoretical_speedup(spec, s)
        for k, m in {0: 133, 3: 16, 6: 7}.items():
            assert r[k] == pytest.approx(s * s * m * m / (s + m) ** 2)


@pytest.mark.parametrize("text,match", [
    ("conv out=1 in=1 k=1 stride=1 weights=seed:1\n", "before input"),
    ("input channels=1\ninput channels=1\n", "duplicate"),
    ("input channels=1\nconv out=1 in=2 k=1 stride=1 weights=seed:1\n", "chain"),
    ("input channels=1\npool kind=min k=2 stride=2\n", "max or avg"),
    ("input channels=1\nconv out=1 in=1 k=0 stride=2 weights=seed:1\n", ">= 1"),
    ("input channels=1\nconv out=1 in=1 k=x stride=1 weights=seed:1\n", "integer"),
    ("input channels=1\nfoo\n", "unknown directive"),
    ("", "missing input"),
])
def test_spec_errors(text, match):
    with pytest.raises(SpecError, match=match):
        dp.parse_spec(text)


def test_spec_round_trip_and_weight_files(tmp_path):
    w = np.random.default_rng(0).uniform(-0.5, 0.5, (2, 3, 3, 3))
    b = np.random.default_rng(1).uniform(-0.5, 0.5, 2)
    path = tmp_path / "c.fmap"
    from paper_1412_4526_b200.netspec import save_weight_file
    save_weight_file(str(path), w, b)
    text = "input channels=3\nconv out=2 in=3 k=3 stride=1 weights=c.fmap\n"
    spec = dp.parse_spec(text, base_dir=str(tmp_path))
    assert np.allclose(spec.layers[0].weights, w.astype(np.float32))
    assert dp.format_spec(spec) == text


def test_fmap_io(tmp_path):
    m = np.random.default_rng(2).normal(size=(2, 3, 4)).astype(np.float32)
    p = str(tmp_path / "m.fmap")
    fmap.write_fmap(p, m)
    assert np.array_equal(fmap.read_fmap(p), m)
    assert fmap.pad_rect(m, 1, 2, 3, 0).shape == (2, 6, 7)
    assert np.array_equal(fmap.crop_patch(fmap.pad(m, 2), 2 + 1, 2 + 1, 3), m[:, 0:3, 0:3])


def test_error_mask():
    mask = dp.ErrorMask.parse("1 2\n3 0\n", 4, 4)
    assert mask.selected == {(1, 2), (3, 0)}
    assert len(dp.ErrorMask.parse("all", 3, 3)) == 9
    with pytest.raises(ValueError):
        dp.ErrorMask.of(4, 4, [(4, 0)])
    delta = np.random.default_rng(3).normal(size=(3, 4, 4))
    out = dp.apply_mask(delta, dp.ErrorMask.of(4, 4, [(0, 0)]))
    assert np.array_equal(out[:, 0, 0], delta[:, 0, 0])
    out[:, 0, 0] = 0
    assert not out.any()
    bm = dp.ErrorMask.from_bitmap(mask.bitmap)
    assert bm.selected == mask.selected


def test_bucket_layout_round_trip():
    spec = dp.parse_spec(_fixture_text("plain", channels=(4, 5, 2), pool1=(2, 2)))
    layout, total = trainer.bucket_layout(spec)
    assert total == sum(l.weights.size + l.bias.size for _, l in spec.conv_layers())
    ks = [l.weights if hasattr(l, "weights") else None for l in spec.layers]
    bs = [l.bias if hasattr(l, "bias") else None for l in spec.layers]
    k2, b2 = trainer.unflatten(spec, trainer.flatten(spec, ks, bs))
    for a, b in zip(ks + bs, k2 + b2):
        assert (a is None and b is None) or np.array_equal(a, b)
    assert [list(trainer.shard(10, r, 3)) for r in range(3)] == [[0, 1, 2, 3], [4, 5, 6], [7, 8, 9]]


# ------------------------------------------------------------------ C ABI library

def _header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(dp_\w+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()  # builds are done by __graft_entry__.build(); load must succeed here
    syms = _header_symbols()
    assert len(syms) >= 26
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, f"{s} declared in the header but not typed in _lib"
    assert set(_lib.SIGNATURES) == set(syms)
    assert lib.dp_abi_version() == _lib.ABI_VERSION


def test_no_device_means_loud_failure(monkeypatch):
    if _lib.device_count() >= 1:
        pytest.skip("a CUDA device is present")
    with pytest.raises(_lib.KernelUnavailable):
        backend.kernels()
    with pytest.raises(_lib.KernelUnavailable):
        dp.dense_forward(dp.compile_plan(dp.parse_spec(_fixture_text("example"))),
                         np.zeros((1, 5, 5)))
    assert backend.available() == []


def test_backend_selection_api():
    assert backend.active() == "cuda"
    with pytest.raises(ValueError):
        backend.use("gpu")
    with pytest.raises(ValueError):
        backend.use("compiled")
    backend.use("auto")
    assert backend.active() == "cuda"
    assert backend.registered() == ["cuda", "cuda-fast"]
    backend.use("cuda-fast")
    assert backend.active() == "cuda-fast"
    backend.use("cuda")


def test_cuda_fast_backend_has_the_module_contract():
    """"cuda-fast" exposes exactly the boundary functions "cuda" does (reference
    backend.py:25-48) and fails as loudly without a device."""
    from paper_1412_4526_b200 import cuda_fast_kernels, cuda_kernels
    names = ["conv_forward", "conv_backward_data", "conv_backward_kernel", "maxpool_forward",
             "maxpool_backward", "avgpool_forward", "avgpool_backward", "nonlin_forward",
             "nonlin_backward"]
    for n in names:
        assert callable(getattr(cuda_fast_kernels, n)) and callable(getattr(cuda_kernels, n))
    if _lib.device_count() == 0:
        with pytest.raises(_lib.KernelUnavailable):
            cuda_fast_kernels.conv_forward(np.zeros((1, 5, 5), np.float32),
                                           np.zeros((1, 1, 3, 3), np.float32),
                                           np.zeros(1, np.float32), 1)


def test_default_threads_env(monkeypatch):
    monkeypatch.delenv("DENSEPROP_THREADS", raising=False)
    assert backend.default_threads() == 1
    monkeypatch.setenv("DENSEPROP_THREADS", "6")
    assert backend.default_threads() == 6
    monkeypatch.setenv("DENSEPROP_THREADS", "0")
    assert backend.default_threads() == 1
    monkeypatch.setenv("DENSEPROP_THREADS", "lots")
    with pytest.warns(RuntimeWarning):
        assert backend.default_threads() == 1


def test_product_never_imports_oracle():
    pkg = os.path.join(REPO, "paper_1412_4526_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(root, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f
