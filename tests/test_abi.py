"""CPU-side checks of the drop-in boundary: libfsgg.so loads, exports every
symbol include/*.h declares, validates like the reference, and refuses to
compute without a device (no CPU fallback). No kernel is launched here."""
import json
import os

import numpy as np
import pytest

import paper_2310_13870_b200 as F
from paper_2310_13870_b200 import _native as N
from paper_2310_13870_b200 import datasets
from conftest import GOLDEN, load_golden


def test_library_exports_every_header_symbol():
    names = N.header_functions()
    assert len(names) >= 25
    lib = N.lib()
    missing = [f for f in names if not hasattr(lib, f)]
    assert missing == []
    # every declared function has a ctypes signature on the Python side
    assert set(names) <= set(N._SIGS)


def test_library_is_sm100a_only():
    # the fatbin embeds sm_100a SASS and nothing else
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.LIB_PATH],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = {line.split(".")[-2] for line in out.stdout.split() if line.endswith(".cubin")}
    assert arches == {"sm_100a"}


@pytest.mark.skipif(F.device_available(), reason="a device is present")
def test_no_device_means_device_error():
    with pytest.raises(F.DeviceError) as e:
        F.Dataset(np.zeros((8, 2), np.float32))
    assert e.value.exit_code == 5


def test_kernel_and_config_validation():
    # proj/src/kernel.cpp:23-26
    with pytest.raises(F.InvalidConfig):
        F.Kernel(F.KernelFamily.gaussian, 0.0)
    with pytest.raises(F.InvalidConfig):
        F.Kernel(F.KernelFamily.gaussian, -1.0)
    assert F.InvalidConfig("x").exit_code == 2
    assert F.NumericError("x").exit_code == 4


def test_rounds_for_and_epsilon_via_abi():
    meta = json.load(open(os.path.join(GOLDEN, "golden_meta.json")))["kat"]
    cfg = F.SparsifierConfig()
    assert cfg.rounds_for(1024) == meta["rounds_for"]["1024"] == 60
    assert cfg.rounds_for(1000) == meta["rounds_for"]["1000"] == 60
    assert F.SparsifierConfig(C=2.0).rounds_for(1024) == meta["rounds_for"]["1024_C2"]
    assert (F.SparsifierConfig(lambda_k1_estimate=0.5).rounds_for(1024)
            == meta["rounds_for"]["1024_lambda_half"])
    assert F.SparsifierConfig(rounds=7).rounds_for(1024) == 7
    assert F.default_epsilon(1024) == meta["default_epsilon_1024"]
    assert F.default_epsilon(2) == meta["default_epsilon_2"]
    with pytest.raises(F.InvalidConfig):
        F.SparsifierConfig(lambda_k1_estimate=-1.0).rounds_for(100)


def test_generators_match_reference_golden():
    g = np.load(os.path.join(GOLDEN, "generators.npz"))
    mp, _ = datasets.make_moons(1000, 0.05, 1)
    bp, _ = datasets.make_blobs(1000, [[-2.0, 0.0], [2.0, 0.0]], 0.5, 1)
    assert np.array_equal(mp, g["moons1000"])
    assert np.array_equal(bp, g["blobs1000"])
    c1 = load_golden("c1_blobs")
    assert np.array_equal(datasets.config("C1").points, c1["points"])


def test_generators_reject_bad_arguments():
    with pytest.raises(F.InvalidConfig):
        datasets.make_moons(1, 0.05, 1)
    with pytest.raises(F.InvalidConfig):
        datasets.make_blobs(1, [[0.0, 0.0], [1.0, 1.0]], 0.1, 1)


def test_harness_configs_shapes():
    c4 = datasets.config("C4")
    assert c4.points.shape == (154401, 5) and c4.points.dtype == np.float32
    assert c4.points[:, 0].min() >= 0 and c4.points[:, 0].max() < 1
    assert len(np.unique(c4.labels)) <= 8
    c5 = datasets.config("C5", n=2000)
    assert c5.points.shape == (2000, 784)
    assert c5.points.min() >= 0.0 and c5.points.max() <= 1.0
    assert 5.0 < c5.sigma < 20.0


def test_edge_list_text_format(tmp_path):
    g = F.WeightedGraph(n=3, u=np.array([0, 1], np.uint32), v=np.array([1, 2], np.uint32),
                        w=np.array([0.5, 1.0 / 3.0]), row_ptr=np.array([0, 1, 2, 2], np.uint64),
                        degrees=np.array([0.5, 0.5 + 1 / 3, 1 / 3]), total_weight=0.5 + 1 / 3)
    p = tmp_path / "g.txt"
    g.write_edge_list(str(p))
    lines = p.read_text().splitlines()
    assert lines[0] == "3 2"
    assert lines[2] == "1 2 0.33333333333333331"  # %.17g (proj/src/graph.cpp:237)
