"""The C-ABI library loads and exports exactly what include/avec_cuda.h declares (CPU)."""
import ctypes
import pathlib
import re
import subprocess

import pytest

from paper_2103_04930_b200 import _lib

ROOT = pathlib.Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "avec_cuda.h"
SO = ROOT / "paper_2103_04930_b200" / "lib" / "libavec_cuda.so"


def header_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(avec_[a-z0-9_]+)\s*\(", text)))


def test_header_matches_python_binding_list():
    assert header_functions() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    assert SO.exists(), "run build() first"
    out = subprocess.run(["nm", "-D", "--defined-only", str(SO)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (avec_[a-z0-9_]+)", out))
    missing = set(header_functions()) - exported
    assert not missing, missing


def test_library_loads_and_binds_without_gpu():
    L = _lib.load()
    for name in _lib.EXPORTS:
        assert callable(getattr(L, name))
    assert L.avec_version().decode().startswith("avec-b200")


def test_kernels_are_sm100a_tcgen05():
    sass = subprocess.run(["cuobjdump", "-sass", str(SO)], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass, "conv kernel must issue tcgen05.mma"
    assert "UTMALDG" in sass, "conv kernel must use TMA"
    assert "LDTM" in sass, "epilogue must read TMEM"
    assert "HMMA" not in re.sub(r"UTCHMMA", "", sass)


def test_synth_weights_deterministic_and_sized():
    from paper_2103_04930_b200 import netspec, synth_posenet_weights
    w1 = synth_posenet_weights(netspec.spec(seed=3))
    w2 = synth_posenet_weights(netspec.spec(seed=3))
    assert w1.size == netspec.weight_floats(netspec.coco_layers()) == 52311446
    assert (w1 == w2).all()
    assert not (w1 == synth_posenet_weights(netspec.spec(seed=4))).all()


def test_invalid_spec_is_invalid_model():
    from paper_2103_04930_b200 import AvecError, synth_posenet_weights
    with pytest.raises(AvecError) as e:
        synth_posenet_weights(b"avecnet 1\nfamily nope\n")
    assert e.value.name == "invalid_model"


def test_input_precision_spec_key():
    """`input tf32` selects the tf32 first layer (test_gpu_tf32.py); it does not
    change the weights blob; anything but bf16 / tf32 is an invalid model."""
    from paper_2103_04930_b200 import AvecError, netspec, synth_posenet_weights
    s32 = netspec.spec(input_dtype="tf32")
    assert b"input tf32" in s32 and b"input" not in netspec.spec()
    assert (synth_posenet_weights(s32) == synth_posenet_weights(netspec.spec())).all()
    with pytest.raises(AvecError):
        synth_posenet_weights(b"avecnet 1\nfamily openpose_coco\ninput fp8\n")


def test_host_library_exports_frame_groups():
    """The split policy's partition is exported from the C++ host library
    (b200_backend.hpp) and is what sharding.py binds."""
    host = ROOT / "paper_2103_04930_b200" / "lib" / "libavec_host.so"
    out = subprocess.run(["nm", "-D", "--defined-only", str(host)], capture_output=True, text=True,
                         check=True).stdout
    assert " T avec_frame_groups" in out
    from paper_2103_04930_b200.sharding import frame_groups
    assert frame_groups(32, 8) == [(4 * i, 4) for i in range(8)]
