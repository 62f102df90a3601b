"""CPU tests of the drop-in boundary: the C-ABI library loads, exports every
symbol include/cascade_gpu.h declares, fails loudly without a GPU, and the
host-side trace generator is bit-identical to the reference generator."""
import os
import re

import numpy as np
import pytest

from parity_util import ROOT
from paper_2506_04203_b200 import engine as eng
from paper_2506_04203_b200 import workloads as W


def header_functions():
    src = open(os.path.join(ROOT, "include", "cascade_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = eng.library()
    declared = header_functions()
    assert len(declared) >= 12
    missing = [f for f in declared if not hasattr(lib, f)]
    assert not missing, missing
    assert set(eng.EXPORTED) <= set(declared)


def test_version_string():
    assert b"sm_100a" in eng.library().cg_version()


def test_engine_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(eng.CascadeError) as ei:
        eng.Engine(0)
    assert ei.value.code == 100
    assert "no CPU fallback" in ei.value.message


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C5"])
def test_generate_trace_bit_identical_to_reference(name):
    from oracle import refpy
    for spec, seed in W.trace_specs(name, 3000)[:2]:
        a = eng.generate_trace(spec, seed)
        b = refpy.generate_trace(spec, seed)
        for k in a:
            assert np.array_equal(a[k].view(np.uint64), b[k].view(np.uint64)), k


def test_generate_trace_all_distributions():
    from oracle import refpy
    spec = {"count": 500, "arrival_rate": 3.0,
            "input_tokens": {"dist": "uniform", "min": 10, "max": 900},
            "stages": [{"output_tokens": {"dist": "fixed", "value": 64.4},
                        "score": {"dist": "normal", "mean": 50, "std": 40, "min": 5, "max": 95}},
                       {"output_tokens": {"dist": "choice", "values": [8, 16, 32]},
                        "score": {"dist": "exponential", "mean": 30}}]}
    a = eng.generate_trace(spec, 77)
    b = refpy.generate_trace(spec, 77)
    for k in a:
        assert np.array_equal(a[k].view(np.uint64), b[k].view(np.uint64)), k


@pytest.mark.parametrize("bad,msg", [
    ({"dist": "gamma"}, "unknown distribution: gamma"),
    ({"dist": "exponential", "mean": -1}, "exponential mean must be >= 0"),
    ({"dist": "choice", "values": []}, "choice needs values"),
    ({"dist": "choice", "values": [1, 2], "weights": [1]}, "choice weights length != values length"),
])
def test_generate_trace_errors_match_reference(bad, msg):
    from oracle import refpy
    spec = {"count": 10, "arrival_rate": 1.0, "input_tokens": bad,
            "stages": [{"output_tokens": {"dist": "fixed", "value": 1}, "score": {"dist": "fixed", "value": 1}}]}
    with pytest.raises(eng.CascadeError) as ei:
        eng.generate_trace(spec, 1)
    with pytest.raises(refpy.RefError) as er:
        refpy.generate_trace(spec, 1)
    assert ei.value.code == er.value.code == 0
    assert ei.value.message == er.value.message == msg


def test_product_path_never_imports_oracle():
    """The shipped package must not reference oracle/ (checker only)."""
    pkg = os.path.join(ROOT, "paper_2506_04203_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                text = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "from oracle" not in text and "import oracle" not in text, f
                assert "refpy" not in text and "libcascade_ref" not in text, f
