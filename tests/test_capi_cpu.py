"""CPU: the C-ABI library loads, exports every symbol include/double_b200.h declares, and fails loudly
(no CPU fallback) when no GPU is present."""
import os
import re

import pytest

from conftest import ROOT


def _declared():
    text = open(os.path.join(ROOT, "include", "double_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int)\s+(dbl_\w+)\(", text, re.M)))


def test_header_declares_the_boundary():
    names = _declared()
    assert len(names) >= 25
    for must in ("dbl_store_lookup", "dbl_store_insert", "dbl_forward_argmax", "dbl_run", "dbl_run_ar"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2601_05524_b200 import _capi
    L = _capi.lib()
    missing = [n for n in _declared() if not hasattr(L, n)]
    assert not missing, missing
    assert set(_declared()) <= set(_capi.PROTOTYPES), set(_declared()) - set(_capi.PROTOTYPES)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2601_05524_b200 import HierarchicalDatastore, _capi
    assert _capi.lib().dbl_device_ok() == 0
    with pytest.raises(_capi.CudaError):
        HierarchicalDatastore(3, 10)


def test_model_v1_and_dstore_v1_parsers():
    from paper_2601_05524_b200.specpar import parse_dstore_v1, parse_model_v1
    g = os.path.join(ROOT, "tests", "golden")
    order, vocab, w, p, f = parse_model_v1(open(os.path.join(g, "config1_target.model-v1")).read())
    assert (order, vocab) == (2, 32) and w.shape[1] == 2 and p.shape == (len(w), 32) and len(f) == 32
    assert abs(p.sum(axis=1) - 1).max() < 1e-12
    mo, seqs = parse_dstore_v1(open(os.path.join(g, "config1_prior.dstore-v1")).read())
    assert mo == 3 and len(seqs) == 10 and all(len(s) == 64 for s in seqs)
