"""The planner / scheduler parity checks of test_hetsim_parity.py, repeated under the gpu marker so
the GPU box's record carries them too (the box has no /root/reference: the 300-case
differential dump is checked against the committed digest of the compiled reference's dump, and
the reference tests' known answers are re-asserted)."""
import hashlib
import json
import os

import pytest

from tests import test_hetsim_parity as P

pytestmark = pytest.mark.gpu


def test_differential_dump_matches_reference_digest(native):
    P.make(os.path.join(P.REF_OUT, "hetsim_diff_new"))
    new = P.run_driver("hetsim_diff_new")
    g = json.load(open(P.GOLDEN))
    assert (g["cases"], g["seed"]) == (P.CASES, P.SEED)
    assert hashlib.sha256(new.encode()).hexdigest() == g["sha256"]


def test_reference_known_answers(native):
    P.test_golden_kats_from_reference_tests(native)
    P.test_golden_trace_prefix(native)
