"""BASELINE configs[4]: HITS on the uk-union-shaped graph (R-MAT scale 28,
133.6 M vertices, 5.5 B edges; the HITS block [[0, A^T], [A, 0]] has 11.0 B entries), Eq. 8
(PAPER.md L436-L440), on one B200 as 8 row slices through the loopback transport
(bench/experiment_c5.py: device generator -> bitonic partition -> per-slice rows -> local solvers).

Parity: one HITS step from the GPU's iterate k-1, computed by the fp64 oracle on every block row
(halves normalised to sum 1, L440), against the GPU's iterate k: L1 < 1e-6 per half.

The full size takes about 10 minutes and ~100 GB of host memory (the slices stay on the host for
the oracle), so it runs only with TCSPMV_TEST_C5=1 (log: profiles/r02_c5*.log); the same route at
1/64 size (c5_s22) runs in the default GPU suite."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "bench"))

pytestmark = pytest.mark.gpu


def _check(rec, config):
    assert rec["config"] == config
    assert rec["iterations"] == rec["iters"]
    assert rec["block_entries"] == 2 * rec["m"] and sum(rec["slice_entries"]) == rec["block_entries"]
    p = rec["parity"]
    assert p["ok"] and p["l1_a"] < 1e-6 and p["l1_h"] < 1e-6 and p["zero_rows_exact"], p
    assert p["max_rel_a"] < 1e-5 and p["max_rel_h"] < 1e-5, p


@pytest.mark.parametrize("transport", ["slices", "loopback"])
def test_c5_route_s22(transport, gpu):
    import experiment_c5
    _check(experiment_c5.run("c5_s22", P=8, iters=6, transport=transport), "c5_s22")


@pytest.mark.slow
@pytest.mark.skipif(not os.environ.get("TCSPMV_TEST_C5"), reason="full c5: set TCSPMV_TEST_C5=1 (~10 min)")
def test_c5_full_size(gpu):
    import experiment_c5
    rec = experiment_c5.run("c5", P=8, iters=6)
    _check(rec, "c5")
    assert rec["n"] == 133_633_040 and rec["m"] == 5_507_679_822
