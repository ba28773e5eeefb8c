"""GPU Monte-Carlo harness: the reference's published acceptance numbers
(test_output.txt:156: F(4,3), C=(3,2), 13x14, N(0,1), seed 424242, 1000 trials)
reproduced by the B200 layer, which is bit-exact with the reference per trial."""

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2004_11077_b200.harness import ErrorExperiment, run_error_benchmark  # noqa: E402


def test_known_answer_means():
    rows = run_error_benchmark(ErrorExperiment(trials=1000, seed=424242))
    got = {(r["mode"], r["qconfig"]): r["mean"] for r in rows if r["metric"] == "rel_l2_err"}
    want = {("canonical", "8b"): 2.72492, ("canonical", "8b+9b"): 1.52523,
            ("legendre", "8b"): 4.20480, ("legendre", "8b+9b"): 3.58458}
    for k, v in want.items():
        assert got[k] == pytest.approx(v, abs=1.5e-5), (k, got[k])
