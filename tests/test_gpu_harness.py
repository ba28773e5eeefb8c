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


def _golden():
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "mc_report.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("name", ["acceptance100", "uniform40"])
def test_full_report_matches_reference(name):
    """Every row of the reference's ErrorReport (tests/golden/make_mc_golden.py): quantized, direct and
    stage-stat rows bit-exact (identical per-trial outputs and ground truth); the float rows are the
    fp32 GPU path (|mean| <= 1e-5 relative-L2, reference ~1e-15); the condition table to 1e-12."""
    from paper_2004_11077_b200.quantize import QuantConfig

    g = _golden()[name]
    c = g["config"]
    qcs = tuple((q["name"], QuantConfig(**{k: v for k, v in q.items() if k != "name"})) for q in c["qconfigs"])
    cfg = ErrorExperiment(trials=c["trials"], seed=c["seed"], channels=tuple(c["channels"]),
                          spatial=tuple(c["spatial"]), modes=tuple(c["modes"]), qconfigs=qcs,
                          distribution=c["input_distribution"])
    run_error_benchmark(cfg)
    rep = cfg.json_dict()
    assert rep["config"] == c
    assert len(rep["rows"]) == len(g["rows"])
    for got, want in zip(rep["rows"], g["rows"]):
        assert (got["mode"], got["qconfig"], got["metric"]) == (want["mode"], want["qconfig"], want["metric"])
        if got["qconfig"] == "float" and got["mode"] != "direct":
            assert got["mean"] <= (1e-5 if got["metric"] == "rel_l2_err" else 1e-4), got
        else:
            for k in ("mean", "std", "median", "max", "trials", "seed"):
                assert got[k] == want[k], (got, want, k)
    assert rep["stage_stats"] == g["stage_stats"]
    for got, want in zip(rep["condition_numbers"], g["condition_numbers"]):
        assert got["matrix"] == want["matrix"]
        assert got["two_norm"] == pytest.approx(want["two_norm"], rel=1e-12)
        assert got["frobenius"] == pytest.approx(want["frobenius"], rel=1e-12)
