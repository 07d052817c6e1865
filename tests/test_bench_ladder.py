"""tools/bench_ladder.py: the port of the reference
bench's slope fit and CSV writers. The cases mirror the reference's own
tests (proj/tests/test_bench.cpp:194-260), and the fit is pinned against the
compiled reference (oracle/_ref/libbitsort_ref.so: bws_bench_run's records
and slopes, proj/src/bench.cpp:162-231)."""
from __future__ import annotations

import ctypes
import math
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))
import bench_ladder as bl  # noqa: E402


def _synthetic(exponent, alg):
    return [(alg, 32, n, 1, t, int(50.0 * n ** exponent), int(50.0 * n ** exponent) / n)
            for n in (1024, 2048, 4096, 8192, 16384) for t in range(3)]


def test_fit_recovers_exact_power_laws():  # test_bench.cpp:194-218
    reports = bl.fit_scaling(_synthetic(1.0, "bitwise") + _synthetic(2.0, "insertion"))
    assert [r[0] for r in reports] == ["bitwise", "insertion"]
    assert reports[0][1] == pytest.approx(1.0, rel=1e-6)
    assert reports[1][1] == pytest.approx(2.0, rel=1e-6)
    assert reports[0][2] < 1e-6 and len(reports[0][3]) == 5


def test_fit_takes_the_median_over_trials():  # test_bench.cpp:220-232
    recs = [("merge", 32, n, 1, t, v * n, float(v)) for n in (16, 32, 64, 128)
            for t, v in enumerate((900, 100, 500))]
    reports = bl.fit_scaling(recs)
    assert len(reports) == 1
    assert reports[0][3][0][1] == pytest.approx(500.0 * 16)
    assert reports[0][1] == pytest.approx(1.0, rel=1e-9)
    # an even trial count: mean of the middle two (bench.cpp:186-189)
    recs = [("merge", 32, n, 1, t, v * n, float(v)) for n in (16, 32, 64, 128)
            for t, v in enumerate((900, 100, 500, 300))]
    assert bl.fit_scaling(recs)[0][3][0][1] == pytest.approx(400.0 * 16)


def test_fit_rejects_fewer_than_four_sizes():  # test_bench.cpp:234-240
    with pytest.raises(bl.ConfigError):
        bl.fit_scaling([("bitwise", 32, n, 1, 0, n * 10, 10.0) for n in (16, 32, 64)])
    assert bl.fit_scaling([]) == []


def test_csv_rendering():  # test_bench.cpp:242-254
    csv = bl.records_csv([("bitwise", 32, 16384, 42, 0, 123456, 7.535)])
    assert csv.startswith("algorithm,width,n,seed,trial,elapsed_ns,ns_per_element\n")
    assert "bitwise,32,16384,42,0,123456,7.535\n" in csv and "\r" not in csv
    slopes = bl.reports_csv([("bitwise", 1.0125, 0.003, [(16384, 1.0)])])
    assert slopes.startswith("algorithm,slope,residual\n")
    assert "bitwise,1.012500,0.003000\n" in slopes


def _reference():
    import oracle

    if oracle.REFERENCE is None:
        pytest.skip("oracle/_ref/libbitsort_ref.so not built")
    lib = ctypes.CDLL(str(oracle.REFERENCE_PATH))
    vp = ctypes.c_void_p
    lib.bws_bench_config_new.restype = vp
    lib.bws_bench_config_free.argtypes = [vp]
    lib.bws_bench_config_set_sizes.argtypes = [vp, ctypes.POINTER(ctypes.c_uint64), ctypes.c_size_t]
    lib.bws_bench_config_set_trials.argtypes = [vp, ctypes.c_uint32]
    lib.bws_bench_config_set_algorithms.argtypes = [vp, ctypes.c_char_p]
    lib.bws_bench_run.argtypes = [vp, ctypes.POINTER(vp)]
    lib.bws_bench_result_free.argtypes = [vp]
    for f in ("bws_bench_result_records_csv", "bws_bench_result_slopes_csv"):
        getattr(lib, f).argtypes = [vp]
        getattr(lib, f).restype = ctypes.c_char_p
    return lib


def test_fit_matches_the_compiled_reference():
    """The reference's own harness (bws_bench_run) times its sorts and fits the
    slopes; re-fitting its records CSV with the port reproduces its slopes CSV
    digit for digit."""
    lib = _reference()
    cfg = lib.bws_bench_config_new()
    try:
        sizes = (ctypes.c_uint64 * 5)(1024, 2048, 4096, 8192, 16384)
        assert lib.bws_bench_config_set_sizes(cfg, sizes, 5) == 0
        assert lib.bws_bench_config_set_trials(cfg, 3) == 0
        assert lib.bws_bench_config_set_algorithms(cfg, b"bitwise,merge,platform") == 0
        res = ctypes.c_void_p()
        assert lib.bws_bench_run(cfg, ctypes.byref(res)) == 0
        try:
            rec_csv = lib.bws_bench_result_records_csv(res).decode()
            slopes_csv = lib.bws_bench_result_slopes_csv(res).decode()
        finally:
            lib.bws_bench_result_free(res)
    finally:
        lib.bws_bench_config_free(cfg)
    rows = [l.split(",") for l in rec_csv.strip().splitlines()[1:]]
    records = [(r[0], int(r[1]), int(r[2]), int(r[3]), int(r[4]), int(r[5]), float(r[6])) for r in rows]
    assert len(records) == 3 * 5 * 3
    # the port's CSV writer reproduces the reference's records CSV
    assert bl.records_csv(records) == rec_csv
    assert bl.reports_csv(bl.fit_scaling(records)) == slopes_csv
    for alg, slope, resid, pts in bl.fit_scaling(records):
        assert math.isfinite(slope) and len(pts) == 5
