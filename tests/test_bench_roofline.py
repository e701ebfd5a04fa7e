"""The bench line's roofline is reproducible by hand (round-1
verdict item 2): the committed final bench line's E || D fraction equals
§8(d)'s algorithmic bytes -- D (Type-II) = 4 D_b + 8 D_b + 8 D_b + 8 n and
E (Type-I) = 4 B per probed entry + 16 B per matched triad -- computed here
from the counts the line itself carries, divided by the phase's CUDA-event time
and the measured HBM peak. CPU only: reads profiles/, runs nothing on a GPU."""
import json
import os

import pytest

import bench

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LINE = os.path.join(REPO, "profiles", "r02h_bench_matched.json")


def _line():
    with open(LINE) as fh:
        return json.loads(fh.read().strip().splitlines()[-1])


def test_survey_bytes_terms():
    # §8(d) table, row by row, on round numbers
    n, D, Db, k, ntri, nprobe = 1000, 50_000, 12_000, 5, 700, 90_000
    b = bench.survey_bytes(n, D, Db, k, ntri, nprobe)
    A = (4 * D + 8 * n + D + 4 * n + 8 * k * n + 8 * n)            # border + histogram + weights
    B = (4 * D + 8 * n + D + 4 * Db + 8 * n)                        # P-list build
    C = (4 * Db + 8 * Db + 8 * k * n)                               # B_w table
    assert b["A"] == A + B + C
    assert b["ED"] == 20 * Db + 8 * n + 4 * nprobe + 16 * ntri      # Type-II + Type-I
    assert b["F"] == 24 * n


@pytest.mark.skipif(not os.path.exists(LINE), reason="no committed bench line")
def test_final_line_frac_by_hand():
    d = _line()
    cfg, roof = d["config"], d["roofline"]
    n, Db = cfg["n"], cfg["pred_entries"]
    alg = 20 * Db + 8 * n + 4 * cfg["probes"] + 16 * cfg["triangles"]
    ed = roof["phases"]["ED_type1_type2"]
    assert ed["survey_bytes"] == alg
    gbps = alg / (ed["ms"] * 1e-3) / 1e9
    assert abs(gbps - roof["achieved"]) <= 0.1
    assert abs(gbps / roof["peak"] - roof["frac"]) <= 1e-4
    # the ncu traffic ratio is traffic / algorithmic bytes, from the capture of this build
    assert abs(roof["traffic"] / alg - roof["traffic_over_alg"]) <= 1e-3
    assert "matches this build: True" in roof["traffic_source"]
    # whole-job value = m / step time
    assert abs(cfg["m"] / (d["ms_per_step"] * 1e-3) / 1e9 - d["value"]) <= 1e-3
