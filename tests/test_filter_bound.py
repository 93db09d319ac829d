"""CPU check of K1's conservative filter (paper_1405_7461_b200/csrc/filter.cuh).

tools/filter_check.cpp evaluates the reference's discriminant with the
vectorised pair arithmetic of core.py:490-537 on adversarial pairs (thresholds
at each pair's own flip point, near-parallel and constant-offset motion,
zero-length spans, waypoints, planar data, epoch-scale times, head-on motion
at the segment-distance flip point) and asserts that every pair with a
non-negative reference discriminant is flagged by the FP64 filter in every
clip case K1 can route it through, and that every reference hit is flagged
by the FP32 pre-filter (with the item origin at the query and at a shifted
point), also in K1's lane form (one threshold from the largest of four speed
bounds, a NaN-propagating min of four norms, then the candidate's own compare), and
that no reference hit is removed by the box cull of the K1 layout (segment
boxes rounded outward to FP32, box_gap2 vs box_cull_r2).  Mutated margins of
the two filters must produce misses, so the generator is known to
reach both bounds.  Mode 8 builds the "absorbed offset" pairs: long motion
crossing the query with a perpendicular offset below the rounding of
|U|^2, which the reference reports as hits at any threshold; the box cull's
radius needs its box-diagonal term for them.
"""

from __future__ import annotations

import json
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tools", "filter_check.cpp")
HDR = os.path.join(ROOT, "paper_1405_7461_b200", "csrc", "filter.cuh")


def _build(tmp_path, header=HDR):
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    src = open(SRC).read().replace('"../paper_1405_7461_b200/csrc/filter.cuh"', '"%s"' % header)
    cpp = tmp_path / "fc.cpp"
    cpp.write_text(src)
    exe = tmp_path / "fc"
    # -ffp-contract=off: the library is built with -fmad=false
    # -frounding-math: the FP32 pre-filter's directed roundings use fesetround
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-frounding-math", "-std=c++17", "-o", str(exe), str(cpp)],
                   check=True)
    return exe


def _run(exe, iters):
    p = subprocess.run([str(exe), str(iters)], capture_output=True, text=True)
    return p.returncode, json.loads(p.stdout.strip().splitlines()[-1]), p.stderr


def test_filter_flags_every_nonnegative_reference_discriminant(tmp_path):
    rc, out, err = _run(_build(tmp_path), 150_000)
    assert rc == 0, err
    assert out["edge"]["misses"] == 0 and out["random"]["misses"] == 0
    assert out["edge"]["disc_pos"] > 100_000 and out["edge"]["skipped"] == 0
    # FP32 pre-filter: every reference hit is flagged
    assert out["edge"]["f32_misses"] == 0 and out["random"]["f32_misses"] == 0
    # box cull: no reference hit is culled, and the radius's diagonal term is
    # needed (without it the absorbed-offset pairs of mode 8 are culled)
    assert out["edge"]["box_checks"] > 1_000_000 and out["edge"]["box_misses"] == 0
    assert out["edge"]["box_mutation_misses"] > 0
    # separating-axis stage: rejects pairs, never a reference hit; a
    # margin-free radius does reject hits (the generator reaches the bound)
    assert out["edge"]["sep_checks"] > 1_000_000 and out["edge"]["sep_rejected"] > 100_000
    assert out["edge"]["sep_misses"] == 0 and out["edge"]["sep_mutation_misses"] > 0
    # the K1 layout's re-based FP32 records (group origin -> item origin)
    assert out["edge"]["rebase_checks"] > 1_000_000 and out["edge"]["rebase_misses"] == 0
    assert out["edge"]["hits"] > 100_000 and out["edge"]["f32_checks"] > 1_000_000


def test_filter_check_detects_a_too_small_margin(tmp_path):
    src = open(HDR).read()
    mutated = re.sub(r"0x1p-40 \* c2", "0.0 * c2", src)
    mutated = mutated.replace("fma(0x1p-34, d2, ka)", "ka").replace("0x1p-35 - 1.0", "-1.0")
    assert mutated != src
    hdr = tmp_path / "filter_mut.cuh"
    hdr.write_text(mutated)
    rc, out, _ = _run(_build(tmp_path, str(hdr)), 150_000)
    assert rc == 1 and out["edge"]["misses"] > 0


def test_filter_check_detects_a_missing_fp32_margin(tmp_path):
    src = open(HDR).read()
    mutated = src.replace("it.delta = 0x1p-18 * M + 0x1p-38 * cmax + 0x1p-100;", "it.delta = 0.0;")
    mutated = mutated.replace("(1.0 + 0x1p-8) * (dthr + lq)", "(dthr + lq)")
    assert mutated != src
    hdr = tmp_path / "filter_mut32.cuh"
    hdr.write_text(mutated)
    rc, out, _ = _run(_build(tmp_path, str(hdr)), 150_000)
    assert rc == 1 and out["edge"]["f32_misses"] > 0
