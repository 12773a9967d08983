"""The GPU-box configuration: no /root/reference there. The bench's timed legs read the committed
config-2 step fixture (never the reference), and the reference scheduler loads from the offline
install under baseline/_ref that __graft_entry__.build() creates and that travels with the repo."""

import json
import os
import subprocess
import sys

import pytest

from conftest import refsim_or_skip  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    sys.path.insert(0, ROOT)
    import bench

    return bench


def test_step_fixture_matches_reference_generate_trace():
    """tests/golden/config2_step_trace.jsonl == the head of generate_trace(config 2, rate 8,
    300 s, seed 7) (workload.py:162-198), request for request."""
    bench = _bench()
    ps = refsim_or_skip()
    classes = [ps.TaskClass(*c) for c in bench.CONFIG2_CLASSES]
    tr = ps.generate_trace(classes, 8.0, 300.0, 7)
    got = bench.step_requests(1, 0)
    with open(bench.STEP_TRACE) as fh:
        fixture = [json.loads(ln) for ln in fh if ln.strip()]
    assert len(fixture) == 128
    for r, d in zip(tr.requests[:128], fixture):
        assert (r.id, r.task, r.num_tokens, r.arrival_time, r.ttft_slo) == (
            d["id"], d["task"], d["num_tokens"], d["arrival_s"], d["ttft_slo_s"])
    assert [r.num_tokens for r in got] == [r.num_tokens for r in tr.requests[:16]]


def test_step_requests_round_robin_without_reference(monkeypatch):
    """Rank r of N gets requests i = r mod N of the first 16 N; no reference import needed."""
    bench = _bench()
    monkeypatch.setenv("FP_REFSIM_NO_SRC", "1")
    monkeypatch.setenv("PREFILLSIM_PATH", "/nonexistent")
    for n in (1, 2, 4, 8):
        parts = [bench.step_requests(n, r) for r in range(n)]
        assert all(len(p) == 16 for p in parts)
        ids = sorted(x.id for p in parts for x in p)
        assert ids == sorted(json.loads(ln)["id"] for ln in open(bench.STEP_TRACE).readlines()[: 16 * n])
        pos = {json.loads(ln)["id"]: i for i, ln in enumerate(open(bench.STEP_TRACE))}
        assert all(pos[x.id] % n == r for r, p in enumerate(parts) for x in p)


def test_refsim_loads_from_baseline_install_only():
    """With the source-tree candidate disabled (as on the GPU box), prefillsim resolves to the
    baseline/_ref install."""
    from paper_2602_16603_b200 import refsim

    if not os.path.isdir(os.path.join(refsim.INSTALL_DIR, "prefillsim")):
        pytest.skip("baseline/_ref not installed here (run __graft_entry__.build())")
    code = ("import sys; sys.path.insert(0, %r); from paper_2602_16603_b200 import refsim; "
            "ps = refsim.load(); print(ps.__file__)" % ROOT)
    env = dict(os.environ, FP_REFSIM_NO_SRC="1")
    env.pop("PREFILLSIM_PATH", None)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         cwd="/tmp", timeout=120)
    assert out.returncode == 0, out.stderr[-1500:]
    assert out.stdout.strip().startswith(refsim.INSTALL_DIR), out.stdout


def test_refsim_install_is_idempotent():
    from paper_2602_16603_b200 import refsim

    if not os.path.isdir(refsim.REFERENCE_SRC) and not os.path.isdir(
            os.path.join(refsim.INSTALL_DIR, "prefillsim")):
        pytest.skip("neither the reference source nor an install is present")
    assert refsim.install() is True
