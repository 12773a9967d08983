"""Multi-instance results in the reference artifact formats: merged
run.csv / summary.json / sweep.csv and the reference goodput bisection over a round-robin
deployment. At one instance every artifact must be byte-identical to the reference CLI's."""

from conftest import refsim_or_skip  # noqa: E402
import filecmp
import json
import os

import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
TRACE = os.path.join(GOLDEN, "config1_trace.jsonl")


def _ps():
    from paper_2602_16603_b200 import refsim

    return refsim_or_skip()


def test_single_instance_artifacts_match_reference_cli(tmp_path):
    ps = _ps()
    from prefillsim import cli

    from paper_2602_16603_b200 import dispatch

    ref_dir = tmp_path / "ref"
    assert cli.main(["run", "--trace", TRACE, "--out", str(ref_dir), "--seed", "0"]) == 0
    cfg = cli.resolve_config(cli.make_parser().parse_args(
        ["run", "--trace", TRACE, "--out", str(ref_dir), "--seed", "0"]))
    tr = ps.load_trace(TRACE)
    res = dispatch.run_instances(tr, 1, cli.build_policy(cfg), cli.build_cost_params(cfg), 0)
    ours = tmp_path / "ours"
    dispatch.write_run_artifacts(res, str(ours), config_hash=cli.config_hash(cfg))
    for f in ("run.csv", "summary.json"):
        assert filecmp.cmp(ref_dir / f, ours / f, shallow=False), f


def test_merged_artifacts_two_instances(tmp_path):
    ps = _ps()
    from paper_2602_16603_b200 import dispatch

    tr = ps.load_trace(TRACE)
    params = ps.CostParams(num_layers=4)
    res = dispatch.run_instances(tr, 2, ps.PolicyConfig(), params, 0, record_events=True)
    summary = dispatch.write_run_artifacts(res, str(tmp_path))
    merged = dispatch.merge_results(res)
    assert summary["instances"] == 2
    assert summary["requests"] == len(tr)
    assert summary["attainment"] == ps.slo_attainment(merged.outcomes)
    assert summary["rounds"] == res[0].rounds + res[1].rounds
    assert summary["blocking"] == ps.blocking_stats(res[0].blocking_log + res[1].blocking_log)
    from prefillsim import metrics

    rows = open(tmp_path / "run.csv").read().splitlines()
    assert rows[0] == ",".join(metrics.RUN_COLUMNS)
    assert len(rows) == len(tr) + 1
    for k in range(2):
        d = tmp_path / f"instance{k}"
        s = json.loads(open(d / "summary.json").read())
        assert s["instance"] == k and s["requests"] == len(res[k].outcomes)
        assert os.path.exists(d / "events.jsonl")
    with pytest.raises(ValueError):
        dispatch.merge_results([res[0], ps.run(dispatch.round_robin(tr, 2)[1], ps.PolicyConfig(),
                                               params, 1)])


def test_sweep_and_goodput_one_instance_equal_reference():
    ps = _ps()
    from prefillsim import metrics

    from paper_2602_16603_b200 import dispatch

    tr = ps.load_trace(TRACE)
    params = ps.CostParams(num_layers=4)
    rows = dispatch.sweep_instances(tr, 1, ps.PolicyConfig(), params, [1.0, 3.0])
    for rate, row in zip([1.0, 3.0], rows):
        ref = metrics.sweep_row("rate", rate, ps.run(ps.scale_rate(tr, rate / tr.base_rate()),
                                                      ps.PolicyConfig(), params, 0))
        assert row == ref
        assert set(row) == set(metrics.SWEEP_COLUMNS)
    rc = ps.RunConfig(policy=ps.PolicyConfig(), cost=params, seed=0)
    ours = dispatch.goodput_search_instances(tr, rc, 1, rate_bounds=(0.5, 8.0), tol=0.1)
    ref = ps.goodput_search(tr, rc, rate_bounds=(0.5, 8.0), tol=0.1)
    assert ours == ref
    assert metrics.run is not None and metrics.run.__module__ == "prefillsim.engine"  # restored


def test_goodput_scales_with_instances():
    ps = _ps()
    from paper_2602_16603_b200 import dispatch

    tr = ps.load_trace(TRACE)
    rc = ps.RunConfig(policy=ps.PolicyConfig(), cost=ps.CostParams(num_layers=4), seed=0)
    g1 = dispatch.goodput_search_instances(tr, rc, 1, rate_bounds=(0.5, 16.0), tol=0.1)
    g2 = dispatch.goodput_search_instances(tr, rc, 2, rate_bounds=(0.5, 16.0), tol=0.1)
    assert g2.value >= g1.value


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    from paper_2602_16603_b200 import dispatch, refsim

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ps = refsim_or_skip()
    tr = ps.load_trace(TRACE)
    mine = dispatch.round_robin(tr, world)[rank]
    local = ps.run(mine, ps.PolicyConfig(), ps.CostParams(num_layers=4), 0)
    results = dispatch.gather_results(local)
    if rank == 0:
        dispatch.write_run_artifacts(results, out_dir)
    dist.destroy_process_group()


def test_gloo_gathered_artifacts(tmp_path):
    import multiprocessing as mp
    import socket

    ps = _ps()
    from paper_2602_16603_b200 import dispatch

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, 2, port, str(tmp_path / "dist")))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    tr = ps.load_trace(TRACE)
    local = dispatch.run_instances(tr, 2, ps.PolicyConfig(), ps.CostParams(num_layers=4), 0)
    dispatch.write_run_artifacts(local, str(tmp_path / "local"))
    for f in ("run.csv", "summary.json", "instance0/run.csv", "instance1/summary.json"):
        assert filecmp.cmp(tmp_path / "dist" / f, tmp_path / "local" / f, shallow=False), f
