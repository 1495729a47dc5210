"""Host-side logic of bench.py (CPU): ncu traffic units, the --gpus self-launch command, the
queue shards of every workload at world 1/2/4/8, the whole-job counters over a world-2 gloo
group, the like-for-like configuration of the oracle leg."""
import json
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

import bench


def test_ncu_traffic_converts_each_metric_with_its_own_unit(tmp_path):
    # MRIQ: 25.23 Mbyte read + 22.53 Kbyte written (profiles/r01_ncu_summary.json) = 25.25 MB,
    # not 47.76 MB (the write counted in the read's unit)
    row = {"kernel": "void k_persistent<BodyMRIQ>(...)",
           "dram__bytes_read.sum": {"value": "25.23", "unit": "Mbyte"},
           "dram__bytes_write.sum": {"value": "22.53", "unit": "Kbyte"}}
    (tmp_path / "r09_ncu_summary.json").write_text(json.dumps({"rep": [row]}))
    t = bench.ncu_traffic("MRIQ", str(tmp_path))
    assert abs(t["bytes_per_instance"] - (25.23e6 + 22.53e3)) < 1
    assert abs(t["write"] - 22.53e3) < 1e-6
    # the committed round-1 capture: MRIQ about 25.25 MB per launch
    t = bench.ncu_traffic("MRIQ")
    assert t is not None and 25.0e6 < t["bytes_per_instance"] < 25.5e6


def test_spawn_cmd(monkeypatch):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    a = bench.parse(["--gpus", "4", "--steps", "2"])
    cmd = bench.spawn_cmd(a, ["--gpus", "4", "--steps", "2"])
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-3:] == ["--gpus", "4", "--steps", "2"][-3:]
    assert bench.spawn_cmd(bench.parse(["--gpus", "1"]), []) is None
    assert bench.spawn_cmd(bench.parse([]), []) is None
    assert bench.spawn_cmd(bench.parse(["--gpus", "8", "--impl", "reference"]), []) is None
    monkeypatch.setenv("WORLD_SIZE", "4")
    assert bench.spawn_cmd(a, []) is None          # already under a launcher


@pytest.mark.parametrize("workload", ["c2", "c4", "c5"])
def test_shards_partition_the_global_queue(workload):
    for world in (1, 2, 4, 8):
        g = bench.global_queue(workload, 4, world)
        parts = [bench.build_queue(r, world, 4, workload) for r in range(world)]
        assert sorted(sum(parts, [])) == sorted(g)
        n = len(g)
        assert n == {"c2": 32 * world, "c4": 1000 * world, "c5": 10000}[workload]
        # round robin per kind: shard sizes differ by at most the number of kinds
        assert max(map(len, parts)) - min(map(len, parts)) <= len(set(g))


def test_c4_mix_variants():
    import kl_inputs as G
    for mix in ("CI", "MI", "MIX", "ALL"):
        q = bench.global_queue("c4", 4, 1, mix)
        assert len(q) == 1000 and set(q) == set(G.MIXES[mix])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shard = bench.build_queue(rank, world, 4, "c5")
    # this rank's counters as the kernels leave them; uneven shards (c5 at world 2 is 5000 each,
    # at world 8 1248-1252): the whole-job count is the gathered sum, never len(shard) * world
    c = torch.tensor([len(shard), 0, 0, 0, 0, rank, world, 0], dtype=torch.int64)
    g = torch.zeros(world * 8, dtype=torch.int64)
    dist.all_gather_into_tensor(g, c)
    t = bench.max_over_ranks(10.0 + rank, "cpu", world, "gloo")
    q.put((rank, int(g.view(world, 8)[:, 0].sum()), t))
    dist.barrier()
    dist.destroy_process_group()


def test_whole_job_counters_world2_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_rank, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, n, t in res:
        assert n == 10000 and t == 11.0


def test_oracle_leg_uses_the_gpu_runs_model_config():
    leg = bench.OracleLeg.__new__(bench.OracleLeg)        # configuration only, no kernels generated
    profs, pcfg = bench._oracle_profiles()
    assert profs and set(profs) == set(bench.ALL)
    import oracle as O
    O.build()
    kw = dict(profile_path=None, split_rule=1, levels="four", alpha=None)
    leg.__init__(["PC", "BS"], "small", **kw)
    assert leg.sched_kw == {"ap": pcfg["alpha_p"], "am": pcfg["alpha_m"], "mode": "4", "split_rule": 1,
                            "cp_min": pcfg.get("cp_min", 0.0), "distinct_kinds": False}
    leg2 = bench.OracleLeg.__new__(bench.OracleLeg)
    leg2.__init__(["PC", "BS"], "small", **dict(kw, levels="all", bmax="sat"))
    assert leg2.sched_kw["mode"] == "all" and leg2.sched_kw["distinct_kinds"] is True
    assert leg2.profs["MRIQ"]["bmax"] == leg2.profs["MRIQ"]["bmax_sat"]
    assert abs(leg.cfg.L0 - pcfg["L0"]) < 1e-9 and abs(leg.cfg.B - pcfg["B"]) < 1e-12
    r = leg.run(target_s=0.5)
    assert r["kind"] == "oracle" and r["value"] > 0 and r["cores"] >= 1


def test_pc_reports_both_atoms():
    import kl_inputs as G
    p = G.gen("PC", "small")["params"]
    w = bench.algorithmic_work("PC", p)
    assert w["bytes"] - w["bytes_32B"] == p["n_threads"] * p["hops"] * 32


def test_saturation_bmax_reading_r31():
    """R31 (option --bmax sat): b_max for every whole-warp level is the smallest cap whose solo
    time is within 1 % of the best in the calibration sweep; C2 (quarters of b_max) keeps the
    hardware b_max; the oracle leg sees the same b_max as the GPU run."""
    import json
    import os
    sys_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools")
    import importlib.util
    spec = importlib.util.spec_from_file_location("calibrate", os.path.join(sys_path, "calibrate.py"))
    cal = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(cal)
    assert cal.saturation_bmax({"1": 2.48, "2": 2.03, "3": 1.981, "4": 1.975, "8": 1.973}) == 3
    assert cal.saturation_bmax({1: 1.0, 2: 0.5}) == 2
    assert cal.saturation_bmax({1: 1.0, 2: 0.995}) == 1
    assert cal.saturation_bmax({1: 1.0, 2: 0.9, 3: 0.89}, tol=0.02) == 2
    path = os.path.join(bench.ROOT, "profiles", "kl_profile_b200.json")
    d = json.load(open(path))
    for k, m in d["measured"].items():
        if m.get("cap_sweep_ms") and k in d["profiles"]:
            assert d["profiles"][k]["bmax_sat"] == cal.saturation_bmax(m["cap_sweep_ms"])
    p_all, _ = bench.load_profiles(path, "all", "sat")
    p_hw, _ = bench.load_profiles(path, "all")
    p_four, _ = bench.load_profiles(path, "four")
    assert p_all["MRIQ"]["bmax"] == d["profiles"]["MRIQ"]["bmax_sat"] < d["profiles"]["MRIQ"]["bmax"]
    assert "bmax" not in p_hw["MRIQ"] and "bmax" not in p_four["MRIQ"]   # left to the runtime
    o_all, _ = bench._oracle_profiles(path, "all", "sat")
    o_four, _ = bench._oracle_profiles(path, "four", "sat")
    for k in bench.ALL:
        assert o_all[k]["bmax"] == p_all[k]["bmax"]
        assert o_four[k]["bmax"] == d["profiles"][k]["bmax"]
