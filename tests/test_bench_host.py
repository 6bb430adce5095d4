"""CPU checks of bench.py's host-side pieces: workload selection and scaling labels per config, the per-step timeline
summary, the ncu-traffic lookup, and the reference (oracle) arm's JSON line contract."""
import json
import os
import subprocess
import sys
from types import SimpleNamespace

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


@pytest.mark.parametrize("name,world,G,scaling", [("c2", 1, 1, "weak"), ("c2", 8, 1, "weak"), ("c3", 4, 1, "weak"),
                                                  ("c4", 1, 1, "weak"), ("c4", 8, 8, "strong"),
                                                  ("c5", 1, 8, "weak"), ("c5", 2, 8, "weak")])
def test_workload_for(name, world, G, scaling):
    cfg, g, sc = bench.workload_for(SimpleNamespace(workload=name), world)
    assert (cfg.name, g, sc) == (name, G, scaling)


@pytest.mark.parametrize("G,r", [(1, 0), (2, 1), (4, 3), (8, 0), (8, 7)])
def test_head_shards_one_gpu(G, r):
    """--head-shards G --shard-rank r: one GPU runs rank r's shard of a G-GPU C4 run (per-GPU flatness line)."""
    a = SimpleNamespace(workload="c4", head_shards=G, shard_rank=r)
    cfg, g, sc = bench.workload_for(a, 1)
    assert (cfg.name, g, sc) == ("c4", G, "strong" if G > 1 else "weak")
    assert bench.shard_rank_for(a, 0, g) == r
    assert cfg.block_bytes(g) == cfg.block_bytes(1) // G


@pytest.mark.parametrize("kw,world", [(dict(workload="c3", head_shards=2, shard_rank=0), 1),
                                      (dict(workload="c4", head_shards=3, shard_rank=0), 1),
                                      (dict(workload="c4", head_shards=2, shard_rank=0), 2),
                                      (dict(workload="c4", head_shards=2, shard_rank=2), 1)])
def test_head_shards_rejects(kw, world):
    with pytest.raises(SystemExit):
        a = SimpleNamespace(**kw)
        cfg, g, _ = bench.workload_for(a, world)
        bench.shard_rank_for(a, 0, g)


def test_timeline_summary():
    spans = [(0, "memcpy_h2d", 0.0, 2.0, 10), (0, "memcpy_d2h", 0.1, 2.5, 10), (0, "offload_kernel", 0.01, 0.05, 10),
             (1, "memcpy_h2d", 0.0, 1.0, 10), (1, "memcpy_d2h", 0.3, 1.5, 10)]
    s = bench.timeline_summary(spans)
    assert s["steps"] == 2
    assert s["step_span_ms"] == pytest.approx((2.5 + 1.5) / 2)
    assert s["d2h_start_ms"] == pytest.approx(0.2)
    assert s["tail_after_last_dma_ms"] == pytest.approx(0.0)
    assert bench.timeline_summary([]) is None


def test_ncu_traffic_lookup():
    kd = {"bound": "hbm", "bytes_per_launch": 1000.0}
    t = bench.ncu_traffic("c2", "gather", kd)
    if os.path.exists(os.path.join(ROOT, "profiles", "r01_traffic_c2.json")):
        assert 0.5 < t["traffic_source"]["dram_over_algorithmic"] < 1.5
        assert t["traffic"] == pytest.approx(1000.0 * t["traffic_source"]["dram_over_algorithmic"])
        assert abs(t["traffic_source"]["dram_read_over_algorithmic_read"] - 1.0) < 0.01
    assert bench.ncu_traffic("c2", "gather", {"bound": "host_link", "bytes_per_launch": 1.0}) == {}
    assert bench.ncu_traffic("nosuch", "gather", kd) == {}


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["metric"] == bench.METRIC and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"


def test_choose_retire_lag():
    """bench.py's retire-loop choice: retire-each at the deepest lag <= 4 that fits (1 if none: refused cycles take
    the retire ladder); an explicit --retire / --retire-lag wins."""
    from bench import choose_retire
    # C2-like: 11.8 k free slots, 19 k free blocks, cycles of ~330 blocks -> lag 4
    assert choose_retire("auto", 0, 11796, 19000, 330, 330) == ("each", 4)
    # host buffer for exactly 1 + 2 cycles (x1.1): lag 2
    assert choose_retire("auto", 0, int(1.1 * 3 * 1000) + 1, 10 ** 6, 1000, 1000) == ("each", 2)
    # not even one extra cycle: still retire-each at lag 1 (refused cycles take the retire ladder)
    assert choose_retire("auto", 0, 1500, 10 ** 6, 1000, 1000) == ("each", 1)
    # free blocks bind: up_max + 2 off_max (x1.1) = 3300 > 3000
    assert choose_retire("auto", 0, 10 ** 6, 3000, 1000, 1000) == ("each", 1)
    assert choose_retire("each", 2, 0, 0, 1000, 1000) == ("each", 2)
    assert choose_retire("sync", 0, 10 ** 6, 10 ** 6, 10, 10) == ("sync", 4)


def test_host_enqueue_summary():
    """Per-cycle host enqueue cost from trace records: grouped by call, max enqueue lag, blocks summed."""
    recs = [{"t_call_ns": 1000, "t_enqueued_ns": 41000, "blocks": 10},
            {"t_call_ns": 1000, "t_enqueued_ns": 61000, "blocks": 30},
            {"t_call_ns": 9000, "t_enqueued_ns": 29000, "blocks": 60}]
    s = bench.host_enqueue_summary(recs, step_ms=1.0)
    assert s["cycles"] == 2 and s["p50_us"] == 60.0 and abs(s["mean_us"] - 40.0) < 1e-9
    assert abs(s["ns_per_block"] - 800.0) < 1e-9 and abs(s["share_of_step"] - 0.04) < 1e-12
    assert bench.host_enqueue_summary([], 1.0) is None


def test_per_gpu_summary():
    """Per-rank GB/s = own bytes / own device ms; spread = (max - min) / mean."""
    rows = [[10.0, 11.0, 1e9, 1000, 0.1], [20.0, 21.0, 1e9, 1000, 0.1]]
    s = bench.per_gpu_summary(rows)
    assert [round(x, 6) for x in s["gbs"]] == [100.0, 50.0]
    assert [round(x) for x in s["blocks_per_s"]] == [100000, 50000]
    assert abs(s["spread"] - 50.0 / 75.0) < 1e-12 and s["min_gbs"] == 50.0


@pytest.mark.parametrize("world,name,G,scaling", [(1, "c3", 1, "weak"), (2, "c4", 2, "strong"),
                                                  (8, "c4", 8, "strong")])
def test_default_workload_per_world(world, name, G, scaling):
    """No --workload: C3 (largest single-GPU config) at N = 1, the head-sharded C4 with G = N at N > 1."""
    cfg, g, sc = bench.workload_for(SimpleNamespace(workload=None), world)
    assert (cfg.name, g, sc) == (name, G, scaling)


def test_launch_command_is_loopback_torchrun():
    cmd = bench.launch_command(["--gpus", "4", "--steps", "3"], 4, 29555)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd and "--master-port=29555" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-3:] == ["--gpus", "4", "--steps", "3"][-3:]


def test_self_launch_two_ranks_dry_run():
    """`bench.py --gpus 2` outside torchrun re-launches itself as two ranks (gloo in --dry-run): rank 0 prints one
    line with n_gpus 2, the C4 head split G = 2 (shard ranks 0 and 1), two per-GPU rows and a cpu_baseline."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run",
                          "--cpu-seconds", "1"], capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["head_shards"] == 2 and d["config"]["shard_ranks"] == [0, 1]
    assert d["config"]["workload"].startswith("c4")
    assert len(d["per_gpu"]["gbs"]) == 2
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] > 0


@pytest.mark.parametrize("name,G", [("c2", 1), ("c3", 1), ("c4", 1), ("c4", 2), ("c4", 8), ("c5", 8)])
def test_oracle_host_sample_fits(name, G):
    """The cpu_baseline / reference-arm host sample of every config fits its scaled pool (no refused op), keeps the
    rank's block-shard size and stays within ~1.5 GB of pool bytes."""
    from workloads.configs import CONFIGS
    cfg = CONFIGS[name]
    small = bench.oracle_scaled(cfg, G)
    assert small.block_bytes(G) == cfg.block_bytes(G)
    assert small.N * small.block_bytes(G) <= (3 << 29) + small.block_bytes(G) or small.N == 256
    from workloads.scripts import agent_sizes
    import numpy as np
    sizes = agent_sizes(small, np.random.default_rng(small.seed))
    assert sum(sizes) <= 0.6 * small.N + len(sizes)


def test_step_link_bound():
    """Per drained step: the smaller direction at half the bidirectional peak, the excess at the larger direction's
    unidirectional peak."""
    link = {"h2d_gbs": 50.0, "d2h_gbs": 40.0, "bidir_gbs": 80.0}
    assert bench.step_link_bound_s(40e9, 40e9, link) == pytest.approx(1.0)
    assert bench.step_link_bound_s(100e9, 0.0, link) == pytest.approx(2.0)          # H2D alone at 50
    assert bench.step_link_bound_s(0.0, 80e9, link) == pytest.approx(2.0)           # D2H alone at 40
    assert bench.step_link_bound_s(90e9, 40e9, link) == pytest.approx(1.0 + 1.0)    # 40 both ways + 50 H2D


def test_offload_size_sweep_logic_on_metadata_pool():
    """bench.py's C5 sweep (both directions per tc_cycle, roles swapping each rep) drives a metadata-only pool to
    completion: one row per size, and afterwards no live handle, no pending block and both sweep agents freed."""
    import paper_2510_18586_b200 as tcb
    from workloads.configs import CONFIGS
    cfg = CONFIGS["c5"]
    p = tcb.Pool(cfg.L, cfg.H, cfg.D, cfg.T, cfg.dtype, 256, device=-1, shard_world=cfg.G, host_slots=64,
                 max_agents=1024, max_blocks_per_agent=64)
    before = p.stats()
    out = bench.offload_size_sweep(p, cfg, p.block_bytes, sizes=(1, 2, 8), reps=2)
    assert [r["blocks"] for r in out["rows"]] == [1, 2, 8]
    s = p.stats()
    assert s["live_handles"] == 0 and s["pending"] == 0 and s["alloc"] == before["alloc"]
    assert s["free"] == before["free"] and s["host_free"] == before["host_free"]
