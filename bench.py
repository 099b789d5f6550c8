#!/usr/bin/env python3
"""Layout cost-evals/sec of the B200 hetsched fitness path (BASELINE.json metric).

Workload (BASELINE config 2, the paper setting): N=64 devices, D_PP=8 x
D_DP=8, GPT3-XL volumes (c_pp=1,073,741,824 B, c_dp=301,989,888 B), case-5
world-wide matrix from the reference generator (seed 0).  A step is one
pass of the fitness kernel over one population of P uniformly random
balanced layouts per GPU.  Multi-GPU: the population is sharded (weak
scaling, no data-path collective); time is the max over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
# rank 0 prints exactly one JSON line on stdout.  The ours arm moves fd 1 to
# stderr for its whole run (JSON_FD keeps the real stdout), so NCCL's banner
# and its communicator-init INFO lines (printed on stdout) land on stderr; a
# caller's NCCL_DEBUG / NCCL_DEBUG_SUBSYS win
os.environ.setdefault("NCCL_DEBUG", "INFO")
os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
JSON_FD = 1

METRIC = "layout cost-evals/sec (N=64, D_PP=8xD_DP=8)"
WORKLOAD = ("paper setting: 64 devices, D_PP=8 x D_DP=8, GPT3-XL tasklets "
            "(c_pp=1073741824 B, c_dp=301989888 B), case 5 world_geo matrix (seed 0)")
# algorithmic on-chip work per evaluation at 8x8:
# 2,240 fp64 table gathers (17,920 B) + Held-Karp 3,584 reads + 1,016 writes (36,800 B)
SMEM_BYTES_PER_EVAL = 17_920 + 36_800
HBM_BYTES_PER_EVAL = 64 * 2 + 3 * 8
SMEM_BYTES_PER_CLK_SM = 128


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--population", type=int, default=1 << 20, help="layouts per GPU per step")
    ap.add_argument("--case", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="bounded CPU baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ga", action="store_true", help="skip the GA time-to-converge / island legs")
    ap.add_argument("--islands", type=int, default=0, help="GA islands per GPU (default: 8 per SM, one per warp)")
    ap.add_argument("--island-gens", type=int, default=100)
    ap.add_argument("--no-sweep", action="store_true",
                    help="skip the BASELINE config 3-5 legs (scenario / population sweep, 512 and 1024 devices)")
    return ap.parse_args()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:  # sampler is live before timing starts
                time.sleep(0.02)
            self.skip = len(self.lines)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        for ln in self.lines[getattr(self, "skip", 0):] or self.lines[-1:]:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for _, _, flags in rows for i, f in enumerate(flags) if f.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


def stdout_to_stderr():
    """fd-level: from here on anything written to fd 1 (NCCL's printf
    logging included) goes to stderr; emit() writes to the saved stdout."""
    global JSON_FD
    sys.stdout.flush()
    JSON_FD = os.dup(1)
    os.dup2(2, 1)


def emit(line: dict) -> None:
    os.write(JSON_FD, (json.dumps(line) + "\n").encode())


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def instance():
    from paper_2206_01288_b200 import PAPER_WORKLOAD, scenario_case
    return scenario_case(ARGS.case).graph(), PAPER_WORKLOAD


def ga_instances():
    """The GA time-to-converge anchors of tests/golden/evolve_1000.json:
    the five paper scenarios at 8x8 and BASELINE config 1 (8 devices, 2x4,
    case-1 links on two nodes of four, GPT3-XL at d_pp=2)."""
    from paper_2206_01288_b200 import PAPER_WORKLOAD, scenario_case
    from paper_2206_01288_b200.netmodel import scenario_from_ms_gbps
    from paper_2206_01288_b200.workload import WorkloadSpec
    out = {f"case{c}": (scenario_case(c).graph(), PAPER_WORKLOAD) for c in range(1, 6)}
    out["config1"] = (scenario_from_ms_gbps([(4, 0.1, 100), (4, 0.1, 100)], 0.25, 25, 0).graph(),
                      WorkloadSpec(2, 4, 2_147_483_648, 1_207_959_552))
    return out


def cpu_oracle_rate(g, w, seconds: float, threads: int):
    """Oracle evals/s on a bounded sample (test infrastructure, CPU baseline only)."""
    from oracle import oracle as O
    orc = O.Oracle.of(g, w)
    rng = np.random.default_rng(12345)
    probe = np.sort(rng.permuted(np.tile(np.arange(64, dtype=np.int16), (400, 1)), axis=1).reshape(-1, 8, 8), axis=2)
    t0 = time.perf_counter()
    orc.comm_cost_batch(probe, threads=1)
    per_core = len(probe) / (time.perf_counter() - t0)
    count = int(max(threads * 200, per_core * threads * seconds))
    parts = np.sort(rng.permuted(np.tile(np.arange(64, dtype=np.int16), (count, 1)), axis=1).reshape(-1, 8, 8),
                    axis=2)
    t0 = time.perf_counter()
    orc.comm_cost_batch(parts, threads=threads)
    dt = time.perf_counter() - t0
    return count / dt, count, dt


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip() + f" x {os.cpu_count()} logical CPUs"
    except OSError:
        pass
    return f"unknown x {os.cpu_count()}"


def run_reference():
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    g, w = instance()
    threads = O.cpu_count()
    rates = []
    per_step = max(ARGS.cpu_seconds / max(ARGS.steps, 1), 1.0)
    for i in range(ARGS.warmup + ARGS.steps):
        r, count, dt = cpu_oracle_rate(g, w, per_step if i >= ARGS.warmup else 0.3, threads)
        if i >= ARGS.warmup:
            rates.append((count, dt))
    total = sum(c for c, _ in rates)
    secs = sum(d for _, d in rates)
    value = total / secs
    sample = f"{total} random 8x8 case-{ARGS.case} layouts over {ARGS.steps} steps, C oracle port of comm_cost"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": max(world, ARGS.gpus),
        "steps": ARGS.steps, "warmup": ARGS.warmup, "ms_per_step": 1000 * secs / ARGS.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic random balanced layouts", "config": {"workload": WORKLOAD},
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": threads, "kind": "port", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def run_ours():
    import torch
    import torch.distributed as dist
    from paper_2206_01288_b200 import _native as N
    from paper_2206_01288_b200.costmodel import comm_cost_batch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        print(f"[bench rank {rank}] NCCL_DEBUG={os.environ.get('NCCL_DEBUG')} "
              f"NCCL_DEBUG_SUBSYS={os.environ.get('NCCL_DEBUG_SUBSYS')}", file=sys.stderr, flush=True)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        dist.barrier()
    dev = torch.device(f"cuda:{local}")
    g, w = instance()
    inst = N.instance_for(g, w, local)
    L = N.lib()
    P = ARGS.population
    nbuf = 4  # 4 x P x 128 B rotating inputs: 512 MiB at P=2^20 (> 126 MB L2)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1000 + rank)
    pops = []
    for _ in range(nbuf):
        keys = torch.rand((P, 64), device=dev, generator=gen)
        perm = torch.argsort(keys, dim=1).to(torch.int16).view(P, 8, 8)
        pops.append(torch.sort(perm, dim=2).values.contiguous())
    outs = [torch.empty(P, dtype=torch.float64, device=dev) for _ in range(3)]
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream

    def step(i):
        N.check(L.hs_eval_batch(inst.handle, pops[i % nbuf].data_ptr(), P, outs[0].data_ptr(), outs[1].data_ptr(),
                                outs[2].data_ptr(), None, None, bad.data_ptr(), sp), "hs_eval_batch")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for i in range(ARGS.warmup):
        step(i)
    barrier()
    assert int(bad.item()) == 0
    # spot parity of the last warm-up output (full parity lives in tests/)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(ARGS.steps + 1)]
    with ClockSampler(local) as clocks:
        barrier()
        ev[0].record(stream)
        for i in range(ARGS.steps):
            step(i)
            ev[i + 1].record(stream)
        barrier()
    launch_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(ARGS.steps)]
    t_ms = ev[0].elapsed_time(ev[-1])
    tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_ms = float(tt.item())
    value = P * ARGS.steps * world / (t_ms / 1000.0)

    # the same pricing with the stage order reconstructed (comm_cost's
    # PathResult; the compact-table warp kernel), reported beside the headline
    order_out = torch.empty((P, 8), dtype=torch.int8, device=dev)
    pg_out = torch.empty((P, 8), dtype=torch.float64, device=dev)

    def order_step(i):
        N.check(L.hs_eval_batch(inst.handle, pops[i % nbuf].data_ptr(), P, outs[0].data_ptr(), outs[1].data_ptr(),
                                outs[2].data_ptr(), pg_out.data_ptr(), order_out.data_ptr(), bad.data_ptr(), sp),
                "hs_eval_batch(order)")

    order_step(0)
    barrier()
    oa, ob = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    oa.record(stream)
    for i in range(3):
        order_step(i)
    ob.record(stream)
    barrier()
    order_rate = P * 3 / (oa.elapsed_time(ob) / 1000.0)

    # e2e through the C-ABI host-buffer entry point: pinned host layouts in,
    # totals/datap/pipelinep out, H2D/D2H inside the timed region.
    host_pop = [pops[i].cpu().pin_memory().numpy() for i in range(2)]
    host_out = [torch.empty(P, dtype=torch.float64).pin_memory().numpy() for _ in range(3)]
    inv = np.zeros(1, dtype=np.int32)

    def e2e_step(i):
        N.check(L.hs_eval_batch_host(inst.handle, host_pop[i % 2].ctypes.data, P, host_out[0].ctypes.data,
                                     host_out[1].ctypes.data, host_out[2].ctypes.data, None, None, inv.ctypes.data),
                "hs_eval_batch_host")

    for i in range(ARGS.warmup):
        e2e_step(i)
    barrier()
    t0 = time.perf_counter()
    for i in range(ARGS.steps):
        e2e_step(i)
    barrier()
    e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_value = P * ARGS.steps * world / float(e2e_s.item())
    # public-API check: same numbers through comm_cost_batch on the host array
    last = (ARGS.steps - 1) % 2
    api = comm_cost_batch(g, host_pop[last][:4096], w)
    assert np.array_equal(api["total"], host_out[0][:4096]), "public API disagrees with the C-ABI host path"

    csum = clocks.summary()
    sm_mhz = csum["sm_mhz"] or 1965.0
    kern_ms = sum(launch_ms) / len(launch_ms)
    achieved = SMEM_BYTES_PER_EVAL * P / (kern_ms / 1000.0) / 1e9
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    arch_peak = SMEM_BYTES_PER_CLK_SM * sms * sm_mhz * 1e6 / 1e9
    # measured denominator: conflict-free LDS.128 stream on every SM (hs_probe.cu)
    measured_peak = N.smem_bandwidth(local) / 1e9
    peak = measured_peak
    traffic, traffic_src, smem_wf, pipes = None, None, None, None
    tp = ROOT / "profiles" / "eval_traffic.json"
    if tp.exists():  # ncu --set full capture of this kernel (scripts/gpu_ncu.sh)
        tj = json.loads(tp.read_text())
        traffic = tj["dram_bytes_per_launch"] * P / tj["population"]
        smem_wf = tj["smem_wavefronts_per_launch"] * 128 * P / tj["population"]
        if "alu_pipe_pct" in tj:  # the pipe that actually binds this issue-bound kernel
            pipes = {"bound": "alu pipe (instruction issue)", "alu_pipe_frac": tj["alu_pipe_pct"] / 100.0,
                     "issue_slots_frac": tj["issue_active_pct"] / 100.0, "ipc": tj["ipc"],
                     "smem_pipe_frac": tj["smem_pipe_pct"] / 100.0, "source": tj["source"]}
        traffic_src = (f"{tj['source']}: dram__bytes_read.sum + dram__bytes_write.sum at P={tj['population']}"
                       + ("" if tj["population"] == P else f", scaled to P={P}")
                       + f"; algorithmic HBM bytes per launch = {HBM_BYTES_PER_EVAL * P}")
    line = {
        "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world, "steps": ARGS.steps,
        "warmup": ARGS.warmup, "ms_per_step": t_ms / ARGS.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: uniformly random balanced layouts (device RNG), reference case-5 generator matrix",
        "config": {"workload": WORKLOAD, "population_per_gpu": P,
                   "l2": f"{nbuf} rotating input populations of {P * 128 / 2**20:.0f} MiB (> 126 MB L2)",
                   "parallelism": f"population sharded over {world} GPU(s), no data-path collective"},
        "roofline": {"bound": "smem", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_source": traffic_src,
                     "smem_wavefront_bytes": smem_wf, "pipes": pipes,
                     "per_eval_bytes": SMEM_BYTES_PER_EVAL, "kernel": "hs::eval8_kernel", "kernel_ms": kern_ms,
                     "peak_source": "measured in this run: hs_probe_smem_bandwidth (conflict-free 16-byte LDS on "
                                    f"all {sms} SMs; MEASURED_PEAKS.json has no shared-memory figure); architectural "
                                    f"128 B/clk/SM at the sampled {sm_mhz:.0f} MHz = {arch_peak:.0f} GB/s",
                     "arch_peak": arch_peak,
                     "hbm_achieved_gbs": HBM_BYTES_PER_EVAL * P / (kern_ms / 1000.0) / 1e9},
        "e2e": {"value": e2e_value, "unit": "evals/s", "h2d_bytes_per_step": P * 128, "d2h_bytes_per_step": P * 24,
                "path": "hs_eval_batch_host (C-ABI, pinned host buffers)"},
        "with_stage_order": {"value": order_rate, "unit": "evals/s",
                             "what": "same workload with per_group + pipeline order (comm_cost's full CostBreakdown; "
                                     "eval_warp_kernel, compact Held-Karp table), device-resident, 3 launches"},
        "gpu_launches": ARGS.steps,
        "clocks": {"sm_mhz": csum["sm_mhz"], "sm_max_mhz": csum["sm_max_mhz"], "reasons": csum["reasons"]},
    }
    if not ARGS.no_ga:
        line["ga"] = ga_legs(g, w, rank, world, local, barrier, dist)
    if not ARGS.no_sweep:
        line["config4_island_model"] = config4_island_leg(rank, world, local, barrier, dist)
    if not ARGS.no_sweep and world == 1:
        line["other_configs"] = sweep_legs(local)
    if rank == 0 and world == 1 and not ARGS.no_cpu_baseline:
        from oracle import oracle as O
        threads = O.cpu_count()
        rate, count, dt = cpu_oracle_rate(g, w, ARGS.cpu_seconds, threads)
        rate1, count1, dt1 = cpu_oracle_rate(g, w, min(3.0, ARGS.cpu_seconds), 1)
        line["cpu_baseline"] = {"value": rate, "unit": "evals/s", "cores": threads, "kind": "port",
                                "sample": f"{count} random 8x8 case-{ARGS.case} layouts in {dt:.1f} s "
                                          f"(C oracle restatement of comm_cost, {threads} threads)",
                                "one_core": {"value": rate1, "sample": f"{count1} layouts in {dt1:.1f} s, 1 thread"},
                                "cpu_model": cpu_model(),
                                "python_reference_per_core_build_container": "179-292 evals/s (SURVEY.md §8(d))"}
        if "ga" in line:
            # the same 1000-generation evolve through the C oracle port on one
            # host core (the GA is one sequential chain of generations)
            o = O.Oracle.of(g, w)
            t0 = time.perf_counter()
            ref = o.evolve(64, 1000, "ours", seed=0)
            t_cpu = time.perf_counter() - t0
            line["ga"]["time_to_converge"]["cpu_baseline"] = {
                "seconds": t_cpu, "cores": 1, "kind": "port",
                "same_best_total": bool(float(ref["total"]) == line["ga"]["time_to_converge"]["best_total_s"])}
    if rank == 0:
        emit(line)
    if world > 1:
        dist.destroy_process_group()


def ga_legs(g, w, rank, world, local, barrier, dist):
    """GA time-to-converge (the reference's 1000-generation case-5 run, one
    seed, latency) and island throughput (one GA per SM, elite migration over
    NCCL every 25 generations)."""
    import torch
    from paper_2206_01288_b200 import scheduler as S

    out = {}
    gold_path = ROOT / "tests" / "golden" / "evolve_1000.json"
    gold = {r["inst"]: r for r in json.loads(gold_path.read_text())["runs"]} if gold_path.exists() else {}
    per_case = {}
    for name, (gi, wi) in ga_instances().items():
        cfg = S.ScheduleConfig(pop_size=64, generations=1000, local_search="ours", seed=0)
        S.evolve(gi, wi, S.ScheduleConfig(pop_size=64, generations=2, local_search="ours", seed=0))  # warm-up
        barrier()
        t0 = time.perf_counter()
        res = S.evolve(gi, wi, cfg)
        torch.cuda.synchronize()
        t_ga = time.perf_counter() - t0
        best = [b for _, b, _ in res.trace]
        conv = max([0] + [i for i in range(1, len(best)) if best[i] < best[i - 1]])
        run = gold.get(name)
        ident = None
        if run is not None:
            ident = (res.evaluations == run["evaluations"]
                     and best == [float.fromhex(x) for x in run["trace_best"]]
                     and [m for _, _, m in res.trace] == [float.fromhex(x) for x in run["trace_mean"]]
                     and [list(x) for x in res.best_partition.key()] == run["partition"])
        per_case[name] = {"seconds": t_ga, "last_improving_generation": conv,
                          "seconds_to_last_improvement": t_ga * (conv + 1) / len(best),
                          "best_total_s": res.best_cost.total, "evaluations": res.evaluations,
                          "identical_to_reference": ident,
                          "reference_python_seconds_build_container": run["wall_s"] if run else None}
    head = per_case[f"case{ARGS.case}"]
    out["time_to_converge"] = {
        "workload": f"evolve(pop=64, generations=1000, local_search='ours', seed=0), case {ARGS.case}",
        "seconds": head["seconds"], "generations": 1000,
        "last_improving_generation": head["last_improving_generation"],
        "best_total_s": head["best_total_s"], "evaluations": head["evaluations"],
        "identical_to_reference": head["identical_to_reference"],
        "reference_python_seconds_build_container": head["reference_python_seconds_build_container"],
        "per_case": per_case,
        "timed": "wall clock around evolve() incl. the final result download, after a 2-generation warm-up",
    }
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    I = ARGS.islands or sms * 8
    icfg = S.ScheduleConfig(pop_size=64, generations=ARGS.island_gens, local_search="ours", seed=1)
    # the island sessions (device buffers, seeding) are built untimed: the
    # timed region is the GA itself -- epochs of 25 generations, elite export,
    # the NCCL all-gather, import, and the final result download
    rank_off = (dist.get_rank() if world > 1 else 0) * I
    src = S.migration_sources(dist.get_rank() if world > 1 else 0, world, I)
    runs = []
    for rep in range(4):
        sess = S.GASession(g, w, icfg, S.island_seeds(icfg.seed, I, offset=rank_off), mode="warp")
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        gen = 0
        while gen < icfg.generations:
            gen = min(icfg.generations, gen + 25)
            sess.run(gen)
            if gen < icfg.generations:
                gr, co = sess.export_elites(2)
                all_gr, all_co = S.gather_elites(gr, co)
                sess.import_elites(all_gr, all_co, src)
        sess.results([icfg.seed] * I)
        torch.cuda.synchronize()
        barrier()
        tt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=f"cuda:{local}")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        if rep:  # the first repetition is a warm-up
            runs.append(float(tt.item()))
        del sess
    tt = torch.tensor([statistics.median(runs)], dtype=torch.float64)
    t_isl = float(tt.item())
    out["islands"] = {"islands": I * world, "generations": ARGS.island_gens, "seconds": t_isl,
                      "runs_s": runs,
                      "island_generations_per_s": I * world * ARGS.island_gens / t_isl,
                      "mode": "one warp per island (8 per CTA), case-5, pop 64, ours",
                      "migration": "2 elites every 25 generations, global ring, NCCL all-gather",
                      "timed": "median of 3 runs after a warm-up; session allocation / seeding outside"}
    return out


def config4_island_leg(rank, world, local, barrier, dist):
    """BASELINE config 4's island model: 512 devices, d_pp = 16 x d_dp = 32,
    one CTA island per SM on every GPU (generations batch-priced by the
    stage + cluster Held-Karp kernels), one elite per island migrating
    around the global ring over NCCL every 2 generations; time = max over
    ranks, evaluations from the islands' own counters."""
    import torch
    from paper_2206_01288_b200 import scheduler as S
    from paper_2206_01288_b200.netmodel import config4_scenario
    from paper_2206_01288_b200.workload import WorkloadSpec

    g4 = config4_scenario().graph()
    w4 = WorkloadSpec(16, 32, 268_435_456, 201_326_592)
    icfg = S.ScheduleConfig(pop_size=16, generations=6, local_search="ours", seed=5)
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    r = dist.get_rank() if world > 1 else 0
    src = S.migration_sources(r, world, sms)
    sess = S.GASession(g4, w4, icfg, S.island_seeds(icfg.seed, sms, offset=r * sms))
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    gen = 0
    while gen < icfg.generations:
        gen = min(icfg.generations, gen + 2)
        sess.run(gen)
        if gen < icfg.generations:
            gr, co = sess.export_elites(1)
            all_gr, all_co = S.gather_elites(gr, co)
            sess.import_elites(all_gr, all_co, src)
    res = sess.results()
    torch.cuda.synchronize()
    barrier()
    tt = torch.tensor([time.perf_counter() - t0, float(sum(x.evaluations for x in res))], dtype=torch.float64,
                      device=f"cuda:{local}")
    if world > 1:
        t_max = tt[:1].clone()
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
        dist.all_reduce(tt[1:], op=dist.ReduceOp.SUM)
        tt[0] = t_max[0]
    t_isl, evals = float(tt[0].item()), float(tt[1].item())
    return {"islands": sms * world, "gpus": world, "generations": icfg.generations, "pop_size": icfg.pop_size,
            "seconds": t_isl, "island_generations_per_s": sms * world * icfg.generations / t_isl,
            "evals_per_s": evals / t_isl,
            "migration": "1 elite per island every 2 generations, global ring, NCCL all-gather",
            "what": "one CTA island per SM per GPU, 512 devices 16x32, ours, incl. init pricing, time max over ranks"}


def sweep_legs(local):
    """Device-resident evals/s on the other BASELINE configs (reported beside
    the headline, not as bench lines): config 3 = the five paper scenarios
    at N=64 8x8 over a population sweep; config 4 = 512 devices, 16x32
    (CTA Held-Karp over 2^16 subsets); config 5 = 1024 devices, 16x64 exact
    and 32x32 heuristic pricing, plus one gains-only refinement pass per
    layout (_pass_ours sweep / chains and _pass_kl) on 32x32 groups."""
    import torch
    from paper_2206_01288_b200 import PAPER_WORKLOAD, scenario_case
    from paper_2206_01288_b200 import _native as N
    from paper_2206_01288_b200 import scheduler as S
    from paper_2206_01288_b200.netmodel import config4_scenario, random_graph
    from paper_2206_01288_b200.workload import WorkloadSpec

    dev = torch.device(f"cuda:{local}")
    gen = torch.Generator(device=dev)
    gen.manual_seed(77)

    def layouts(P, n, k, m):
        perm = torch.argsort(torch.rand((P, n), device=dev, generator=gen), dim=1).to(torch.int16).view(P, k, m)
        return torch.sort(perm, dim=2).values.contiguous()

    def rate(g, w, P, reps=3, heuristic=False):
        """device-resident evals/s through hs_eval_batch_ex (CUDA events)"""
        x = layouts(P, g.lat.shape[0], w.d_pp, w.d_dp)
        inst = N.instance_for(g, w, local)
        o = [torch.empty(P, dtype=torch.float64, device=dev) for _ in range(3)]
        pg = torch.empty((P, w.d_pp), dtype=torch.float64, device=dev)
        od = torch.empty((P, w.d_pp), dtype=torch.int8, device=dev)
        sp = torch.cuda.current_stream(dev).cuda_stream

        def call():
            N.check(N.lib().hs_eval_batch_ex(inst.handle, x.data_ptr(), P, o[0].data_ptr(), o[1].data_ptr(),
                                             o[2].data_ptr(), pg.data_ptr() if heuristic else None,
                                             od.data_ptr() if heuristic else None, None, int(heuristic), sp),
                    "hs_eval_batch_ex")
        call()
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            call()
        b.record()
        torch.cuda.synchronize(dev)
        return P * reps / (a.elapsed_time(b) / 1000.0)

    out = {"config3_scenarios_evals_per_s": {}}
    for c in range(1, 6):
        g = scenario_case(c).graph()
        out["config3_scenarios_evals_per_s"][f"case{c}"] = {
            str(P): rate(g, PAPER_WORKLOAD, P) for P in (1 << 10, 1 << 14, 1 << 18, 1 << 20)}
    g4 = config4_scenario().graph()
    w4 = WorkloadSpec(16, 32, 268_435_456, 201_326_592)
    out["config4_512dev_16x32_evals_per_s"] = rate(g4, w4, 16384, reps=2)
    g5 = random_graph(0, 1024)
    out["config5_1024dev_16x64_evals_per_s"] = rate(g5, WorkloadSpec(16, 64, 1 << 30, 3 << 26), 1024, reps=2)
    out["config5_1024dev_32x32_heuristic_evals_per_s"] = rate(g5, WorkloadSpec(32, 32, 1 << 30, 3 << 26), 4096,
                                                              reps=2, heuristic=True)
    w5 = WorkloadSpec(32, 32, 1 << 30, 3 << 26)
    inst = N.instance_for(g5, w5, local)
    B = 1024
    parts = np.ascontiguousarray(layouts(B, 1024, 32, 32).cpu().numpy())
    res = np.empty_like(parts)
    ch = np.zeros(B, dtype=np.int32)
    passes = {}
    for name, kind, phase in (("ours_sweep", 0, 0), ("ours_chains", 0, 1), ("kl", 1, 0)):
        ts = []
        for rep in range(4):  # a warm-up call, then the median of three (host buffers, copies included)
            st = S._states([np.random.default_rng(i) for i in range(B)])
            t0 = time.perf_counter()
            N.check(N.lib().hs_refine_pass(inst.handle, kind, phase, B, parts.ctypes.data, st, res.ctypes.data,
                                           ch.ctypes.data), "hs_refine_pass")
            ts.append(time.perf_counter() - t0)
        passes[name] = B / float(np.median(ts[1:]))
    out["config5_1024dev_32x32_gains_only_passes_per_s"] = passes
    return out


def self_launch(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: re-run this script as N ranks
    (one process per GPU, NCCL) through torch.distributed.run on this node;
    rank 0's JSON line is this process's stdout."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"),
               NCCL_DEBUG=os.environ.get("NCCL_DEBUG", "INFO"),
               NCCL_DEBUG_SUBSYS=os.environ.get("NCCL_DEBUG_SUBSYS", "INIT"))
    return subprocess.call(cmd, env=env)


if __name__ == "__main__":
    ARGS = parse()
    if ARGS.gpus > 1 and "WORLD_SIZE" not in os.environ and ARGS.impl == "ours":
        sys.exit(self_launch(ARGS.gpus))
    if ARGS.impl == "reference":
        run_reference()
    else:
        stdout_to_stderr()
        run_ours()
