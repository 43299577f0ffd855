"""Benchmark: the hpc_benchmark weak-scaling network (BASELINE.json configs[2],
SURVEY.md §8 C3) on N B200s -- construction throughput (synapses/s, the
headline `value`) and the propagation real-time factor.

One "step" is one complete construction of the network through the public
façade: create neurons (per-gid initial V), attach the Poisson drive, two
distributed fixed in-degree projections (E then I), prepare (stable sort by
source, first-index, image maps, rosters, routes).  Per GPU: 1e5 neurons
(80,000 E + 20,000 I), K = 11,250 (9,000 + 2,250) -> 1.125e9 synapses.
Collective spike exchange (group 0 over all ranks) when N > 1.

Launch: python bench.py [--gpus N --steps K --warmup W]  (N > 1 under
torchrun, one rank per GPU, NCCL).  --impl reference times the unmodified
reference package (baseline/_ref: Python + its Cython kernels; the CPU
oracle port of oracle/ when it is not installed) on a bounded sample on
rank 0.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_PEAK_FALLBACK = 6650.0
BYTES_PER_SYN = 20.0  # BASELINE.md §4 / SURVEY §8(d): generation + sort, constant syn


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--neurons", type=int, default=100_000)
    ap.add_argument("--k-exc", type=int, default=9_000)
    ap.add_argument("--k-inh", type=int, default=2_250)
    ap.add_argument("--model-ms", type=float, default=100.0)
    ap.add_argument("--prop-warmup-ms", type=float, default=20.0)
    ap.add_argument("--seed", type=int, default=12345)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: --neurons is the whole network, split over the GPUs")
    ap.add_argument("--cpu-sample-neurons", type=int, default=5_000)
    ap.add_argument("--cpu-sample-k-scale", type=float, default=0.1)
    ap.add_argument("--c4-areas", type=int, default=0,
                    help="C4 areas (default 4 per GPU: the per-GPU load of the 32-area model on 8 GPUs)")
    ap.add_argument("--c4-neurons", type=int, default=129_063)
    ap.add_argument("--c4-k", default="3600,900,44", help="k_intra_exc,k_intra_inh,k_inter (SURVEY §8 C4)")
    ap.add_argument("--workload", default="c3", choices=["c2", "c3", "c4", "c5"],
                    help="c3: the headline (hpc_benchmark weak scaling); c5: construction-only sweep")
    ap.add_argument("--c5-points", default="1e8,3e8,1e9,3e9,1e10")
    ap.add_argument("--c5-rules", default="fixed_indegree,fixed_total")
    return ap.parse_args()


TRAFFIC = {"fused": "profiles/r2/traffic.json", "general": "profiles/r1f/traffic.json"}
KERNELS = {"fused": "pass A (smx_fused_gen: generation + low-digit ranking) + pass B (smx_fused_sort)",
           "general": "generation (smx_gen_draw) + stable sort (smx_sort_records)"}


def traffic_per_synapse(path_kind: str):
    """DRAM bytes (read + write) per synapse of the generation + sort kernels
    of the store path the run took, from the committed ncu capture of one C3
    construction on that path (tools/profile_summary.py)."""
    rel = TRAFFIC.get(path_kind)
    if rel is None:
        return None, None
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), rel)) as f:
            d = json.load(f)
        if d.get("store_path", "general") != path_kind:
            return None, None
        return float(d["bytes_per_synapse"]), rel
    except (OSError, KeyError, ValueError):
        return None, None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return HBM_PEAK_FALLBACK, "fallback"


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        util = [float(r[6]) for r in self.rows if len(r) > 6 and r[6].replace(".", "").isdigit()]
        loaded = [s for s, u in zip(sm, util) if u > 0] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(loaded)) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_info():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def host_info() -> dict:
    model = ""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def reference_package():
    """The unmodified reference (spikemesh, Python + its Cython kernels)
    installed under baseline/_ref; None when it is not there."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(path) and path not in sys.path:
        sys.path.insert(0, path)
    try:
        import spikemesh
        import spikemesh.models  # noqa: F401
        from spikemesh import kernels
        return spikemesh, kernels.backend_name() if hasattr(kernels, "backend_name") else kernels.BACKEND_NAME
    except ImportError:
        return None, None


def cpu_sample(args):
    """The CPU reference arm's workload: the same network scaled down (the
    reference's 40 B records cannot hold C3's 1.125e9 synapses in host RAM)."""
    n = args.cpu_sample_neurons
    k_e = max(1, int(round(args.k_exc * args.cpu_sample_k_scale)))
    k_i = max(1, int(round(args.k_inh * args.cpu_sample_k_scale)))
    return n, k_e, k_i


def cpu_construct(args):
    """One construction of the sampled network on the host: the unmodified
    reference when installed (kind "reference"), else the oracle port."""
    sm, backend = reference_package()
    n, k_e, k_i = cpu_sample(args)
    if sm is not None:
        c = sm.Cluster(sm.SimConfig(n_ranks=1, seed=args.seed))
        sm.models.build_balanced_network(c, sm.models.BalancedParams(neurons_per_rank=n, k_exc=k_e, k_inh=k_i))
        c.prepare()
        return c, "reference", f"unmodified reference spikemesh 0.1.0 ({backend} kernels, baseline/_ref)"
    from oracle.spikemesh_oracle import OracleCluster
    from paper_2512_09502_b200 import api, models
    c = OracleCluster(api.SimConfig(n_ranks=1, seed=args.seed))
    models.build_balanced_network(c, models.BalancedParams(neurons_per_rank=n, k_exc=k_e, k_inh=k_i))
    c.prepare()
    return c, "port", "oracle port (reference not installed)"


def run_reference(args):
    """The reference's CPU implementation on the box's host cores, bounded
    sample, rank 0 only (other ranks exit without work)."""
    world, rank, _ = dist_info()
    if rank != 0:
        return
    n, k_e, k_i = cpu_sample(args)
    times = []
    kind = what = None
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        c, kind, what = cpu_construct(args)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
        del c
        gc.collect()
    syn = n * (k_e + k_i)
    value = syn / float(np.mean(times))
    sample = (f"{what}: 1 rank, {n} neurons, K={k_e}+{k_i} ({syn:.3g} synapses) per step; the GPU workload's "
              f"structure scaled down (neurons x{n / args.neurons:g}, K x{args.cpu_sample_k_scale:g}); "
              f"single-threaded (1 core used)")
    line = {
        "impl": "reference", "metric": "construction_synapses_per_s", "value": value, "unit": "synapses/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(times)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64/f64", "data": "synthetic",
        # the GPU arm's config (the metric is per synapse), with the bounded
        # sample each step actually builds
        "config": {"workload": "hpc_benchmark_C3_strong" if args.strong else "hpc_benchmark_C3_weak",
                   "neurons_per_gpu": args.neurons, "k_in": args.k_exc + args.k_inh,
                   "synapses_per_gpu": args.neurons * (args.k_exc + args.k_inh),
                   "comm": "collective" if args.gpus > 1 else "p2p", "parallelism": f"ranks{args.gpus}",
                   "seed": args.seed, "sample": {"neurons": n, "k_in": k_e + k_i, "synapses": syn}},
        "cpu_baseline": {"value": value, "unit": "synapses/s", "cores": 1, "kind": kind, "sample": sample,
                         "host": host_info()},
        "e2e": {"value": value, "unit": "synapses/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(args):
    """The reference timed on the host for the headline line (rank 0, N=1):
    one construction, then a recorded propagation window (RTF, rate)."""
    n, k_e, k_i = cpu_sample(args)
    t0 = time.perf_counter()
    c, kind, what = cpu_construct(args)
    dt = time.perf_counter() - t0
    rep = c.simulate(20.0, 50.0, record=True)
    rtf = rep.rtf if hasattr(rep, "rtf") else rep["rtf"]
    n_ev = rep.n_spike_events if hasattr(rep, "n_spike_events") else int(c.raster().shape[0])
    syn = n * (k_e + k_i)
    return {"value": syn / dt, "unit": "synapses/s", "cores": 1, "kind": kind,
            "sample": f"{what}: 1 rank, {n} neurons, K={k_e}+{k_i} ({syn:.3g} synapses) construction "
                      f"{dt:.2f} s; propagation RTF {rtf:.2f} over 50 ms after 20 ms warmup",
            "rtf": rtf, "rate_hz": n_ev / (n * 0.05), "host": host_info()}


def propagation_stats(c, rep, rep2, args, world, n_rank, syn_per_rank, max_over_ranks):
    """Event counts and the per-step roofline of propagation (SURVEY §8d:
    B_step = 40 N + 20 E bytes; N neurons, E synaptic events per step).
    rep: unrecorded run (RTF); rep2: recorded window of the same length."""
    import torch
    peak, _ = peaks()
    steps = c.cfg.steps_for(args.model_ms)
    (rank, st), = [(r, st) for r, st in c.ranks.items()][:1]
    ev = c.rank_events(rank)
    nodes = c._gid_to_node(st, ev[:, 1]) if len(ev) else np.empty(0, np.int64)
    fi = st.first_index.cpu().numpy()
    local_events = int((fi[nodes + 1] - fi[nodes]).sum()) if len(nodes) else 0
    spikes = int(max_over_ranks(float(len(ev))) if world == 1 else 0)
    if world > 1:
        t = torch.tensor([float(len(ev)), float(local_events)], dtype=torch.float64, device=st.device)
        torch.distributed.all_reduce(t)
        spikes = int(t[0].item())
    rate = spikes / (world * n_rank * args.model_ms * 1e-3)
    if world == 1:
        e_step = local_events / steps
        how = "exact: sum of the spiking sources' row lengths"
    else:  # every source has the same expected out-degree over all ranks
        e_step = spikes * (syn_per_rank / n_rank) / steps / world
        how = "per GPU, spikes x mean out-degree (K N / N_src)"
    step_s = rep.rtf * c.cfg.resolution_ms * 1e-3
    b_step = 40.0 * n_rank + 20.0 * e_step
    achieved = b_step / step_s / 1e9 if step_s > 0 else 0.0
    return {"spikes": spikes, "model_ms": args.model_ms, "steps": steps, "rate_hz": rate,
            "events_per_step": e_step, "events_how": how, "rtf_recording": max_over_ranks(rep2.rtf),
            "step_us": step_s * 1e6,
            "roofline_prop": {"bound": "hbm", "bytes_per_step": b_step, "achieved": achieved, "peak": peak,
                              "unit": "GB/s", "frac": achieved / peak,
                              "formula": "(40 N + 20 E) / step time (SURVEY 8d)"}}


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2512_09502_b200 import _lib, api, engine, models

    world, rank, local = dist_info()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    cfg = api.SimConfig(n_ranks=world, comm_mode="collective" if world > 1 else "p2p", seed=args.seed)
    n_rank = args.neurons // world if args.strong else args.neurons
    params = models.BalancedParams(neurons_per_rank=n_rank, k_exc=args.k_exc, k_inh=args.k_inh)
    syn_per_rank = n_rank * (args.k_exc + args.k_inh)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def construct():
        c = engine.Cluster(cfg, profile=True)
        models.build_balanced_network(c, params)
        c.prepare()
        return c

    c = None
    for _ in range(args.warmup):
        del c
        gc.collect()
        c = construct()
        barrier()
    step_ms, wall_s, gen_ms, sort_ms, launches, h2d = [], [], [], [], [], []
    with Clocks(dev.index) as clk:
        for _ in range(args.steps):
            del c
            gc.collect()
            barrier()
            L0 = _lib.lib().smx_launch_count()
            H0 = engine.H2D_BYTES[0]
            stream = torch.cuda.current_stream(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record(stream)
            c = construct()
            e1.record(stream)
            # end-to-end: read the result back to the host (records per rank)
            n_rec = int(c.ranks[rank].first_index[-1].item())
            wall = time.perf_counter() - t0
            torch.cuda.synchronize(dev)
            barrier()
            assert n_rec == syn_per_rank, (n_rec, syn_per_rank)
            step_ms.append(max_over_ranks(e0.elapsed_time(e1)))
            wall_s.append(max_over_ranks(wall))
            gen_ms.append(c.kernel_ms("gen"))
            sort_ms.append(c.kernel_ms("sort"))
            launches.append(_lib.lib().smx_launch_count() - L0)
            h2d.append(engine.H2D_BYTES[0] - H0)
        # propagation on the last network: the RTF without recording, then a
        # recorded window of the same length for spikes / events / rate
        rep = c.simulate(args.prop_warmup_ms, args.model_ms, record=False)
        rep2 = c.simulate(0.0, args.model_ms, record=True)
    rtf = max_over_ranks(rep.rtf)
    prop = propagation_stats(c, rep, rep2, args, world, n_rank, syn_per_rank, max_over_ranks)
    clocks = clk.summary()
    ms = float(np.mean(step_ms))
    total_syn = world * syn_per_rank
    value = total_syn / (ms * 1e-3)
    e2e = total_syn / float(np.mean(wall_s))
    peak, peak_kind = peaks()
    k_ms = float(np.mean(gen_ms)) + float(np.mean(sort_ms))
    achieved = BYTES_PER_SYN * syn_per_rank / (k_ms * 1e-3) / 1e9
    store_path = c.ranks[rank].store_path
    tps, traffic_src = traffic_per_synapse(store_path)
    traffic = tps * syn_per_rank if tps is not None else None  # bytes per construction, like achieved
    line = {
        "metric": "construction_synapses_per_s", "value": value, "unit": "synapses/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if args.strong else "weak", "vs_baseline": None, "dtype": "u32/f64",
        "data": "synthetic",
        "config": {"workload": "hpc_benchmark_C3_strong" if args.strong else "hpc_benchmark_C3_weak",
                   "neurons_per_gpu": n_rank,
                   "k_in": args.k_exc + args.k_inh,
                   "synapses_per_gpu": syn_per_rank, "comm": cfg.comm_mode, "parallelism": f"ranks{world}",
                   "l2": "inputs larger than L2 (tables 4.5 GB per GPU)", "seed": args.seed},
        "construction_wall_s": float(np.mean(wall_s)),
        "rtf": rtf, "rtf_model_ms": args.model_ms, "n_spikes_model": prop["spikes"],
        "propagation": prop,
        "gpu_launches": int(np.mean(launches)),
        "e2e": {"value": e2e, "unit": "synapses/s", "h2d_bytes_per_step": int(np.mean(h2d)),
                "d2h_bytes_per_step": 8},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_kind": peak_kind,
                     "kernel": KERNELS.get(store_path, store_path), "store_path": store_path,
                     "kernel_ms": k_ms, "bytes_per_synapse": BYTES_PER_SYN},
        "clocks": clocks,
        "phase_ms": {"gen": float(np.mean(gen_ms)), "sort": float(np.mean(sort_ms))},
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        c.close()
        dist.barrier()
        dist.destroy_process_group()


def run_c5(args):
    """BASELINE configs[4]: construction-only sweep of
    synapses per GPU for fixed_indegree (distributed rule, the fused path)
    and fixed_total (local rule; fused too: targets drawn per record).  N neurons per GPU fixed,
    K or n_total scaled.  One JSON line per point; peak device memory from
    the caching allocator (everything the construction holds at once)."""
    import torch
    import torch.distributed as dist

    from paper_2512_09502_b200 import api, engine

    world, rank, local = dist_info()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    n = args.neurons
    points = [int(float(x)) for x in args.c5_points.split(",")]
    rules = args.c5_rules.split(",")

    def build(rule, syn_per_gpu):
        c = engine.Cluster(api.SimConfig(n_ranks=world, seed=args.seed), profile=True)
        pops = [np.arange(c.create_neurons(r, n).start, n) for r in range(world)]
        if rule == "fixed_indegree":
            k = syn_per_gpu // n
            c.connect_fixed_indegree_distributed([(r, pops[r]) for r in range(world)],
                                                 [(r, pops[r]) for r in range(world)], k, api.SynSpec(0.125, 15))
        else:
            for r in range(world):
                c.connect(r, pops[r], pops[r], api.ConnSpec("fixed_total", n_total=syn_per_gpu), api.SynSpec(0.125, 15))
        c.prepare()
        return c

    for rule in rules:
        for S in points:
            times, gen, srt = [], [], []
            c = None
            for i in range(args.warmup + args.steps):
                del c
                gc.collect()
                torch.cuda.reset_peak_memory_stats(dev)
                if world > 1:
                    dist.barrier()
                torch.cuda.synchronize(dev)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                c = build(rule, S)
                e1.record()
                torch.cuda.synchronize(dev)
                if i >= args.warmup:
                    t = e0.elapsed_time(e1)
                    if world > 1:
                        x = torch.tensor([t], dtype=torch.float64, device=dev)
                        dist.all_reduce(x, op=dist.ReduceOp.MAX)
                        t = float(x.item())
                    times.append(t)
                    gen.append(c.kernel_ms("gen"))
                    srt.append(c.kernel_ms("sort"))
            peak = torch.cuda.max_memory_allocated(dev)
            ok = int(c.ranks[rank].first_index[-1].item()) == S
            path = c.ranks[rank].store_path
            ms = float(np.mean(times))
            line = {"metric": "construction_synapses_per_s", "value": world * S / (ms * 1e-3), "unit": "synapses/s",
                    "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                    "higher_is_better": True, "scaling": "weak", "data": "synthetic",
                    "config": {"workload": f"C5_{rule}_{S:.0e}", "rule": rule, "neurons_per_gpu": n,
                               "synapses_per_gpu": S, "store_path": path},
                    "phase_ms": {"gen": float(np.mean(gen)), "sort": float(np.mean(srt))},
                    "peak_device_bytes": int(peak), "peak_bytes_per_synapse": peak / S, "records_ok": ok}
            if rank == 0:
                print(json.dumps(line), flush=True)
            del c
            c = None
            gc.collect()
            torch.cuda.empty_cache()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_c4(args):
    """BASELINE configs[3]: the multi-area model of
    sm/models.py:349-403 -- areas of ~1.29e5 neurons packed onto the ranks
    by pack_areas (sm/models.py:290-306), local E/I circuits plus k_inter
    remote E inputs for every ordered area pair, point-to-point exchange.
    One JSON line: construction (device span, max over ranks; host wall; the
    host share = time inside the façade calls / wall), then the RTF of a
    propagation window."""
    import torch
    import torch.distributed as dist

    from paper_2512_09502_b200 import api, engine, models

    world, rank, local = dist_info()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    n_areas = args.c4_areas or 4 * world
    ke, ki, kx = (int(x) for x in args.c4_k.split(","))
    per_in = ke + ki + kx * (n_areas - 1)
    areas = [models.AreaSpec(f"A{i:02d}", args.c4_neurons, args.c4_neurons * per_in) for i in range(n_areas)]
    assignment, _ = models.pack_areas(areas, world)
    params = models.MultiAreaParams(k_intra_exc=ke, k_intra_inh=ki, k_inter=kx, delay_steps=15)
    cfg = api.SimConfig(n_ranks=world, comm_mode="p2p", seed=args.seed)
    mine = [a for a in areas if assignment[a.area_id] == rank]
    syn_rank = sum(a.neurons * per_in for a in mine)
    syn_total = sum(a.neurons * per_in for a in areas)

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    c = None
    span, wall, host, kern, gen, srt = [], [], [], [], [], []
    for i in range(args.warmup + args.steps):
        del c
        gc.collect()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        c = engine.Cluster(cfg, profile=True)
        models.build_multi_area(c, areas, assignment, params)
        c.prepare()
        e1.record()
        n_rec = int(c.ranks[rank].first_index[-1].item())
        w = time.perf_counter() - t0
        torch.cuda.synchronize(dev)
        assert n_rec == syn_rank, (n_rec, syn_rank)
        if i >= args.warmup:
            span.append(max_over_ranks(e0.elapsed_time(e1)))
            wall.append(max_over_ranks(w))
            host.append(max_over_ranks(sum(h for _, h, _ in c.timers._pending)))
            gen.append(max_over_ranks(c.kernel_ms("gen")))
            srt.append(max_over_ranks(c.kernel_ms("sort")))
            kern.append(max_over_ranks(c.kernel_ms("gen") + c.kernel_ms("sort")))
    peak = torch.cuda.max_memory_allocated(dev)
    rep = c.simulate(args.prop_warmup_ms, args.model_ms, record=False)
    rtf = max_over_ranks(rep.rtf)
    c.simulate(0.0, args.model_ms, record=True)
    n_spk = len(c.rank_events(rank))
    n_rank_neurons = sum(a.neurons for a in mine)
    ms = float(np.mean(span))
    line = {"metric": "construction_synapses_per_s", "value": syn_total / (ms * 1e-3), "unit": "synapses/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "data": "synthetic",
            "config": {"workload": "multi_area_C4", "areas": n_areas, "areas_per_gpu": len(mine),
                       "neurons_per_area": args.c4_neurons, "k": [ke, ki, kx], "synapses_total": syn_total,
                       "synapses_rank0": syn_rank, "comm": "p2p", "parallelism": f"ranks{world}",
                       "remote_calls": n_areas * (n_areas - 1), "store_path": c.ranks[rank].store_path},
            "construction_wall_s": float(np.mean(wall)),
            "facade_s": float(np.mean(host)),
            "non_kernel_share": 1.0 - float(np.mean(kern)) / (1e3 * float(np.mean(wall))),
            "gen_sort_kernel_ms": float(np.mean(kern)),
            "phase_ms": {"gen": float(np.mean(gen)), "sort": float(np.mean(srt))},
            "peak_device_bytes": int(peak), "rtf": rtf, "rtf_model_ms": args.model_ms,
            "n_spikes_rank0": n_spk, "rate_hz_rank0": n_spk / (n_rank_neurons * args.model_ms * 1e-3)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        c.close()
        dist.barrier()
        dist.destroy_process_group()


def run_c2(args):
    """BASELINE configs[1]: the Potjans-Diesmann microcircuit
    at full scale on one GPU (paper_2512_09502_b200/models.py:
    build_microcircuit; fixed_total per projection, normal weights, uniform
    integer delays -> the wide general path).  Under torchrun every rank
    builds its own copy (replicas; the model is a one-GPU config)."""
    import torch
    import torch.distributed as dist

    from paper_2512_09502_b200 import api, engine, models

    world, rank, local = dist_info()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    p = models.MicrocircuitParams(scale=1.0)
    sizes, k = models.microcircuit_synapse_counts(p)
    n_syn = int(k.sum())

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    c = None
    span, wall, gen, srt = [], [], [], []
    for i in range(args.warmup + args.steps):
        del c
        gc.collect()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        torch.cuda.reset_peak_memory_stats(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        c = engine.Cluster(api.SimConfig(n_ranks=1, comm_mode="p2p", seed=args.seed), profile=True)
        models.build_microcircuit(c, p)
        c.prepare()
        e1.record()
        n_rec = int(c.ranks[0].first_index[-1].item())
        w = time.perf_counter() - t0
        torch.cuda.synchronize(dev)
        assert n_rec == n_syn, (n_rec, n_syn)
        if i >= args.warmup:
            span.append(max_over_ranks(e0.elapsed_time(e1)))
            wall.append(max_over_ranks(w))
            gen.append(c.kernel_ms("gen"))
            srt.append(c.kernel_ms("sort"))
    peak = torch.cuda.max_memory_allocated(dev)
    rep = c.simulate(args.prop_warmup_ms, args.model_ms, record=False)
    c.simulate(0.0, args.model_ms, record=True)
    n_spk = len(c.rank_events(0))
    ms = float(np.mean(span))
    line = {"metric": "construction_synapses_per_s", "value": world * n_syn / (ms * 1e-3), "unit": "synapses/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "data": "synthetic", "dtype": "u32/f64",
            "config": {"workload": "microcircuit_C2", "neurons": int(sum(sizes)), "synapses": n_syn,
                       "parallelism": "replicas" if world > 1 else "ranks1", "seed": args.seed,
                       "store_path": c.ranks[0].store_path},
            "construction_wall_s": float(np.mean(wall)),
            "phase_ms": {"gen": float(np.mean(gen)), "sort": float(np.mean(srt))},
            "peak_device_bytes": int(peak), "peak_bytes_per_synapse": peak / n_syn,
            "rtf": max_over_ranks(rep.rtf), "rtf_model_ms": args.model_ms, "n_spikes": n_spk,
            "rate_hz": n_spk / (sum(sizes) * args.model_ms * 1e-3)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.workload == "c2":
        run_c2(args)
    elif args.workload == "c5":
        run_c5(args)
    elif args.workload == "c4":
        run_c4(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
