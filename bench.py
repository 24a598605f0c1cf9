#!/usr/bin/env python3
"""Benchmark of the sm_100a compress / decompress path (BASELINE.json metric).

One *step* = one compress + one decompress of the workload field through the
library (``paper_2401_05994_b200``, C-ABI ``include/mgrc_gpu.h``):

  * ``value``   device-resident: the input field and the container live in HBM
                when the step starts (compress_to a device buffer, then
                decompress_into a device array).  Reported as the harmonic
                combination 2·N·s_T / (t_compress + t_decompress), i.e. the
                uncompressed GB/s of a round trip; compress and decompress GB/s
                are also reported on their own.
  * ``e2e``     the same step through the public API with pinned HOST buffers:
                H2D of the input + D2H of the container (compress), H2D of the
                container + D2H of the output (decompress), all inside the
                timed region.  ``--e2e-workers`` host threads (default 4,
                each its own library context = stream + workspace) issue
                round trips concurrently, so PCIe H2D, D2H (full duplex) and
                the kernels of different round trips overlap; the
                single-thread figure is reported beside it.

Workload at N=1: BASELINE.json configs[1], 513^3 f32 synthetic multisine
(test_support.hpp:43-62), L-inf REL 1e-4, codec 2 (varint + Huffman).  The
input (540 MB) and output exceed the 126 MB L2, so no L2 flush is needed.
At N>1 (``--gpus N``; the script re-launches itself under torchrun when
WORLD_SIZE is unset) the default workload is BASELINE.json configs[4]: the
2049^3 f32 field chunked into the CLI's 8 slabs [257, 256x7] (chunk_mem =
257*2049^2*4), slab b on rank floor(b*N/8) — strong scaling, total work fixed;
the only collectives are the all-gathers of [min, max] and of the compressed
sizes (sharded.py).  ``--workload`` selects any configuration explicitly.

``--impl reference`` times the reference's own CPU implementation
(oracle/_ref: /root/reference/proj/src compiled unmodified) on the host cores
with all host threads: the full 513^3 field per step for configs[1] (the same
config as the GPU arm), a bounded row sample of the field for the larger
workloads (named in ``cpu_baseline.sample``).
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

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = "compress/decompress GB/s (round trip, uncompressed bytes)"
UNIT = "GB/s"

WORKLOADS = {
    # name: (shape, dtype, tol, norm, s, mode)
    "cfg2_513cubed_f32_inf_rel1e-4": ((513, 513, 513), "f32", 1e-4, 0, 0.0, 1),
    "cfg1_65cubed_f64_inf_rel1e-3": ((65, 65, 65), "f64", 1e-3, 0, 0.0, 1),
    "cfg3_8193sq_f64_s1_rel1e-3": ((8193, 8193), "f64", 1e-3, 1, 1.0, 1),
    "cfg4_1025cubed_f64_inf_rel1e-5": ((1025, 1025, 1025), "f64", 1e-5, 0, 0.0, 1),
}
DEFAULT_WORKLOAD = "cfg2_513cubed_f32_inf_rel1e-4"
# configs[4]: 2049^3 f32, INF REL 1e-4, chunked into 8 slabs [257, 256x7] (chunk_mem = 257*2049^2*4) that
# are split across the ranks (strong scaling: total work fixed) — the multi-GPU sweep of BASELINE.json.
CHUNKED_WORKLOAD = "cfg5_2049cubed_f32_chunked_rel1e-4"
WORKLOADS[CHUNKED_WORKLOAD] = ((2049, 2049, 2049), "f32", 1e-4, 0, 0.0, 1)
CHUNK_MEM = 257 * 2049 * 2049 * 4
# configs[3] as stated: "1025^3 fp64 decompose+recompose round trip" — one step = forward_transform +
# inverse_transform on the device (transform.hpp:24-30), metric = 2·N·8 bytes / step time
TRANSFORM_WORKLOADS = {
    "cfg4_1025cubed_f64_roundtrip": ((1025, 1025, 1025), False),
    "cfg4_1025cubed_f64_roundtrip_l2proj": ((1025, 1025, 1025), True),
}
# the opt-in L2-projection correction (row f3) on configs[1]'s field
L2_WORKLOADS = {"cfg2_513cubed_f32_inf_rel1e-4_l2proj": ((513, 513, 513), "f32", 1e-4, 0, 0.0, 1)}
WORKLOADS.update(L2_WORKLOADS)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# synthetic field: multisine (test_support.hpp:43-62), evaluated in f64


def multisine_torch(shape, device):
    import torch

    d = len(shape)
    t = [torch.linspace(0.0, 1.0, n, dtype=torch.float64, device=device) if n > 1 else
         torch.zeros(1, dtype=torch.float64, device=device) for n in shape]

    def ax(a):
        if a >= d:
            return torch.zeros((1,) * d, dtype=torch.float64, device=device)
        v = t[a]
        return v.reshape([-1 if k == a else 1 for k in range(d)])

    t0, t1, t2, t3 = ax(0), ax(1), ax(2), ax(3)
    two_pi = 2.0 * np.pi
    u = torch.sin(two_pi * (t0 + 0.7 * t1 + 0.4 * t2))
    u = u + 0.5 * torch.sin(two_pi * (3.0 * t0 + 2.2 * t1))
    u = u + 0.25 * torch.sin(two_pi * (7.0 * t0 + 5.0 * t3))
    u = u + 1.5 * t0
    return u.expand(*shape).contiguous()


# dominant phase -> its main kernel (for the ncu DRAM traffic lookup)
PHASE_KERNEL = {"forward": "k_forward", "inverse": "k_inverse_level", "forward_l2": "k_l2_line",
                "inverse_l2": "k_l2_line", "quantize": "k_quant_zz", "check_l2": "k_l2_line", "fine": "k_fine_warp", "huff_maps": "k_tfd_maps", "huff_count": "k_tfd_count", "huff_emit": "k_tfd_emit",
                "recon": "k_recon_warp", "pack": "k_pack_lb", "coarse_check": "k_cq_warp", "crc": "k_crc_coal",
                "stats": "k_stats"}


def ncu_traffic(phase, workload):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the phase's kernel, from the committed
    `ncu --set full` capture summary of THIS workload (profiles/ncu_traffic.json, scripts/ncu_traffic.py);
    None when no capture of the workload exists."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text()).get("workloads", {}).get(workload)
    if not d:
        return None
    k = PHASE_KERNEL.get(phase)
    for name, v in d.get("kernels", {}).items():
        if k and k in name:
            return v["dram_bytes"]
    return None


# ---------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md "clocks DURING the timed region")


class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for name, v in zip(self.NAMES, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# reference arm / cpu baseline: the reference library on host cores


def cpu_reference_step(ref, u_np, tol, norm, s, mode):
    t0 = time.perf_counter()
    blob = ref.compress(u_np, tol, norm, s, mode, 2)
    t1 = time.perf_counter()
    ref.decompress(blob)
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1, len(blob)


def host_info():
    model = None
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count() or 1}


# Largest sample the CPU arm compresses per step: the whole field up to configs[1]'s 540 MB (so the
# reference arm runs the SAME config as the GPU arm there), a leading row slab of the field beyond it.
CPU_SAMPLE_BYTES = 560e6


def cpu_sample_rows(shape, esz, budget=CPU_SAMPLE_BYTES):
    row = int(np.prod(shape[1:])) * esz
    return max(1, min(shape[0], int(budget // row)))


def field_rows_np(shape, rows, dts):
    """First ``rows`` rows (axis 0) of multisine(shape), on the host, in the workload's element type."""
    u = multisine_rows(shape, 0, rows, "cpu").contiguous().numpy()
    return u.astype(np.float32 if dts == "f32" else np.float64)


def ref_oracle():
    from oracle import binding

    kind = "reference" if binding.available("reference") else "restatement"
    return binding.get(kind), ("reference" if kind == "reference" else "port")


def time_cpu(ref, sample, spec, reps_max, budget_s):
    tol, norm, s, mode = spec
    tc = td = 0.0
    reps = 0
    clen = 0
    t_start = time.perf_counter()
    while reps < reps_max and (reps == 0 or time.perf_counter() - t_start < budget_s):
        a, b, clen = cpu_reference_step(ref, sample, tol, norm, s, mode)
        tc += a
        td += b
        reps += 1
    return tc, td, reps, clen


def cpu_baseline_measure(workload, budget_s=20.0):
    """The reference library (oracle/_ref, else the C restatement) on the host cores: all threads on the
    workload's CPU sample (the whole field for configs[1]), plus one thread on a 65-row slab of it."""
    shape, dts, tol, norm, s, mode = WORKLOADS[workload]
    esz = 4 if dts == "f32" else 8
    ref, kind = ref_oracle()
    info = host_info()
    cores = info["nproc"]
    rows = cpu_sample_rows(shape, esz)
    sample = field_rows_np(shape, rows, dts)
    spec = (tol, norm, s, mode)
    ref.set_threads(cores)
    tc, td, reps, _ = time_cpu(ref, sample, spec, 3, budget_s)
    nbytes = sample.nbytes
    whole = rows == shape[0]
    what = ("the whole workload field" if whole else
            f"the first {rows} rows of the workload field (REL bound taken on the sample)")
    out = {
        "value": 2.0 * nbytes * reps / (tc + td) / 1e9, "unit": UNIT, "cores": cores, "kind": kind,
        "sample": f"{reps}x compress+decompress of {what} ({'x'.join(map(str, sample.shape))} {sample.dtype}, "
                  f"{nbytes / 1e6:.1f} MB), codec 2, {cores} threads",
        "same_config": whole,
        "compress_gbs": nbytes * reps / tc / 1e9, "decompress_gbs": nbytes * reps / td / 1e9,
        "cpu_model": info["cpu_model"],
    }
    # one thread, on a bounded slab of the same field
    row_bytes = int(np.prod(shape[1:])) * esz
    r1 = min(shape[0], max(9 if len(shape) >= 3 else 1, min(65, int(70e6 // row_bytes))))
    s1 = np.ascontiguousarray(sample[:r1]) if r1 <= rows else field_rows_np(shape, r1, dts)
    ref.set_threads(1)
    tc1, td1, reps1, _ = time_cpu(ref, s1, spec, 1, budget_s)
    ref.set_threads(cores)
    out["single_thread"] = {
        "value": 2.0 * s1.nbytes * reps1 / (tc1 + td1) / 1e9, "unit": UNIT, "cores": 1,
        "compress_gbs": s1.nbytes * reps1 / tc1 / 1e9, "decompress_gbs": s1.nbytes * reps1 / td1 / 1e9,
        "sample": f"{reps1}x compress+decompress of the first {r1} rows ({'x'.join(map(str, s1.shape))}, "
                  f"{s1.nbytes / 1e6:.1f} MB)"}
    return out


def run_reference_arm(args, workload):
    """The reference's CPU implementation (unmodified library, public API) on all host threads; rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    shape, dts, tol, norm, s, mode = WORKLOADS[workload]
    esz = 4 if dts == "f32" else 8
    ref, kind = ref_oracle()
    info = host_info()
    cores = info["nproc"]
    ref.set_threads(cores)
    rows = cpu_sample_rows(shape, esz)
    sample = field_rows_np(shape, rows, dts)
    whole = rows == shape[0]
    for _ in range(args.warmup):
        cpu_reference_step(ref, sample, tol, norm, s, mode)
    tc = td = 0.0
    clen = 0
    for _ in range(args.steps):
        a, b, clen = cpu_reference_step(ref, sample, tol, norm, s, mode)
        tc += a
        td += b
    nbytes = sample.nbytes
    value = 2.0 * nbytes * args.steps / (tc + td) / 1e9
    what = "the whole workload field" if whole else f"the first {rows} rows of the workload field"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": (tc + td) / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong" if workload == CHUNKED_WORKLOAD else "weak",
        "vs_baseline": None, "dtype": "f64 (f32 data widened)" if dts == "f32" else "f64",
        "data": "synthetic multisine (test_support.hpp:43-62)",
        "config": {"workload": workload, "shape": list(shape), "sample_shape": list(sample.shape),
                   "same_config": whole, "codec": "huffman", "threads": cores},
        "compress_gbs": nbytes * args.steps / tc / 1e9, "decompress_gbs": nbytes * args.steps / td / 1e9,
        "ratio": nbytes / clen,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"compress+decompress of {what} per step "
                                   f"({'x'.join(map(str, sample.shape))} {sample.dtype}, {nbytes / 1e6:.1f} MB)",
                         "cpu_model": info["cpu_model"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def multisine_rows(shape, r0, r1, device):
    """Rows [r0, r1) (axis 0) of multisine(shape), evaluated exactly as multisine_torch."""
    import torch

    d = len(shape)
    t = [torch.linspace(0.0, 1.0, n, dtype=torch.float64, device=device) for n in shape]
    t[0] = t[0][r0:r1]

    def ax(a):
        if a >= d:
            return torch.zeros((1,) * d, dtype=torch.float64, device=device)
        return t[a].reshape([-1 if k == a else 1 for k in range(d)])

    t0, t1, t2, t3 = ax(0), ax(1), ax(2), ax(3)
    two_pi = 2.0 * np.pi
    u = torch.sin(two_pi * (t0 + 0.7 * t1 + 0.4 * t2))
    u = u + 0.5 * torch.sin(two_pi * (3.0 * t0 + 2.2 * t1))
    u = u + 0.25 * torch.sin(two_pi * (7.0 * t0 + 5.0 * t3))
    u = u + 1.5 * t0
    return u.expand(r1 - r0, *shape[1:])


class PhaseAcc:
    """Per-phase CUDA-event times (the library's stream) summed over the calls of the timed region."""

    def __init__(self):
        self.ms, self.bytes, self.n = {}, {}, {}

    def add(self, mg):
        for name, ms, by in mg.last_profile():
            self.ms[name] = self.ms.get(name, 0.0) + ms
            self.bytes[name] = self.bytes.get(name, 0.0) + by
            self.n[name] = self.n.get(name, 0) + 1

    def roofline(self, steps, workload):
        peak, peak_src = peaks()
        kernel_phases = {k: v for k, v in self.ms.items() if not k.startswith(("h2d", "d2h"))}
        dom = max(kernel_phases, key=kernel_phases.get)
        dom_ms = self.ms[dom] / self.n[dom]
        dom_bytes = self.bytes[dom] / self.n[dom]
        achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": ncu_traffic(dom, workload), "alg_bytes_per_launch": dom_bytes,
                "ms_per_launch": dom_ms, "launches_per_step": self.n[dom] / steps, "peak_source": peak_src}
        phases = {k: {"ms": round(self.ms[k] / steps, 4),
                      "gbs": round(self.bytes[k] / (self.ms[k] * 1e-3) / 1e9, 1) if self.ms[k] > 0 else None}
                  for k in sorted(self.ms, key=self.ms.get, reverse=True)}
        return roof, phases


def run_chunked(args, world, rank, local, coll_dev):
    """configs[4]: the chunked driver (paper_2401_05994_b200/sharded.py, tools/mgrc.cpp:363-542) with the
    slabs split across ranks; device-resident containers; NCCL all-gathers of [min,max] and of the sizes.
    Then the same step through the public API from pinned HOST buffers (e2e), and the CPU baseline."""
    import torch
    import torch.distributed as dist

    import paper_2401_05994_b200 as mg
    from paper_2401_05994_b200 import sharded

    mg.set_device(local)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    mg.set_stream(stream.cuda_stream)
    workload = CHUNKED_WORKLOAD
    shape, dts, tol, norm, s, mode = WORKLOADS[workload]
    plan = mg.plan_chunks(shape, mg.DType.f32, CHUNK_MEM)
    nb = plan.shape[0]
    mine = sharded.blocks_of(rank, nb, world)
    r0, r1 = int(plan[mine[0]][0][0]), int(plan[mine[-1]][0][1])
    u = torch.empty((r1 - r0,) + tuple(shape[1:]), dtype=torch.float32, device="cuda")
    for a in range(r0, r1, 64):  # generate in row chunks (bounded f64 temporaries)
        b = min(r1, a + 64)
        u[a - r0:b - r0] = multisine_rows(shape, a, b, "cuda").to(torch.float32)
    slab_bytes = {b: int(np.prod([int(r[1] - r[0]) for r in plan[b]])) * 4 for b in mine}
    cap = {b: slab_bytes[b] // 2 + (64 << 20) for b in mine}  # containers are ~1/4 of the slab at this bound
    dsts = {b: torch.empty(cap[b], dtype=torch.uint8, device="cuda") for b in mine}
    outs = {b: torch.empty(slab_bytes[b] // 4, dtype=torch.float32, device="cuda") for b in mine}
    coords = [np.arange(n, dtype=np.float64) for n in shape]
    grids = {b: mg.make_grid(tuple(int(r[1] - r[0]) for r in plan[b]), sharded.block_coords(plan[b].tolist(), coords))
             for b in mine}
    sizes_local = {}

    def allgather_vec(vals):
        if world == 1:
            return [vals]
        t = torch.tensor(vals, dtype=torch.float64, device=coll_dev)
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        return [p.cpu().tolist() for p in parts]

    def view(b):
        a0, a1 = int(plan[b][0][0]), int(plan[b][0][1])
        return u[a0 - r0:a1 - r0]

    def global_spec(views):
        mn, mx = np.inf, -np.inf
        for v in views:  # REL normalisation (mgrc.cpp:405-418): per-rank stats, one tiny all-gather
            a, c, _ = mg.field_stats(v)
            mn, mx = min(mn, a), max(mx, c)
        st = allgather_vec([mn, mx])
        tau = tol * (max(r[1] for r in st) - min(r[0] for r in st))
        return mg.ErrorSpec(tau, mg.Norm.inf, 0.0, mg.Mode.abs), tau

    def gather_sizes(local_sizes):
        vec = [0.0] * nb
        for b, n in local_sizes.items():
            vec[b] = float(n)
        allv = allgather_vec(vec)
        return [int(sum(r[b] for r in allv)) for b in range(nb)]

    acc = None

    def compress_step():
        spec, _ = global_spec([view(b) for b in mine])
        for b in mine:
            sizes_local[b] = mg.compress_to(view(b), dsts[b], grids[b], spec, mg.Codec.huffman)
            if acc is not None:
                acc.add(mg)
        return gather_sizes(sizes_local)

    def decompress_step():
        for b in mine:
            mg.decompress_into(dsts[b][:sizes_local[b]], outs[b])
            if acc is not None:
                acc.add(mg)

    for _ in range(args.warmup):
        sizes = compress_step()
        decompress_step()
    torch.cuda.synchronize()
    _, tau_abs = global_spec([view(b) for b in mine])
    if world > 1:
        dist.barrier()
    mg.set_profiling(True)
    acc = PhaseAcc()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    l0 = mg.launch_count()
    tc = td = 0.0
    for _ in range(args.steps):
        e[0].record(stream)
        sizes = compress_step()
        e[1].record(stream)
        decompress_step()
        e[2].record(stream)
        torch.cuda.synchronize()
        tc += e[0].elapsed_time(e[1])
        td += e[1].elapsed_time(e[2])
    if world > 1:
        dist.barrier()
    launches = mg.launch_count() - l0
    clk = clocks.stop()
    mg.set_profiling(False)
    t = torch.tensor([tc, td], dtype=torch.float64, device=coll_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tc, td = (float(x) for x in t.tolist())
    total_bytes = int(np.prod(shape)) * 4
    stream_len = len(sharded.frame_header(sizes)) + sum(sizes)
    ms_step = (tc + td) / args.steps
    roof, phases = acc.roofline(args.steps, workload)
    # bound check on this rank's slabs (max over ranks)
    err = 0.0
    for b in mine:  # in row chunks (bounded temporaries)
        ob, ub = outs[b].view(view(b).shape), view(b)
        for a in range(0, ub.shape[0], 16):
            err = max(err, float((ob[a:a + 16].double() - ub[a:a + 16].double()).abs().max()))
    errs = allgather_vec([err])

    # e2e: the same chunked step through the public API from pinned HOST buffers (H2D of every slab, D2H of
    # every container, H2D of the containers, D2H of the decompressed slabs inside the timed region)
    e2e = None
    if not args.no_e2e:
        u_host = torch.empty(u.shape, dtype=torch.float32).pin_memory()
        u_host.copy_(u)
        del dsts, outs, u
        torch.cuda.empty_cache()
        h_dst = {b: torch.empty(sizes_local[b] + (64 << 20), dtype=torch.uint8).pin_memory() for b in mine}
        h_out = torch.empty(max(slab_bytes.values()) // 4, dtype=torch.float32).pin_memory()

        def hview(b):
            a0, a1 = int(plan[b][0][0]), int(plan[b][0][1])
            return u_host[a0 - r0:a1 - r0]

        def e2e_step():
            spec, _ = global_spec([hview(b) for b in mine])
            loc = {b: mg.compress_to(hview(b), h_dst[b], grids[b], spec, mg.Codec.huffman) for b in mine}
            gather_sizes(loc)
            for b in mine:
                mg.decompress_into(h_dst[b][:loc[b]], h_out[:slab_bytes[b] // 4])
            return loc

        e2e_step()
        if world > 1:
            dist.barrier()
        l1 = mg.launch_count()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            loc = e2e_step()
        e_ms = (time.perf_counter() - t0) * 1e3
        e_launch = mg.launch_count() - l1
        t = torch.tensor([e_ms], dtype=torch.float64, device=coll_dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
        my_in = sum(slab_bytes[b] for b in mine)
        my_c = sum(loc.values())
        e2e = {"value": 2.0 * total_bytes * args.steps / (e_ms * 1e-3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": my_in + my_c, "d2h_bytes_per_step": my_c + my_in,
               "per_rank": True, "ms_per_step": e_ms / args.steps, "gpu_launches": int(e_launch),
               "timing": "wall clock per rank (every call returns after its D2H copy), max over ranks"}
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline_measure(workload)
    if world > 1:
        dist.barrier()
    if rank == 0:
        line = {
            "metric": METRIC, "value": 2.0 * total_bytes / (ms_step * 1e-3) / 1e9, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64 (f32 data widened to f64 in registers)",
            "data": "synthetic multisine field (test_support.hpp:43-62), generated on the GPUs",
            "config": {"workload": workload, "shape": list(shape), "elem": dts, "tol": tol, "norm": "inf",
                       "mode": "rel", "codec": "huffman", "chunk_mem": CHUNK_MEM, "slabs": nb,
                       "slab_rows": [int(r[0][1] - r[0][0]) for r in plan], "parallelism": f"slabs over {world} ranks",
                       "l2": "inputs/outputs exceed the 126 MB L2; no flush"},
            "compress_gbs": total_bytes * args.steps / (tc * 1e-3) / 1e9,
            "decompress_gbs": total_bytes * args.steps / (td * 1e-3) / 1e9,
            "ratio": total_bytes / stream_len, "stream_bytes": stream_len,
            "max_err": max(r[0] for r in errs), "tau_abs": tau_abs,
            "bound_met": max(r[0] for r in errs) <= tau_abs,
            "step_alg_roofline_frac": 2 * (total_bytes + stream_len) / (ms_step * 1e-3) / 1e9 / roof["peak"] / world,
            "roofline": roof, "phases_ms_per_step_rank0": phases,
            "gpu_launches": int(launches), "clocks": clk,
            "e2e": e2e, "cpu_baseline": cpu, "host": host_info(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_transform(args, world, rank, local, coll_dev):
    """configs[3]: decompose + recompose round trip of the 1025^3 fp64 multisine field on the device
    (forward_transform then inverse_transform, transform.hpp:24-30; ``_l2proj``: with the L2-projection
    correction).  Metric: 2·N·8 bytes per step (the field is read once and written once per direction) / time;
    the reconstruction is checked against the input every run.  One field per rank (weak)."""
    import torch
    import torch.distributed as dist

    import paper_2401_05994_b200 as mg

    mg.set_device(local)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    mg.set_stream(stream.cuda_stream)
    shape, l2 = TRANSFORM_WORKLOADS[args.workload]
    N = int(np.prod(shape))
    u = multisine_torch(shape, "cuda")
    grid = mg.make_grid(shape)
    c = mg.forward_transform(u, grid, l2=l2)
    back = mg.inverse_transform(c, grid, l2=l2)
    rel_err = float((back - u).abs().max()) / float(u.max() - u.min())
    for _ in range(args.warmup - 1):
        c = mg.forward_transform(u, grid, l2=l2)
        back = mg.inverse_transform(c, grid, l2=l2)
    acc = PhaseAcc()
    mg.set_profiling(True)
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = mg.launch_count()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(stream)
    for _ in range(args.steps):
        c = mg.forward_transform(u, grid, l2=l2)
        acc.add(mg)
        back = mg.inverse_transform(c, grid, l2=l2)
        acc.add(mg)
    g1.record(stream)
    torch.cuda.synchronize()
    launches = mg.launch_count() - l0
    clk = clocks.stop()
    mg.set_profiling(False)
    ms = g0.elapsed_time(g1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    roof, phases = acc.roofline(args.steps, args.workload)
    if rank == 0:
        line = {
            "metric": "decompose+recompose round trip GB/s (2 x N x 8 bytes per step)",
            "value": 2.0 * N * 8 * world / (ms_step * 1e-3) / 1e9, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic multisine field (test_support.hpp:43-62), generated on the GPU",
            "config": {"workload": args.workload, "shape": list(shape), "l2_projection": l2,
                       "l2": "inputs/outputs exceed the 126 MB L2; no flush"},
            "max_rel_roundtrip_err": rel_err, "roofline": roof, "phases_ms_per_step": phases,
            "gpu_launches": int(launches), "clocks": clk, "host": host_info(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------
# GPU arm


def e2e_measure(mg, u_host, shape, tdt, cap, grid, spec, local, steps, workers, world, coll_dev, gather_sizes):
    """Round trips through the public API with pinned HOST buffers (H2D input, D2H container, H2D container,
    D2H output inside the timed region).  ``workers`` host threads, each with its own library context
    (stream + workspace, capi.cpp: one per thread and device), run ``steps`` round trips each on the same
    input, so one worker's copies overlap another's kernels and H2D overlaps D2H (PCIe is full duplex).
    Wall clock between a start barrier and the last completed call (every call returns after its
    device->host copy has landed), max over ranks."""
    import threading
    import torch
    import torch.distributed as dist

    nbytes = u_host.numel() * u_host.element_size()
    bufs = [(torch.empty(cap, dtype=torch.uint8).pin_memory(), torch.empty(shape, dtype=tdt).pin_memory())
            for _ in range(workers)]
    sizes = [[] for _ in range(workers)]
    launches = [0] * workers
    go = threading.Barrier(workers + 1)
    done = threading.Barrier(workers + 1)
    errs = []

    def work(w):
        try:
            mg.set_device(local)
            dst_h, out_h = bufs[w]
            for _ in range(2):  # warm-up: this thread's context, workspaces, hierarchy tables
                n_h = mg.compress_to(u_host, dst_h, grid, spec, mg.Codec.huffman)
                mg.decompress_into(dst_h[:n_h], out_h)
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(e)
        go.wait()
        try:
            l0 = mg.launch_count()
            for _ in range(steps):
                n_h = mg.compress_to(u_host, dst_h, grid, spec, mg.Codec.huffman)
                if workers == 1:
                    gather_sizes(n_h)
                sizes[w].append(n_h)
                mg.decompress_into(dst_h[:n_h], out_h)
            launches[w] = mg.launch_count() - l0
        except Exception as e:  # pragma: no cover
            errs.append(e)
        done.wait()

    ths = [threading.Thread(target=work, args=(w,)) for w in range(workers)]
    for t in ths:
        t.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    go.wait()
    t0 = time.perf_counter()
    done.wait()
    e_ms = (time.perf_counter() - t0) * 1e3
    for t in ths:
        t.join()
    if errs:
        raise errs[0]
    if workers > 1:  # the per-block size exchange of the sharded placement, once for all round trips
        for n_h in (n for per in sizes for n in per):
            gather_sizes(n_h)
    if world > 1:
        t = torch.tensor([e_ms], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
    n_h = sizes[0][-1]
    rt = steps * workers
    return {"value": 2.0 * nbytes * world * rt / (e_ms * 1e-3) / 1e9, "unit": UNIT,
            "h2d_bytes_per_step": nbytes + n_h, "d2h_bytes_per_step": n_h + nbytes,
            "ms_per_step": e_ms / rt, "workers": workers, "round_trips": rt, "gpu_launches": int(sum(launches)),
            "timing": "wall clock, start barrier to last call returned (each call ends after its D2H copy)"}


def self_launch(args):
    """`bench.py --gpus N` without torchrun: start N ranks (one per GPU) under torch.distributed.run on
    127.0.0.1, with the same arguments; rank 0 prints the JSON line."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # the NCCL init lines show the N ranks / devices in the log
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=sorted(list(WORKLOADS) + list(TRANSFORM_WORKLOADS)),
                    help="default: configs[1] (513^3 f32) at N=1, configs[4] (2049^3 f32 chunked) at N>1")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-workers", type=int, default=4,
                    help="host threads issuing round trips concurrently in the e2e measurement")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if args.workload is None:
        args.workload = CHUNKED_WORKLOAD if max(args.gpus, world_env) > 1 else DEFAULT_WORKLOAD

    if args.impl == "reference":
        return run_reference_arm(args, args.workload)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    shared_gpu = world > 1 and ndev < world  # test mode: several ranks on one device (gloo for the collective)
    local = local % ndev
    torch.cuda.set_device(local)
    coll_dev = "cpu" if shared_gpu else "cuda"
    if world > 1:
        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.workload == CHUNKED_WORKLOAD:
        return run_chunked(args, world, rank, local, coll_dev)
    if args.workload in TRANSFORM_WORKLOADS:
        return run_transform(args, world, rank, local, coll_dev)

    import paper_2401_05994_b200 as mg

    mg.set_device(local)
    # one non-default stream shared by torch and the library, so the CUDA
    # events below are recorded on the stream the kernels are launched on
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    mg.set_stream(stream.cuda_stream)

    shape, dts, tol, norm, s, mode = WORKLOADS[args.workload]
    tdt = torch.float32 if dts == "f32" else torch.float64
    N = int(np.prod(shape))
    esz = 4 if dts == "f32" else 8
    nbytes = N * esz
    u = multisine_torch(shape, f"cuda:{local}").to(tdt)
    grid = mg.make_grid(shape)
    spec = mg.ErrorSpec(tol, mg.Norm(norm), s, mg.Mode(mode))
    cap = nbytes * 2 + (1 << 20)
    dst = torch.empty(cap, dtype=torch.uint8, device="cuda")
    out = torch.empty(shape, dtype=tdt, device="cuda")

    def gather_sizes(n):
        if world == 1:
            return [n]
        t = torch.tensor([n], dtype=torch.int64, device=coll_dev)
        allt = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        return [int(x.item()) for x in allt]

    l2 = args.workload in L2_WORKLOADS

    def step_device():
        n = mg.compress_to(u, dst, grid, spec, mg.Codec.huffman, l2=l2)
        sizes = gather_sizes(n)
        mg.decompress_into(dst[:n], out)
        return n, sizes

    # warm-up (also builds the hierarchy tables / workspaces)
    for _ in range(args.warmup):
        clen, sizes = step_device()
    torch.cuda.synchronize()
    mg.compress_to(u, dst, grid, spec, mg.Codec.huffman, l2=l2)
    cstats = mg.last_compress_stats()  # the accept decision (tau_abs, achieved error, passes)

    # correctness of the measured path: the error bound on the reconstruction, in the reference's own
    # semantics (container.cpp:93-123): INF / S(0) compare the true max / RMS error with tau_abs; for
    # S(s!=0) the reference accepts on its level-weighted estimator (error_control.cpp:72-101, not a
    # certified L2 bound), so that estimator is the check and the true RMS is reported beside it
    u64 = u.double()
    diff = out.double() - u64
    max_err = float(diff.abs().max())
    rms_err = float(diff.square().mean().sqrt())
    del u64, diff
    tau = cstats["tau_abs"]
    if norm == 0:
        bound = {"norm": "inf", "tau_abs": tau, "max_err": max_err, "bound_met": max_err <= tau}
    elif s == 0.0:
        bound = {"norm": "s=0 (L2)", "tau_abs": tau, "rms_err": rms_err, "max_err": max_err,
                 "bound_met": rms_err <= tau}
    else:
        est = cstats["achieved"]
        bound = {"norm": f"s={s}", "tau_abs": tau, "estimator": est,
                 "estimator_semantics": "reference level-weighted aggregate (error_control.cpp:72-101)",
                 "bound_met": est <= tau * (1 - 1e-9), "true_rms_err": rms_err, "true_max_err": max_err}
    bound.update({"passes": cstats["passes"], "decided_by": cstats["decided_by"]})

    # timed region: K steps, device-resident, per-phase CUDA events on the launching stream
    mg.set_profiling(True)
    phase_ms, phase_bytes, phase_n = {}, {}, {}
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = mg.launch_count()
    g0 = torch.cuda.Event(enable_timing=True)
    g1 = torch.cuda.Event(enable_timing=True)
    g0.record(stream)
    for k in range(args.steps):
        a, b, c = ev[k]
        a.record(stream)
        n = mg.compress_to(u, dst, grid, spec, mg.Codec.huffman, l2=l2)
        for name, ms, by in mg.last_profile():
            phase_ms[name] = phase_ms.get(name, 0.0) + ms
            phase_bytes[name] = phase_bytes.get(name, 0.0) + by
            phase_n[name] = phase_n.get(name, 0) + 1
        gather_sizes(n)
        b.record(stream)
        mg.decompress_into(dst[:n], out)
        for name, ms, by in mg.last_profile():
            phase_ms[name] = phase_ms.get(name, 0.0) + ms
            phase_bytes[name] = phase_bytes.get(name, 0.0) + by
            phase_n[name] = phase_n.get(name, 0) + 1
        c.record(stream)
    g1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = mg.launch_count() - l0
    clk = clocks.stop()
    mg.set_profiling(False)
    total_ms = g0.elapsed_time(g1)
    tc = sum(ev[k][0].elapsed_time(ev[k][1]) for k in range(args.steps))
    td = sum(ev[k][1].elapsed_time(ev[k][2]) for k in range(args.steps))
    if world > 1:
        t = torch.tensor([total_ms, tc, td], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, tc, td = (float(x) for x in t.tolist())
    ms_step = total_ms / args.steps
    value = 2.0 * nbytes * world / (ms_step * 1e-3) / 1e9
    comp_gbs = nbytes * world * args.steps / (tc * 1e-3) / 1e9
    decomp_gbs = nbytes * world * args.steps / (td * 1e-3) / 1e9
    clen = n

    # dominant kernel phase (CUDA events on the library stream = the torch stream)
    peak, peak_src = peaks()
    kernel_phases = {k: v for k, v in phase_ms.items() if not k.startswith(("h2d", "d2h"))}
    dom = max(kernel_phases, key=kernel_phases.get)
    dom_ms = phase_ms[dom] / phase_n[dom]
    dom_bytes = phase_bytes[dom] / phase_n[dom]
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic = ncu_traffic(dom, args.workload)
    step_alg = (2 * nbytes + 2 * clen)  # B_c + B_d
    phases = {k: {"ms": round(phase_ms[k] / args.steps, 4),
                  "gbs": round(phase_bytes[k] / args.steps / (phase_ms[k] / args.steps * 1e-3) / 1e9, 1)
                  if phase_ms[k] > 0 else None}
              for k in sorted(phase_ms, key=phase_ms.get, reverse=True)}

    # e2e: public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        u_host = u.cpu().pin_memory()
        single = e2e_measure(mg, u_host, shape, tdt, cap, grid, spec, local, args.steps, 1, world, coll_dev,
                             gather_sizes)
        e2e = single
        # concurrent round trips only while their pinned buffers stay modest (cfg4's 8.6 GB field runs one)
        workers = max(1, min(args.e2e_workers, int(32e9 // (cap + nbytes))))
        if workers > 1:
            multi = e2e_measure(mg, u_host, shape, tdt, cap, grid, spec, local, args.steps, workers, world,
                                coll_dev, gather_sizes)
            multi["single_worker"] = {"value": single["value"], "ms_per_step": single["ms_per_step"]}
            e2e = multi

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline_measure(args.workload)

    if world > 1:
        dist.barrier()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64 (f32 data widened to f64 in registers)",
            "data": "synthetic multisine field (test_support.hpp:43-62), generated on the GPU",
            "config": {"workload": args.workload, "shape": list(shape), "elem": dts, "tol": tol,
                       "norm": "inf" if norm == 0 else f"s={s}", "mode": "rel" if mode else "abs",
                       "codec": "huffman", "per_rank": "one field per rank (independent containers)",
                       "l2": "inputs/outputs exceed the 126 MB L2; no flush"},
            "compress_gbs": comp_gbs, "decompress_gbs": decomp_gbs,
            "ratio": nbytes / clen, "compressed_bytes": clen,
            "max_err": max_err, "tau_abs": tau, "bound_met": bound["bound_met"], "bound": bound,
            "step_alg_roofline_frac": step_alg * world / (ms_step * 1e-3) / 1e9 / peak / world,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "alg_bytes_per_launch": dom_bytes,
                         "ms_per_launch": dom_ms, "peak_source": peak_src},
            "phases_ms_per_step": phases,
            "gpu_launches": int(launches),
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "host": host_info(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
