#!/usr/bin/env python
"""Benchmark: GR-KAN group-rational fwd+bwd throughput at KAT-B shape on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--dtype fp32|bf16|fp64]
                    [--config kat-b|kat-s|kat-t] [--mode fast|exact] [--impl b200|reference]
                    [--batch B --seqlen L --dim D --groups G --num-coeffs M1 --den-coeffs N
                     --seed S --block-size S --strategy blocked|naive|both --dump PATH]

``--gpus N`` without a launcher re-executes itself under torch.distributed.run
with N ranks (one per GPU); under a launcher WORLD_SIZE must equal N.  The
shape / degree / seed flags are run_bench's (pkg/src/grkan/cli.py:341-361);
inputs follow its draw order (x, upstream, numerator, denominator from
default_rng(seed), cli.py:143-158; rank r > 0 draws from default_rng([seed, r])).

One step = one forward (K1) + one backward (K2 + K3) of the group-rational
unit over one synthetic [B, L, D] batch (run_bench --include-forward,
pkg/src/grkan/cli.py:178-185), plus, when N > 1, the NCCL all-reduce of the
per-group da/db (the path's only exchange).  Weak scaling: every rank owns a
full KAT-B batch (B=256), so per-GPU work is fixed as N grows.

``value``  elements/s over all ranks, inputs already resident in HBM, device
           time (CUDA events) max over ranks.  Warm-up: >= W steps and >= 150 ms (GRKAN_BENCH_WARM_S);
           the timed K steps are enqueued behind a short device-side spin
           (--hold-ms) so host launch jitter cannot open gaps inside them;
           NVML clocks are then sampled by the (idle) host thread from the
           first timed step to the last.
           ``--collective`` picks the da/db exchange for N > 1 (NCCL
           all-reduce on a side stream, the world-size-invariant block path,
           or the peer-memory fused reduce); its time is ``kernels.collective_us``.
``e2e``    the same metric through the public streaming API
           (streaming.HostPipeline.fwd_bwd) with x, dy copied from pinned host
           memory and y, dx, da, db copied back every step; the plain
           autograd path (GroupRationalFn + backward) is reported beside it, and
           ``e2e.reference_api``: the reference-facing functions themselves
           (shim forward_tensor + backward_blocked on pageable NumPy arrays).
``roofline`` the dominant kernel (the backward call: K2 + its tiny K3 fold),
           algorithmic bytes 3*s*E per launch / its CUDA-event duration.
``cpu_baseline`` the reference itself (``grkan`` installed from /root/reference
           into baseline/_ref, kind "reference"; the oracle port, kind "port",
           only if that install is absent): forward_tensor + backward_blocked
           with all host threads on a bounded sample of the same workload
           (rank 0, N=1).

``--impl reference`` times only that CPU path (rank 0; other ranks exit 0).
Inputs exceed L2 (KAT-B fp32: 620 MB per tensor vs 126 MB L2), so no flush.
"""

from __future__ import annotations

import argparse
import math
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "GR-KAN fwd+bwd elements/sec & HBM GB/s (KAT-B shape) at 1/2/4/8 B200 vs CPU"
UNIT = "elements/s"
CONFIGS = {  # (batch per GPU, seq, dim, groups)
    "kat-t": (8, 197, 192, 8),
    "kat-s": (128, 197, 1536, 8),
    "kat-b": (256, 197, 3072, 8),
}
TRAIN_CONFIGS = {"kat-b-train": "kat_b", "kat-s-train": "kat_s", "kat-t-train": "kat_t"}
TRAIN_METRIC = "KAT training throughput, images/s (synthetic 224x224 batch, bf16 autocast, AdamW)"
M1, NDEN = 6, 4
FALLBACK_HBM_GBS = 6650.0


def parse_args(argv=None):
    p = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)  # repeats 100, as the paper and run_bench (cli.py:73-74)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=("b200", "reference"), default="b200")
    p.add_argument("--dtype", choices=("fp32", "bf16", "fp64"), default="fp32")
    p.add_argument("--config", choices=tuple(CONFIGS) + tuple(TRAIN_CONFIGS), default="kat-b")
    # run_bench's workload flags (pkg/src/grkan/cli.py:341-361); unset = the --config preset
    p.add_argument("--batch", type=int, default=None,
                   help="batch per GPU (the config's B; images per GPU for the *-train configs, default 128)")
    p.add_argument("--seqlen", type=int, default=None)
    p.add_argument("--dim", type=int, default=None)
    p.add_argument("--groups", type=int, default=None)
    p.add_argument("--num-coeffs", type=int, default=6, help="numerator coefficients per group (m + 1)")
    p.add_argument("--den-coeffs", type=int, default=4, help="denominator coefficients per group (n)")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--block-size", type=int, default=256,
                   help="row block of the CPU reference's blocked strategy (backward.py:48)")
    p.add_argument("--fused-step", action="store_true",
                   help="time grkan_fwd_bwd -- forward and backward of the same x in one pass (x read once, "
                        "y from the backward's own P and 1/Q) -- as the step; the default times grkan_fwd then "
                        "grkan_bwd and reports the fused step beside it")
    p.add_argument("--strategy", choices=("blocked", "naive", "both"), default="both",
                   help="blocked: K2+K3 timed; naive: the Alg.-1 atomic comparator (K4) timed as the "
                        "backward; both: blocked timed, the comparator reported beside it")
    p.add_argument("--dump", default=None, help="write the final dx as a GRKB tensor dump (cli.py:105-118)")
    p.add_argument("--mode", choices=("fast", "exact"), default="fast")
    p.add_argument("--scaling", choices=("weak", "strong"), default="weak")
    p.add_argument("--e2e-steps", type=int, default=None)
    p.add_argument("--hold-ms", type=float, default=8.0,
                   help="device-side spin before the timed region while the host enqueues it")
    p.add_argument("--collective", choices=("allreduce", "deterministic", "p2p"), default="allreduce",
                   help="da/db exchange: NCCL all-reduce of the 320 B da||db; the world-size-invariant "
                        "path (per-block partials, all-gather, fixed-order fold; SURVEY 8e); or p2p: K3 "
                        "fused with the exchange over CUDA-IPC peer memory (grkan_bwd_p2p, no NCCL)")
    p.add_argument("--e2e-chunks", type=int, default=16,
                   help="row chunks of the streaming e2e pipeline (fill + drain cost one chunk each)")
    p.add_argument("--cpu-sample-batch", type=int, default=64,
                   help="rows B of the bounded CPU-reference sample (KAT-B: 64 of 256)")
    p.add_argument("--cpu-passes", type=int, default=3)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--single-thread-baseline", action=argparse.BooleanOptionalAction, default=True,
                   help="--impl reference: also time the CPU path with one worker (SURVEY 8d)")
    p.add_argument("--fused-mlp", action="store_true",
                   help="*-train configs: GR-KAN rational->Linear pairs with the fused tcgen05 backward")
    p.add_argument("--dist-backend", default="nccl",
                   help="torch.distributed backend for N > 1 (gloo only to exercise the multi-rank "
                        "code path when several ranks share one GPU)")
    args = p.parse_args(argv)
    if args.gpus < 1:
        p.error("--gpus must be >= 1")
    return args


def workload(args):
    """(batch per GPU, seq, dim, groups): the --config preset with run_bench's overrides."""
    batch, seq, dim, groups = CONFIGS[args.config]
    batch = args.batch if args.batch is not None else batch
    seq = args.seqlen if args.seqlen is not None else seq
    dim = args.dim if args.dim is not None else dim
    groups = args.groups if args.groups is not None else groups
    if min(batch, seq, dim, groups) < 1:
        raise SystemExit("error: dimensions must be positive")
    if dim % groups:
        raise SystemExit("error: layout mismatch: dim %d not divisible by groups %d" % (dim, groups))
    if args.num_coeffs < 1 or args.den_coeffs < 0:
        raise SystemExit("error: need at least one numerator coefficient and den_coeffs >= 0")
    return batch, seq, dim, groups


def is_preset(args):
    return (args.batch, args.seqlen, args.dim, args.groups) == (None,) * 4 and \
        (args.num_coeffs, args.den_coeffs) == (M1, NDEN)


def ncu_traffic(args, kind):
    """DRAM bytes per launch for this workload from the committed ncu capture, or None."""
    if not is_preset(args):
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            d = json.load(fh)
        return d["%s/%s/%s/%s" % (args.config, args.dtype, args.mode, kind)]["bytes_per_launch"]
    except Exception:
        return None


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy bandwidth)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# CPU path: the oracle port of the reference (forward_tensor + backward_blocked)
# ---------------------------------------------------------------------------

def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def reference_module():
    """The reference package installed into baseline/_ref (build() / oracle/install_reference.sh),
    or None when that install is absent (then the oracle port stands in)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isfile(os.path.join(ref, "grkan", "backward.py")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import grkan.backward
    import grkan.rational
    return grkan


def cpu_reference_rate(args, shape, batch, passes, warmup=1, workers=None):
    """elements/s of the reference's CPU path (forward_tensor + backward_blocked,
    run_bench --include-forward, pkg/src/grkan/cli.py:178-193) on this host."""
    from oracle import grkan_oracle as orc

    _, seq, dim, groups = shape
    x, u, num, den = orc.bench_inputs(batch, seq, dim, groups, args.num_coeffs, args.den_coeffs, seed=args.seed)
    workers = workers or os.cpu_count() or 1
    ref = reference_module()
    if ref is not None:
        R, B = ref.rational, ref.backward
        layout = R.GroupLayout(dim, groups)
        xt, ut = R.ActivationTensor(x, validated=True), R.ActivationTensor(u, validated=True)
        params = R.GroupRationalParams(num, den)
        plan = B.ExecutionPlan.blocked(batch, seq, layout, args.block_size)

        def step():
            R.forward_tensor(xt, params, layout, validate=False)
            B.backward_blocked(xt, ut, params, plan, workers=workers, validate=False)
        kind, what = "reference", "the reference package grkan (pkg/src/grkan, installed into baseline/_ref)"
    else:
        def step():
            orc.cpu_step(x, u, num, den, block_size=args.block_size, workers=workers)
        kind, what = "port", "the NumPy port of the reference (oracle/grkan_oracle.py)"
    for _ in range(warmup):
        step()
    times = []
    for _ in range(passes):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    mean = statistics.fmean(times)
    return x.size / mean, workers, times, kind, what


def run_reference(args, rank):
    if rank != 0:
        return
    shape = workload(args)
    batch = min(args.cpu_sample_batch, shape[0])
    # each step = one reference fwd+bwd pass over a bounded sample
    rate, workers, times, kind, what = cpu_reference_rate(args, shape, batch, max(1, args.steps),
                                                          warmup=args.warmup)
    ms = statistics.fmean(times) * 1e3
    sample = "%s rows B=%d of %d (E=%d): %s, forward_tensor + backward_blocked (block %d), workers=%d" % (
        args.config, batch, shape[0], batch * shape[1] * shape[2], what, args.block_size, workers)
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f64" if args.dtype == "fp64" else "f32",
        "data": "synthetic (run_bench draw order, seed %d)" % args.seed,
        "config": config_block(args, shape, args.gpus),
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": workers, "kind": kind,
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if args.single_thread_baseline:  # also time workers=1 (one pass, B=4 rows sample)
        r1, _, t1, _, _ = cpu_reference_rate(args, shape, min(4, batch), 1, warmup=0, workers=1)
        line["cpu_baseline"]["single_thread"] = {
            "value": r1, "unit": UNIT, "cores": 1,
            "sample": "%s rows B=%d, workers=1, one pass (%.2f s)" % (args.config, min(4, batch), t1[0])}
    print(json.dumps(line), flush=True)


def config_block(args, shape, world=1):
    batch, seq, dim, groups = shape
    if args.scaling == "strong":  # the global batch is fixed and split over the ranks
        global_batch, batch = batch, max(1, batch // world)
    else:
        global_batch = batch * world
    es = {"fp32": 4, "bf16": 2, "fp64": 8}[args.dtype]
    name = args.config.upper() if is_preset(args) else "custom (%s-based)" % args.config.upper()
    return {
        "workload": "GR-KAN group-rational fwd+bwd, %s shape [B=%d, L=%d, D=%d] per GPU, %d groups, "
                    "degrees (%d,%d)" % (name, batch, seq, dim, groups, args.num_coeffs - 1, args.den_coeffs),
        "batch_per_gpu": batch, "global_batch": global_batch, "seq_len": seq, "dim": dim, "groups": groups,
        "degrees": [args.num_coeffs - 1, args.den_coeffs], "seed": args.seed, "mode": args.mode,
        "io_dtype": args.dtype, "strategy": args.strategy,
        "parallelism": "dp%d" % world, "collective": args.collective,
        "step": ("fused: grkan_fwd_bwd (forward and backward of the same x in one pass)"
                 if getattr(args, "fused_step", False) else "two passes: grkan_fwd then grkan_bwd"),
        "l2": ("inputs larger than L2 (no flush): %d MB per tensor vs 126 MB L2"
               % (batch * seq * dim * es // 2**20)) if batch * seq * dim * es > 126 * 2**20 else
              ("inputs smaller than L2: a >=256 MB buffer is written between timed steps (L2 flush)"),
    }


# ---------------------------------------------------------------------------
# Clock sampling during the timed region (NVML)
# ---------------------------------------------------------------------------

def nvml_index(dev):
    """NVML index of a torch CUDA device (honours CUDA_VISIBLE_DEVICES)."""
    import torch
    try:
        return torch.cuda._get_nvml_device_index(dev)
    except Exception:
        return dev.index or 0


class ClockSampler:
    REASONS = {
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
        0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle",
        0x2: "applications_clocks_setting", 0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.samples = []
        self.mem_mhz = []
        self.power_mw = []
        self.power_inst_mw = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._thr = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
        self.temp_start = None
        if self._nv is not None:  # the first queries are slow (NVML lazy init): not inside the region
            self._sample()
            self.samples, self.power_mw, self.power_inst_mw, self.reasons = [], [], [], 0
            self.mem_mhz = []
            self.temp_start = self._temps()

    def _temps(self):
        """GPU and HBM temperature (C), read outside the timed region: HBM refreshes
        more often when hot, which costs bandwidth without any clock-event reason."""
        nv = self._nv
        out = {}
        try:
            out["gpu"] = nv.nvmlDeviceGetTemperature(self._h, nv.NVML_TEMPERATURE_GPU)
        except Exception:
            pass
        try:
            fv = nv.nvmlDeviceGetFieldValues(self._h, [getattr(nv, "NVML_FI_DEV_MEMORY_TEMP", 82)])[0]
            if fv.nvmlReturn == 0:
                out["mem"] = int(fv.value.uiVal)
        except Exception:
            pass
        return out

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            self._sample()
            time.sleep(0.002)

    def _sample(self):
        nv = self._nv
        try:
            self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
            self.mem_mhz.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_MEM))
            self.reasons |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(self._h))
            self.power_mw.append(nv.nvmlDeviceGetPowerUsage(self._h))
        except Exception:
            pass
        try:  # instantaneous board power (nvmlDeviceGetPowerUsage is a ~1 s average)
            fv = nv.nvmlDeviceGetFieldValues(self._h, [nv.NVML_FI_DEV_POWER_INSTANT])[0]
            if fv.nvmlReturn == 0:
                self.power_inst_mw.append(fv.value.uiVal)
        except Exception:
            pass

    def poll_until(self, begin, end, period_s=0.0005):
        """Sample in the calling thread from when the device reaches event `begin`
        until it completes event `end` (host otherwise idle)."""
        if self._nv is None:
            return
        while not begin.query():
            time.sleep(period_s / 4)
        if os.environ.get("GRKAN_BENCH_NVML_POLL", "1") == "0":  # diagnostic: one sample, then wait
            self._sample()
            while not end.query():
                time.sleep(period_s)
            return
        while not end.query():
            self._sample()
            time.sleep(period_s)
        if not self.samples:
            self._sample()

    def start(self):
        if self._nv is not None:
            self._thr = threading.Thread(target=self._run, daemon=True)
            self._thr.start()

    def stop(self):
        if self._thr is not None:
            self._stop.set()
            self._thr.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        reasons = [name for bit, name in self.REASONS.items() if self.reasons & bit and bit != 0x1]
        out = {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
               "reasons": reasons, "reasons_mask": hex(self.reasons), "samples": len(self.samples)}
        try:  # power draw vs the enforced limit: a power-capped run shows median power at the limit
            out["power_w_median"] = statistics.median(self.power_mw) / 1e3 if self.power_mw else None
            if self.power_inst_mw:
                out["power_inst_w_median"] = statistics.median(self.power_inst_mw) / 1e3
                out["power_inst_w_max"] = max(self.power_inst_mw) / 1e3
            out["power_limit_w"] = self._nv.nvmlDeviceGetEnforcedPowerLimit(self._h) / 1e3
        except Exception:
            pass
        if self.mem_mhz:
            out["mem_mhz"] = statistics.median(self.mem_mhz)
            out["mem_mhz_min"] = min(self.mem_mhz)
        if self.temp_start is not None:
            out["temp_c"] = {"before": self.temp_start, "after": self._temps()}
        return out


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def world_ok(args):
    return args.scaling == "weak" or args.gpus == 1


def run_b200(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2505_13813_b200 import _native as N
    from paper_2505_13813_b200 import ops
    from paper_2505_13813_b200.module import GroupRationalFn

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    # diagnostic (profiles/r2/s4/temp): GRKAN_BENCH_PREALLOC_GB=N maps, touches and
    # releases N GB before the workload's own buffers are allocated
    pre_gb = float(os.environ.get("GRKAN_BENCH_PREALLOC_GB", "0"))
    if pre_gb > 0:
        tmp = torch.empty(int(pre_gb * 2**30), dtype=torch.uint8, device=dev)
        tmp.fill_(0)
        torch.cuda.synchronize()
        del tmp
        torch.cuda.empty_cache()
    shape = workload(args)
    batch, seq, dim, groups = shape
    if args.scaling == "strong":
        batch = max(1, batch // world)
    m1, nden = args.num_coeffs, args.den_coeffs
    tdt = {"fp32": torch.float32, "bf16": torch.bfloat16, "fp64": torch.float64}[args.dtype]
    es = {"fp32": 4, "bf16": 2, "fp64": 8}[args.dtype]
    cdt = torch.float64 if args.dtype == "fp64" else torch.float32  # coefficient / gradient dtype
    ces = 8 if args.dtype == "fp64" else 4
    E = batch * seq * dim
    rows = batch * seq
    dt_code = {"fp32": N.DT_F32, "bf16": N.DT_BF16, "fp64": N.DT_F64}[args.dtype]
    flags = N.FLAG_EXACT if args.mode == "exact" else N.FLAG_FAST

    # run_bench's inputs (pkg/src/grkan/cli.py:143-158): x, upstream, numerator,
    # denominator from one default_rng(seed) -- rank 0 gets exactly the reference's
    # draw; rank r > 0 draws from default_rng([seed, r]) (independent shards).
    # bf16 runs round the fp32 draw.  The coefficients are identical on every rank.
    rng = np.random.default_rng(args.seed if rank == 0 else [args.seed, rank])
    host_dt = np.float64 if args.dtype == "fp64" else np.float32

    def draw():
        t = torch.empty((batch, seq, dim), dtype=tdt, device=dev)
        step_b = max(1, (64 << 20) // (seq * dim))  # chunked: bounded host memory
        for b0 in range(0, batch, step_b):
            nb = min(step_b, batch - b0)
            t[b0:b0 + nb].copy_(torch.from_numpy(rng.standard_normal((nb, seq, dim)).astype(host_dt)))
        return t

    x = draw()
    dy = draw()
    crng = np.random.default_rng(args.seed)
    if rank == 0:
        crng = rng  # continue the reference's stream after x and upstream
    num = crng.standard_normal((groups, m1))
    den = crng.standard_normal((groups, nden))
    if world > 1:  # every rank must use rank 0's coefficients
        import torch.distributed as dist_
        cbuf = torch.from_numpy(np.concatenate([num.ravel(), den.ravel()])).to(dev)
        dist_.broadcast(cbuf, 0)
        cbuf = cbuf.cpu().numpy()
        num, den = cbuf[: groups * m1].reshape(groups, m1), cbuf[groups * m1:].reshape(groups, nden)
    a = torch.from_numpy(num).to(cdt).to(dev)
    b = torch.from_numpy(den).to(cdt).to(dev).reshape(groups, nden)
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    grads = torch.empty(groups * (m1 + nden), dtype=cdt, device=dev)  # da || db, one buffer
    da = grads[: groups * m1].view(groups, m1)
    db = grads[groups * m1:].view(groups, nden)
    ws_bytes = ops.workspace_bytes(rows, dim, groups, m1, nden, tdt)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    L = N.lib()
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    # workloads smaller than L2 (126 MB): write a 256 MB buffer between timed steps
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if 3 * es * E <= 256 << 20 else None
    st_naive = torch.zeros(ops.STATUS_WORDS, dtype=torch.int32, device=dev)

    def fwd():
        rc = L.grkan_fwd(x.data_ptr(), y.data_ptr(), a.data_ptr(), ops._ptr(b), rows, dim, groups,
                         m1, nden, dt_code, flags, None, sp)
        assert rc == 0, N.last_error()

    def bwd():
        join_comm()  # the previous step's all-reduce still reads grads
        if args.strategy == "naive":  # the paper's Alg. 1: per-element atomics (K4) as the backward
            rc = L.grkan_bwd_atomic(x.data_ptr(), dy.data_ptr(), a.data_ptr(), ops._ptr(b), dx.data_ptr(),
                                    da.data_ptr(), ops._ptr(db), rows, dim, groups, m1, nden, dt_code,
                                    flags, None, sp)
        else:
            rc = L.grkan_bwd(x.data_ptr(), dy.data_ptr(), a.data_ptr(), ops._ptr(b), dx.data_ptr(),
                             da.data_ptr(), ops._ptr(db), ws.data_ptr(), ws_bytes, rows, dim, groups,
                             m1, nden, dt_code, flags, sp)
        assert rc == 0, N.last_error()

    # da||db all-reduce on a side stream: it overlaps the next step's forward
    # (the next K3 waits for it before overwriting the buffer); the timed
    # region ends only after the last one completes.
    # (NCCL only: gloo -- several ranks sharing one GPU in tests -- stages CUDA
    # tensors through the host and runs in stream order on the main stream)
    comm = torch.cuda.Stream(dev) if world > 1 and args.dist_backend == "nccl" else None
    bwd_done = torch.cuda.Event()

    comm_ev = []  # (start, end) on the comm stream, timed steps only

    def allreduce(timed=False):
        if world > 1 and comm is None:
            dist.all_reduce(grads)
        elif world > 1:
            bwd_done.record(stream)
            comm.wait_event(bwd_done)
            with torch.cuda.stream(comm):
                if timed:
                    comm_ev.append((torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)))
                    comm_ev[-1][0].record(comm)
                dist.all_reduce(grads)
                if timed:
                    comm_ev[-1][1].record(comm)

    def join_comm():
        if comm is not None:
            stream.wait_stream(comm)

    if args.collective == "p2p":
        from paper_2505_13813_b200.parallel import PeerExchange

        pex = PeerExchange(groups, m1, nden, dev)
        ws_p2p = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)

        def bwd():
            pex.epoch += 1
            rc = L.grkan_bwd_p2p(x.data_ptr(), dy.data_ptr(), a.data_ptr(), b.data_ptr(), dx.data_ptr(),
                                 da.data_ptr(), db.data_ptr(), ws_p2p.data_ptr(), ws_bytes, rows, dim, groups,
                                 m1, nden, dt_code, flags, pex.ptrs.data_ptr(), pex.rank, pex.world, pex.epoch, sp)
            assert rc == 0, N.last_error()

        def allreduce(timed=False):
            pass  # the exchange happened inside bwd's reduce kernel

    if args.collective == "deterministic":
        # world-size-invariant da/db: K2 writes one partial per 128-row block,
        # the ranks all-gather them (global block order = rank order) and every
        # rank runs the same fixed-order K3 fold (parallel.deterministic_backward)
        rb = ops.det_block_rows(dim, groups, tdt)
        n_blk = -(-rows // rb)
        part = torch.empty((n_blk, groups, m1 + nden), dtype=cdt, device=dev)
        gathered = torch.empty((world * n_blk, groups, m1 + nden), dtype=cdt, device=dev)
        parts_list = list(gathered.chunk(world))
        st = torch.zeros(ops.STATUS_WORDS, dtype=torch.int32, device=dev)

        def bwd():
            rc = L.grkan_bwd_partials(x.data_ptr(), dy.data_ptr(), a.data_ptr(), b.data_ptr(), dx.data_ptr(),
                                      part.data_ptr(), part.numel() * ces, rows, dim, groups, m1, nden, dt_code,
                                      flags, None, sp)
            assert rc == 0, N.last_error()

        def allreduce(timed=False):
            src = part
            if world > 1:
                if args.dist_backend == "nccl":
                    dist.all_gather_into_tensor(gathered, part)
                else:
                    dist.all_gather(parts_list, part)
                src = gathered
            rc = L.grkan_reduce_partials(src.data_ptr(), src.shape[0], groups, m1, nden, da.data_ptr(),
                                         ops._ptr(db), N.DT_F64 if args.dtype == "fp64" else N.DT_F32, st.data_ptr(), sp)
            assert rc == 0, N.last_error()

    def fused():
        join_comm()
        rc = L.grkan_fwd_bwd(x.data_ptr(), dy.data_ptr(), a.data_ptr(), ops._ptr(b), y.data_ptr(), dx.data_ptr(),
                             da.data_ptr(), ops._ptr(db), ws.data_ptr(), ws_bytes, rows, dim, groups, m1, nden,
                             dt_code, flags, sp)
        assert rc == 0, N.last_error()

    fused_ok = args.strategy != "naive" and args.collective == "allreduce"
    if args.fused_step:
        if not fused_ok:
            raise SystemExit("--fused-step needs the blocked strategy and --collective allreduce")

        def fwd():
            pass

        bwd = fused

    # warm-up: at least W steps and at least WARM_S of device work (clocks and
    # memory settled on a fresh box), untimed.  (A 1 s warm-up was tried: the
    # fp32 backward then met sw_power_cap inside the timed steps more, not less.)  Every step carries a collective,
    # so every rank must run the same number: the time-based extension is
    # agreed across ranks (the slowest rank's count) before it runs.
    def warm(n):
        for i in range(n):
            fwd(); bwd(); allreduce()
            if (i + 1) % 20 == 0:
                torch.cuda.synchronize()
        join_comm()
        torch.cuda.synchronize()

    n_min = max(3, args.warmup)
    t_w = time.perf_counter()
    warm(n_min)
    el = time.perf_counter() - t_w
    extra = 0 if el >= WARM_S else int(math.ceil((WARM_S - el) / max(el / n_min, 1e-6)))
    if world > 1:
        t_extra = torch.tensor([extra], dtype=torch.int64, device=dev)
        dist.all_reduce(t_extra, op=dist.ReduceOp.MAX)
        extra = int(t_extra.item())
    warm(extra)
    # host cost of enqueueing one step (events included), to size the hold below
    t_h = time.perf_counter()
    for _ in range(4):
        e_tmp = torch.cuda.Event(enable_timing=True)
        e_tmp.record(stream)
        fwd(); bwd(); allreduce()
    host_step_ms = (time.perf_counter() - t_h) / 4 * 1e3
    torch.cuda.synchronize()

    K = args.steps
    # two events per step in the timed region: at the step boundary and between
    # the forward and the backward (each event record drains the stream, ~1-2 us;
    # the four per step of round 1 added ~10 us to a KAT-B step)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    evm = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    eve = [torch.cuda.Event(enable_timing=True) for _ in range(K)] if flush_buf is not None else None
    # an exchange on the compute stream (N > 1 without the side stream): its own event
    evc = [torch.cuda.Event(enable_timing=True) for _ in range(K)] if world > 1 and comm is None else None
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(nvml_index(dev))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # hold the stream with a short device-side spin while the host enqueues all
    # K steps, so host-side jitter cannot open launch gaps inside the timed region
    hold_ms = max(args.hold_ms, 2.0 * K * host_step_ms + 2.0)
    torch.cuda._sleep(int(hold_ms * 1e-3 * 1.965e9))
    t_enq = time.perf_counter()
    t_start.record(stream)
    for k in range(K):
        if flush_buf is not None:  # L2 flush outside the step's events (workload < L2)
            flush_buf.zero_()
        evs[k].record(stream)
        fwd()
        evm[k].record(stream)
        bwd()
        if evc is not None:
            evc[k].record(stream)
        allreduce(timed=True)
        if eve is not None:
            eve[k].record(stream)
    if args.collective == "allreduce":
        join_comm()
    t_end.record(stream)
    host_enqueue_ms = (time.perf_counter() - t_enq) * 1e3
    # the host is idle now: sample the clocks from this thread until the timed
    # region has drained (only while the device is past the hold)
    sampler.poll_until(t_start, t_end)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ends = eve if eve is not None else evs[1:] + [t_end]
    step_ms = [evs[k].elapsed_time(ends[k]) for k in range(K)]
    ms_total = sum(step_ms) if eve is not None else t_start.elapsed_time(t_end)
    fwd_ms = statistics.fmean(evs[k].elapsed_time(evm[k]) for k in range(K))
    bwd_end = evc if evc is not None else ends
    bwd_ms = statistics.fmean(evm[k].elapsed_time(bwd_end[k]) for k in range(K))  # K2 + K3
    if comm_ev:  # overlapped all-reduce: its own duration on the comm stream
        coll_ms = statistics.fmean(c0.elapsed_time(c1) for c0, c1 in comm_ev)
    elif evc is not None:
        coll_ms = statistics.fmean(evc[k].elapsed_time(ends[k]) for k in range(K))
    else:
        coll_ms = 0.0
    if world > 1:
        t = torch.tensor([ms_total, fwd_ms, bwd_ms, coll_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total, fwd_ms, bwd_ms, coll_ms = t.tolist()
    ms_step = ms_total / K
    # after the timed region: every rank must hold the same da||db (the
    # deterministic and peer-memory paths bitwise by construction)
    coll_check = None
    if world > 1:
        torch.cuda.synchronize()
        mine = grads.detach().cpu()
        allg = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather_object(allg, mine)
        same = all(torch.equal(g, allg[0]) for g in allg)
        coll_check = {"ranks": world, "bitwise_identical": same,
                      "max_abs_diff": max(float((g - allg[0]).abs().max()) for g in allg)}
    # per-step device times (step boundary to step boundary): mean +- CI95 with
    # the normal approximation, as the reference reports (verification.py:344-349)
    ci95_ms = 1.96 * statistics.stdev(step_ms) / math.sqrt(len(step_ms)) if len(step_ms) > 1 else None
    value = world * E / (ms_step / 1e3)

    # ---- the fused forward + backward step beside the two-pass step (same inputs) ---------
    fused_us = None
    if fused_ok and not args.fused_step and world == 1:
        for _ in range(3):
            fused()
        torch.cuda.synchronize()
        fe = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        for k in range(K):
            if flush_buf is not None:  # L2 flush outside the step's events (workload < L2)
                flush_buf.zero_()
            fe[k][0].record(stream)
            fused()
            fe[k][1].record(stream)
        torch.cuda.synchronize()
        fused_us = statistics.fmean(e0.elapsed_time(e1) for e0, e1 in fe) * 1e3
    elif args.fused_step:
        fused_us = bwd_ms * 1e3

    if args.dump and rank == 0:  # run_bench --dump: the final dx as a GRKB tensor dump
        from paper_2505_13813_b200 import grkb
        grkb.save(args.dump, dx.float() if args.dtype == "bf16" else dx)

    # ---- the paper's Alg. 1 comparator (per-element atomicAdd), same inputs ----------------
    alg1_us = None
    if world == 1 and args.strategy == "both":
        st = torch.zeros(ops.STATUS_WORDS, dtype=torch.int32, device=dev)
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for it in range(2):
            ea.record(stream)
            rc = L.grkan_bwd_atomic(x.data_ptr(), dy.data_ptr(), a.data_ptr(), ops._ptr(b), dx.data_ptr(),
                                    da.data_ptr(), ops._ptr(db), rows, dim, groups, m1, nden, dt_code,
                                    flags, st.data_ptr(), sp)
            eb.record(stream)
            assert rc == 0, N.last_error()
        torch.cuda.synchronize()
        alg1_us = ea.elapsed_time(eb) * 1e3

    # ---- e2e with host buffers: pinned x, dy in; y, dx, da, db out every step ----------
    # (a) streaming API: chunked, copy-in / compute / copy-out overlapped on 3 streams
    # (b) plain autograd on the whole tensor (GroupRationalFn.apply + backward)
    from paper_2505_13813_b200.streaming import HostPipeline

    Ke = args.e2e_steps or min(K, 10)
    xh = torch.empty((batch, seq, dim), dtype=tdt, pin_memory=True)
    dyh = torch.empty_like(xh, pin_memory=True)
    xh.copy_(x.cpu())
    dyh.copy_(dy.cpu())
    yh = torch.empty_like(xh, pin_memory=True)
    dxh = torch.empty_like(xh, pin_memory=True)
    gh = torch.empty(groups * (m1 + nden), dtype=cdt, pin_memory=True)
    exact = args.mode == "exact"
    del y, dx, ws
    torch.cuda.empty_cache()
    pipe = HostPipeline(dev, dim, groups, m1, nden, tdt,
                        chunk_rows=max(rows // args.e2e_chunks, -(-(4 << 20) // (dim * es))))

    def e2e_stream():
        da_, db_ = pipe.fwd_bwd(xh, dyh, a, b, yh, dxh, exact=exact)
        g = torch.cat([da_.reshape(-1), db_.reshape(-1)])
        if world > 1:
            dist.all_reduce(g)
        gh.copy_(g, non_blocking=True)

    ap = torch.nn.Parameter(a.clone())
    bp = torch.nn.Parameter(b.clone())

    def e2e_autograd():
        xd = xh.to(dev, non_blocking=True).requires_grad_(True)
        dyd = dyh.to(dev, non_blocking=True)
        yd = GroupRationalFn.apply(xd, ap, bp, exact)
        yd.backward(dyd)
        g = torch.cat([ap.grad.reshape(-1), bp.grad.reshape(-1)])
        if world > 1:
            dist.all_reduce(g)
        yh.copy_(yd.detach(), non_blocking=True)
        dxh.copy_(xd.grad, non_blocking=True)
        gh.copy_(g, non_blocking=True)
        ap.grad = None
        bp.grad = None

    def time_e2e(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(Ke):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / Ke
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = t.item()
        return ms

    e2e_ms = time_e2e(e2e_stream)
    e2e_auto_ms = time_e2e(e2e_autograd)
    e2e_value = world * E / (e2e_ms / 1e3)

    # (c) the reference-facing API itself: the shim's forward_tensor + backward_blocked
    # on pageable NumPy arrays (what a caller of the reference holds), host-synchronous,
    # wall clock; fp32 only (the reference has no bf16), one process
    shim = None
    if args.dtype == "fp32" and world == 1:
        from paper_2505_13813_b200 import grkan as G
        xt = G.ActivationTensor(np.array(xh.numpy()))
        ut = G.ActivationTensor(np.array(dyh.numpy()))
        params = G.GroupRationalParams(a.double().cpu().numpy(), b.double().cpu().numpy())
        layout = G.GroupLayout(dim, groups)
        plan = G.ExecutionPlan.blocked(batch, seq, layout)

        def shim_step():
            G.forward_tensor(xt, params, layout, validate=False, exact=exact)
            G.backward_blocked(xt, ut, params, plan, validate=False, exact=exact)

        shim_step()
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            shim_step()
            ts.append(time.perf_counter() - t0)
        shim_ms = statistics.fmean(ts) * 1e3
        shim = {"value": E / (shim_ms / 1e3), "ms_per_step": shim_ms, "steps": len(ts),
                "h2d_bytes_per_step": 3 * es * E, "d2h_bytes_per_step": 2 * es * E + 4 * groups * (m1 + nden),
                "api": "paper_2505_13813_b200.grkan.forward_tensor + backward_blocked (the reference's "
                       "functions and types; pageable NumPy in/out, wall clock)"}
        del xt, ut
    del xh, dyh, yh, dxh, pipe

    if rank != 0:
        return
    peak, peak_src = peaks()
    bwd_bytes = (4 if args.fused_step else 3) * es * E  # fused step: x, dy read once; y, dx written
    fwd_bytes = 2 * es * E
    bwd_gbs = bwd_bytes / (bwd_ms / 1e3) / 1e9
    fwd_gbs = fwd_bytes / (fwd_ms / 1e3) / 1e9 if not args.fused_step else 0.0
    fused_blk = None if fused_us is None else {
        "us": fused_us, "elements_per_s": world * E / (fused_us / 1e6),
        "algorithmic_bytes": 4 * es * E, "gbs": 4 * es * E / (fused_us / 1e6) / 1e9,
        "frac": 4 * es * E / (fused_us / 1e6) / 1e9 / peak,
        "gbs_fwd_plus_bwd_bytes": 5 * es * E / (fused_us / 1e6) / 1e9,
        "api": "grkan_fwd_bwd / ops.rational_forward_backward (y, dx, da, db of the same x in one pass)"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms_step, "ms_per_step_ci95": ci95_ms,
        "timing": {"hold_ms": hold_ms, "host_enqueue_ms": host_enqueue_ms,
                   "note": "timed steps enqueued behind a device-side hold longer than the host enqueue; "
                           "two CUDA events per step (step boundary, forward | backward)"},
        "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f32" if args.dtype == "fp32" else "bf16-io/f32-math",
        "data": "synthetic: x, dy ~ N(0,1) (torch seeded per rank), coefficients ~ N(0,1) "
                "(run_bench protocol, pkg/src/grkan/cli.py:146-158)",
        "config": config_block(args, shape, world),
        "hbm_gbs": (5 * es * E) / (ms_step / 1e3) / 1e9,
        "roofline": {
            "bound": "hbm", "kernel": ("grkan_fwd_bwd (K2 with the forward fused + K3 reduce)" if args.fused_step
                                       else "grkan_bwd (K2 bwd_main + K3 reduce)"),
            "achieved": bwd_gbs, "peak": peak, "unit": "GB/s", "frac": bwd_gbs / peak,
            "peak_source": peak_src, "traffic": ncu_traffic(args, "bwd") if world_ok(args) else None,
            "algorithmic_bytes_per_launch": bwd_bytes, "launch_us": bwd_ms * 1e3,
        },
        "kernels": {
            "fwd_us": fwd_ms * 1e3, "fwd_gbs": fwd_gbs, "fwd_frac": fwd_gbs / peak,
            "fwd_traffic": ncu_traffic(args, "fwd"),
            "bwd_us": bwd_ms * 1e3, "bwd_gbs": bwd_gbs, "bwd_frac": bwd_gbs / peak,
            "collective": args.collective, "collective_us": coll_ms * 1e3,
            "collective_check": coll_check,
            "fused_step": fused_blk,
        },
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 2 * es * E,
                "d2h_bytes_per_step": 2 * es * E + ces * groups * (m1 + nden),
                "ms_per_step": e2e_ms,
                "api": "paper_2505_13813_b200.streaming.HostPipeline.fwd_bwd (pinned host x, dy -> "
                       "y, dx, da, db; chunked, copies overlapped with compute)",
                "autograd_ms_per_step": e2e_auto_ms,
                "autograd_value": world * E / (e2e_auto_ms / 1e3),
                "reference_api": shim},
        "clocks": sampler.summary(),
        "gpu_launches": (2 if args.strategy == "naive" or args.fused_step else 3) * K,
        "dist": None if world == 1 else {
            "backend": dist.get_backend(), "world_size": dist.get_world_size(),
            "nccl_version": ".".join(map(str, torch.cuda.nccl.version())) if args.dist_backend == "nccl" else None},
        "alg1_atomic_comparator": None if alg1_us is None else {
            "bwd_us": alg1_us, "speedup_of_staged_bwd": alg1_us / (bwd_ms * 1e3),
            "note": "paper: FlashKAT bwd 140.5x faster than KAT's atomic bwd on RTX 4060 Ti (PAPER.md:402)"},
    }
    if world == 1 and not args.no_cpu_baseline:
        sb = min(args.cpu_sample_batch, shape[0])
        rate, workers, times, kind, what = cpu_reference_rate(args, shape, sb, args.cpu_passes)
        line["cpu_baseline"] = {
            "value": rate, "unit": UNIT, "cores": workers, "kind": kind, "cpu_model": cpu_model(),
            "sample": "%s with B=%d (E=%d): %s, forward_tensor + backward_blocked (block %d, %d threads), "
                      "%d timed passes after 1 warm-up"
                      % (args.config, sb, sb * shape[1] * shape[2], what, args.block_size, workers, len(times)),
        }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# Config 4: full KAT training step -- images/s, not the headline
# ---------------------------------------------------------------------------

def run_train(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2505_13813_b200 import kat

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    torch.manual_seed(1234 + rank)
    model = getattr(kat, TRAIN_CONFIGS[args.config])(fused_mlp=args.fused_mlp).to(dev)
    if world > 1:
        model = torch.nn.parallel.DistributedDataParallel(model, device_ids=[local_rank])
    opt = torch.optim.AdamW(model.parameters(), lr=1e-4, weight_decay=0.05, fused=True)
    B = args.batch or 128
    imgs = torch.randn(B, 3, 224, 224, device=dev)
    labels = torch.randint(0, 1000, (B,), device=dev)
    loss_fn = torch.nn.CrossEntropyLoss()

    def step():
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = loss_fn(model(imgs), labels)
        loss.backward()
        opt.step()
        opt.zero_grad(set_to_none=True)
        return loss

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(nvml_index(dev))
    sampler.start()
    e0.record()
    for _ in range(args.steps):
        loss = step()
    e1.record()
    torch.cuda.synchronize()
    sampler.stop()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    if rank == 0:
        n_params = sum(p.numel() for p in model.parameters())
        print(json.dumps({
            "metric": TRAIN_METRIC, "value": world * B / (ms / 1e3), "unit": "images/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic images N(0,1), random labels",
            "config": {"workload": args.config, "model": TRAIN_CONFIGS[args.config], "params": n_params,
                       "batch_per_gpu": B, "global_batch": B * world, "parallelism": "ddp%d" % world,
                       "fused_mlp": bool(args.fused_mlp)},
            "final_loss": float(loss.item()), "clocks": sampler.summary(),
            "paper_h200_images_s": {"kat_b": 1801.75, "kat_s": 3741.91, "kat_t": 6317.90}[TRAIN_CONFIGS[args.config]],
        }), flush=True)


# minimum warm-up of device work before the timed steps (seconds)
WARM_S = float(os.environ.get("GRKAN_BENCH_WARM_S", "0.15"))

# a rank that never arrives fails the collective (and the run) instead of hanging it
PG_TIMEOUT = __import__("datetime").timedelta(seconds=float(os.environ.get("GRKAN_PG_TIMEOUT_S", "600")))


def free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_ranks(args, argv):
    """--gpus N with no launcher: re-execute this script under torch.distributed.run
    with N ranks on this node (127.0.0.1 rendezvous), forwarding its output."""
    import subprocess

    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)]
    cmd += list(sys.argv[1:] if argv is None else argv)
    env = dict(os.environ, GRKAN_BENCH_SPAWNED="1")
    if args.dist_backend == "gloo":
        # single node: gloo's transport on loopback (its default device follows the
        # hostname, which need not resolve to this box inside a container)
        env.setdefault("GLOO_SOCKET_IFNAME", "lo")
    return subprocess.run(cmd, env=env).returncode


def main(argv=None):
    args = parse_args(argv)
    if os.environ.get("GRKAN_BENCH_TRACE_AFTER"):  # diagnostics: dump every thread's stack, then exit
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["GRKAN_BENCH_TRACE_AFTER"]), exit=True)
    env_world = os.environ.get("WORLD_SIZE")
    world = int(env_world or "1")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":  # rank 0 alone times the CPU path, however it was launched
        run_reference(args, rank)
        return 0
    if env_world is None and args.gpus > 1:
        return spawn_ranks(args, argv)
    if world != args.gpus:
        print("error: --gpus %d but WORLD_SIZE=%d: launch one rank per GPU (or omit the launcher and let "
              "bench.py spawn --gpus ranks itself)" % (args.gpus, world), file=sys.stderr)
        return 2
    if world > 1:
        import torch
        import torch.distributed as dist

        ngpu = torch.cuda.device_count()
        if args.dist_backend == "nccl" and ngpu < world:
            print("error: %d ranks over NCCL need %d GPUs, this node has %d" % (world, world, ngpu),
                  file=sys.stderr)
            return 2
        local_rank = local_rank % ngpu  # ranks may share a GPU when testing with gloo
        torch.cuda.set_device(local_rank)
        if args.dist_backend == "nccl":
            # communicator setup (ranks, NVLink/NVLS transport) goes to stderr, not the JSON stdout
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank), timeout=PG_TIMEOUT)
        else:
            dist.init_process_group(args.dist_backend, timeout=PG_TIMEOUT)
        assert dist.get_world_size() == args.gpus, (dist.get_world_size(), args.gpus)
    try:
        if args.config in TRAIN_CONFIGS:
            run_train(args, rank, world, local_rank)
            return 0
        run_b200(args, rank, world, local_rank)
        return 0
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
