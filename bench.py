#!/usr/bin/env python
"""bench.py -- XPipe hot path on B200: pipeline samples/s (BASELINE.json metric) with the
dominant kernel's roofline, the end-to-end number through the public API, and the CPU oracle
as the reported baseline.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload vgg16|mlp|sweep] [--minibatches M] [--stages S]

A step = one xpipe_step call feeding M mini-batches (N=128 samples, T=4 micro-batches of 32)
into the running pipeline: every row of the hot path (schedule, Eq. (1)/(2) staleness, W_hat
materialisation, stage conv/linear compute under W_hat, hand-offs, loss, backward, the fused
Adam+prediction sweep) runs on the GPU.  Inputs already resident in HBM for `value`; `e2e`
feeds host (pinned) buffers through the same API call with the H2D copies inside.
Stages K = number of GPUs unless --stages is given (config C2 names 4 stages: --stages 4 on
one GPU maps the 4 stages onto one device).
"""
import argparse
import json
import os

# the library's default (paper_1911_04610_b200/xpipe.py): 32 hardware work queues, set before
# torch creates the CUDA context
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "pipeline samples/sec (VGG-16 synthetic CIFAR-10, XPipe Adam+prediction)"
METRICS = {"resnet101": "pipeline samples/sec (ResNet-101 synthetic Tiny-ImageNet 64x64, XPipe Adam+prediction)",
           "inception": "pipeline samples/sec (Inception-V3 synthetic Tiny-ImageNet 64x64, XPipe Adam+prediction)",
           "mlp": "pipeline samples/sec (MLP 784-256-256-256-10, XPipe Adam+prediction)"}
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


class Clocks:
    """Sample nvidia-smi clocks and throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.samples, self.stop_ev = device, [], threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop_ev.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    self.samples.append([x.strip() for x in line.split(",")])
            except Exception:
                pass
            self.stop_ev.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop_ev.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 5 + i and s[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# BASELINE.json configs: default stage count on one GPU (the config's K) and the workload text
DEFAULT_STAGES = {"mlp": 2, "vgg16": 4, "resnet101": 8, "inception": 4}
WORKLOAD_TEXT = {"mlp": "MLP 784-256-256-256-10 (configs[0])",
                 "vgg16": "VGG-16 on synthetic CIFAR-10 32x32 (BASELINE configs[1])",
                 "resnet101": "ResNet-101 on synthetic Tiny-ImageNet 64x64 (BASELINE configs[2])",
                 "inception": "Inception-V3 on synthetic Tiny-ImageNet 64x64 (BASELINE configs[3])"}


def workload_model(name, K=1, image=64, micro=0, T=0):
    """(layers, input shape, classes, input kind, mini-batch N, micro-batches T, precision) of a
    BASELINE config; DAG models get explicit unit-based stages for K (R17).  image=224: the
    paper's upscaled Tiny-ImageNet with the unmodified Inception stem;
    micro / T override the micro-batch size and count (50*T on 2 GPUs, 100*T on 4)."""
    import synthetic as S
    from synthetic.models import resnet101, inception_v3, assign_stages
    if name == "mlp":
        return S.mlp(), (784, 1, 1), 10, "mnist", 32, 4, "fp32"
    if name in ("resnet101", "inception"):
        if name == "resnet101":
            L, units = resnet101(classes=200)
            T0, n0 = 8, 32
        else:
            L, units = inception_v3(classes=200, stem_pad=image < 75)
            T0, n0 = 4, 32
        T = T or T0
        n = micro or n0
        return assign_stages(L, units, K), (3, image, image), 200, "imagenet", n * T, T, "bf16"
    return S.vgg16_cifar(), (3, 32, 32), 10, "cifar", 128, 4, "bf16"


def measured_unit_costs(L, units, shape, classes, kind, N, T, prec, sched, minibatches=8, max_groups=16):
    """Per-unit device cost for the cost-balanced partition ("a contiguous linear
    partition minimising max_k(t_compute,k + t_sweep,k), with per-unit times measured on the
    device").  The model runs on this GPU with every unit its own pipeline stage (or, beyond
    max_groups units, every group of a forward-MAC-balanced max_groups-way split), all stages on
    one stream (cfg.serialize: no overlap, so a stage's busy time is its own cost), with per-op
    timing: busy_ms[g] = the union of stage g's forward / backward op intervals including its
    hand-offs and its Adam + prediction sweep.  A group's time is shared among its units by
    their forward MACs.  Returns the per-unit cost in ms per step."""
    import synthetic as S
    from synthetic.models import unit_macs, balanced_stages
    from paper_1911_04610_b200 import XPipe
    nu = max(units) + 1
    macs = unit_macs(L, units, shape)
    G = min(nu, max_groups)
    if G == nu:
        Lg = [l.with_stage(units[i]) for i, l in enumerate(L)]
        group_of_unit = list(range(nu))
    else:
        Lg = balanced_stages(L, units, macs, G)
        group_of_unit = [0] * nu
        for i, l in enumerate(Lg):
            group_of_unit[units[i]] = l.stage
    P = S.make_params(Lg, 1)
    x, y = S.make_inputs(minibatches * N, shape, classes, 1, kind=kind)
    m = XPipe(Lg, G, T, N, 1e-4, (0.9, 0.999), 1e-8, shape, classes, params=P, precision=prec, serialize=True,
              timing=1, graphs=False, watchdog_ms=300000, **{k: v for k, v in sched.items() if k != "fb_overlap"})
    try:
        m.step(x, y, minibatches)          # fill the pipeline (allocations, first captures)
        m.step(x, y, minibatches)          # steady state, timed per op on the device
        busy = m.last_stats.timing(G)["busy_ms"]
    finally:
        m.close()
    gmacs = [0.0] * G
    for u in range(nu):
        gmacs[group_of_unit[u]] += macs[u]
    return [busy[group_of_unit[u]] * (macs[u] / gmacs[group_of_unit[u]] if gmacs[group_of_unit[u]] else 1.0)
            for u in range(nu)]


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline_single_thread(workload, seconds=8.0):
    """The same oracle measurement on one host thread (1 thread and all cores), in a
    subprocess so OpenMP starts with OMP_NUM_THREADS=1; samples/s or None."""
    code = ("import sys, json; sys.path.insert(0, %r); import bench; "
            "r = bench.cpu_baseline(%r, seconds=%r, single_thread=False); print(json.dumps(r['value']))"
            % (os.path.dirname(os.path.abspath(__file__)), workload, seconds))
    env = dict(os.environ, OMP_NUM_THREADS="1")
    try:
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=120)
        v = float(out.stdout.strip().splitlines()[-1])
        return {"value": v, "unit": "samples/s", "cores": 1}
    except Exception:
        return None


def cpu_baseline(workload, seconds=20.0, single_thread=True):
    """The oracle as it stands, on this host's cores: one micro-batch at a time of the same
    workload (K=1 stage, bf16 emulation for VGG-16 / fp32 for the MLP), bounded to ~seconds."""
    import oracle
    import synthetic as S
    L, shape, classes, kind, N, T, prec = workload_model(workload)
    n = N // T
    P = S.make_params(L, 1)
    o = oracle.Oracle(L, 1, 1, n, 1e-4, (0.9, 0.999), 1e-8, shape, classes, P, mode=prec)
    x, y = S.make_inputs(n, shape, classes, 1, kind=kind)
    done, t0 = 0, time.perf_counter()
    while True:
        o.step(x, y, 1, flush=True)
        done += 1
        el = time.perf_counter() - t0
        if el >= seconds or (done >= 1 and el * (done + 1) / done > 3 * seconds):
            break
    cores = int(os.environ.get("OMP_NUM_THREADS") or len(os.sched_getaffinity(0)))
    one = cpu_baseline_single_thread(workload) if single_thread else None
    return {"value": done * n / el, "unit": "samples/s", "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(), "single_thread": one,
            "sample": "%d micro-batch(es) of %d samples through the oracle (%s, K=1, fwd+bwd+update), %.1f s"
                      % (done, n, "bf16 emulation" if prec == "bf16" else "fp32", el)}


def stage_costs(g, L, shape, K):
    """Per stage: training flops per sample (2 x (fwd + dgrad + wgrad) MACs; the first layer
    needs no dgrad) and parameters, from the layer list and the library's stage assignment
    (SURVEY 8d "algorithmic work")."""
    from synthetic.models import infer_shapes, LINEAR, CONV2D, BATCHNORM2D
    shapes = infer_shapes(L, shape)
    flops = [0.0] * K
    params = [0] * K
    first = True
    for i, l in enumerate(L):
        k = g.stage_of(i)
        if l.kind == LINEAR:
            mac = l.in_c * l.out_c
            params[k] += mac + (l.out_c if l.bias else 0)
        elif l.kind == CONV2D:
            c, h, w = shapes[i]
            mac = c * h * w * l.in_c * l.kh * l.kw
            params[k] += l.out_c * l.in_c * l.kh * l.kw + (l.out_c if l.bias else 0)
        elif l.kind == BATCHNORM2D:
            params[k] += 2 * l.in_c
            continue
        else:
            continue
        flops[k] += 2.0 * mac * (2 if first else 3)
        first = False
    return flops, params


def pipeline_roofline(flops, params, N, M, ms_per_step, peaks, one_device, sweep_bytes=32.0):
    """ideal time per mini-batch at the measured peaks (stage GEMM/conv flops at the
    sustained bf16 tensor peak + the K1 sweep's bytes at the HBM copy peak), the bottleneck stage
    when every stage has its own GPU, the sum when they share one, over the measured time per
    mini-batch.  BN / elementwise traffic, launch latency and hand-offs are not in the ideal."""
    tp = peaks.get("bf16_tflops_sustained", 1400.0) * 1e12
    hb = peaks["hbm_gbs"] * 1e9
    per = [f * N / tp + p * sweep_bytes / hb for f, p in zip(flops, params)]
    ideal = sum(per) if one_device else max(per)
    meas = ms_per_step * 1e-3 / M
    return {"frac": ideal / meas, "ideal_ms_per_minibatch": ideal * 1e3, "measured_ms_per_minibatch": meas * 1e3,
            "per_stage_ideal_ms": [x * 1e3 for x in per],
            "note": "ideal = %s of per-stage (flops/sustained tensor peak + 32 B/param sweep/HBM peak)"
                    % ("sum (all stages share one GPU)" if one_device else "max (one stage per GPU)")}


def run_reference(args):
    """--impl reference: the CPU oracle timed as it stands (the reference arm of this tier)."""
    ws, rank, local = dist_env()
    if rank != 0:
        return 0
    import oracle
    import synthetic as S
    oracle.build()
    L, shape, classes, kind, N, T, prec = workload_model(args.workload)
    n = N // T
    P = S.make_params(L, 1)
    o = oracle.Oracle(L, 1, 1, n, 1e-4, (0.9, 0.999), 1e-8, shape, classes, P, mode=prec)
    x, y = S.make_inputs(n, shape, classes, 1, kind=kind)
    for _ in range(args.warmup):
        o.step(x, y, 1, flush=True)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        o.step(x, y, 1, flush=True)
    el = time.perf_counter() - t0
    v = args.steps * n / el
    K = args.stages or (DEFAULT_STAGES[args.workload] if args.gpus == 1 else args.gpus)
    cfg = {"workload": "%s, K=%d stages, mini-batch %d, T=%d micro-batches" % (WORKLOAD_TEXT[args.workload], K, N, T),
           "global_batch": N, "stages": K, "micro_batches": T,
           "sample": "oracle (bf16 emulation, fp64 accumulation): one %d-sample micro-batch fwd+bwd+update per "
                     "step; the per-sample work equals the K-stage pipeline's" % n}
    line = {"impl": "reference", "metric": METRICS.get(args.workload, METRIC), "value": v, "unit": "samples/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": el * 1000 / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": v, "unit": "samples/s", "cores": os.cpu_count(), "kind": "oracle",
                             "sample": "%d steps x %d samples" % (args.steps, n)},
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_sweep(args, peaks, peak_kind, n=None, steps=None):
    """Config 5: the fused Adam+prediction sweep alone (kernel-level metric)."""
    import torch
    from paper_1911_04610_b200 import adam_predict
    n = n or args.sweep_params
    steps = steps or args.steps
    dev = torch.device("cuda", 0)
    W = torch.rand(n, device=dev) * 0.1 - 0.05
    g = torch.rand(n, device=dev) * 2e-2 - 1e-2
    m = (torch.rand(n, device=dev) * 2e-2 - 1e-2) * 0.1
    v = torch.rand(n, device=dev) * 9.9e-5 + 1e-6
    pf = torch.empty(n, dtype=torch.bfloat16, device=dev)
    pb = torch.empty(n, dtype=torch.bfloat16, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    for i in range(args.warmup):
        adam_predict(W, g, m, v, pf, pb, i + 1, 1e-4, (0.9, 0.999), 1e-8, 3, 1, True, stream=st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(0) as ck:
        e0.record()
        for i in range(steps):
            adam_predict(W, g, m, v, pf, pb, args.warmup + i + 1, 1e-4, (0.9, 0.999), 1e-8, 3, 1, True, stream=st)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    del W, g, m, v, pf, pb
    torch.cuda.empty_cache()
    gbs = n * 32 / (ms * 1e-3) / 1e9
    peak = peaks["hbm_gbs"]
    return {"metric": "Adam+predict sweep HBM GB/s (config 5)", "value": gbs, "unit": "GB/s", "n_gpus": 1,
            "steps": steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "sweep P=%d, s_f=3, s_b=1, bf16 W_hat, 32 B/param" % n,
                       "l2": "working set %d MB > 126 MB L2" % (n * 32 // 2**20)},
            "gpu_launches": steps, "clocks": ck.summary(),
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                         "traffic": sweep_traffic(n), "peak_source": peak_kind}}


def sweep_traffic(n):
    """DRAM bytes per launch from the committed ncu --set full capture of the sweep, scaled to P
    (the capture's P is recorded beside it), or None."""
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(tp):
        return None
    with open(tp) as f:
        d = json.load(f)
    if "sweep" not in d:
        return None
    return d["sweep"] * n / d.get("sweep_params", 1 << 28)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="vgg16", choices=["vgg16", "mlp", "resnet101", "inception", "sweep"])
    ap.add_argument("--minibatches", type=int, default=16,
                    help="mini-batches fed per step, i.e. per xpipe_step call; a call starts from the "
                         "previous call's completed work, so fewer, larger calls amortise that drain "
                         "(4 -> 16 per call measured +3%%)")
    ap.add_argument("--stages", type=int, default=0,
                    help="pipeline stages (default: the BASELINE config's -- VGG-16 4, MLP 2 -- on one GPU, "
                         "else one per GPU)")
    ap.add_argument("--sweep-params", type=int, default=1 << 28)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the embedded config-5 sweep measurement")
    ap.add_argument("--recompute", action="store_true", help="activation recomputation (P:167, SURVEY f3)")
    ap.add_argument("--no-fb-overlap", action="store_true",
                    help="one stream per stage (default: a forward stream per stage, F(u+S) overlaps B(u))")
    ap.add_argument("--partition", default="layer-count", choices=["layer-count", "balanced", "macs"],
                    help="stage split: the paper's layer-count rule (R17), cost-balanced on per-unit device "
                         "times measured first (SURVEY 8e), or balanced on forward MACs")
    ap.add_argument("--image", type=int, default=64, help="Tiny-ImageNet side for resnet101/inception (224: f4)")
    ap.add_argument("--micro-batch", type=int, default=0, help="micro-batch size override (resnet101/inception)")
    ap.add_argument("--micro-batches", type=int, default=0, help="T override (resnet101/inception)")
    ap.add_argument("--optimizer", default="adam", choices=["adam", "sgd"],
                    help="sgd: Momentum SGD (0.9, wd 5e-4) + the paper-literal prediction (SURVEY 8f f2)")
    ap.add_argument("--schedule", default="xpipe", choices=["xpipe", "gpipe"],
                    help="gpipe: synchronous GPipe with a flush per mini-batch (prediction off), same kernels")
    ap.add_argument("--no-graphs", action="store_true", help="enqueue every kernel from the host (no CUDA graphs)")
    ap.add_argument("--sync-calls", action="store_true",
                    help="every xpipe_step call waits for its work (no chained asynchronous graph replays)")
    ap.add_argument("--timing", type=int, default=-1,
                    help="stamp every p-th call of the timed run (cfg.timing: bubble, steady rate, hand-offs); "
                         "0 = off, default = --steps (one stamped call per timed run).  A stamped call carries "
                         "a timestamp kernel around every op: every 4th call stamped cost 5.9%% at ResNet-101 K=8, "
                         "0.9%% at VGG-16 K=4")
    ap.add_argument("--no-timing", dest="timing", action="store_const", const=0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.timing < 0:
        args.timing = max(1, args.steps)

    if args.impl == "reference":
        return run_reference(args)

    ws, rank, local = dist_env()
    import torch
    peaks, peak_kind = load_peaks()
    if ws > 1:
        import torch.distributed as dist
        if os.environ.get("XPIPE_BENCH_ONE_GPU"):
            # development dry run of the multi-process path on a one-GPU box: every rank on
            # device 0 (CUDA IPC within one device), gloo for the host plumbing
            local = 0
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.workload == "sweep":
        line = run_sweep(args, peaks, peak_kind)
        if rank == 0:
            print(json.dumps(line), flush=True)
        return 0

    import numpy as np
    import synthetic as S
    from paper_1911_04610_b200 import XPipe, connect_pipeline
    M = args.minibatches
    mp_mode = ws > 1
    # each BASELINE config names its stage count (VGG-16 4, ResNet-101 8, Inception-V3 4, MLP 2):
    # on one GPU all stages share the device (one stream each); on N GPUs one stage per GPU
    K = ws if mp_mode else (args.stages or (DEFAULT_STAGES[args.workload] if args.gpus == 1 else args.gpus))
    L, shape, classes, kind, N, T, prec = workload_model(args.workload, K, args.image, args.micro_batch,
                                                         args.micro_batches)
    # f1: the GPipe-flush schedule (prediction off) through the same kernels, for the paper's
    # XPipe/GPipe throughput comparison (Figs. 7-8)
    sched = dict(schedule="gpipe", predict="off") if args.schedule == "gpipe" else {}
    # f2: the paper's Momentum-SGD training with the literal Eq. (3)/(4) prediction
    if args.optimizer == "sgd":
        sched.update(optimizer="sgd", delta="paper", momentum=0.9, weight_decay=5e-4)
    if args.recompute:  # f3: activation recomputation in every backward
        sched.update(recompute=True)
    if not args.no_fb_overlap:  # forwards on a second stream per stage (F(u+S) overlaps B(u))
        sched.update(fb_overlap=True)
    unit_cost = None
    if args.partition in ("balanced", "macs") and K > 1:
        # contiguous partition minimising the largest stage cost -- per-unit device
        # times measured first (every rank measures the same model on its own GPU and takes the
        # same deterministic split; rank 0's costs are broadcast so all ranks agree exactly)
        from synthetic.models import chain_units, unit_macs, balanced_stages
        if args.workload in ("resnet101", "inception"):
            from synthetic.models import resnet101, inception_v3
            units = (resnet101(classes=200)[1] if args.workload == "resnet101" else
                     inception_v3(classes=200, stem_pad=args.image < 75)[1])
        else:
            units = chain_units(L)
        if args.partition == "macs":
            unit_cost = unit_macs(L, units, shape)
        else:
            if mp_mode:
                torch.cuda.set_device(local if not os.environ.get("XPIPE_BENCH_ONE_GPU") else 0)
            unit_cost = measured_unit_costs(L, units, shape, classes, kind, N, T, prec, sched) if rank == 0 else None
            if mp_mode:
                import torch.distributed as dist
                box = [unit_cost]
                dist.broadcast_object_list(box, src=0)
                unit_cost = box[0]
        L = balanced_stages(L, units, unit_cost, K)
    dev = local if mp_mode else 0
    P = S.make_params(L, 1)
    from synthetic.models import param_count
    nparams = param_count(L, shape)
    def make_model(profile):
        if mp_mode:
            # one process per GPU: this rank owns stage `rank`; rings/flags are CUDA IPC-mapped
            import torch.distributed as dist
            m = XPipe(L, K, T, N, 1e-4, (0.9, 0.999), 1e-8, shape, classes, params=P, precision=prec,
                      profile=profile, watchdog_ms=300000, my_stage=rank, timing=0 if profile else args.timing,
                      graphs=not args.no_graphs, **sched)
            connect_pipeline(m, dist.new_group(backend="gloo"))
        else:
            # the profiled pass runs every stage on one stream (serialize): each launch then runs
            # alone, so its event-timed duration is the kernel's own (as in ncu's launch list)
            m = XPipe(L, K, T, N, 1e-4, (0.9, 0.999), 1e-8, shape, classes, params=P, precision=prec,
                      devices=list(range(args.gpus)), profile=profile, watchdog_ms=300000,
                      graphs=not args.no_graphs, serialize=profile and args.gpus == 1,
                      timing=0 if profile else args.timing, **sched)
        return m

    x, y = S.make_inputs(M * N, shape, classes, 1, kind=kind)
    last_dev = dev if mp_mode else (K - 1) % args.gpus
    xd = torch.from_numpy(x).cuda(dev)
    yd = torch.from_numpy(y).cuda(last_dev)

    def barrier():
        if mp_mode:
            import torch.distributed as dist
            dist.barrier()

    def warm(m):
        # warm-up: at least --warmup steps, and (with CUDA graphs) until every step signature of
        # the steady state has been captured -- the ring-slot phase repeats with a period of up
        # to K calls -- so no capture/instantiation lands in the timed region
        streak, w = 0, 0
        if mp_mode:
            # every rank must run the same number of calls (the stages are coupled): a fixed count
            # that covers eligibility, the first sighting, the capture and a few replays
            for _ in range(args.warmup + (0 if args.no_graphs else 2 * K + 4 + 2 * max(1, args.timing))):
                m.step(xd, yd, M)
            barrier()
            return
        # (the calls stamped for xpipe_stats -- every --timing-th -- have a graph of their own: the
        # streak must cover one of them too, or the timed region would enqueue it from the host)
        tp = max(1, args.timing)
        while w < args.warmup or (not args.no_graphs and streak < K + 1 + tp and w < args.warmup + 4 * K + 8 + 3 * tp):
            m.step(xd, yd, M)
            streak = streak + 1 if m.last_stats.graph_replays else 0
            w += 1
        barrier()

    # ---- the timed run: no profiling events inside (they would split the PDL chains)
    g = make_model(False)
    warm(g)
    launches = 0
    replays = 0
    tim = []
    with Clocks(dev) as ck:
        g.timer_start()
        for _ in range(args.steps):
            # asynchronous calls: consecutive graph replays chain on the device (no host wait at
            # the call boundary); stamped calls complete synchronously; timer_stop waits for all
            g.step(xd, yd, M, losses=False, async_=not args.sync_calls)
            st = g.last_stats
            launches += st.kernel_launches
            replays += st.graph_replays
            if args.timing and st.ops_timed:
                tim.append(st.timing(K))
        ms = g.timer_stop()
        barrier()
    flops, params = stage_costs(g, L, shape, K)
    clocks = ck.summary()
    e2e_s = None
    if not args.no_e2e:
        xh = torch.from_numpy(x).pin_memory()
        yh = torch.from_numpy(y).pin_memory()
        lh = torch.empty(M * T, dtype=torch.float32).pin_memory()  # every step's losses (D2H)
        xh_np, yh_np = xh.numpy(), yh.numpy()
        g.step(xh_np, yh_np, M)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            g.step(xh_np, yh_np, M, async_=not args.sync_calls, loss_out=lh)
        g.sync()
        barrier()
        e2e_s = time.perf_counter() - t0
    # ---- a separate profiled pass (CUDA events around every kernel class) for the roofline and
    # the per-class shares; its step time is not the metric
    g.close()
    gp = make_model(True)
    warm(gp)
    prof = {}
    gp.timer_start()
    for _ in range(args.steps):
        gp.step(xd, yd, M, losses=False)
        for name, d in gp.last_stats.profile().items():
            q = prof.setdefault(name, {"ms": 0.0, "launches": 0, "work": 0.0})
            q["ms"] += d["ms"]; q["launches"] += d["launches"]; q["work"] += d["work"]
    prof_step_ms = gp.timer_stop() / args.steps
    barrier()
    g = gp
    if mp_mode:
        import torch.distributed as dist
        allp = [None] * ws
        dist.all_gather_object(allp, {"ms": ms, "prof": prof, "launches": launches, "e2e_s": e2e_s, "tim": tim})
        ms = max(p["ms"] for p in allp)                       # max over ranks
        # each rank timed its own stage: merge per step (busy of stage r from rank r, the span as
        # the max over ranks, the steady rate from stage 0's rank)
        if args.timing:
            merged = []
            for i in range(len(tim)):
                t = dict(allp[0]["tim"][i])
                t["span_ms"] = max(p["tim"][i]["span_ms"] for p in allp)
                for key in ("busy_ms", "p2p_fwd_ms", "p2p_bwd_ms", "p2p_fwd_bytes", "p2p_bwd_bytes"):
                    t[key] = [allp[r]["tim"][i][key][r] for r in range(ws)]
                merged.append(t)
            tim = merged
        e2e_s = None if e2e_s is None else max(p["e2e_s"] for p in allp)
        launches = sum(p["launches"] for p in allp)
        prof = {}
        for p in allp:
            for name, d in p["prof"].items():
                q = prof.setdefault(name, {"ms": 0.0, "launches": 0, "work": 0.0})
                q["ms"] += d["ms"]; q["launches"] += d["launches"]; q["work"] += d["work"]
        dist.barrier()
    g.close()
    if rank != 0:
        return 0
    value = args.steps * M * N / (ms * 1e-3)
    e2e = None
    if e2e_s is not None:
        e2e = {"value": args.steps * M * N / e2e_s, "unit": "samples/s",
               "h2d_bytes_per_step": int(x.nbytes + y.nbytes), "d2h_bytes_per_step": int(M * T * 4)}
    # ---- roofline of the dominant kernel class (CUDA events on the launching streams)
    from paper_1911_04610_b200.xpipe import BYTE_CLASSES
    prof = {k: v for k, v in prof.items() if v["launches"]}
    total_prof_ms = sum(v["ms"] for v in prof.values())
    dom = max(prof, key=lambda k: prof[k]["ms"])
    d = prof[dom]
    if dom in BYTE_CLASSES:
        roof = {"bound": "hbm", "achieved": d["work"] / (d["ms"] * 1e-3) / 1e9, "peak": peaks["hbm_gbs"],
                "unit": "GB/s"}
    else:
        roof = {"bound": "tensor", "achieved": d["work"] / (d["ms"] * 1e-3) / 1e12,
                "peak": peaks.get("bf16_tflops_sustained", 1400.0), "unit": "TFLOP/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"] = None
    roof["kernel"] = dom
    roof["launches_per_step"] = d["launches"] / args.steps
    roof["work_per_launch"] = d["work"] / d["launches"]
    roof["peak_source"] = peak_kind + (" (sustained)" if roof["bound"] == "tensor" else "")
    roof["note"] = ("CUDA-event launch durations from a profiled pass of the same step with all K stages "
                    "serialised on one stream (each launch runs alone, as in the ncu launch list); the timed "
                    "run overlaps the stages' kernels, so its step is shorter than the sum of these")
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tr = json.load(f).get(dom)
        if tr is not None:
            roof["traffic"] = tr
    shares = {k: {"ms_per_step": v["ms"] / args.steps, "share_of_step": v["ms"] / (prof_step_ms * args.steps * (ws if mp_mode else 1)),
                  "share_norm": v["ms"] / total_prof_ms,
                  "achieved": (v["work"] / (v["ms"] * 1e-3) / (1e9 if k in BYTE_CLASSES else 1e12)) if v["ms"] else 0,
                  "unit": "GB/s" if k in BYTE_CLASSES else "TFLOP/s", "launches": v["launches"]}
              for k, v in prof.items()}
    result = dict(ms=ms, clocks=clocks, roof=roof, shares=shares, launches=launches, replays=replays)
    # bubble fraction and hand-offs of the timed run itself (xpipe_stats from per-op CUDA events,
    # also inside the replayed graphs): 1 - sum_k busy_k / (K * span) over all timed steps
    bubble = None
    if tim:
        span = sum(t["span_ms"] for t in tim)
        busy = [sum(t["busy_ms"][k] for t in tim) for k in range(K)]
        gp_ = args.schedule == "gpipe"
        ideal = (K - 1) / (T + K - 1) if gp_ else (K - 1) / (M * T + K - 1)  # SURVEY A.3 closed forms
        steady = [t["steady_samples_per_s"] for t in tim if t["steady_samples_per_s"] > 0]
        edges = []
        for k in range(K):
            fb = sum(t["p2p_fwd_bytes"][k] for t in tim)
            fm = sum(t["p2p_fwd_ms"][k] for t in tim)
            bb = sum(t["p2p_bwd_bytes"][k] for t in tim)
            bm = sum(t["p2p_bwd_ms"][k] for t in tim)
            # sampled on the bellwether micro-batches (1 in T): per-step time and the share of the
            # span during which the stage's stream is copying = T x the sampled figures
            if fb:
                edges.append({"edge": "%d->%d" % (k, k + 1), "GB_per_s": fb / (fm * 1e-3) / 1e9 if fm else None,
                              "ms_per_step": T * fm / len(tim), "stream_blocked_frac_of_span": T * fm / span})
            if bb:
                edges.append({"edge": "%d->%d" % (k, k - 1), "GB_per_s": bb / (bm * 1e-3) / 1e9 if bm else None,
                              "ms_per_step": T * bm / len(tim), "stream_blocked_frac_of_span": T * bm / span})
        bubble = {"bubble_fraction": 1.0 - sum(busy) / (K * span), "ideal_uniform": ideal,
                  "busy_frac_per_stage": [b / span for b in busy],
                  "span_ms_per_step": span / len(tim),
                  "steady_samples_per_s": statistics.median(steady) if steady else None,
                  "p2p": edges,
                  "timed_calls": len(tim), "of_calls": args.steps,
                  "source": "xpipe_stats of the timed run (cfg.timing: %globaltimer stamps per op on its "
                            "stream, replayed inside the graphs); a stage's busy time is the union of its F/B "
                            "op intervals (input arrival to hand-off end; B(t,T) to the update's end); "
                            "hand-offs sampled on bellwether micro-batches"}
    one_dev = (not mp_mode) and args.gpus == 1
    proof = pipeline_roofline(flops, params, N, M, result["ms"] / args.steps, peaks, one_dev,
                              sweep_bytes=32.0 if prec == "bf16" else 36.0)
    # the oracle baseline is timed on rank 0 at N=1 only (the contract); N>1 lines omit it
    cpu = None if (args.no_cpu_baseline or mp_mode) else cpu_baseline(args.workload)
    sweep = None
    if not args.no_sweep and not mp_mode:
        # the BASELINE metric's second half: the fused Adam+prediction sweep alone (config 5)
        sl = run_sweep(args, peaks, peak_kind, n=1 << 27, steps=20)
        sweep = {k: sl[k] for k in ("value", "unit", "ms_per_step", "roofline")}
        sweep["config"] = sl["config"]["workload"]
    # first layer of every stage where the split is explicit (DAG models, balanced partitions);
    # None = the library's layer-count rule (R17)
    stage_first = ([min((i for i, l in enumerate(L) if l.stage == k), default=-1) for k in range(K)]
                   if K > 1 and all(l.stage >= 0 for l in L) else None)
    line = {"metric": METRICS.get(args.workload, METRIC), "value": value, "unit": "samples/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": result["ms"] / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": prec, "data": "synthetic",
            "config": {"workload": "%s, K=%d stages, mini-batch %d, T=%d micro-batches, %d mini-batches per step"
                                   % (WORKLOAD_TEXT[args.workload], K, N, T, M),
                       "processes": "one per GPU (CUDA IPC rings)" if ws > 1 else "one process",
                       "global_batch": N, "stages": K, "micro_batches": T, "minibatches_per_step": M,
                       "parallelism": "pipeline K=%d (%s)" % (K, "GPipe-flush" if args.schedule == "gpipe" else "XPipe"),
                       "schedule": args.schedule, "optimizer": args.optimizer, "recompute": args.recompute,
                       "partition": args.partition, "stage_first_layer": stage_first,
                       "unit_cost": ([round(c, 4) for c in unit_cost] if unit_cost else None),
                       "fb_overlap": not args.no_fb_overlap,
                       "image": list(shape),
                       "l2": "working set > L2: optimizer state 16 B/param x %.1fM params = %d MB (126 MB L2)"
                             % (nparams / 1e6, nparams * 16 // 10**6)},
            "e2e": e2e, "gpu_launches": result["launches"], "graph_replays": result.get("replays"),
            "clocks": result["clocks"],
            "roofline": result["roof"], "kernel_shares": result["shares"],
            "profiled_step_ms": prof_step_ms if not mp_mode else None, "bubble": bubble,
            "pipeline_roofline": proof, "cpu_baseline": cpu,
            "adam_predict": sweep}
    print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
