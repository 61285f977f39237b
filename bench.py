#!/usr/bin/env python
"""EasySpec decode benchmark on B200 (BASELINE.json configs[1] at one GPU).

One *step* = one EasySpec decode iteration of the reference's loop
(Generation::run_iteration_speculative, proj/src/orchestrator.cpp:407-436):
bonus-calibration pass -> (n-1) fuzzy layer-parallel draft passes -> base
verification of the n+1 rows -> greedy acceptance -> KV commit/discard.

Workload "c2": Llama-3-70B-shaped base + Llama-3-8B-shaped drafter, bf16
weights and KV, random init (device N(0, sd) with the reference's sd rules),
layer-parallel width 4 (plan 0|1-3|4-7|...|28-30|31), n = 5, batch 1,
greedy, synthetic prompt of --ctx uniform-random token ids. The full pair
(157 GB) is resident on one B200; at N>1 the pair is tensor-parallel over
the N GPUs (one rank per GPU, Megatron-sharded base AND drafter, partial sums
exchanged by the engine's own one-shot all-reduce kernels over NVLink peer
memory) and one generation stream is decoded by the whole job
(scaling "strong").

Prints ONE JSON line (rank 0). `value` is decode tokens/s of EasySpec with
inputs resident in HBM; `e2e` the same metric through the C ABI
(espec_generate_tokens: host token ids in, host tokens out, prefill included).
The weights (157 GB) exceed L2 (126 MB) many times over: every timed step
streams them from HBM, so no L2 flush is needed.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "c2": dict(
        name="llama3-70b-base(tp1)+llama3-8b-drafter, lp4, n5, batch1, greedy",
        base=dict(vocab_size=128256, d_model=8192, n_layers=80, n_heads=64, n_kv_heads=8, d_head=128, d_mlp=28672,
                  rope_theta=500000.0),
        draft=dict(vocab_size=128256, d_model=4096, n_layers=32, n_heads=32, n_kv_heads=8, d_head=128, d_mlp=14336,
                   rope_theta=500000.0),
        lp=4, n=5),
    # BASELINE.json configs[2]: Qwen2-72B base + Qwen2-7B drafter shapes, lp 8
    # (plan 0|1-7|8-15|16-23|24-26|27); vocab 152064 (no QKV bias: the
    # reference model family has none)
    "c3": dict(
        name="qwen2-72b-base(tp1)+qwen2-7b-drafter, lp8, n5, batch1, greedy",
        base=dict(vocab_size=152064, d_model=8192, n_layers=80, n_heads=64, n_kv_heads=8, d_head=128, d_mlp=29568,
                  rope_theta=1000000.0),
        draft=dict(vocab_size=152064, d_model=3584, n_layers=28, n_heads=28, n_kv_heads=4, d_head=128, d_mlp=18944,
                   rope_theta=1000000.0),
        lp=8, n=5),
    # BASELINE.json configs[3]: Qwen2.5-32B base + Qwen2.5-0.5B drafter, lp 4
    "c4": dict(
        name="qwen2.5-32b-base(tp1)+qwen2.5-0.5b-drafter, lp4, n5, batch1, greedy",
        base=dict(vocab_size=152064, d_model=5120, n_layers=64, n_heads=40, n_kv_heads=8, d_head=128, d_mlp=27648,
                  rope_theta=1000000.0),
        draft=dict(vocab_size=152064, d_model=896, n_layers=24, n_heads=14, n_kv_heads=2, d_head=64, d_mlp=4864,
                   rope_theta=1000000.0),
        lp=4, n=5),
    # small shapes for quick functional runs of this script
    "mini": dict(
        name="mini pair (functional check only)",
        base=dict(vocab_size=32000, d_model=1024, n_layers=8, n_heads=16, n_kv_heads=4, d_head=64, d_mlp=2816,
                  rope_theta=500000.0),
        draft=dict(vocab_size=32000, d_model=512, n_layers=6, n_heads=8, n_kv_heads=2, d_head=64, d_mlp=1408,
                   rope_theta=500000.0),
        lp=4, n=5),
}
PAPER_ALPHA = 0.82  # Llama-3-70B/8B, MMLU, T=0


def pass_bytes(cfg, ctx, tp=1):
    """Algorithmic HBM bytes of one decode pass of a model (bf16 weights
    streamed once: QKV, O, gate/up, down per layer + the LM head; the KV
    cache read once; embeddings are a row gather), per GPU at TP degree tp."""
    d, L, H, kv, dh, f, V = (cfg[k] for k in ("d_model", "n_layers", "n_heads", "n_kv_heads", "d_head", "d_mlp",
                                              "vocab_size"))
    per_layer = d * (H + 2 * kv) * dh + H * dh * d + d * 2 * f + f * d
    weights = 2.0 * (L * per_layer + d * V) / tp
    kv_bytes = 2.0 * 2 * ctx * kv * dh * L / tp
    return weights + kv_bytes


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ----------------------------------------------------------------------------
# CPU baseline: the unmodified reference core (oracle/_ref/ref_bench)
# ----------------------------------------------------------------------------

def _ref_bench(*args):
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_bench")
    out = subprocess.run([exe, *map(str, args)], capture_output=True, text=True, timeout=600)
    if out.returncode != 0:
        raise RuntimeError(f"ref_bench {args} failed: {out.stderr[-400:]}")
    return json.loads(out.stdout.strip().splitlines()[-1])


def _mha_equiv(cfg):
    # the reference is MHA-only: d_model = n_heads * d_head, wk/wv are d x d
    return cfg["d_model"], cfg["n_heads"], cfg["d_head"], cfg["d_mlp"]


def _plan_sizes(n_layers, lp):
    """Group sizes of plan_groups(n_layers, lp) (proj/src/layer_plan.cpp:54-82,
    through the engine's C ABI: host logic only, no GPU needed)."""
    from paper_2502_02493_b200 import espec as E
    return [int(g.split("-")[-1]) - int(g.split("-")[0]) + 1 for g in E.plan_groups(n_layers, lp).split("|")]


def cpu_iteration_seconds(wl, ctx, workers=1, reps=1, cache=None):
    """Extrapolated wall time of one EasySpec iteration of the reference CPU
    path with m = 0 accepted drafts: calibration = one precise drafter pass
    over 1 row; n-1 fuzzy draft passes over 1 row, each = the plan's groups
    through forward_fuzzy with a WorkerPool of `workers` threads (singleton
    groups = one layer); base verification over n+1 rows; plus the LM head
    rows each pass scores."""
    n, lp = wl["n"], wl["lp"]
    b, d = wl["base"], wl["draft"]
    cache = cache if cache is not None else {}

    def layer(cfg, T):
        key = ("layer", cfg["d_model"], T)
        if key not in cache:
            r = _ref_bench("layer", *_mha_equiv(cfg), T, ctx, reps)
            cache[key] = (r["mask_ms"] + r["attn_ms"] + r["mlp_ms"] + r["rest_ms"]) / 1000.0
        return cache[key]

    def group(cfg, g, T):
        if g == 1:
            return layer(cfg, T)
        key = ("group", cfg["d_model"], g, T, workers)
        if key not in cache:
            cache[key] = _ref_bench("group", *_mha_equiv(cfg), g, T, ctx, workers, reps)["group_ms"] / 1000.0
        return cache[key]

    def head(cfg, T):
        key = ("head", cfg["d_model"], T)
        if key not in cache:
            cache[key] = _ref_bench("head", cfg["d_model"], cfg["vocab_size"], T, reps)["head_ms"] / 1000.0
        return cache[key]

    calib = d["n_layers"] * layer(d, 1) + head(d, 1)
    fuzzy_pass = sum(group(d, g, 1) for g in _plan_sizes(d["n_layers"], lp))
    draft = (n - 1) * (fuzzy_pass + head(d, 1))
    verify = b["n_layers"] * layer(b, n + 1) + head(b, n + 1)
    return calib + draft + verify, {"calibrate_s": calib, "draft_s": draft, "verify_s": verify}


def cpu_baseline(wl, ctx):
    """The reference CPU path at its stock worker count (RunConfig.workers = 0
    -> the largest plan group = lp, proj/src/orchestrator.cpp:152,
    proj/src/worker_pool.cpp:73-84) and at workers = 1."""
    t0 = time.time()
    cache = {}
    lp = wl["lp"]
    it_lp, parts_lp = cpu_iteration_seconds(wl, ctx, workers=lp, cache=cache)
    it_1, parts_1 = cpu_iteration_seconds(wl, ctx, workers=1, cache=cache)
    return {"value": 1.0 / it_lp, "unit": "tokens/s", "cores": lp, "kind": "reference",
            "sample": (f"oracle/_ref/ref_bench (unmodified reference core): one layer per shape at ctx {ctx} "
                       f"(base T={wl['n'] + 1}, drafter T=1, MHA-equivalent widths) and each fuzzy group through "
                       f"forward_fuzzy + WorkerPool, + LM head rows, extrapolated to "
                       f"{wl['base']['n_layers']}/{wl['draft']['n_layers']} layers, 1 token per iteration (m=0); "
                       f"value at workers={lp} (the reference's auto setting); {time.time() - t0:.1f}s of CPU work"),
            "stage_s": parts_lp,
            "workers_1": {"value": 1.0 / it_1, "cores": 1, "stage_s": parts_1}}


def run_reference(args, wl):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    cache = {}
    times = []
    lp = wl["lp"]
    t_start = time.time()
    for i in range(args.warmup + args.steps):
        # each step re-samples the dominant term (one base layer at T=n+1);
        # drafter layers, fuzzy groups and LM heads are sampled once (warm-up)
        cache.pop(("layer", wl["base"]["d_model"], wl["n"] + 1), None)
        it_s, parts = cpu_iteration_seconds(wl, args.ctx, workers=lp, cache=cache)
        if i >= args.warmup:
            times.append(it_s)
    it = statistics.median(times)
    value = 1.0 / it
    line = {"metric": "decode tokens/s (EasySpec, greedy)", "value": value, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": it * 1000.0,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": wl["name"], "ctx": args.ctx, "n": wl["n"], "lp": wl["lp"],
                       "note": "reference CPU core; 1 token per iteration (m=0)"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": lp, "kind": "reference",
                             "sample": f"per step: one base layer (T={wl['n'] + 1}, ctx {args.ctx}) timed, "
                                       f"extrapolated; drafter layers, fuzzy groups (forward_fuzzy, "
                                       f"WorkerPool({lp})) + heads sampled once; {time.time() - t_start:.0f}s total"},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "stage_s": parts}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------
# GPU arms
# ----------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--ctx", type=int, default=512)
    ap.add_argument("--e2e-tokens", type=int, default=128)  # the paper protocol: 128 new tokens
    ap.add_argument("--no-arms", action="store_true", help="skip the vanilla / sd comparison arms")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--tp-proxy", type=int, default=0,
                    help="shard proxy: run rank 0 of a TP-N group alone on one GPU, collectives looped back "
                         "(per-GPU step time at TP-N shard shapes; outputs are not the model's)")
    ap.add_argument("--draft-layout", default="tp", choices=["tp", "lp"],
                    help="drafter across the GPUs: tensor-parallel (tp) or the paper's layer-parallel placement "
                         "(lp: fuzzy-group slot j on GPU j, MLP / head tensor-parallel)")
    ap.add_argument("--temperature", type=float, default=0.0,
                    help="sampling temperature of every arm (0 = greedy, the BASELINE metric)")
    args = ap.parse_args()
    assert args.warmup >= 1
    wl = WORKLOADS[args.workload]
    # --gpus N without a torchrun environment: launch the N ranks ourselves
    # (one process per GPU), exactly as the driver's torchrun line would
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    ws_env = int(os.environ.get("WORLD_SIZE", "1"))
    if ws_env != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws_env}")
    if args.impl == "reference":
        return run_reference(args, wl)

    import numpy as np
    import torch
    from paper_2502_02493_b200 import espec as E

    ws, rank, local = dist_env()
    one_gpu = os.environ.get("ESPEC_BENCH_ONE_GPU") == "1"
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo" if one_gpu else "nccl")
    # ESPEC_BENCH_ONE_GPU=1: every rank on cuda:0 (functional check of the
    # multi-rank path on a 1-GPU box; timings are then meaningless)
    dev = 0 if one_gpu else local
    torch.cuda.set_device(dev)

    n, lp = wl["n"], wl["lp"]
    steps, warm = args.steps, args.warmup
    max_pos = args.ctx + (warm + steps + 4) * (n + 1) + args.e2e_tokens + 64
    base = E.ModelConfig(max_positions=max_pos, seed=7, tied_head=False, weight_dtype=E.BF16, kv_dtype=E.BF16,
                         **wl["base"])
    draft = E.ModelConfig(max_positions=max_pos, seed=9, tied_head=False, weight_dtype=E.BF16, kv_dtype=E.BF16,
                          **wl["draft"])
    run = E.RunConfig(algorithm="easyspec", n=n, lp_size=lp, temperature=args.temperature,
                      max_new_tokens=(warm + steps + 2) * (n + 1))
    proxy = args.tp_proxy if ws == 1 else 0
    tp = proxy or ws  # tensor-parallel degree whose per-GPU shard this process runs
    layout = args.draft_layout if tp > 1 else "tp"
    eng = E.Engine(base, draft, run, device=dev, tp_size=tp, tp_rank=rank, draft_layout=layout)
    if ws > 1:
        eng.link_process_group()  # all-gather the NVLink receive-region IPC handles
    elif proxy > 1:
        eng.link_loopback()
    eng.init_weights(E.Engine.BASE, base.seed, parity=False)
    eng.init_weights(E.Engine.DRAFT, draft.seed, parity=False)
    rng = np.random.default_rng(1234)  # the same prompt on every TP rank
    prompt = [int(t) for t in rng.integers(0, base.vocab_size, size=args.ctx)]
    stream = torch.cuda.ExternalStream(eng.stream(), device=dev)

    def barrier():
        if ws > 1:
            torch.distributed.barrier()

    def max_over_ranks(x):
        if ws == 1:
            return x
        t = torch.tensor([x], device="cpu" if one_gpu else f"cuda:{dev}", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        # tensor parallel: every rank emits the SAME tokens of one stream
        return x

    def arm(alg, site=None, clocks=False):
        eng.set_run(E.RunConfig(algorithm=alg, n=n, lp_size=lp, temperature=args.temperature,
                                max_new_tokens=(warm + steps + 2) * (n + 1)))
        eng.begin(prompt)
        for _ in range(warm):  # first warm-up step includes the prompt prefill
            eng.step()
        if site is not None:
            eng.time_site(*site)
        eng.reset_kernel_launches()
        barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sampler = ClockSampler(dev) if clocks else None
        if sampler:
            sampler.__enter__()
        prof = os.environ.get("ESPEC_PROFILE_REGION") == "1" and alg == "easyspec"
        if prof:  # ncu --profile-from-start off: capture only the timed decode steps
            torch.cuda.profiler.start()
        ev0.record(stream)
        traces, emitted = [], 0
        for _ in range(steps):
            em, tr = eng.step()
            emitted += len(em)
            traces.append(tr)
        ev1.record(stream)
        torch.cuda.synchronize()
        if prof:
            torch.cuda.profiler.stop()
        if sampler:
            sampler.__exit__()
        barrier()
        ms = ev0.elapsed_time(ev1)
        launches = eng.kernel_launches()
        site_stats = eng.site_stats() if site is not None else None
        if site is not None:
            eng.time_site(-1, -1)
        return dict(ms=ms, emitted=emitted, traces=traces, launches=launches, site=site_stats,
                    clocks=sampler.summary() if sampler else None)

    # main arm: EasySpec. Roofline site: the base gate/up GEMV (the largest
    # launch of the step)
    site_kind = 3
    # headline: no per-launch events inside the timed region (they would
    # break PDL overlap of the timed kernel site); the roofline comes from a
    # separate pass of the same arm below
    es = arm("easyspec", clocks=True)
    t_max = max_over_ranks(es["ms"])
    tokens_all = sum_over_ranks(es["emitted"])
    value = tokens_all / (t_max / 1000.0)
    m_list = [t.m for t in es["traces"]]
    alpha = sum(m_list) / (n * len(m_list))
    calib_ms = sum(t.calibrate_ms for t in es["traces"])
    draft_ms = sum(t.draft_ms for t in es["traces"])
    verify_ms = sum(t.verify_ms for t in es["traces"])
    per_tok = 1.0 / max(es["emitted"], 1)

    arms = {}
    if not args.no_arms:
        for alg in ("vanilla", "sd"):
            r = arm(alg)
            arms[alg] = dict(tokens_per_s=sum_over_ranks(r["emitted"]) / (max_over_ranks(r["ms"]) / 1000.0),
                             ms_per_step=r["ms"] / steps,
                             draft_ms_per_token=sum(t.draft_ms for t in r["traces"]) / max(r["emitted"], 1),
                             verify_ms_per_step=sum(t.verify_ms for t in r["traces"]) / steps)

    # roofline of the dominant kernel (base gate/up GEMV, bf16 weights streamed
    # once): its launches timed with CUDA events on the engine stream during a
    # separate pass of the EasySpec arm (same steps, same shapes)
    rf = arm("easyspec", site=(1, site_kind))
    hbm, peak_kind = peaks()
    cnt, site_ms, site_bytes = rf["site"]
    achieved = site_bytes / (site_ms / cnt / 1000.0) / 1e9 if cnt else None
    gu_shape = f"{wl['base']['d_model']}x{2 * wl['base']['d_mlp'] // tp}"
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(tpath) and tp == 1:
        try:  # ncu --set full dram__bytes of this workload's gate/up launch
            ent = json.load(open(tpath)).get("workloads", {}).get(args.workload)
            if ent and ent.get("shape") == gu_shape:
                traffic, traffic_src = ent["dram_bytes_per_launch"], ent["source"]
        except Exception:
            traffic = None

    # e2e through the C ABI: host prompt ids -> host tokens, prefill included
    e2e = None
    if args.e2e_tokens > 0:
        eng.set_run(E.RunConfig(algorithm="easyspec", n=n, lp_size=lp, temperature=args.temperature,
                                max_new_tokens=args.e2e_tokens))
        eng.generate_tokens(prompt)  # warm-up request
        h0, d0 = eng.io_bytes()
        reps = 2
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        got = 0
        for _ in range(reps):
            out, _tr = eng.generate_tokens(prompt)
            got += len(out)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        h1, d1 = eng.io_bytes()
        e_ms = max_over_ranks(e0.elapsed_time(e1))
        e2e = {"value": sum_over_ranks(got) / (e_ms / 1000.0), "unit": "tokens/s",
               "h2d_bytes_per_step": (h1 - h0) // reps, "d2h_bytes_per_step": (d1 - d0) // reps + 4 * args.e2e_tokens,
               "step": f"one espec_generate_tokens request: {args.ctx}-token prompt (prefill included) -> "
                       f"{args.e2e_tokens} new tokens"}

    cpu = None
    if rank == 0 and not args.no_cpu:
        try:
            cpu = cpu_baseline(wl, args.ctx)
        except Exception as ex:  # the checker binary is built here, not on the box
            cpu = {"value": None, "unit": "tokens/s", "cores": 1, "kind": "reference", "sample": f"unavailable: {ex}"}

    if rank == 0:
        it_ms = t_max / steps
        # alpha-projected: tokens/iteration = n*alpha + 1 at the
        # paper's alpha; calibration then covers m+1 rows (same weight bytes).
        proj_tok_s = (n * PAPER_ALPHA + 1) / (it_ms / 1000.0)
        line = {
            "metric": "decode tokens/s (EasySpec, greedy)" if args.temperature == 0 else
                      f"decode tokens/s (EasySpec, T={args.temperature})",
            "value": value, "unit": "tokens/s", "n_gpus": ws, "steps": steps, "warmup": warm,
            "ms_per_step": it_ms, "higher_is_better": True, "scaling": "strong" if ws > 1 else "weak",
            "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic (random-init weights, uniform-random prompt ids)",
            "config": {"workload": wl["name"], "ctx": args.ctx, "n": n, "lp": lp,
                       "plan": E.plan_groups(draft.n_layers, lp), "tp": tp,
                       "draft_layout": layout,
                       "parallelism": (f"tp{ws} (base + drafter)" if layout == "tp" else
                                       f"base tp{ws}, drafter layer-parallel over {ws} GPUs (MLP / head tp{ws})")
                       if ws > 1 else
                       (f"tp{proxy} shard proxy: rank 0 of a TP-{proxy} group alone on one GPU, collectives "
                        f"looped back (per-GPU step at TP-{proxy} shard shapes; tokens are not the model's)"
                        if proxy > 1 else "single GPU"),
                       "l2": "no flush: the weights streamed per step (GBs) >> 126 MB L2"},
            "speedup_vs_vanilla": (value / arms["vanilla"]["tokens_per_s"]) if "vanilla" in arms else None,
            "draft_ms_per_token": (calib_ms + draft_ms) * per_tok,
            "calibrate_ms_per_token": calib_ms * per_tok, "fuzzy_draft_ms_per_token": draft_ms * per_tok,
            "verify_ms_per_token": verify_ms * per_tok,
            # per-stage roofline: algorithmic bytes of the stage's
            # passes / the stage's device time; calibrate = 1 drafter pass + head,
            # draft = (n-1) fuzzy passes + heads, verify = 1 base pass + head
            "stage_roofline": {
                "calibrate": pass_bytes(wl["draft"], args.ctx, tp) / (calib_ms / steps / 1e3) / 1e9 / hbm,
                "draft": (n - 1) * pass_bytes(wl["draft"], args.ctx, tp) / (draft_ms / steps / 1e3) / 1e9 / hbm,
                "verify": pass_bytes(wl["base"], args.ctx, tp) / (verify_ms / steps / 1e3) / 1e9 / hbm,
                "vanilla": (pass_bytes(wl["base"], args.ctx, tp) / (arms["vanilla"]["ms_per_step"] / 1e3) / 1e9 / hbm)
                if "vanilla" in arms else None,
                "unit": "fraction of measured HBM GB/s"},
            "stage_ms_per_step": {"calibrate": calib_ms / steps, "draft": draft_ms / steps,
                                  "verify": verify_ms / steps},
            "mean_accept_len": es["emitted"] / steps, "alpha": alpha,
            "arms": arms,
            "alpha_projected": {"alpha": PAPER_ALPHA, "tokens_per_s": proj_tok_s,
                                "speedup_vs_vanilla": (proj_tok_s / arms["vanilla"]["tokens_per_s"])
                                if "vanilla" in arms else None,
                                "note": "projection, tokens/iteration = n*alpha+1 (proj/src/cli.cpp:403)"},
            "roofline": {"kernel": f"sgemv_kernel<8,EPI_SILU> (stream-K bf16 GEMV, base gate/up {gu_shape}, "
                                   f"T={n + 1})",
                         "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": (achieved / hbm) if achieved else None, "traffic": traffic,
                         "traffic_source": traffic_src,
                         "launches_timed": cnt, "bytes_per_launch": site_bytes, "peak_source": peak_kind,
                         "timing": "CUDA events around each launch on the engine stream, in a separate pass of "
                                   "the EasySpec arm (the headline pass runs without them)"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": es["launches"],
            "clocks": es["clocks"],
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
