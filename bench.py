"""PPO experience-making benchmark (BASELINE.json metric: rollout tokens/s +
experience samples/s, 1/2/4/8 B200 vs the host-CPU reference).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2|c1|c3|c4]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, NCCL)

A step = one experience step (ppo_step's experience half, src/ppo.cpp:302-393,
+ advantage whitening) for this rank's prompts: batched rollout decode,
policy + reference log-probs, critic values, scripted reward, KL shaping, GAE
and whitening through ONE all-gather of 6 fp64 partials.  Weak scaling: every
rank owns B prompts (global indices rank*B ...).

value        = rollout tokens/s (generated tokens incl. EOT / generation-phase
               device time, CUDA events, max over ranks), inputs resident in HBM.
e2e          = the same metric through the C ABI with HOST buffers
               (ppoexp_engine_generate, prompts H2D + tokens/log-probs D2H inside
               the timed region), plus experience samples/s through
               ppoexp_make_experience with HOST buffers.
cpu_baseline = the reference itself (oracle/_ref, compiled from its sources)
               on the host cores, bounded sample, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (V, d, L, H, f, S, B per rank, P, N, sampling, description)
    "c1": (1024, 128, 2, 4, 512, 128, 8, 9, 64, "greedy", "tiny GPT policy 2x128, vocab 1k, 8 prompts x 64 greedy"),
    "c2": (50257, 768, 12, 12, 3072, 512, 64, 64, 256, "top_p", "GPT-style 125M policy+reference+critic, 64 prompts x 256 tokens, top-p"),
    "c3": (32000, 2048, 24, 16, 8192, 1024, 32, 128, 512, "top_p", "1.3B policy/critic, 256x512 global (32 per rank at 8 GPUs), vocab 32k"),
    "c4": (128256, 4096, 32, 32, 14336, 2048, 64, 128, 1024, "top_p", "8B-shape reference block, paged KV, 64 prompts x 1024 per GPU"),
}
TOP_P = 0.9
SEED = 20240809


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "fallback": True}


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu, self.p = gpu, None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.p:
            time.sleep(0.25)
            self.p.terminate()
            out, _ = self.p.communicate(timeout=5)
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None, "reasons": sorted(reasons),
                "samples": len(sm)}


def init_weights(cfg, seed, device, head=False):
    """Random-init weights of the reference architecture (N(0,0.02) projections
    and embeddings, LayerNorm 1/0, scalar head N(0,0.1); src/model.cpp:156-184,
    tests/test_ppo.cpp:40-44), generated on the device in bf16."""
    import torch
    from paper_2405_01481_b200 import ppoexp as px
    g = torch.Generator(device=device).manual_seed(seed)
    out = {}
    for name, shape in px.expected_names(cfg.with_head(head)):
        if "norm.weight" in name:
            t = torch.ones(shape, device=device, dtype=torch.bfloat16)
        elif "norm.bias" in name:
            t = torch.zeros(shape, device=device, dtype=torch.bfloat16)
        elif name == "scalar_head.weight":
            t = (torch.randn(shape, generator=g, device=device) * 0.1).to(torch.bfloat16)
        else:
            t = (torch.randn(shape, generator=g, device=device) * 0.02).to(torch.bfloat16)
        out[name] = t
    return out


def prompts_for(rank, B, P, V, seed):
    """Synthetic byte-range prompts (ids < 256), fixed per global index."""
    rng = np.random.default_rng([seed, rank])
    return [rng.integers(0, 256, size=P).astype(np.int32) for _ in range(B)]


def reference_sample(cfg_t, threads, n_new, steps=1, seed=SEED):
    """Times the REFERENCE itself (oracle/_ref = /root/reference sources compiled
    in place) on the host: Engine::generate_batch with n_workers = threads,
    one sequence per worker, P-token prompts, n_new sampled tokens.  Returns
    (tokens/s, seconds per step)."""
    from oracle.oracle import ModelCfg, RefLib
    V, d, L, H, f, S, B, P, N, _, _ = cfg_t
    ref = RefLib()
    cfg = ModelCfg(V, d, L, H, f, S)
    w = ref.init_params(cfg, seed)
    prompts = prompts_for(0, threads, P, V, seed)
    seeds = [ref.mix_seed(seed, i) for i in range(threads)]
    rates, secs = [], []
    for _ in range(steps):
        toks, _, s = ref.generate_batch(cfg, w, prompts, n_new, greedy=False, temperature=1.0, seeds=seeds,
                                        n_workers=threads)
        n = sum(len(t) for t in toks)
        rates.append(n / s)
        secs.append(s)
    return float(np.median(rates)), secs


def workload_config(args, world, B=None):
    """The `config` object of the JSON line (identical for both arms)."""
    V, d, L, H, f, S, Bc, P, N, samp, desc = CONFIGS[args.config]
    B = B if B is not None else (args.batch or Bc)
    return {"workload": args.config, "description": desc, "vocab": V, "d_model": d, "n_layers": L,
            "n_heads": H, "d_ff": f, "max_seq_len": S, "prompts_per_rank": B, "global_batch": B * world,
            "prompt_len": P, "max_new": N, "sampling": samp if samp == "greedy" else f"top_p={TOP_P}",
            "models": "policy+reference+critic, scripted reward", "parallelism": f"dp{world}",
            "l2": "flushed between timed steps (256 MiB write); weights+KV > L2"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg_t = CONFIGS[args.config]
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    threads = max(1, min(threads, 128))
    n_new = args.ref_new_tokens
    # warmup + timed steps; each step is a bounded sample of the workload
    reference_sample(cfg_t, threads, n_new, steps=max(0, min(args.warmup, 1)))
    val, secs = reference_sample(cfg_t, threads, n_new, steps=args.steps)
    V, d, L, H, f, S, B, P, N, samp, desc = cfg_t
    sample = (f"{threads} sequences (one per host thread) x {P}-token prompt x {n_new} sampled tokens through the "
              f"reference's Engine::generate_batch (n_workers={threads}, fp64) per step; prompts fed token-by-token "
              f"as the reference does")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    line = {"impl": "reference", "metric": "rollout_tokens_per_s", "value": val, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * float(np.mean(secs)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, world),
            "note": "the reference's own CPU path on this box's host cores (no GPU used)",
            "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": threads, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _dbg(*a):
    if os.environ.get("PPOEXP_BENCH_DEBUG"):
        print(f"[rank {os.environ.get('RANK', '0')}]", *a, file=sys.stderr, flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2405_01481_b200 import ppoexp as px

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    V, d, L, H, f, S, B, P, N, samp, desc = CONFIGS[args.config]
    if args.batch:
        B = args.batch
    cfg = px.ModelConfig(V, d, L, H, f, S)
    ctx = px.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    w_pol = init_weights(cfg, SEED, dev)
    w_ref = init_weights(cfg, SEED + 1, dev)
    w_crit = init_weights(cfg, SEED + 101, dev, head=True)
    policy = px.DeviceModel(ctx, cfg, w_pol, px.BF16)
    engine = px.Engine(policy, px.EngineOptions(max_batch=max(B, 1), page_size=64,
                                                 max_total_tokens=B * (-(-(P + N) // 64)) * 64))
    reference = px.DeviceModel(ctx, cfg, w_ref, px.BF16)
    critic = px.DeviceModel(ctx, cfg.with_head(), w_crit, px.BF16)
    del w_pol, w_ref, w_crit
    torch.cuda.synchronize()

    # the single collective: all-gather of the 6 fp64 partials, summed in rank
    # order on every rank (paper_2405_01481_b200/dist.py)
    from paper_2405_01481_b200.dist import allgather_sum_fn
    allreduce = allgather_sum_fn(device=dev) if world > 1 else None

    xm = px.ExperienceMaker(engine, reference, critic, scripted_target=ord("e"),
                            hyper=px.PpoHyper(0.003, 1.0, 0.95), allreduce=allreduce)
    sampling = (px.SamplingSpec.greedy_spec() if samp == "greedy"
                else px.SamplingSpec.temperature_spec(1.0, 0, 0, TOP_P))
    prompts = prompts_for(rank, B, P, V, SEED)
    flat = np.concatenate(prompts).astype(np.int32)
    offs = np.concatenate([[0], np.cumsum([len(p) for p in prompts])]).astype(np.int64)
    prompts_d = torch.from_numpy(flat).to(dev)
    offs_d = torch.from_numpy(offs).to(dev)
    out = px.ExperienceMaker.alloc_device_outputs(B, N, dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()

    def step(i):
        xm.run_device(prompts_d, offs_d, out, max_new=N, sampling=sampling, seed=SEED, step_index=i, gidx0=rank * B)

    _dbg("models ready")
    for i in range(args.warmup):
        step(i)
        _dbg("warmup step", i)
    ctx.synchronize()
    roof_cls = args.roofline_class
    live_classes = ["logprob_gather", "gemm_tc"]  # launched eagerly: events here do not perturb the graphs
    if args.profile_classes:
        ctx.profile_filter(live_classes)
        ctx.profile(True)
    launches0 = ctx.launch_count
    gen_ms, step_ms, tokens, seqs = [], [], 0, 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()  # L2 flush between timed iterations (outside the events)
            barrier()
            ctx.synchronize()
            torch.cuda.synchronize()
            ev0.record(stream)
            step(args.warmup + i)
            ev1.record(stream)
            ev1.synchronize()
            st = out["stats"].cpu().numpy()
            gen_ms.append(float(st[6]))
            step_ms.append(ev0.elapsed_time(ev1))
            tokens += int(out["lengths"].sum().item())
            seqs += B
            _dbg("timed step", i)
    barrier()
    launches = ctx.launch_count - launches0
    roof = None
    prof = {}
    live = {}
    if args.profile_classes:
        live = {k: ctx.profile_query(k) for k in live_classes}
        # one extra, fully profiled step (outside the timed region) for the breakdown
        ctx.profile_filter(None)
        ctx.profile(True)
        step(args.warmup + args.steps)
        for cls in ("gemm_decode", "decode_attention", "gemm_tc", "gemm_simt", "logprob_gather", "sampler",
                    "attention_prefill", "layernorm", "embed", "kv_scatter", "shape_gae", "convert", "meta"):
            q = ctx.profile_query(cls)
            if q["launches"]:
                prof[cls] = q
        ctx.profile(False)
        ctx.profile_filter(None)

    # max over ranks
    def gmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def gsum(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        return float(t.item())

    total_gen_s = gmax(sum(gen_ms)) / 1000.0
    total_step_s = gmax(sum(step_ms)) / 1000.0
    all_tokens = gsum(tokens)
    all_seqs = gsum(seqs)
    value = all_tokens / total_gen_s
    samples_per_s = all_seqs / total_step_s
    max_launches = int(gmax(launches))  # collective: every rank participates

    # ---- e2e through the C ABI with HOST buffers (pinned staging inside the library)
    e2e_tok, e2e_xp, h2d, d2h = None, None, 0, 0
    if args.e2e_steps > 0:
        tasks = [px.GenTask(p, N, px.SamplingSpec.temperature_spec(1.0, 1000 + rank * B + i, 0, TOP_P)
                            if samp != "greedy" else px.SamplingSpec.greedy_spec()) for i, p in enumerate(prompts)]
        walls, ntok = [], 0
        for i in range(args.e2e_steps):
            barrier()
            t0 = time.perf_counter()
            res = engine.generate_batch(tasks)
            walls.append(time.perf_counter() - t0)
            ntok += sum(len(r.tokens) for r in res)
        e2e_tok = gsum(ntok) / gmax(sum(walls))
        walls = []
        for i in range(args.e2e_steps):
            barrier()
            t0 = time.perf_counter()
            xm.run(prompts, max_new=N, sampling=sampling, seed=SEED, step_index=100 + i, gidx0=rank * B)
            walls.append(time.perf_counter() - t0)
        e2e_xp = gsum(B * args.e2e_steps) / gmax(sum(walls))
        h2d = int(flat.nbytes + offs.nbytes + B * 8 * 3)
        d2h = int(B * N * (4 + 8) + B * 8)

    if rank == 0:
        pk = peaks()
        line = {"metric": "rollout_tokens_per_s", "value": value, "unit": "tokens/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_step_s * 1000 / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic prompts, random-init weights",
                "config": workload_config(args, world, B),
                "experience_samples_per_s": samples_per_s,
                "gen_ms_per_step": total_gen_s * 1000 / args.steps,
                "gpu_launches": max_launches,
                "clocks": clk.summary()}
        if e2e_tok is not None:
            line["e2e"] = {"value": e2e_tok, "unit": "tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                           "experience_samples_per_s": e2e_xp,
                           "api": "ppoexp_engine_generate / ppoexp_make_experience, HOST buffers"}
        def rf(v, tensor):
            if tensor:
                ach, peak, unit = v["flops"] / v["ms"] / 1e9, pk.get("bf16_tflops_sustained", 1400.0), "TFLOP/s"
            else:
                ach, peak, unit = v["bytes"] / v["ms"] / 1e6, pk.get("hbm_gbs", 6650.0), "GB/s"
            return {"bound": "tensor" if tensor else "hbm", "achieved": ach, "peak": peak, "unit": unit,
                    "frac": ach / peak, "per_launch_ms": v["ms"] / v["launches"], "launches": v["launches"],
                    "algorithmic_per_launch": (v["flops"] if tensor else v["bytes"]) / v["launches"]}
        # measured DRAM traffic per launch of the roofline class, from the newest
        # committed ncu launch list (profiles/<round>/traffic.json)
        traffic, traffic_src = None, None
        try:
            import glob
            tj = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "*",
                                               "traffic.json")))
            if tj:
                tdoc = json.load(open(tj[-1]))
                traffic = tdoc["bytes_per_launch"].get(roof_cls)
                traffic_src = os.path.relpath(tj[-1], os.path.dirname(os.path.abspath(__file__)))
        except Exception:
            pass
        if prof.get(roof_cls, {}).get("launches"):
            line["roofline"] = {"kernel": roof_cls, **rf(prof[roof_cls], roof_cls in ("gemm_tc",)), "traffic": traffic,
                                "traffic_source": traffic_src,
                                "peak_source": "MEASURED_PEAKS.json" + (" (fallback)" if pk.get("fallback") else ""),
                                "timing": "CUDA events on the library stream around every launch of this class, "
                                          "one extra step of the same workload after the timed region (events inside "
                                          "the decode CUDA graph break its PDL overlap, so the timed region carries "
                                          "events only on eagerly launched classes: see roofline_live)"}
        if live:
            line["roofline_live"] = {k: rf(v, k in ("gemm_tc",)) for k, v in live.items() if v["launches"]}
            line["roofline_live_note"] = ("per-launch CUDA events in the timed region; the reference and critic "
                                          "scoring forwards run on two extra streams concurrently with the policy "
                                          "forward, so these durations include overlap with the other streams")
        if prof:
            line["kernel_classes"] = {k: {"ms": v["ms"], "launches": v["launches"],
                                          "GB_s": v["bytes"] / v["ms"] / 1e6 if v["ms"] else None,
                                          "TF_s": v["flops"] / v["ms"] / 1e9 if v["ms"] else None}
                                      for k, v in prof.items()}
            line["kernel_classes_note"] = "one extra fully-profiled step after the timed region (events perturb PDL)"
            line["roofline_by_kernel"] = {k: rf(prof[k], k in ("gemm_tc",)) for k in
                                          ("logprob_gather", "decode_attention", "gemm_decode", "gemm_tc")
                                          if k in prof and prof[k]["ms"]}
        if not args.no_cpu_baseline and world == 1:
            try:
                threads = len(os.sched_getaffinity(0))
                cpu_val, secs = reference_sample(CONFIGS[args.config], threads, args.ref_new_tokens, steps=1)
                line["cpu_baseline"] = {"value": cpu_val, "unit": "tokens/s", "cores": threads, "kind": "reference",
                                        "sample": f"{threads} seqs x {P}-token prompt x {args.ref_new_tokens} sampled "
                                                  f"tokens, reference Engine::generate_batch n_workers={threads}, "
                                                  f"{secs[0]:.1f} s"}
            except Exception as e:  # reference build absent
                line["cpu_baseline"] = {"value": None, "unit": "tokens/s", "cores": 0, "kind": "reference",
                                        "sample": f"unavailable: {e}"}
        print(json.dumps(line), flush=True)
    # Ordered teardown: torch tensors that lived on the library stream, then the
    # library objects (engine before its models, models before the context),
    # then the process group.
    torch.cuda.synchronize()
    del out, flush, prompts_d, offs_d, stream
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    xm = None
    engine.close()
    policy.close()
    reference.close()
    critic.close()
    ctx.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--profile-classes", action="store_true", default=True)
    ap.add_argument("--no-profile", dest="profile_classes", action="store_false")
    ap.add_argument("--roofline-class", default="gemm_decode")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-new-tokens", type=int, default=8)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
    # everything is torn down explicitly above; skip interpreter-exit
    # destructors (torch / NCCL module teardown order is not ours to control)
    sys.stdout.flush()
    sys.stderr.flush()
    os._exit(0)


if __name__ == "__main__":
    main()
