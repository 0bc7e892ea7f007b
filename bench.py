"""Bench: MPIC-k partial-reuse prefill (BASELINE.json metric: prefill tokens/s and p50 TTFT).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]

One step = one MPIC-k request end to end on one GPU: select_tokens -> assemble the
request's KV from its cached image chunks (K2) -> selective recompute of the text tokens
plus the first k tokens of every image through all layers (K3-K8) -> first-token logits.
Default workload is config C: LLaVA-1.6-7B shape, 32 layers x 32 heads x
128, vocab 32000, 4 images of 2304 tokens each preceded by 32+7i text tokens, 32-token
tail, k=32 => n=9418 prompt tokens, m=330 recomputed rows. bf16 weights synthesised on
the device from seed 1 (bit-exact build_model, rounded to bf16); synthetic chunk KV.

value : prompt tokens/s with the chunks resident in HBM (the store's Device tier),
        device-timed with CUDA events; each rank serves its own requests (request
        sharding, no collective) and value = all ranks' tokens / max-over-ranks time.
e2e   : the same request through mpic_request_prefill_host with the chunk KV in pinned
        HOST memory (fp32, as the .mpic store holds it): the per-layer H2D copies, the
        ids upload and the logits download are inside the timed region.
--impl reference: the unmodified reference (oracle/_ref, built from proj/src) on the
        host cores, same workload, bounded sample (2 of 32 layers, scaled x16).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (L, H, D, V, [image tokens], k, text prefix fn)
    "A": (2, 8, 64, 4096, [576, 576], 32),
    "B": (32, 32, 128, 32000, [576], 32),
    "C": (32, 32, 128, 32000, [2304] * 4, 32),
    "D": (32, 32, 128, 32000, [2304] * 8, 32),
    "E16": (32, 32, 128, 32000, [2304] * 16, 32),
    "E": (32, 32, 128, 32000, [576], 32),  # images per request vary: see serving_requests()
}
WORKLOAD_NAMES = {
    "A": "A: tiny decoder L2 H8 D64 V4096, 2x576-token images + text, MPIC-k k=32",
    "B": "B: LLaVA-1.5-7B shape L32 H32 D128 V32000, 1x576-token image + text, MPIC-k k=32",
    "C": "C: LLaVA-1.6-7B shape L32 H32 D128 V32000, 4x2304-token images interleaved with "
         "text (32+7i prefix tokens, 32-token tail), MPIC-k k=32, AsStored",
    "D": "D: MRAG 8x2304-token retrieved images, LLaVA-1.6 shape, MPIC-k k=32",
    "E16": "E: one long request, 16x2304-token images, LLaVA-1.6 shape, MPIC-k k=32",
    "E": "E: batched serving, 256 requests of 1-4 images (U{1..4}, seeded) drawn from a pool of 64 "
         "distinct 576-token chunks resident in HBM, text prefixes 32+7i and a 32-token tail, "
         "LLaVA-1.5 shape L32 H32 D128 V32000, MPIC-k k=32; requests sharded over the ranks",
}

E_REQUESTS, E_POOL = 256, 64


def serving_requests(V, n_req=E_REQUESTS, pool=E_POOL, seed=7):
    """Config E: the same seeded request list on every rank. Returns the pool's
    content hashes and, per request, (segments, pool indices of its images)."""
    rng = np.random.default_rng(seed)
    hashes = [rng.bytes(32) for _ in range(pool)]
    reqs = []
    for _ in range(n_req):
        imgs = rng.integers(0, pool, int(rng.integers(1, 5))).tolist()
        segs = []
        for i, c in enumerate(imgs):
            segs.append(("text", rng.integers(0, V - 1, 32 + 7 * i).tolist()))
            segs.append(("image", hashes[c], 576))
        segs.append(("text", rng.integers(0, V - 1, 32).tolist()))
        reqs.append((segs, imgs))
    return hashes, reqs


def shard_requests(reqs, world, rank):
    """Request sharding without a collective: longest-processing-time-first over the ranks by
    the predicted cost (recomputed rows x layers dominate; images add attention keys)."""
    cost = [(len(im) * 32 + sum(len(sg[1]) for sg in segs if sg[0] == "text")) for segs, im in reqs]
    load = [0.0] * world
    mine = []
    for i in sorted(range(len(reqs)), key=lambda i: (-cost[i], i)):
        r = min(range(world), key=lambda w: (load[w], w))
        load[r] += cost[i]
        if r == rank:
            mine.append(i)
    return sorted(mine)


def run_serving(args, world, rank, local):
    """Config E: this rank's share of the 256 requests, each an MPIC-k request over pooled
    device-resident chunks. One step = the rank's whole share; value = all ranks' prompt
    tokens / max-over-ranks device time."""
    import torch

    import paper_2502_01960_b200 as mp

    L, H, D, V, _, k = CONFIGS["E"]
    h = H * D
    torch.cuda.set_device(local)
    stream = torch.cuda.Stream(device=local)
    cfg = mp.config(L, H, D, vocab_size=V, image_token_count=576, seed=1)
    model = mp.Model(cfg, mp.BF16, device=local)
    hashes, reqs = serving_requests(V)
    mine = shard_requests(reqs, world, rank)
    prompts = [mp.Prompt.from_segments(reqs[i][0]) for i in mine]
    used = sorted({c for i in mine for c in reqs[i][1]})
    g = np.random.default_rng(1234)
    host = [(np.ascontiguousarray(np.broadcast_to(g.random((576, h), dtype=np.float32) - 0.5, (L, 576, h))),
             np.ascontiguousarray(np.broadcast_to(g.random((576, h), dtype=np.float32) - 0.5, (L, 576, h))))
            for _ in range(4)]
    pool = {}
    for c in used:  # chunk c holds one of four synthetic payloads (timing only)
        kv = mp.KV(L, 576, H, D, mp.BF16, local)
        kv.upload(*host[c % 4])
        pool[c] = kv
    del host
    ns = [p.n for p in prompts]
    ms = [len(mp.select_tokens(p, mp.POLICY_MPIC_K, k)) for p in prompts]
    B = max(1, args.batch)
    batches = [list(range(j, min(j + B, len(mine)))) for j in range(0, len(mine), B)]
    if B > 1:  # batched varlen requests (mpic_request_prefill_batch): one cache holds a batch
        ws = mp.Workspace(model, max(sum(ms[j] for j in b) for b in batches),
                          max(sum(ns[j] for j in b) for b in batches))
        big = mp.KV(L, max(sum(ns[j] for j in b) for b in batches), H, D, mp.BF16, local)
    else:
        ws = mp.Workspace(model, max(ms) if ms else 1, max(ns) if ns else 1)
        linked = {n: mp.KV(L, n, H, D, mp.BF16, local) for n in sorted(set(ns))}

    batch_ms = []

    def step(ttft=None, clk=None):
        for b in batches:
            t0 = time.perf_counter()
            if ttft is not None:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            if B > 1:
                mp.request_prefill_batch(model, ws, [prompts[j] for j in b],
                                         [[pool[c] for c in reqs[mine[j]][1]] for j in b], big, k=k, stream=stream)
            else:
                (j,) = b
                mp.request_prefill(model, ws, prompts[j], [pool[c] for c in reqs[mine[j]][1]], linked[prompts[j].n],
                                   k=k, stream=stream)
            if ttft is not None:  # every request of a batch gets its logits when the batch ends
                ttft.extend([(time.perf_counter() - t0) * 1e3] * len(b))
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(stream)
                if clk is not None:
                    clk.probe(stream)  # the SM clock right after the batch (device-side)
                e1.synchronize()
                batch_ms.append(round(e0.elapsed_time(e1), 2))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(world)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ttft = []
    clk = ClockSampler(local, args.steps * len(batches))
    import gc
    gc.collect()
    gc.disable()  # a full Python GC inside the region stalled single steps by 0.3-1.2 s (MPIC_BENCH_GC=1 keeps it)
    if os.environ.get("MPIC_BENCH_GC") == "1":
        gc.enable()
    with clk, torch.cuda.stream(stream):
        ev[0].record(stream)
        for _ in range(args.steps):
            step(ttft, clk)
        ev[1].record(stream)
    torch.cuda.synchronize()
    gc.enable()
    ms_total = allreduce_max(ev[0].elapsed_time(ev[1]), world)
    tok_all = sum(mp.Prompt.from_segments(sg).n for sg, _ in reqs)
    rows_all = sum(len(mp.select_tokens(mp.Prompt.from_segments(sg), mp.POLICY_MPIC_K, k)) for sg, _ in reqs)
    return dict(value=tok_all * args.steps / (ms_total / 1e3), ms_per_step=ms_total / args.steps,
                ttft_p50=float(statistics.median(ttft)) if ttft else None, n=tok_all, m=rows_all,
                rows_per_s=rows_all * args.steps / (ms_total / 1e3), mine=len(mine), world=world,
                batch_ms=batch_ms, clocks=clk.summary(),
                batch_sm_mhz=[round(x) for x in clk.buf[:clk.i].cpu().tolist()])



def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return (float(p["hbm_gbs"]), float(p["bf16_tflops"]), float(p["bf16_tflops_sustained"]),
                "measured")
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


def build_prompt(cfg_name, V, seed=42):
    L, H, D, _, images, k = CONFIGS[cfg_name]
    rng = np.random.default_rng(seed)
    segs = []
    for i, t in enumerate(images):
        segs.append(("text", rng.integers(0, V - 1, 32 + 7 * i).tolist()))
        segs.append(("image", rng.bytes(32), t))
    segs.append(("text", rng.integers(0, V - 1, 32).tolist()))
    return segs


def prompt_stats(cfg_name, k=None):
    """(n prompt tokens, m recomputed rows) of the config's request under MPIC-k
    (select_tokens, linker.cpp:209-258: every text token + the first k of each image)."""
    L, H, D, V, images, kk = CONFIGS[cfg_name]
    k = kk if k is None else k
    segs = build_prompt(cfg_name, V)
    n = sum(len(sg[1]) if sg[0] == "text" else sg[2] for sg in segs)
    m = sum(len(sg[1]) if sg[0] == "text" else min(k, sg[2]) for sg in segs)
    return n, m


def config_json(args):
    """The `config` object of the JSON line: identical in both arms (--impl ours|reference)."""
    L, H, D, V, images, k = CONFIGS[args.config]
    cj = {"workload": WORKLOAD_NAMES[args.config], "layers": L, "heads": H, "head_dim": D,
          "vocab": V, "image_tokens": images, "k": k,
          "parallelism": f"request-sharded x{args.gpus} (no collective)",
          "l2": "inputs larger than L2: 12.9 GB bf16 weights + 4.8 GB chunk KV stream "
                "through HBM every step"}
    if args.config == "E":
        _, reqs = serving_requests(V)
        cj.update(requests=E_REQUESTS, pool_chunks=E_POOL, batch=max(1, args.batch),
                  n_tokens_total=sum(sum(len(sg[1]) if sg[0] == "text" else sg[2] for sg in segs)
                                     for segs, _ in reqs),
                  parallelism=f"request-sharded x{args.gpus} (LPT by predicted cost, no collective)",
                  l2="inputs larger than L2: 12.9 GB bf16 weights stream through HBM per request")
    else:
        n, m = prompt_stats(args.config, k)
        cj.update(n_tokens=n, recompute_rows=m)
    if args.mode == "head-parallel":
        cj["parallelism"] = f"head-parallel x{args.gpus} (NCCL reduce-scatter + all-gather per layer)"
    return cj


class ClockSampler:
    """Clocks and throttle reasons of the timed region.

    On these VM-hosted B200s every NVML query (nvidia-smi or pynvml) stalls GPU work
    submission: sampling at 50-250 ms periods inside the timed region produced 30-770 ms
    step outliers (profiles/r1_clock_sampling.md). So the SM clock is measured ON THE
    DEVICE during the region — a 5 us clock64 / %globaltimer probe kernel on the timed
    stream after every step (mpic_clock_probe) — and nvidia-smi is queried for the clocks
    and the throttle reasons right before and right after the region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device_index=0, steps=1):
        import torch
        self.dev = device_index
        self.rows = []
        self.buf = torch.zeros(max(steps, 1), dtype=torch.float32, device=f"cuda:{device_index}")
        self.i = 0

    def _query(self):
        import subprocess
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                 timeout=20).stdout
            for line in out.splitlines():
                parts = [p.strip() for p in line.split(",")]
                if len(parts) == 6:
                    self.rows.append(parts)
        except Exception:
            pass

    def probe(self, stream):
        """Enqueue one on-device clock measurement (after a step, on the timed stream)."""
        from paper_2502_01960_b200 import _lib
        if self.i < self.buf.numel():
            _lib.check(_lib.lib().mpic_clock_probe(self.buf.data_ptr() + 4 * self.i, 5000,
                                                   _stream_handle(stream)))
            self.i += 1

    def __enter__(self):
        self._query()
        return self

    def __exit__(self, *a):
        self._query()

    def summary(self):
        dev_mhz = [float(x) for x in self.buf[:self.i].cpu().tolist()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({n for r in self.rows for n, v in zip(self.NAMES, r[2:]) if v.lower() == "active"})
        return {"sm_mhz": float(statistics.median(dev_mhz)) if dev_mhz else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(dev_mhz), "sm_mhz_min": min(dev_mhz) if dev_mhz else None,
                "method": "device clock64/globaltimer probe after every timed step; nvidia-smi "
                          "reasons before+after the region",
                "nvidia_smi_sm_mhz": [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]}


def _stream_handle(stream):
    return int(getattr(stream, "cuda_stream", stream))


def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def allreduce_max(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def algorithmic(cfg_name, n, m, sel, elt=2):
    """Algorithmic bytes / FLOPs per step."""
    L, H, D, V, images, _ = CONFIGS[cfg_name]
    h = H * D
    img = sum(images)
    asm_bytes = 2 * img * L * 2 * h * elt  # read chunks + write assembled K and V
    attn_flops_layer = 4.0 * h * float(np.sum(sel.astype(np.float64) + 1))
    gemm = {"qkv": 2.0 * m * 3 * h * h, "wo": 2.0 * m * h * h, "w1": 2.0 * m * 4 * h * h,
            "w2": 2.0 * m * 4 * h * h}
    gemm_bytes = {"qkv": 3 * h * h * elt, "wo": h * h * elt, "w1": 4 * h * h * elt,
                  "w2": 4 * h * h * elt}
    return asm_bytes, attn_flops_layer, gemm, gemm_bytes, 2.0 * h * V


def linked_blocks(segs, sel, n, head_dim, elt=2):
    """Number of 128-row cache blocks that attention reads straight from a cached chunk and
    stores into the request cache itself (capi.cu plan_attn_link): the block lies inside one
    image segment and holds no recomputed row. The assembly kernel skips them, so its
    algorithmic bytes cover only the other image rows (MPIC_ATTN_LINK=0 assembles all)."""
    if head_dim != 128 or elt != 2 or os.environ.get("MPIC_ATTN_LINK", "1") == "0":
        return 0
    spans, at = [], 0
    for sg in segs:
        t = len(sg[1]) if sg[0] == "text" else sg[2]
        if sg[0] == "image":
            spans.append((at, at + t))
        at += t
    if not spans or len(spans) > 8:
        return 0
    rec = np.zeros(n, bool)
    rec[np.asarray(sel, np.int64)] = True
    nb = 0
    for b in range(n // 128):
        a0 = b * 128
        for s0, s1 in spans:
            if s0 <= a0 and a0 + 128 <= s1:
                nb += int(not rec[a0:a0 + 128].any())
                break
    return nb


def run_ours(args, world, rank, local):
    import torch

    import paper_2502_01960_b200 as mp

    L, H, D, V, images, k = CONFIGS[args.config]
    h = H * D
    dev = local
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(device=dev)
    cfg = mp.config(L, H, D, vocab_size=V, image_token_count=images[0], seed=1)
    model = mp.Model(cfg, mp.BF16, device=dev)
    segs = build_prompt(args.config, V, seed=42 + rank)
    prompt = mp.Prompt.from_segments(segs)
    n = prompt.n
    sel = mp.select_tokens(prompt, mp.POLICY_MPIC_K, k)
    m = len(sel)
    ws = mp.Workspace(model, m, n)

    # chunk KV: pinned host fp32 (Host tier / .mpic payload) and a bf16 HBM copy (Device tier)
    host_k, host_v, host_kf, host_vf, dev_chunks = [], [], [], [], []
    g = np.random.default_rng(1234 + rank)
    for t in images:
        rk = g.random((t, h), dtype=np.float32) - 0.5  # U(-0.5, 0.5), one draw per chunk
        rv = g.random((t, h), dtype=np.float32) - 0.5
        kv = mp.KV(L, t, H, D, mp.BF16, dev)
        kv.upload(np.broadcast_to(rk, (L, t, h)), np.broadcast_to(rv, (L, t, h)))
        dev_chunks.append(kv)
        if not args.no_e2e:  # the Host tier copies the e2e legs stream from (pinned)
            hk, hv = mp.HostBuffer((L, t, h), np.uint16), mp.HostBuffer((L, t, h), np.uint16)
            hk.array[:] = mp.to_bf16_bits(rk)  # model-dtype Host tier (bf16)
            hv.array[:] = mp.to_bf16_bits(rv)
            host_k.append(hk)
            host_v.append(hv)
            if args.e2e_fp32:  # .mpic v1 payload (fp32), reported beside it
                fk, fv = mp.HostBuffer((L, t, h)), mp.HostBuffer((L, t, h))
                fk.array[:] = rk
                fv.array[:] = rv
                host_kf.append(fk)
                host_vf.append(fv)
    linked = mp.KV(L, n, H, D, mp.BF16, dev)

    def step_device():
        logits, _ = mp.request_prefill(model, ws, prompt, dev_chunks, linked, k=k, stream=stream)
        return mp.last_launch_count()

    def step_host(ks=None, vs=None):
        logits, _ = mp.request_prefill_host(model, ws, prompt, [x.array for x in ks or host_k],
                                            [x.array for x in vs or host_v], linked, k=k,
                                            stream=stream)
        return mp.last_launch_count()

    # ---- device-resident path (value) ----
    # Same-shape requests replay a CUDA graph of the whole request (mpic_workspace_set_graphs):
    # warm-up request 2 records it, the timed requests replay it with their inputs re-staged.
    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    launches = 0
    per_step = []
    host_ms = []
    import gc
    gc.collect()
    gc.disable()  # a full collection inside a timed region stalls submission for 100s of ms
    with ClockSampler(dev, args.steps) as clk:
        with torch.cuda.stream(stream):
            ev[0].record(stream)
            for i in range(args.steps):
                h0 = time.perf_counter()
                launches += step_device()
                clk.probe(stream)
                ev[i + 1].record(stream)
                host_ms.append((time.perf_counter() - h0) * 1e3)
        torch.cuda.synchronize()
    gc.enable()
    barrier(world)
    for i in range(args.steps):
        per_step.append(ev[i].elapsed_time(ev[i + 1]))
    # per-phase device times (CUDA events around every phase: eager launches, so a separate
    # pass after the timed region; kernel durations are the same as in the graph)
    mp.profile_enable(True)
    mp.profile_collect()
    for _ in range(args.steps):
        step_device()
    torch.cuda.synchronize()
    mp.profile_enable(False)
    phases = mp.profile_collect()
    # the standalone assembly kernel over the whole request (every image row of every layer,
    # the MPIC_ATTN_LINK=0 form): the HBM-roofline evidence for K2 on its own
    refs = []
    at, ci = 0, 0
    for sg in segs:
        t = len(sg[1]) if sg[0] == "text" else sg[2]
        if sg[0] == "image":
            refs.append((dev_chunks[ci], 0, at, t, 0))
            ci += 1
        at += t
    asm_full = None
    if refs:
        for _ in range(2):
            mp.assemble(refs, linked, stream=stream)
        ea = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        reps = 5
        with torch.cuda.stream(stream):
            ea[0].record(stream)
            for _ in range(reps):
                mp.assemble(refs, linked, stream=stream)
            ea[1].record(stream)
        torch.cuda.synchronize()
        asm_full = ea[0].elapsed_time(ea[1]) / reps
    total_ms = ev[0].elapsed_time(ev[-1])
    total_ms = allreduce_max(total_ms, world)
    ms_per_step = total_ms / args.steps
    value = world * n * args.steps / (total_ms / 1e3)

    # ---- end-to-end through the host-buffer C ABI call (e2e) ----
    def time_host_leg(ks, vs, label):
        for _ in range(max(1, min(args.warmup, 2))):
            step_host(ks, vs)
        torch.cuda.synchronize()
        barrier(world)
        import gc
        gc.collect()
        gc.disable()
        t0 = time.perf_counter()
        ev2 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        with torch.cuda.stream(stream):
            ev2[0].record(stream)
            for i in range(args.steps):
                step_host(ks, vs)
                ev2[i + 1].record(stream)
        torch.cuda.synchronize()
        gc.enable()
        wall = time.perf_counter() - t0
        e2e_steps = [ev2[i].elapsed_time(ev2[i + 1]) for i in range(args.steps)]
        e_ms = allreduce_max(ev2[0].elapsed_time(ev2[-1]), world)
        # the loader skips each chunk's leading recomputed rows (its first k under MPIC-k)
        lead = sum(min(k, sg[2]) for sg in segs if sg[0] == "image")
        skipped = 2 * lead * L * h * ks[0].array.itemsize if ks else 0
        h2d = sum(x.array.nbytes for x in ks + vs) - skipped + 2 * 4 * m
        return {"value": world * n * args.steps / (e_ms / 1e3), "unit": "prompt tokens/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(4 * V),
                "ttft_p50_ms": float(statistics.median(e2e_steps)), "wall_s": wall,
                "path": f"mpic_request_prefill_host ({label} chunks in pinned host memory -> "
                        "per-layer H2D on a side stream overlapped with the layer loop; ids "
                        "H2D, logits D2H)"}

    e2e = e2e_fp32 = e2e_disk = None
    if args.disk:
        # MRAG-style: every chunk read from its .mpic v3 (bf16, per-layer CRCs) file by the disk loader
        # (reader thread -> pinned ring -> HBM per layer, CRC checked); the files are written
        # first, so the reads are served by the page cache (warm), as after a recent fetch.
        import shutil
        import tempfile
        ddir = tempfile.mkdtemp(prefix="mpic_chunks_", dir=args.disk_dir)
        try:
            paths = []
            gd = np.random.default_rng(1234 + rank)
            for i, (seg, t) in enumerate([(sg, sg[2]) for sg in segs if sg[0] == "image"]):
                rk = gd.random((t, h), dtype=np.float32) - 0.5
                rv = gd.random((t, h), dtype=np.float32) - 0.5
                path = os.path.join(ddir, f"chunk{i}.mpic")
                mp.write_mpic(path, cfg, seg[1], np.broadcast_to(rk, (L, t, h)), np.broadcast_to(rv, (L, t, h)),
                              bf16=True)
                paths.append(path)
            fbytes = sum(os.path.getsize(x) for x in paths)
            for _ in range(2):
                mp.request_prefill_files(model, ws, prompt, paths, linked, k=k, stream=stream)
            torch.cuda.synchronize()
            barrier(world)
            t0 = time.perf_counter()
            ttft = []
            for _ in range(args.steps):
                s0 = time.perf_counter()
                mp.request_prefill_files(model, ws, prompt, paths, linked, k=k, stream=stream)
                ttft.append((time.perf_counter() - s0) * 1e3)
            wall = allreduce_max(time.perf_counter() - t0, world)
            e2e_disk = {"value": world * n * args.steps / wall, "unit": "prompt tokens/s",
                        "ttft_p50_ms": float(statistics.median(ttft)), "file_bytes_per_step": int(fbytes),
                        "path": "mpic_request_prefill_files (.mpic v3 bf16 files with per-layer CRCs, page cache warm -> "
                                "reader thread -> pinned ring -> HBM per layer, CRC32 verified)",
                        "timing": "host wall clock per request (the loader is host I/O)"}
        finally:
            shutil.rmtree(ddir, ignore_errors=True)
    sweep = None
    if args.disk and args.k_sweep:
        sweep = disk_k_sweep(args, mp, torch, model, cfg, prompt, segs, dev_chunks, stream, L, H, D, h, n, world,
                             rank, [int(x) for x in args.k_sweep.split(",")])
    if not args.no_e2e:
        e2e = time_host_leg(host_k, host_v, "bf16 Host-tier")
        if args.e2e_fp32:
            e2e_fp32 = time_host_leg(host_kf, host_vf, "fp32 .mpic-v1")

    # ---- decode after the prefill (decode_step, proj/src/model.cpp:356-367 = extend_rows of
    # one row at the end of the cache): bf16 tensor-core path (tcgen05 GEMMs at one token,
    # tcgen05 attention over the whole cache), synchronous per token (host id in, logits out).
    # Per token it must stream every weight (12.9 GB at config C) and the cache's K/V: an
    # HBM-bound step, reported against the measured copy rate.
    decode = None
    if args.decode_steps and rank == 0:
        D_ = args.decode_steps
        kvd = mp.KV(L, n + D_ + 1, H, D, mp.BF16, dev)
        wsd = mp.Workspace(model, 16, n + D_ + 1)
        tok = [int(x) for x in np.random.default_rng(5).integers(0, V - 1, D_ + 1)]
        mp.prefill_extend(model, wsd, [tok[0]], n, 0, kvd, stream=stream)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e_d = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e_d[0].record(stream)
        for i in range(D_):
            mp.prefill_extend(model, wsd, [tok[i + 1]], n + 1 + i, 0, kvd, stream=stream)
        e_d[1].record(stream)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / D_ * 1e3
        dev_ms = e_d[0].elapsed_time(e_d[1]) / D_
        ctx = n + 1 + D_ / 2
        wbytes = L * 12 * h * h * 2 + V * h * 2  # bf16 projection weights + lm_head
        kvbytes = L * ctx * 2 * h * 2            # the cache's K and V (bf16) read by attention
        hbm, _, _, _ = load_peaks()
        decode = {"value": 1e3 / wall, "unit": "tokens/s", "ms_per_token": round(wall, 3),
                  "device_ms_per_token": round(dev_ms, 3), "context_tokens": int(ctx), "steps": D_,
                  "bytes_per_token": int(wbytes + kvbytes),
                  "hbm_frac": round((wbytes + kvbytes) / (wall / 1e3) / 1e9 / hbm, 4),
                  "path": "mpic_prefill_extend of one row at the end of a bf16 cache (decode_step): tcgen05 GEMMs at "
                          "M = 1 token, tcgen05 attention over the cache; host id in, logits out per token"}
        del kvd, wsd

    # ---- miss path: compute_entry of one image chunk on the device
    # (prefill_extend of its token ids at position base 0, transfer.cpp:41-58: a full causal
    # prefill of the chunk's tokens on the tcgen05 kernels), and the request with every chunk
    # missing (mpic_request_prefill_files with no files: the loader's compute lane prefills all
    # chunks on a side stream while the request consumes them layer by layer)
    miss = None
    if args.miss and rank == 0:
        T0 = images[0]
        img_hashes = [sg[1] for sg in segs if sg[0] == "image"]
        wsm = mp.Workspace(model, T0, T0)
        kvm = mp.KV(L, T0, H, D, mp.BF16, dev)
        ids0 = mp.image_token_ids(cfg, img_hashes[0], T0)
        mp.prefill_extend(model, wsm, ids0, 0, 0, kvm, stream=stream)  # warm-up
        torch.cuda.synchronize()
        nrep = 3
        e_m = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e_m[0].record(stream)
        for _ in range(nrep):
            mp.prefill_extend(model, wsm, ids0, 0, 0, kvm, stream=stream)
        e_m[1].record(stream)
        torch.cuda.synchronize()
        chunk_ms = e_m[0].elapsed_time(e_m[1]) / nrep
        fl = L * (2 * T0 * 12 * h * h + 4 * h * T0 * (T0 + 1) / 2)
        _, _, tf_s, _ = load_peaks()
        linked_m = mp.KV(L, n, H, D, mp.BF16, dev)
        none_paths = [None] * len(img_hashes)
        mp.request_prefill_files(model, ws, prompt, none_paths, linked_m, k=k, stream=stream)  # warm-up
        torch.cuda.synchronize()
        walls = []
        for _ in range(2):
            t0 = time.perf_counter()
            mp.request_prefill_files(model, ws, prompt, none_paths, linked_m, k=k, stream=stream)
            torch.cuda.synchronize()
            walls.append((time.perf_counter() - t0) * 1e3)
        miss = {"chunk_prefill_ms": round(chunk_ms, 3), "chunk_tokens": T0,
                "chunk_tflops": round(fl / (chunk_ms / 1e3) / 1e12, 1),
                "chunk_tensor_frac": round(fl / (chunk_ms / 1e3) / 1e12 / tf_s, 4),
                "request_all_miss_ms": round(statistics.median(walls), 3), "chunks": len(img_hashes),
                "path": "prefill_extend of an image chunk's token ids at base 0 (compute_entry) on the tcgen05 "
                        "kernels; the all-miss request through mpic_request_prefill_files (compute lane concurrent "
                        "with the request), host wall time"}
        del wsm, kvm, linked_m

    # ---- fp32 mode: the same request at the reference's own precision (fp32 weights, KV and
    # arithmetic: 3xTF32 tcgen05 GEMMs with segmented accumulation + fp32 online-softmax
    # attention; parity 1e-4 vs the reference in tests/test_gpu_llava.py), device-resident
    # chunks. Two untimed requests: the second records the request's CUDA graph ----
    fp32_mode = None
    if args.fp32_mode and rank == 0:
        model32 = mp.Model(cfg, mp.F32, device=dev)
        ws32 = mp.Workspace(model32, m, n)
        g32 = np.random.default_rng(1234 + rank)
        chunks32 = []
        for t in images:
            rk = g32.random((t, h), dtype=np.float32) - 0.5
            rv = g32.random((t, h), dtype=np.float32) - 0.5
            kv = mp.KV(L, t, H, D, mp.F32, dev)
            kv.upload(np.broadcast_to(rk, (L, t, h)), np.broadcast_to(rv, (L, t, h)))
            chunks32.append(kv)
        linked32 = mp.KV(L, n, H, D, mp.F32, dev)
        for _ in range(2):
            mp.request_prefill(model32, ws32, prompt, chunks32, linked32, k=k, stream=stream)
        torch.cuda.synchronize()
        n32 = 3
        e32 = [torch.cuda.Event(enable_timing=True) for _ in range(n32 + 1)]
        with torch.cuda.stream(stream):
            e32[0].record(stream)
            for i in range(n32):
                mp.request_prefill(model32, ws32, prompt, chunks32, linked32, k=k, stream=stream)
                e32[i + 1].record(stream)
        torch.cuda.synchronize()
        ms32 = [e32[i].elapsed_time(e32[i + 1]) for i in range(n32)]
        fp32_mode = {"value": n / (statistics.mean(ms32) / 1e3), "unit": "prompt tokens/s",
                     "ms_per_step": round(statistics.mean(ms32), 3), "steps": n32, "dtype": "f32",
                     "path": "mpic_request_prefill, fp32 model: 3xTF32 tcgen05 GEMMs (tf32 hi/lo split, "
                             "accumulation drained to fp32 registers every 32 K) + fp32 online-softmax SIMT "
                             "attention, fp32 chunks HBM-resident (the reference's precision; parity <= 1e-4 in "
                             "tests/test_gpu_llava.py; MPIC_F32_GEMM=simt: SIMT FFMA GEMMs)"}
        del model32, ws32, chunks32, linked32

    # ---- roofline of the dominant phase ----
    hbm, tf_burst, tf_sust, peak_src = load_peaks()
    asm_bytes, attn_fl, gemm_fl, gemm_b, lm_fl = algorithmic(args.config, n, m, sel)
    nlink = linked_blocks(segs, sel, n, D)
    link_bytes = 2 * nlink * 128 * L * 2 * h * 2  # read chunk + write request cache, K and V
    asm_full_bytes = asm_bytes
    asm_bytes = asm_bytes - link_bytes  # what the assembly kernel itself moves
    steps = args.steps
    per_phase = {}
    for p, (ms, cnt) in phases.items():
        if cnt == 0:
            continue
        avg = ms / cnt
        if p == "assemble":
            algo, unit = asm_bytes / (cnt / steps), "GB/s"
            ach = algo / (avg / 1e3) / 1e9
            pk = hbm
            bound = "hbm"
        elif p == "attn":
            algo, unit = attn_fl, "TFLOP/s"
            ach = algo / (avg / 1e3) / 1e12
            pk = tf_sust
            bound = "tensor"
        elif p in gemm_fl:
            algo, unit = gemm_fl[p], "TFLOP/s"
            ach = algo / (avg / 1e3) / 1e12
            pk = tf_sust
            bound = "tensor"
            per_phase.setdefault("weight_stream_GBps", {})[p] = round(
                gemm_b[p] / (avg / 1e3) / 1e9, 1)
        else:
            per_phase[p] = {"ms_per_step": round(ms / steps, 4), "launches": cnt}
            continue
        per_phase[p] = {"ms_per_step": round(ms / steps, 4), "launches": cnt,
                        "avg_launch_ms": round(avg, 5), "achieved": round(ach, 2), "unit": unit,
                        "bound": bound, "frac": round(ach / pk, 4)}
    if "attn" in per_phase and nlink:
        per_phase["attn"]["linked_blocks"] = nlink
        per_phase["attn"]["link_bytes_per_step"] = int(link_bytes)
    if asm_full is not None:
        per_phase["assemble_standalone"] = {
            "ms": round(asm_full, 4), "bytes": int(asm_full_bytes),
            "achieved": round(asm_full_bytes / (asm_full / 1e3) / 1e9, 2), "unit": "GB/s",
            "bound": "hbm", "frac": round(asm_full_bytes / (asm_full / 1e3) / 1e9 / hbm, 4),
            "what": "mpic_assemble of every image row of every layer (one launch), timed alone"}
    cand = [(v["ms_per_step"], p) for p, v in per_phase.items()
            if isinstance(v, dict) and "achieved" in v and "ms_per_step" in v]
    dom = max(cand)[1]
    d = per_phase[dom]
    traffic = None
    try:  # DRAM bytes per launch of this kernel from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(dom)
    except Exception:
        pass
    roofline = {"bound": d["bound"], "achieved": d["achieved"],
                "peak": hbm if d["bound"] == "hbm" else tf_sust, "unit": d["unit"],
                "frac": d["frac"], "traffic": traffic, "kernel": dom,
                "traffic_source": "profiles/traffic.json (ncu --set full, one launch)",
                "peak_source": peak_src + (" HBM copy" if d["bound"] == "hbm"
                                           else " bf16 sustained"),
                "per_launch_algorithmic": (asm_bytes if dom == "assemble" else
                                           attn_fl if dom == "attn" else gemm_fl.get(dom))}
    # whole-request fraction: sum over phases of max(F/P, B/BW) / step time
    floor_ms = (asm_full_bytes / (hbm * 1e9) + L * (
        max(sum(gemm_fl.values()) / (tf_sust * 1e12), sum(gemm_b.values()) / (hbm * 1e9)) +
        attn_fl / (tf_sust * 1e12))) * 1e3
    return dict(value=value, ms_per_step=ms_per_step, per_step=per_step, host_ms=host_ms, e2e=e2e,
                e2e_fp32=e2e_fp32, e2e_disk=e2e_disk, fp32_mode=fp32_mode, k_sweep=sweep, decode=decode, miss=miss,
                launches=launches, roofline=roofline, phases=per_phase, clocks=clk.summary(),
                n=n, m=m, floor_ms=floor_ms, world=world)


def disk_k_sweep(args, mp, torch, model, cfg, prompt, segs, dev_chunks, stream, L, H, D, h, n, world, rank, ks):
    """MRAG sweep (SURVEY config D): for each MPIC-k budget (k >= the image length = full
    recompute), the request with its chunks read from .mpic v3 files — warm (page cache, the
    files were just written) and cold (posix_fadvise DONTNEED on every file before each
    request, so the reads come from the device) — beside the device-resident time of the
    same request. Host wall clock per request (the loader is host I/O)."""
    import shutil
    import tempfile
    ddir = tempfile.mkdtemp(prefix="mpic_sweep_", dir=args.disk_dir)
    out = {"k": [], "recompute_rows": [], "device_ms": [], "warm_ttft_ms": [], "cold_ttft_ms": [],
           "what": "per k: device-resident request (CUDA events), then from .mpic v3 bf16 files warm and cold "
                   "(host wall clock, median of the timed requests)"}
    try:
        paths = []
        gd = np.random.default_rng(1234 + rank)
        for i, seg in enumerate([sg for sg in segs if sg[0] == "image"]):
            t = seg[2]
            rk = gd.random((t, h), dtype=np.float32) - 0.5
            rv = gd.random((t, h), dtype=np.float32) - 0.5
            path = os.path.join(ddir, f"chunk{i}.mpic")
            mp.write_mpic(path, cfg, seg[1], np.broadcast_to(rk, (L, t, h)), np.broadcast_to(rv, (L, t, h)), bf16=True)
            paths.append(path)
        out["file_bytes_per_request"] = int(sum(os.path.getsize(x) for x in paths))

        def drop_cache():
            for pth in paths:
                fd = os.open(pth, os.O_RDONLY)
                try:
                    os.fsync(fd)
                    os.posix_fadvise(fd, 0, 0, os.POSIX_FADV_DONTNEED)
                finally:
                    os.close(fd)

        reps = max(2, min(args.steps, 3))
        for kk in ks:
            sel = mp.select_tokens(prompt, mp.POLICY_MPIC_K, kk)
            m = len(sel)
            ws = mp.Workspace(model, m, n)
            linked = mp.KV(L, n, H, D, mp.BF16, torch.cuda.current_device())
            mp.request_prefill(model, ws, prompt, dev_chunks, linked, k=kk, stream=stream)
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
            with torch.cuda.stream(stream):
                ev[0].record(stream)
                for i in range(reps):
                    mp.request_prefill(model, ws, prompt, dev_chunks, linked, k=kk, stream=stream)
                    ev[i + 1].record(stream)
            torch.cuda.synchronize()
            dev_ms = statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(reps))
            mp.request_prefill_files(model, ws, prompt, paths, linked, k=kk, stream=stream)  # page cache warm
            torch.cuda.synchronize()
            warm, cold = [], []
            for _ in range(reps):
                t0 = time.perf_counter()
                mp.request_prefill_files(model, ws, prompt, paths, linked, k=kk, stream=stream)
                warm.append((time.perf_counter() - t0) * 1e3)
            for _ in range(reps):
                drop_cache()
                t0 = time.perf_counter()
                mp.request_prefill_files(model, ws, prompt, paths, linked, k=kk, stream=stream)
                cold.append((time.perf_counter() - t0) * 1e3)
            out["k"].append(kk)
            out["recompute_rows"].append(m)
            out["device_ms"].append(round(dev_ms, 3))
            out["warm_ttft_ms"].append(round(statistics.median(warm), 2))
            out["cold_ttft_ms"].append(round(statistics.median(cold), 2))
            del ws, linked
            torch.cuda.empty_cache()
    finally:
        shutil.rmtree(ddir, ignore_errors=True)
    return out


def run_head_parallel(args, world, rank, local):
    """One long request split by attention head over the ranks: per layer a
    reduce-scatter of the Wo partials and an all-gather of the FFN rows over NCCL."""
    import torch

    import paper_2502_01960_b200 as mp
    from paper_2502_01960_b200 import headpar

    L, H, D, V, images, k = CONFIGS[args.config]
    h = H * D
    torch.cuda.set_device(local)
    stream = torch.cuda.current_stream()
    cfg = mp.config(L, H, D, vocab_size=V, image_token_count=images[0], seed=1)
    segs = build_prompt(args.config, V, seed=42)  # the same request on every rank
    prompt = mp.Prompt.from_segments(segs)
    n = prompt.n
    m_est = len(mp.select_tokens(prompt, mp.POLICY_MPIC_K, k))
    eng = headpar.HeadParallelRank(cfg, rank, world, device=local, max_rows=m_est + world,
                                   max_ctx=n)
    g = np.random.default_rng(1234)
    chunks = []
    for t in images:
        rk = g.random((t, h), dtype=np.float32) - 0.5
        rv = g.random((t, h), dtype=np.float32) - 0.5
        kv = mp.KV(L, t, H, D, mp.BF16, local)
        kv.upload(np.broadcast_to(rk, (L, t, h)), np.broadcast_to(rv, (L, t, h)))
        chunks.append(kv)
    linked = eng.linked_cache(n)
    sh = stream.cuda_stream
    if args.hp_driver == "library":
        # the production path: mpic_hp_request (layer loop + NCCL collectives in C++, the loop
        # replayed as one CUDA graph) on a library-created communicator
        comm = headpar.NcclComm(rank, world, local)

        def step():
            eng.request(prompt, chunks, linked, k=k, stream=sh, comm=comm)
    else:
        comm = headpar.TorchComm() if world > 1 else headpar.SoloComm()

        def step():
            eng.prepare(prompt, chunks, linked, mp.POLICY_MPIC_K, k, sh)
            headpar.prefill_layers(eng, comm, L)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(world)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    clk = ClockSampler(local, args.steps)
    import gc
    gc.collect()
    gc.disable()
    if os.environ.get("MPIC_BENCH_GC") == "1":
        gc.enable()
    with clk:
        ev[0].record(stream)
        for i in range(args.steps):
            step()
            ev[i + 1].record(stream)
            clk.probe(stream)
        torch.cuda.synchronize()
    gc.enable()
    barrier(world)
    per_step = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
    total = allreduce_max(ev[0].elapsed_time(ev[-1]), world)
    return dict(value=n * args.steps / (total / 1e3), ms_per_step=total / args.steps,
                per_step=per_step, n=n, m=eng.m, world=world, clocks=clk.summary(),
                step_sm_mhz=[round(x) for x in clk.buf[:clk.i].cpu().tolist()])


def cpu_reference(cfg_name, steps, warmup, threads=None, layers_sample=2, seed=42):
    """Time the unmodified reference's assemble_linked_cache + selective_prefill on the
    host cores (oracle/_ref). Bounded sample: `layers_sample` of L layers, scaled."""
    import oracle
    L, H, D, V, images, k = CONFIGS[cfg_name]
    h = H * D
    if not oracle.have_ref():
        return None, "oracle/_ref not built"
    r = oracle.RefLib()
    threads = threads or os.cpu_count()
    r.set_threads(threads)
    ls = min(layers_sample, L)
    cfg = oracle.Config(ls, H, D, h, V, images[0], 10000.0, 1)
    rm = r.model(cfg)
    if cfg_name == "E":
        return cpu_reference_serving(r, rm, L, ls, H, D, V, k, threads, steps)
    segs = build_prompt(cfg_name, V, seed)
    p = oracle.make_prompt(segs, "")
    g = np.random.default_rng(1234)
    for t in images:
        p.chunk_k.append((g.random((ls, t, h), dtype=np.float32) - 0.5))
        p.chunk_v.append((g.random((ls, t, h), dtype=np.float32) - 0.5))
        p.chunk_base.append(0)
    sel = rm.select(p, 0, k)
    ents = rm.entries(p)
    times = []
    try:
        for i in range(warmup + steps):
            res = rm.link_and_prefill(p, sel=sel, want_asm=False, want_final=False, entries=ents)
            if i >= warmup:
                times.append((res["ms_assemble"] + res["ms_selective"]) * (L / ls))
    finally:
        r.lib.ref_entries_free(ents)
    return dict(ms=float(statistics.median(times)), n=p.n, m=len(sel), threads=threads,
                sample=f"{ls} of {L} layers of config {cfg_name} (n={p.n}, m={len(sel)}), "
                       f"per-request time scaled x{L / ls:g}; assemble_linked_cache + "
                       f"selective_prefill, OpenBLAS {threads} threads"), None


def cpu_reference_serving(r, rm, L, ls, H, D, V, k, threads, steps, sample=6):
    """Config E on the reference: it serves requests one at a time, so the 256-request time
    is extrapolated from the first `sample` requests of the seeded list (ls of L layers each,
    scaled by L/ls) by prompt tokens."""
    import oracle
    h = H * D
    _, reqs = serving_requests(V)
    g = np.random.default_rng(1234)
    pool = {}
    ms, n_s = 0.0, 0
    for segs, imgs in reqs[:sample]:
        p = oracle.make_prompt(segs, "")
        for c in imgs:
            if c not in pool:
                pool[c] = (g.random((ls, 576, h), dtype=np.float32) - 0.5, g.random((ls, 576, h), dtype=np.float32) - 0.5)
            p.chunk_k.append(pool[c][0])
            p.chunk_v.append(pool[c][1])
            p.chunk_base.append(0)
        sel = rm.select(p, 0, k)
        ents = rm.entries(p)
        try:
            best = None
            for _ in range(max(1, min(steps, 2))):
                res = rm.link_and_prefill(p, sel=sel, want_asm=False, want_final=False, entries=ents)
                t = (res["ms_assemble"] + res["ms_selective"]) * (L / ls)
                best = t if best is None else min(best, t)
        finally:
            r.lib.ref_entries_free(ents)
        ms += best
        n_s += p.n
    n_all = sum(oracle.make_prompt(segs, "").n for segs, _ in reqs)
    return dict(ms=ms * n_all / n_s, n=n_all, m=None, threads=threads,
                sample=f"first {sample} of the 256 config-E requests (n={n_s}) at {ls} of {L} layers, scaled "
                       f"x{L / ls:g} and by prompt tokens to all 256 (n={n_all}); requests one at a time; "
                       f"assemble_linked_cache + selective_prefill, OpenBLAS {threads} threads"), None


def cpu_baseline_legs(cfg_name, thread_counts):
    """The reference on the host cores, each leg in its own process (so the reference build's
    .so files never map into the GPU arm). The first count is the headline (None = all
    cores); the others (1 thread) are reported beside it."""
    import subprocess
    out = None
    for th in thread_counts:
        one = th == 1
        cmd = [sys.executable, os.path.abspath(__file__), "--cpu-leg", "--config", cfg_name,
               "--steps", "1" if (one or cfg_name == "E") else "2", "--warmup", "0" if (one or cfg_name == "E") else "1",
               "--layers-sample", "1" if one else "2"]
        if th:
            cmd += ["--threads", str(th)]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        try:
            res = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception:
            res = {"unavailable": (r.stderr or r.stdout)[-300:]}
        if "ms" not in res:
            leg = {"value": None, "unavailable": res.get("unavailable")}
        else:
            leg = {"value": res["n"] / (res["ms"] / 1e3), "unit": "prompt tokens/s", "cores": res["threads"],
                   "kind": "reference", "sample": res["sample"], "ttft_ms": res["ms"]}
        if out is None:
            out = leg
        else:
            out[f"threads_{th}"] = leg
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS))
    ap.add_argument("--mode", default="request", choices=["request", "head-parallel"],
                    help="request: every rank serves its own requests (request sharding); "
                         "head-parallel: one long request split by attention head over the ranks")
    ap.add_argument("--hp-driver", default="library", choices=["library", "python"],
                    help="head-parallel: mpic_hp_request with NCCL inside the library, or the "
                         "Python layer loop over torch.distributed")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-fp32", action="store_true", default=True,
                    help="also time the e2e leg from fp32 (.mpic v1) host chunks")
    ap.add_argument("--no-e2e-fp32", dest="e2e_fp32", action="store_false")
    ap.add_argument("--disk", action="store_true",
                    help="also time the request with every chunk read from its .mpic file")
    ap.add_argument("--disk-dir", default=None, help="where the .mpic files are written")
    ap.add_argument("--k-sweep", default=None,
                    help="with --disk: comma-separated MPIC-k budgets timed device-resident, warm and cold "
                         "(config D: 0,16,32,64,2304)")
    ap.add_argument("--k", type=int, default=None, help="MPIC-k budget (default: the config's)")
    ap.add_argument("--batch", type=int, default=64,
                    help="config E: requests per batched varlen pass (1 = one request at a time)")
    ap.add_argument("--fp32-mode", action="store_true", default=True,
                    help="also time the request in fp32 mode (the reference's precision)")
    ap.add_argument("--no-fp32-mode", dest="fp32_mode", action="store_false")
    ap.add_argument("--no-miss", dest="miss", action="store_false", default=True,
                    help="skip the miss-path key (chunk prefill + all-miss request)")
    ap.add_argument("--decode-steps", type=int, default=8,
                    help="decode tokens timed after the prefill (0: skip)")
    ap.add_argument("--no-serving", action="store_true",
                    help="skip the config-E serving key of the default (config C) line")
    ap.add_argument("--cpu-leg", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--threads", type=int, default=None, help=argparse.SUPPRESS)
    ap.add_argument("--layers-sample", type=int, default=2, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.config is None:
        args.config = "E16" if args.mode == "head-parallel" else "C"
    if args.k is not None:
        c = CONFIGS[args.config]
        CONFIGS[args.config] = c[:5] + (args.k,)

    if args.cpu_leg:  # child process of the cpu_baseline leg (keeps oracle/_ref out of the GPU arm)
        res, why = cpu_reference(args.config, args.steps, args.warmup, threads=args.threads,
                                 layers_sample=args.layers_sample)
        print(json.dumps(res if res is not None else {"unavailable": why}))
        return
    args.warmup = max(args.warmup, 3)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one rank per GPU: relaunch this command under torch.distributed.run
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        os.execv(sys.executable, cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch with torchrun "
                         f"--nproc-per-node {args.gpus} (or without torchrun: bench.py spawns the ranks)")
    L, H, D, V, images, k = CONFIGS[args.config]
    cfg_json = config_json(args)

    if args.impl == "reference":
        if rank != 0:
            return
        res, why = cpu_reference(args.config, args.steps, args.warmup)
        if res is None:
            print(json.dumps({"impl": "reference", "unavailable": why}))
            return
        val = res["n"] / (res["ms"] / 1e3)
        line = {"metric": "MPIC-k prefill tokens/s (p50 TTFT alongside)", "impl": "reference",
                "value": val, "unit": "prompt tokens/s", "n_gpus": 0, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": res["ms"], "ttft_p50_ms": res["ms"],
                "higher_is_better": True, "scaling": "strong" if args.config == "E" else "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded ids, U(-0.5,0.5) chunk KV)",
                "config": cfg_json,
                "cpu_baseline": {"value": val, "unit": "prompt tokens/s", "cores": res["threads"],
                                 "kind": "reference", "sample": res["sample"]},
                "e2e": {"value": val, "unit": "prompt tokens/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    world, rank, local = dist_setup(args.gpus)
    if args.mode == "head-parallel":
        r = run_head_parallel(args, world, rank, local)
        if rank == 0:
            print(json.dumps({
                "metric": "MPIC-k prefill tokens/s (p50 TTFT alongside)", "value": r["value"],
                "unit": "prompt tokens/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
                "ttft_p50_ms": float(statistics.median(r["per_step"])), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (seeded ids and hashes, U(-0.5,0.5) chunk KV, weights synthesised from seed 1)",
                "config": cfg_json,
                "step_ms": [round(x, 3) for x in r["per_step"]], "step_sm_mhz": r["step_sm_mhz"],
                "clocks": r["clocks"]}))
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    if args.config == "E":
        r = run_serving(args, world, rank, local)
        cpu = None
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline_legs("E", [None])
        if rank == 0:
            print(json.dumps({
                "metric": "MPIC-k prefill tokens/s (p50 TTFT alongside)", "value": r["value"],
                "unit": "prompt tokens/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
                "ttft_p50_ms": r["ttft_p50"], "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (seeded requests and hashes, U(-0.5,0.5) pooled chunk KV, weights "
                        "synthesised from seed 1)",
                "config": cfg_json, "recompute_rows_total": r["m"], "requests_rank0": r["mine"],
                "recompute_rows_per_s": r["rows_per_s"], "cpu_baseline": cpu, "batch_ms": r["batch_ms"],
                "batch_sm_mhz": r["batch_sm_mhz"], "clocks": r["clocks"],
                "ttft": "host wall time per request (submission -> logits on the host), p50 over rank 0's requests"}))
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    r = run_ours(args, world, rank, local)
    assert (r["n"], r["m"]) == (cfg_json["n_tokens"], cfg_json["recompute_rows"])
    serving = None
    if args.config == "C" and not args.no_serving:
        # config E (256 requests sharded over the ranks: the 1/2/4/8 strong-scaling workload)
        # as an extra key of the default line
        import copy
        ea = copy.copy(args)
        ea.steps, ea.warmup = 2, 3
        e = run_serving(ea, world, rank, local)
        serving = {"workload": WORKLOAD_NAMES["E"], "value": e["value"], "unit": "prompt tokens/s",
                   "ms_per_256_requests": e["ms_per_step"], "steps": ea.steps, "warmup": ea.warmup,
                   "n_gpus": world, "scaling": "strong", "batch": max(1, args.batch),
                   "recompute_rows_per_s": e["rows_per_s"], "ttft_p50_ms": e["ttft_p50"],
                   "batch_ms_rank0": e["batch_ms"], "clocks": e["clocks"]}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_legs(args.config, [None, 1])
    if rank == 0:
        line = {"metric": "MPIC-k prefill tokens/s (p50 TTFT alongside)", "value": r["value"],
                "unit": "prompt tokens/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
                "ttft_p50_ms": float(statistics.median(r["per_step"])),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "bf16", "data": "synthetic (seeded ids and hashes, U(-0.5,0.5) chunk "
                                         "KV, weights synthesised from seed 1)",
                "config": cfg_json,
                "e2e": r["e2e"], "e2e_fp32_host": r["e2e_fp32"], "e2e_disk": r["e2e_disk"],
                "fp32_mode": r.get("fp32_mode"), "k_sweep": r.get("k_sweep"), "decode": r.get("decode"),
                "miss": r.get("miss"),
                "gpu_launches": r["launches"],
                "roofline": r["roofline"],
                "request_roofline_frac": round(r["floor_ms"] / r["ms_per_step"], 4),
                "phases": r["phases"], "cpu_baseline": cpu, "serving_E": serving, "clocks": r["clocks"],
                "step_ms": [round(x, 3) for x in r["per_step"]],
                "host_ms": [round(x, 3) for x in r["host_ms"]]}
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
