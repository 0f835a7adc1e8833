#!/usr/bin/env python
"""ScMoE layer benchmark (BASELINE.json metric: ScMoE layer tokens/sec).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config prefill|decode]

N=1 workload = BASELINE config 2 ("prefill"): one LongCat-Flash-shape MoE
layer (d=6144, 512 FFN experts with inter 2048 + 256 zero experts, top-12,
K_e=8), 8192 tokens, bf16 expert GEMMs on tcgen05, exact fp32 router.  A step
is one full ScMoE MoE-branch forward through the C ABI
(scmoe_layer_forward: rmsnorm -> exact router -> permutation -> grouped GEMM1
(+SiLU) -> grouped GEMM2 -> combine with zero-expert identity + residual).

For N>1 (torchrun, one process per GPU) every rank runs the same layer on its
own 8192-token shard with the full expert set resident (replicated experts,
token-sharded; no data-path collective) -> "scaling": "weak".

`value` is device-timed (CUDA events on the layer's stream, inputs resident in
HBM, inputs + weights larger than L2); `e2e` is the same metric through the
host tier (scmoe_layer_forward_host_batches) with pinned host buffers, H2D
of every step's inputs and D2H of its outputs inside the timed region (the
copies of neighbouring steps overlap compute, as in a serving loop).
`--impl reference` times the reference's own CPU code (oracle/_ref, compiled
from /root/reference headers; the C restatement when absent) on this host's
cores on a bounded token sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ScMoE layer tokens/sec"
D, N_FFN, N_ZERO, TOPK, KE, INTER = 6144, 512, 256, 12, 8, 2048
CONFIGS = {
    "prefill": dict(tokens=8192, workload="LongCat-Flash ScMoE MoE layer prefill (BASELINE config 2)"),
    "decode": dict(tokens=256, workload="LongCat-Flash ScMoE MoE layer decode step (BASELINE config 3)"),
}
SEED_W, SEED_X = 5, 99


def log(*a):
    print(*a, file=sys.stderr, flush=True)


_JSON_FD = None


def emit(line: dict):
    """The one JSON line on stdout (libraries' banners are routed to stderr)."""
    data = (json.dumps(line) + "\n").encode()
    if _JSON_FD is not None:
        os.write(_JSON_FD, data)
    else:
        sys.stdout.write(data.decode())
        sys.stdout.flush()


def stdout_to_stderr():
    """Keep fd 1 for the JSON line only: NCCL prints its version banner on stdout."""
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------
def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        os.environ.setdefault("NCCL_DEBUG", "WARN")  # keep stdout to the one JSON line
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v: float, ws: int) -> float:
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
_NVML_POLL = r"""
import sys, time
import pynvml as n
gpu, out, period = int(sys.argv[1]), sys.argv[2], float(sys.argv[3])
n.nvmlInit()
h = n.nvmlDeviceGetHandleByIndex(gpu)
mx = n.nvmlDeviceGetMaxClockInfo(h, n.NVML_CLOCK_SM)
bits = [n.nvmlClocksEventReasonHwSlowdown, n.nvmlClocksEventReasonHwThermalSlowdown,
        n.nvmlClocksEventReasonSwThermalSlowdown, n.nvmlClocksEventReasonSwPowerCap]
with open(out, "w", buffering=1) as f:
    f.write("ready\n")
    while True:
        sm = n.nvmlDeviceGetClockInfo(h, n.NVML_CLOCK_SM)
        pw = n.nvmlDeviceGetPowerUsage(h) / 1000.0
        r = n.nvmlDeviceGetCurrentClocksEventReasons(h)
        f.write(f"{sm} {mx} {pw} " + "".join("1" if r & b else "0" for b in bits) + "\n")
        time.sleep(period)
"""


class ClockSampler:
    """SM clocks, power and throttle reasons polled through NVML every 5 ms
    during the timed region by a separate process (a thread of this process
    starves behind the GIL while the timed region blocks in CUDA calls: one
    run got no sample at all); falls back to nvidia-smi when NVML is absent."""
    PERIOD_S = 0.005
    REASONS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self._proc = None
        self._smi = None
        self.error = None
        self._src = None

    def __enter__(self):
        self._f = tempfile.NamedTemporaryFile("w+", suffix=".txt", delete=False)
        try:
            self._proc = subprocess.Popen([sys.executable, "-c", _NVML_POLL, str(self.gpu),
                                           self._f.name, str(self.PERIOD_S)],
                                          stdout=subprocess.DEVNULL, stderr=subprocess.PIPE)
            t0 = time.time()
            while time.time() - t0 < 20:
                if self._proc.poll() is not None:
                    raise RuntimeError(self._proc.stderr.read().decode()[-160:])
                if open(self._f.name).read().startswith("ready"):
                    break
                time.sleep(0.01)
            else:
                raise RuntimeError("NVML poller did not start")
            self._src = "nvml 5 ms (separate process)"
        except Exception as ex:
            self.error = f"{type(ex).__name__}: {ex}"[:160]
            if self._proc:
                self._proc.kill()
            self._proc = None
            try:
                q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                     "clocks_event_reasons.hw_thermal_slowdown,"
                     "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
                self._smi = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + q,
                                              "--format=csv,noheader,nounits", "-lms", "50"],
                                             stdout=self._f, stderr=subprocess.DEVNULL)
                self._src = "nvidia-smi 50 ms"
            except FileNotFoundError:
                self._smi = None
        time.sleep(0.02)
        return self

    def __exit__(self, *a):
        time.sleep(0.01)
        if self._proc:
            self._proc.terminate()
            self._proc.wait()
            for line in open(self._f.name).read().splitlines()[1:]:
                p = line.split()
                if len(p) == 4 and len(p[3]) == 4:
                    self.rows.append((float(p[0]), float(p[1]), float(p[2]),
                                      [nm for nm, b in zip(self.REASONS, p[3]) if b == "1"]))
        if self._smi:
            self._smi.terminate()
            self._smi.wait()
            for r in open(self._f.name).read().strip().splitlines():
                r = r.split(", ")
                if len(r) >= 7:
                    self.rows.append((float(r[0]), float(r[1]), float(r[2]),
                                      [nm for nm, v in zip(self.REASONS, r[3:7])
                                       if v.strip() == "Active"]))
        try:
            os.unlink(self._f.name)
        except OSError:
            pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"],
                    "error": self.error}
        sm = [r[0] for r in self.rows]
        mx = max(r[1] for r in self.rows)
        reasons = sorted({x for r in self.rows for x in r[3]})
        loaded = [v for v in sm if v > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_min_mhz": min(loaded), "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(self.rows), "source": self._src,
                "power_w_max": max(r[2] for r in self.rows)}


def energy_block(gpu: int, fn, ms_per_step: float, seconds: float = 1.5):
    """Energy per step from NVML's total-energy counter (mJ) around ~`seconds`
    of the same schedule (after the timed region; the counter lags ~0.1 s, so
    the short timed region itself is not used).  power_floor_ms = J per step /
    the enforced power limit: the step time a schedule with this energy per
    step cannot beat on this board; floor / ms_per_step ~ 1 means the step is
    power-bound, not HBM- or tensor-bound.  None when NVML is absent."""
    try:
        import pynvml as n
        import torch
        n.nvmlInit()
        h = n.nvmlDeviceGetHandleByIndex(gpu)
        limit = n.nvmlDeviceGetEnforcedPowerLimit(h) / 1e3
        torch.cuda.synchronize()
        time.sleep(0.3)
        e, t = n.nvmlDeviceGetTotalEnergyConsumption(h), time.perf_counter()
        time.sleep(0.7)
        idle_w = (n.nvmlDeviceGetTotalEnergyConsumption(h) - e) / 1e3 / (time.perf_counter() - t)
        steps = max(8, int(seconds * 1e3 / ms_per_step))
        fn(steps)  # same load before the counted run
        torch.cuda.synchronize()
        e0, w0 = n.nvmlDeviceGetTotalEnergyConsumption(h), time.perf_counter()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        fn(steps)
        t1.record()
        torch.cuda.synchronize()
        time.sleep(0.25)
        e1, w1 = n.nvmlDeviceGetTotalEnergyConsumption(h), time.perf_counter()
        ms = t0.elapsed_time(t1) / steps
        idle_s = max(0.0, (w1 - w0) - ms * steps / 1e3)
        j = ((e1 - e0) / 1e3 - idle_w * idle_s) / steps
        return {"power_limit_w": limit, "idle_w": round(idle_w, 1), "steps": steps,
                "ms_per_step": round(ms, 4), "j_per_step": round(j, 4),
                "avg_w": round(j / ms * 1e3, 1), "power_floor_ms": round(j / limit * 1e3, 4),
                "frac_of_power_bound": round(j / limit * 1e3 / ms, 3),
                "source": "NVML total energy counter over the run, idle energy of the "
                          "counter lag subtracted"}
    except Exception as ex:  # reported, not fatal
        return {"unavailable": str(ex)[:200]}


def pcie_h2d_gbs(nbytes: int, reps: int = 4, trials: int = 3) -> float:
    """Pinned host -> device copy bandwidth of one nbytes buffer (the e2e
    tier's bound: every step copies its fp32 inputs over PCIe); best of
    `trials` runs of `reps` back-to-back copies (the link is shared and noisy
    on these boxes: 42-56 GB/s run to run)."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h.fill_(1)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(trials):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            d.copy_(h, non_blocking=True)
        e1.record()
        e1.synchronize()
        best = max(best, nbytes * reps / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return best


def pcie_duplex_gbs(nbytes: int, reps: int = 4, trials: int = 3) -> float:
    """H2D bandwidth while a D2H of the same size runs on another stream (the
    e2e tier copies outputs back while the next inputs come in); best of
    `trials`."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    best = 0.0
    for _ in range(trials):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s1)
        s2.wait_event(e0)
        for _ in range(reps):
            with torch.cuda.stream(s1):
                d.copy_(h, non_blocking=True)
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
        e1.record(s1)
        e1.synchronize()
        torch.cuda.synchronize()
        best = max(best, nbytes * reps / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return best


def nvlink_bytes(gpu: int):
    """Cumulative NVLink data bytes (tx, rx) of one GPU from NVML's throughput
    counters (summed over links), or None when unavailable."""
    try:
        import pynvml as n
        n.nvmlInit()
        h = n.nvmlDeviceGetHandleByIndex(gpu)
        tx = rx = 0
        for link in range(18):
            try:
                v = n.nvmlDeviceGetFieldValues(h, [(n.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, link),
                                                   (n.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, link)])
            except Exception:
                break
            if v[0].nvmlReturn != 0 or v[1].nvmlReturn != 0:
                continue
            tx += v[0].value.ullVal
            rx += v[1].value.ullVal
        return (tx * 1024, rx * 1024)  # the DATA counters count KiB
    except Exception:
        return None


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref = the reference's own code) on a bounded sample
# ---------------------------------------------------------------------------
_CPU_WEIGHTS = {}


def reference_cpu_sample(threads=None, route_tokens=1024, shard_tokens=8, shard_distinct=1,
                         log_fn=log):
    """tokens/s of the reference's route_topk + moe_forward at the LongCat
    shape on this host.  ONE definition for both the cpu_baseline leg and the
    --impl reference arm (same sample, same threads).

    route_topk (router.hpp:133-141) runs on `route_tokens` tokens,
    token-sharded over `threads` (bitwise one call).  moe_forward
    (blocks.hpp:372-394) runs one shard per thread; a shard holds
    `shard_tokens` tokens made of `shard_distinct` routed tokens, each repeated:
    the reference's per-row cost does not depend on how many rows an expert
    gathers (mm_into re-streams W per row), while its per-CALL copy of every hit
    expert's weights into the graph (blocks.hpp:387-391, ~200 MB per expert)
    amortises over the repeats as it does over the ~128 tokens per expert of a
    full 8192-token call -- without the 100 GB of host RAM such a call needs.
    The sampled tokens are routed tokens with exactly K_e = 8 FFN slots, the
    workload's mean (7.98-8.01 per token at configs B/C), so the per-token
    work equals the workload's.  Weights of the hit experts are generated
    (untimed) once per process."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import _oracle as O
    from _oracle import ptr, ptr_array

    threads = threads or os.cpu_count() or 1
    kind = "reference" if O.ref_available() else "port"
    E = N_FFN + N_ZERO
    x = O.normal_f32(O.stream_seed(SEED_X, 0), route_tokens * D).reshape(route_tokens, D)
    w = O.uniform_f32(O.stream_seed(SEED_W, 0), D * E, 1.0 / D).reshape(D, E)
    idx = np.empty(route_tokens * TOPK, np.uint32)
    g = np.empty(route_tokens * TOPK)
    cnt = np.empty(route_tokens, np.uint32)
    b = np.zeros(E)
    t0 = time.perf_counter()
    if kind == "reference":
        rc = O.ref().ref_route_topk_f32(ptr(x), route_tokens, D, ptr(w), N_FFN, N_ZERO, TOPK, KE,
                                        0.0, ptr(b), ptr(idx), ptr(g), ptr(cnt), None, threads)
    else:
        rc = O.orc().orc_route_topk_f32(ptr(x), route_tokens, D, ptr(w), N_FFN, N_ZERO, TOPK, KE,
                                        0.0, ptr(b), ptr(idx), ptr(g), ptr(cnt), None)
    t_route = time.perf_counter() - t0
    assert rc == 0
    # moe sample: shard i holds tokens [i*distinct, (i+1)*distinct) of the
    # routed batch, each repeated shard_tokens/distinct times
    n_shards = threads
    rep = max(1, shard_tokens // shard_distinct)
    mean_tok = np.nonzero(cnt == KE)[0]
    src = np.concatenate([np.repeat(mean_tok[(np.arange(i * shard_distinct, (i + 1) *
                                                        shard_distinct)) % mean_tok.size], rep)
                          for i in range(n_shards)])
    M = src.size
    mx = np.ascontiguousarray(x[src])
    mi = np.ascontiguousarray(idx.reshape(-1, TOPK)[src].ravel())
    mg = np.ascontiguousarray(g.reshape(-1, TOPK)[src].ravel())
    hit = sorted({int(e) for e in mi if e < N_FFN})

    def gen(e):
        a = np.empty(D * INTER, np.float32)
        bb = np.empty(D * INTER, np.float32)
        O.orc().orc_seeded_uniform_f32(O.stream_seed(SEED_W, 100 + 2 * e), 0, D * INTER, 1.0 / D,
                                       ptr(a))
        O.orc().orc_seeded_uniform_f32(O.stream_seed(SEED_W, 101 + 2 * e), 0, D * INTER, 1.0 / D,
                                       ptr(bb))
        return e, a, bb

    from concurrent.futures import ThreadPoolExecutor
    todo = [e for e in hit if e not in _CPU_WEIGHTS]
    with ThreadPoolExecutor(threads) as ex:
        for e, a, bb in ex.map(gen, todo):
            _CPU_WEIGHTS[e] = (a, bb)
    w_in = [_CPU_WEIGHTS[e][0] if e in _CPU_WEIGHTS and e in hit else None for e in range(N_FFN)]
    w_out = [_CPU_WEIGHTS[e][1] if e in _CPU_WEIGHTS and e in hit else None for e in range(N_FFN)]
    out = np.empty((M, D), np.float32)
    t0 = time.perf_counter()
    if kind == "reference":
        rc = O.ref().ref_moe_forward_f32(ptr(mx), M, D, ptr(mi), ptr(mg), TOPK, N_FFN, N_ZERO,
                                         ptr_array(w_in), ptr_array(w_out), INTER, 1, 0, ptr(out),
                                         n_shards)
        used = n_shards
    else:
        rc = O.orc().orc_moe_forward_f32(ptr(mx), M, D, ptr(mi), ptr(mg), TOPK, N_FFN, N_ZERO,
                                         ptr_array(w_in), ptr_array(w_out), INTER, 1.0, 1.0, 0,
                                         ptr(out))
        used = 1
    t_moe = time.perf_counter() - t0
    assert rc == 0
    route_tps = route_tokens / t_route
    moe_tps = M / t_moe
    value = 1.0 / (1.0 / route_tps + 1.0 / moe_tps)
    sample = (f"route_topk on {route_tokens} tokens over {threads} threads ({t_route:.2f}s, "
              f"{route_tps:.0f} tok/s) + moe_forward on {M} tokens = {n_shards} shards x "
              f"{shard_distinct} routed tokens x {rep} repeats, one shard per thread "
              f"({t_moe:.2f}s, {moe_tps:.2f} tok/s, {len(hit)} experts materialised, "
              f"{float((mi < N_FFN).sum()) / M:.2f} FFN slots/token); LongCat shape fp32")
    log_fn("cpu reference:", sample, f"-> {value:.2f} tok/s")
    return {"value": value, "unit": "tokens/s", "cores": used if kind == "reference" else 1,
            "route_threads": threads if kind == "reference" else 1, "kind": kind,
            "route_tokens_per_s": route_tps, "moe_tokens_per_s": moe_tps,
            "tokens_sampled": {"route": route_tokens, "moe": M, "moe_distinct": n_shards *
                               shard_distinct},
            "experts_materialised": len(hit), "sample": sample}


def tiny_config_a(ctx, stream, iters, with_cpu):
    """T=512, d=256, 8 FFN + 4 zero experts, top-2,
    K_e=1, I=128, exact fp32 (the bit-exact kernels).  Device time per layer
    call (stream-launched, back to back) and the reference's route_topk +
    moe_forward on the same shape, one thread, on this host."""
    import torch
    from paper_2509_01322_b200.layer import TINY, DeviceLayer
    s, T = TINY, 512
    lay = DeviceLayer(ctx, s, seed=11)
    a1 = torch.randn(T, s.d, device="cuda")
    a3 = torch.randn(T, s.d, device="cuda")
    idx = torch.empty(T * s.top_k, dtype=torch.int32, device="cuda")
    g = torch.empty(T * s.top_k, dtype=torch.float64, device="cuda")
    cnt = torch.empty(T, dtype=torch.int32, device="cuda")
    out = torch.empty(T, s.d, device="cuda")

    def run(n):
        for _ in range(n):
            lay.forward(a1.data_ptr(), a3.data_ptr(), None, T, idx.data_ptr(), g.data_ptr(),
                        cnt.data_ptr(), out.data_ptr())
    with torch.cuda.stream(stream):
        run(10)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        ev0.record(stream)
        run(iters)
        ev1.record(stream)
    ev1.synchronize()
    us = ev0.elapsed_time(ev1) / iters * 1e3
    res = {"workload": "SURVEY config A: tiny fp32 layer (T=512, d=256, 8+4 experts, top-2, "
                       "I=128), exact fp32 kernels", "us_per_call": round(us, 2),
           "tokens_per_s": T / (us * 1e-6)}
    # the same call captured once in a CUDA graph and replayed (launch-bound shape)
    try:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            run(1)
        with torch.cuda.stream(stream):
            for _ in range(10):
                graph.replay()
            ev0.record(stream)
            for _ in range(iters):
                graph.replay()
            ev1.record(stream)
        ev1.synchronize()
        res["us_per_call_cuda_graph"] = round(ev0.elapsed_time(ev1) / iters * 1e3, 2)
    except Exception as e:  # capture is an optimisation; report why it was skipped
        res["us_per_call_cuda_graph"] = None
        res["cuda_graph_error"] = str(e)[:200]
    if with_cpu:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import _oracle as O
        from _oracle import ptr, ptr_array
        E = s.n_ffn + s.n_zero
        x = O.normal_f32(7, T * s.d).reshape(T, s.d)
        w = O.uniform_f32(8, s.d * E, 1.0 / s.d).reshape(s.d, E)
        wi = [O.uniform_f32(9 + e, s.d * s.inter, 1.0 / s.d) for e in range(s.n_ffn)]
        wo = [O.uniform_f32(50 + e, s.d * s.inter, 1.0 / s.d) for e in range(s.n_ffn)]
        ix = np.empty(T * s.top_k, np.uint32)
        gg = np.empty(T * s.top_k)
        cc = np.empty(T, np.uint32)
        o = np.empty((T, s.d), np.float32)
        kind = "reference" if O.ref_available() else "port"
        reps = 20
        t0 = time.perf_counter()
        for _ in range(reps):
            if kind == "reference":
                O.ref().ref_route_topk_f32(ptr(x), T, s.d, ptr(w), s.n_ffn, s.n_zero, s.top_k,
                                           s.k_expected, 0.0, ptr(np.zeros(E)), ptr(ix), ptr(gg),
                                           ptr(cc), None, 1)
                O.ref().ref_moe_forward_f32(ptr(x), T, s.d, ptr(ix), ptr(gg), s.top_k, s.n_ffn,
                                            s.n_zero, ptr_array(wi), ptr_array(wo), s.inter, 1, 0,
                                            ptr(o), 1)
            else:
                O.orc().orc_route_topk_f32(ptr(x), T, s.d, ptr(w), s.n_ffn, s.n_zero, s.top_k,
                                           s.k_expected, 0.0, ptr(np.zeros(E)), ptr(ix), ptr(gg),
                                           ptr(cc), None)
                O.orc().orc_moe_forward_f32(ptr(x), T, s.d, ptr(ix), ptr(gg), s.top_k, s.n_ffn,
                                            s.n_zero, ptr_array(wi), ptr_array(wo), s.inter, 1.0,
                                            1.0, 0, ptr(o))
        cpu_us = (time.perf_counter() - t0) / reps * 1e6
        res["cpu_reference"] = {"us_per_call": round(cpu_us, 1), "kind": kind, "cores": 1}
        res["speedup_vs_cpu_reference"] = round(cpu_us / us, 1)
    return res


def run_reference_arm(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    vals = []
    base = None
    for i in range(args.warmup + args.steps):
        r = reference_cpu_sample()
        if i >= args.warmup:
            vals.append(r["value"])
            base = r
    v = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup,
        # the time this rate implies for one full 8192-token step of the workload
        "ms_per_step": cfg["tokens"] / v * 1e3 if v else None,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (CounterRng normal inputs, seeded_init Uniform weights)",
        "config": {"workload": cfg["workload"], "tokens": cfg["tokens"], "d_model": D,
                   "n_ffn": N_FFN, "n_zero": N_ZERO, "top_k": TOPK, "inter": INTER,
                   "parallelism": f"cpu x{base['cores']}",
                   "same_config": ("same layer shape, weights and inputs as the B200 arm; each "
                                   "step is a bounded token sample (see cpu_baseline.sample), "
                                   "the same function as the B200 line's cpu_baseline leg")},
        "cpu_baseline": {**base, "value": v},
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def gemm_algorithmic_bytes(idx: np.ndarray, T: int):
    """Algorithmic bytes of the two grouped-GEMM launches of one step: the
    bf16 weights of every hit expert once + activations in/out once."""
    ffn = idx[idx < N_FFN]
    S = int(ffn.size)
    n_hit = int(np.unique(ffn).size)
    w_bytes = n_hit * D * INTER * 2
    g1 = w_bytes + S * D * 2 + S * INTER * 2
    g2 = w_bytes + S * INTER * 2 + S * D * 2
    flops = 2 * 2 * S * D * INTER
    return g1, g2, S, n_hit, flops


def run_b200(args):
    import torch
    ws, rank, local = dist_init()
    torch.cuda.set_device(local)
    import paper_2509_01322_b200 as P
    from paper_2509_01322_b200.layer import LONGCAT, DeviceLayer

    cfg = CONFIGS[args.config]
    T = args.tokens or cfg["tokens"]
    ctx = P.Context(local)
    stream = torch.cuda.Stream()
    ctx.set_stream(stream.cuda_stream)
    t0 = time.time()
    layer = DeviceLayer(ctx, LONGCAT, seed=SEED_W)
    # inputs: a1 (shortcut stream) and a3 (dense-branch output / residual)
    a1_h = P.fill_normal(P.stream_seed(SEED_X, rank), T * D, threads=os.cpu_count() or 8)
    a3_h = P.fill_normal(P.stream_seed(SEED_X + 1, rank), T * D, threads=os.cpu_count() or 8)
    a1 = torch.from_numpy(a1_h).cuda()
    a3 = torch.from_numpy(a3_h).cuda()
    # two output sets: consecutive micro-batches of the pipelined schedule must not alias
    sets = [dict(idx=torch.empty(T * TOPK, dtype=torch.int32, device="cuda"),
                 gates=torch.empty(T * TOPK, dtype=torch.float64, device="cuda"),
                 cnt=torch.empty(T, dtype=torch.int32, device="cuda"),
                 out=torch.empty(T, D, dtype=torch.float32, device="cuda")) for _ in range(2)]
    torch.cuda.synchronize()
    log(f"[rank {rank}] setup {time.time() - t0:.1f}s; bank {layer.bank_bytes() / 1e9:.2f} GB")

    def step(s):
        b = sets[s & 1]
        layer.forward(a1.data_ptr(), a3.data_ptr(), None, T, b["idx"].data_ptr(),
                      b["gates"].data_ptr(), b["cnt"].data_ptr(), b["out"].data_ptr())

    def batches(n):
        sel = [sets[i & 1] for i in range(n)]
        layer.forward_batches([a1.data_ptr()] * n, [a3.data_ptr()] * n, None, T,
                              [b["idx"].data_ptr() for b in sel],
                              [b["gates"].data_ptr() for b in sel],
                              [b["cnt"].data_ptr() for b in sel],
                              [b["out"].data_ptr() for b in sel])

    def timed(fn, n):
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        barrier(ws)
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            ev0.record(stream)
            fn(n)
            ev1.record(stream)
        ev1.synchronize()
        torch.cuda.synchronize()
        barrier(ws)
        return ev0.elapsed_time(ev1) / n

    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            step(i)
        ctx.synchronize()
    idx_h = sets[0]["idx"].cpu().numpy().view(np.uint32)
    g1b, g2b, S, n_hit, flops = gemm_algorithmic_bytes(idx_h, T)
    w_hit_bytes = n_hit * D * INTER * 2 * 2
    ffn_mean = float(sets[0]["cnt"].cpu().numpy().mean())

    # ---- serial schedule: one batch after the other (per-batch latency) ----
    ctx.profile(True)
    ctx.profile_flush()
    ms_serial = timed(lambda n: [step(i) for i in range(n)], args.steps)
    stages_serial = ctx.profile_flush()

    # ---- pipelined schedule (headline): front half of batch i+1 under the
    # expert GEMMs of batch i; device-timed over K batches -------------------
    pipelined = args.schedule == "pipelined"
    if pipelined:
        with torch.cuda.stream(stream):
            batches(max(args.warmup, 2))
        ctx.synchronize()
    ctx.profile_flush()
    l0 = ctx.kernel_launches()
    with ClockSampler(local) as clk:
        if pipelined:
            ms = timed(batches, args.steps)
        else:
            ms = timed(lambda n: [step(i) for i in range(n)], args.steps)
    launches = ctx.kernel_launches() - l0
    stages = ctx.profile_flush()
    ctx.profile(False)
    ms_max = max_over_ranks(ms, ws)
    ms_serial_max = max_over_ranks(ms_serial, ws)
    value = T * ws / (ms_max / 1e3)
    # energy per step of the same schedule (is the step power-bound?)
    energy = None
    if ws == 1 and args.energy:
        with torch.cuda.stream(stream):
            energy = energy_block(local, batches if pipelined else
                                  (lambda n: [step(i) for i in range(n)]), ms_max)

    # ---- e2e through the host tier (pinned buffers, copies in the region) --
    # scmoe_layer_forward_host_batches: every step copies its a1/a3 in and its
    # output + routing out; the copies of neighbouring steps overlap compute.
    # Two pinned host slots alternate (inputs re-read, outputs overwritten).
    def pinned(shape, dt):
        return torch.empty(shape, dtype=dt).pin_memory().numpy()
    hs = []
    for _ in range(2):
        h = dict(a1=pinned((T, D), torch.float32), a3=pinned((T, D), torch.float32),
                 idx=pinned((T * TOPK,), torch.int32), gat=pinned((T * TOPK,), torch.float64),
                 cnt=pinned((T,), torch.int32), out=pinned((T, D), torch.float32))
        h["a1"][:] = a1_h.reshape(T, D)
        h["a3"][:] = a3_h.reshape(T, D)
        hs.append(h)

    def host_run(n):
        sl = [hs[i % 2] for i in range(n)]
        layer.forward_host_batches([h["a1"] for h in sl], [h["a3"] for h in sl], None, T,
                                   [h["idx"] for h in sl], [h["gat"] for h in sl],
                                   [h["cnt"] for h in sl], [h["out"] for h in sl])
    e_steps = max(4, args.steps)
    host_run(2)
    e2e_ms = timed(host_run, e_steps)
    e2e_ms = max_over_ranks(e2e_ms, ws)
    e2e_val = T * ws / (e2e_ms / 1e3)
    h2d = 2 * T * D * 4
    d2h = T * D * 4 + T * TOPK * (4 + 8) + T * 4
    h2d_gbs = pcie_h2d_gbs(T * D * 4)
    duplex_gbs = pcie_duplex_gbs(T * D * 4)
    # the step moves h2d bytes in and d2h bytes out; while both directions are
    # busy the H2D runs at the duplex rate: floor = d2h at the duplex rate +
    # the remaining H2D at the solo rate
    both = min(h2d, d2h) / (duplex_gbs * 1e9)
    floor_duplex = both + max(0, h2d - min(h2d, d2h)) / (h2d_gbs * 1e9)
    e2e_roof = {"bound": "pcie_h2d", "h2d_gbs_measured": h2d_gbs,
                "h2d_gbs_with_concurrent_d2h": duplex_gbs,
                "floor_ms": floor_duplex * 1e3, "floor_ms_h2d_alone": h2d / (h2d_gbs * 1e9) * 1e3,
                "frac": floor_duplex * 1e3 / e2e_ms,
                "note": "floor = the step's D2H bytes moved at the measured duplex H2D rate "
                        "(both directions busy) + the remaining H2D bytes at the solo rate"}

    # ---- SURVEY config C (decode: 256 tokens per step, HBM-bound weight
    # streaming) on the same layer, serial steps; reported beside the headline
    config_c = None
    if args.decode_tokens > 0:
        Tc = args.decode_tokens
        dsets = dict(idx=torch.empty(Tc * TOPK, dtype=torch.int32, device="cuda"),
                     gates=torch.empty(Tc * TOPK, dtype=torch.float64, device="cuda"),
                     cnt=torch.empty(Tc, dtype=torch.int32, device="cuda"),
                     out=torch.empty(Tc, D, dtype=torch.float32, device="cuda"))

        def dstep(n):
            for i in range(n):  # consecutive 256-token windows of the prefill input
                off = (i % (T // Tc)) * Tc * D * 4
                layer.forward(a1.data_ptr() + off, a3.data_ptr() + off, None, Tc,
                              dsets["idx"].data_ptr(), dsets["gates"].data_ptr(),
                              dsets["cnt"].data_ptr(), dsets["out"].data_ptr())
        with torch.cuda.stream(stream):
            dstep(3)
        ctx.synchronize()
        ctx.profile(True)
        ctx.profile_flush()
        ms_c = max_over_ranks(timed(dstep, args.steps), ws)
        st_c = ctx.profile_flush()
        ctx.profile(False)
        idx_c = dsets["idx"].cpu().numpy().view(np.uint32)
        # two independent decode micro-batches in flight (scmoe_layer_forward_batches:
        # batch i+1's routing beside batch i's expert-weight stream)
        psets = [dict(idx=torch.empty(Tc * TOPK, dtype=torch.int32, device="cuda"),
                      gates=torch.empty(Tc * TOPK, dtype=torch.float64, device="cuda"),
                      cnt=torch.empty(Tc, dtype=torch.int32, device="cuda"),
                      out=torch.empty(Tc, D, dtype=torch.float32, device="cuda"))
                 for _ in range(2)]

        def dbatches(n):
            sel = [psets[i & 1] for i in range(n)]
            offs = [(i % (T // Tc)) * Tc * D * 4 for i in range(n)]
            layer.forward_batches([a1.data_ptr() + o for o in offs],
                                  [a3.data_ptr() + o for o in offs], None, Tc,
                                  [b["idx"].data_ptr() for b in sel],
                                  [b["gates"].data_ptr() for b in sel],
                                  [b["cnt"].data_ptr() for b in sel],
                                  [b["out"].data_ptr() for b in sel])
        with torch.cuda.stream(stream):
            dbatches(3)
        ctx.synchronize()
        ms_cp = max_over_ranks(timed(dbatches, args.steps), ws)
        c1, c2, Sc, hit_c, _ = gemm_algorithmic_bytes(idx_c, Tc)
        tg = (st_c["gemm1_tcgen05"][0] + st_c["gemm2_tcgen05"][0]) / st_c["gemm1_tcgen05"][1]
        config_c = {"workload": "SURVEY config C: LongCat MoE layer decode step, 256 tokens, "
                                "1xB200 (expert weights streamed from HBM)",
                    "tokens": Tc, "ms_per_step": ms_c, "tokens_per_s": Tc * ws / (ms_c / 1e3),
                    "pipelined_ms_per_step": ms_cp,
                    "pipelined_tokens_per_s": Tc * ws / (ms_cp / 1e3),
                    "pipelined_note": "independent decode micro-batches, scmoe_layer_forward_batches",
                    "ffn_slots": Sc, "experts_hit": hit_c,
                    "gemm_ms_per_step": tg, "gemm_bytes_per_step": c1 + c2,
                    "gemm_achieved_gbs": (c1 + c2) / (tg / 1e3) / 1e9,
                    "stages_ms": {k: round(v[0] / v[1], 4) for k, v in st_c.items()}}
        # e2e of the decode step through the host tier (pinned buffers, H2D of
        # the step's a1/a3 and D2H of its output + routing inside the region)
        hc = [dict(a1=pinned((Tc, D), torch.float32), a3=pinned((Tc, D), torch.float32),
                   idx=pinned((Tc * TOPK,), torch.int32), gat=pinned((Tc * TOPK,), torch.float64),
                   cnt=pinned((Tc,), torch.int32), out=pinned((Tc, D), torch.float32))
              for _ in range(2)]
        for i, h in enumerate(hc):
            h["a1"][:] = a1_h.reshape(T, D)[i * Tc:(i + 1) * Tc]
            h["a3"][:] = a3_h.reshape(T, D)[i * Tc:(i + 1) * Tc]

        def host_dec(n):
            sl = [hc[i % 2] for i in range(n)]
            layer.forward_host_batches([h["a1"] for h in sl], [h["a3"] for h in sl], None, Tc,
                                       [h["idx"] for h in sl], [h["gat"] for h in sl],
                                       [h["cnt"] for h in sl], [h["out"] for h in sl])
        host_dec(2)
        ms_ce = max_over_ranks(timed(host_dec, e_steps), ws)
        config_c["e2e"] = {"value": Tc * ws / (ms_ce / 1e3), "unit": "tokens/s",
                           "h2d_bytes_per_step": 2 * Tc * D * 4,
                           "d2h_bytes_per_step": Tc * D * 4 + Tc * TOPK * (4 + 8) + Tc * 4,
                           "ms_per_step": ms_ce,
                           "api": "scmoe_layer_forward_host_batches (pinned host buffers)"}

    # ---- TPOT from measured latencies -- one GPU holding all
    # 512 experts serving a decode batch of tpot_batch tokens (the reference
    # row's batch_per_device); no all-to-all at N=1, so dispatch / combine
    # stay the row's values (measured at N>1 by the EP arm)
    tpot = None
    if args.tpot_batch > 0:
        Tb = args.tpot_batch
        bsets = dict(idx=torch.empty(Tb * TOPK, dtype=torch.int32, device="cuda"),
                     gates=torch.empty(Tb * TOPK, dtype=torch.float64, device="cuda"),
                     cnt=torch.empty(Tb, dtype=torch.int32, device="cuda"),
                     out=torch.empty(Tb, D, dtype=torch.float32, device="cuda"))

        def bstep(n):
            for _ in range(n):
                layer.forward(a1.data_ptr(), None, None, Tb, bsets["idx"].data_ptr(),
                              bsets["gates"].data_ptr(), bsets["cnt"].data_ptr(),
                              bsets["out"].data_ptr())
        with torch.cuda.stream(stream):
            bstep(3)
        ctx.synchronize()
        ctx.profile(True)
        ctx.profile_flush()
        ms_b = timed(bstep, args.steps)
        st_b = ctx.profile_flush()
        ctx.profile(False)
        moe_us = sum(st_b[k][0] / st_b[k][1] for k in ("permute", "gather", "gemm1_tcgen05",
                                                       "gemm2_tcgen05") if k in st_b) * 1e3
        tpot = tpot_block(moe_us, source=f"1xB200 holding all {N_FFN} experts, decode batch of "
                                         f"{Tb} tokens ({ms_b:.3f} ms per layer call incl. routing "
                                         "and combine); moe = permute + gather + GEMM1 + GEMM2")
        tpot["layer_ms_measured"] = ms_b

    # ---- SURVEY config A (tiny fp32, bit-exact path, latency-bound): device
    # time per layer call beside the reference's own CPU time on the same shape
    config_a = None
    if ws == 1 and args.config_a:
        config_a = tiny_config_a(ctx, stream, args.steps * 20, not args.no_cpu_baseline)

    # ---- the full ScMoE layer (Model::build_layer, model.hpp:355-409)
    # at LongCat widths with the tensor-core MLA, on the same router / experts
    full_layer = None
    if ws == 1 and args.full_layer:
        full_layer = run_full_layer(P, ctx, stream, layer, a1, T, args.steps)

    # ---- 4-layer ScMoE stack, 100 router steps of 1024 tokens with
    # PID bias control (K_e = 6, mu = 0.2, decay 0.999); the main layer's
    # 25.8 GB are released first (the stack holds 4 x 25.8 GB)
    e5 = None
    if ws == 1 and args.e5_steps > 0:
        layer.close()
        torch.cuda.synchronize()
        e5 = run_e5(P, ctx, stream, args.e5_steps)

    if rank != 0:
        return
    peaks = measured_peaks()
    hbm_peak = peaks["hbm_gbs"] if peaks else 6650.0
    if config_c:
        config_c["gemm_frac_of_measured_hbm"] = config_c["gemm_achieved_gbs"] / hbm_peak
        config_c["gemm_frac_of_8tbs_nominal"] = config_c["gemm_achieved_gbs"] / 8000.0

    # algorithmic bytes per SURVEY 8(d): every hit expert's bf16 weights once
    # + the token rows in (x) and out, bf16 -- the unfused kernels' extra
    # traffic (the permuted copy, h, per-slot rows) is NOT counted as useful
    alg_bytes = w_hit_bytes + 2 * T * D * 2

    def gemm_roofline(st):
        g1 = st.get("gemm1_tcgen05", (0.0, 1))
        g2 = st.get("gemm2_tcgen05", (0.0, 1))
        t = (g1[0] + g2[0]) / max(1, g1[1])  # per step (one launch of each per step)
        return t, (alg_bytes / (t / 1e3) / 1e9 if t > 0 else None)

    t_gemm, achieved = gemm_roofline(stages)
    # dram bytes per step of the same kernels from the committed ncu --set full
    # capture (profiles/); compare with algorithmic_bytes_per_step
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r02_traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath))["dram_bytes_per_step"]
    t_gemm_serial, achieved_serial = gemm_roofline(stages_serial)
    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        try:
            cpu = reference_cpu_sample()
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": "tokens/s", "cores": 0, "kind": "reference",
                   "sample": f"failed: {e}"}
    if config_c and cpu and cpu.get("value"):
        # the reference's per-token cost (route_topk + moe_forward) does not depend
        # on the batch size once its per-call weight copy is amortised: the same
        # sample is the decode step's CPU baseline
        config_c["cpu_baseline"] = {**cpu, "note": "same per-token sample as the headline line"}
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (CounterRng normal inputs, seeded_init Uniform weights, random-init)",
        "config": {"workload": cfg["workload"], "tokens_per_gpu": T, "d_model": D, "n_ffn": N_FFN,
                   "n_zero": N_ZERO, "top_k": TOPK, "k_expected": KE, "inter": INTER,
                   "router": "exact fp32 (bit-exact vs reference)", "expert_gemm": "bf16 tcgen05",
                   "schedule": ("pipelined batches (scmoe_layer_forward_batches): the front "
                                "half of batch i+1 (rmsnorm, exact fp32 router on a 256-thread "
                                "kernel co-resident with the GEMM CTA on every SM, top-K, "
                                "permute, gather) runs on the FP32 pipes while the HBM-bound "
                                "expert GEMMs + combine of batch i run (2 streams); every batch "
                                "still passes the whole path") if pipelined
                   else "serial", "serial_ms_per_batch": ms_serial_max,
                   "parallelism": f"replicated experts, token-sharded x{ws}",
                   "l2": "inputs + weights (25.8 GB) larger than L2 every step",
                   "mean_ffn_per_token": ffn_mean, "ffn_slots": S, "experts_hit": n_hit},
        "e2e": {"value": e2e_val, "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms, "steps": e_steps,
                "roofline": e2e_roof,
                "api": "scmoe_layer_forward_host_batches (pinned host buffers; H2D of step i+1 "
                       "and D2H of step i-1 overlap compute of step i)"},
        "gpu_launches": launches,
        "roofline": {"kernel": "grouped_gemm_bf16 (GEMM1+GEMM2, tcgen05)", "bound": "hbm",
                     "note": ("achieved = SURVEY 8(d) algorithmic bytes (hit experts' bf16 "
                              "weights + x + out) / the GEMM pair's event time inside the timed "
                              "region (pipelined: the co-resident router shares the SMs); "
                              "achieved_serial: the same kernels timed alone (serial schedule); "
                              "kernel_io_bytes_per_step adds the unfused design's permuted x, h "
                              "and per-slot rows"),
                     "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": (achieved / hbm_peak) if achieved else None, "traffic": traffic,
                     "traffic_source": "profiles/r02_traffic.json (ncu dram__bytes_read+write of the pair GEMMs)",
                     "algorithmic_bytes_per_step": alg_bytes,
                     "kernel_io_bytes_per_step": g1b + g2b, "ms_per_step": t_gemm,
                     "achieved_serial": achieved_serial, "ms_per_step_serial": t_gemm_serial,
                     "tflops": flops / (t_gemm / 1e3) / 1e12 if t_gemm > 0 else None,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650",
                     "binding_constraint": ("board power: the step's energy over the 1000 W cap "
                                            "(see `energy`: frac_of_power_bound); streaming the "
                                            "expert weights alone costs ~3.2 J per pass "
                                            "(profiles/r02_energy_split.json)")},
        "stages_ms": {k: round(v[0] / v[1], 4) for k, v in stages.items()},
        "stages_ms_serial": {k: round(v[0] / v[1], 4) for k, v in stages_serial.items()},
        "clocks": clk.summary(),
        "energy": energy,
        "cpu_baseline": cpu,
        "config_c": config_c,
        "config_a": config_a,
        "tpot": tpot,
        "e5": e5,
        "full_layer": full_layer,
    }
    emit(line)


def run_full_layer(P, ctx, stream, layer, a1, T, steps, seq=4096):
    """One full ScMoE layer (model.hpp:355-409): a1 = x + MLA1(rmsnorm x);
    dd = a1 + FFN(rmsnorm a1) (dense_inter 12288); a3 = dd + MLA2(rmsnorm dd);
    out = a3 + moe(rmsnorm a1) -- LongCat MLA widths (d_q 1536, d_kv 512, 64 heads
    x (128 + 64)), tensor-core MLA (csrc/mla_tc.cu), T tokens as T/seq causal
    sequences, device-timed per layer call; the MoE branch alone for scale."""
    import torch
    from paper_2509_01322_b200.layer import DenseFFN
    from paper_2509_01322_b200.mla import MlaParams, ScMoELayer
    dq, dkv, H, dhc, dhr = 1536, 512, 64, 128, 64

    def mla(seed):
        ws_ = []
        for i, (r, c) in enumerate([(D, dq), (dq, H * dhc), (dq, H * dhr), (D, dkv),
                                    (dkv, H * dhc), (dkv, H * dhc), (D, dhr), (H * dhc, D)]):
            t = torch.empty(r * c, dtype=torch.float32, device="cuda")
            ctx._check(P.lib().scmoe_rng_fill_uniform(ctx.handle, P.stream_seed(seed, i), 0, r * c,
                                                      1.0 / D, t.data_ptr()))
            ws_.append(t.view(r, c))
        return MlaParams(D, dq, dkv, H, dhc, dhr, weights=ws_, rope_base=1.0e6,
                         precision=P.PREC_BF16)

    class _Handle:  # the bench layer's device router / bank
        def __init__(self, h, top_k=None):
            self.h, self.top_k = h, top_k

        def device(self, c):
            return self.h

    dense = DenseFFN(ctx, D, 12288, seed=SEED_W + 3)
    full = ScMoELayer(mla(SEED_W + 4), mla(SEED_W + 5), dense, _Handle(layer.router, TOPK),
                      _Handle(layer.bank), *[np.ones(D, np.float32)] * 4, ctx=ctx)
    x = a1.view(T, D)
    res = {"workload": "full ScMoE layer (MLA1, dense FFN 12288, MLA2, MoE branch), LongCat "
                       f"widths, {T} tokens as {T // seq} causal sequences of {seq}, "
                       "tensor-core MLA (bf16 operands, rel-L2 ~7e-3 vs the exact oracle)"}
    for overlap in (False, True):
        with torch.cuda.stream(stream):  # the context's stream: the layer runs there
            full.forward(x, seq, overlap=overlap)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = max(2, steps // 4)
            e0.record(stream)
            for _ in range(n):
                full.forward(x, seq, overlap=overlap)
            e1.record(stream)
            e1.synchronize()
        ms = e0.elapsed_time(e1) / n
        res["overlap" if overlap else "serial"] = {"ms_per_layer": ms, "tokens_per_s": T / ms * 1e3}
    ctx.profile(True)
    ctx.profile_flush()
    with torch.cuda.stream(stream):
        full.forward(x, seq, overlap=False)
    st = ctx.profile_flush()
    ctx.profile(False)
    res["stages_ms"] = {k: round(v[0], 3) for k, v in st.items()}
    moe_keys = ("rmsnorm", "router_gemm", "softmax_topk", "permute", "gather", "gemm1_tcgen05",
                "gemm2_tcgen05", "combine")
    moe_ms = sum(st[k][0] for k in moe_keys if k in st)
    res["moe_branch_ms"] = moe_ms
    res["layer_over_moe_branch"] = res["serial"]["ms_per_layer"] / moe_ms if moe_ms else None
    dense.close()
    return res


def run_e5(P, ctx, stream, steps, T=1024, n_layers=4):
    """SURVEY 8(d) E5 (BASELINE config 5): 4 ScMoE layers (LongCat shape,
    bf16 experts) x `steps` router steps of T tokens, rmsnorm before each
    router, accumulate + bias_update every step (Model::accumulate_routing /
    update_biases).  Device-timed steps/s; the activated-FFN trace shows the
    zero-expert fraction tracking 1 - K_e/K.  Bitwise routing / bias parity of
    this exact run against the reference is tests/test_gpu_stack.py."""
    import torch
    from paper_2509_01322_b200.layer import LayerShape
    from paper_2509_01322_b200.stack import ScMoEStack
    shape = LayerShape(d=D, n_ffn=N_FFN, n_zero=N_ZERO, top_k=TOPK, k_expected=6, inter=INTER,
                       precision=P.PREC_BF16)
    t0 = time.time()
    with torch.cuda.stream(stream):
        stack = ScMoEStack(ctx, shape, n_layers, seed=11, mu=0.2, mu_decay=0.999)
        xs = [torch.from_numpy(P.fill_normal(P.stream_seed(99, s), T * D,
                                             threads=os.cpu_count() or 8)).cuda().view(T, D)
              for s in range(steps)]
        torch.cuda.synchronize()
        setup = time.time() - t0
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for s in range(steps):  # fresh inputs every step (CounterRng stream(step))
            stack.step(xs[s], T, record=True)
        ev1.record(stream)
        ev1.synchronize()
    ms = ev0.elapsed_time(ev1) / steps
    means = np.array(stack.trace.mean_ffn)
    tail = means[-20:].mean(0)
    for l in stack.layers:
        l.close()
    return {"workload": "SURVEY E5 / BASELINE config 5: 4-layer ScMoE stack (LongCat layer, "
                        "bf16 experts), PID bias control K_e=6, mu=0.2, decay 0.999, bias_update "
                        "every step", "tokens_per_step": T, "layers": n_layers, "steps": steps,
            "ms_per_step": ms, "steps_per_s": 1e3 / ms, "tokens_per_s": T / (ms / 1e3),
            "setup_s": setup, "first_step_mean_ffn": [round(v, 4) for v in means[0]],
            "final_tail20_mean_ffn": [round(v, 4) for v in tail],
            "final_zero_expert_fraction": [round(1 - v / TOPK, 4) for v in tail],
            "target_zero_expert_fraction": 1 - 6 / TOPK,
            "timing": "device events around all steps; includes the per-step host reads of the "
                      "ffn counts and bias_update's StateError check (one sync per layer)"}


def tpot_block(moe_us, dispatch_us=None, combine_us=None, source=""):
    """the reference's TPOT calculator (analytics.hpp:211-253,
    costmodel.py) on its LongCat SBO row (data/costmodels/sbo_28l.json: 28
    layers, 96 tokens per device, accept 1.8 -> 16.05 ms) with the module
    latencies measured here substituted; attention stays the row's value (the
    exact-fp32 MLA is not a decode-serving path)."""
    from paper_2509_01322_b200.costmodel import CostModel, tpot_theoretical, with_measured
    row = CostModel(264, 236, 60, 472, 28, 1.8, "sbo", 96, 2.0)
    meas = {"moe_us": moe_us}
    if dispatch_us is not None:
        meas["dispatch_us"] = dispatch_us
    if combine_us is not None:
        meas["combine_us"] = combine_us
    out = {"reference_row": "sbo_28l (analytics.hpp:232-253, data/costmodels/sbo_28l.json)",
           "measured_us": {k: round(v, 2) for k, v in meas.items()}, "measured_on": source}
    for strat in ("sbo", "tbo"):
        ref = tpot_theoretical(CostModel(**{**row.__dict__, "strategy": strat}))
        b200 = tpot_theoretical(with_measured(CostModel(**{**row.__dict__, "strategy": strat}),
                                              **meas))
        out[strat] = {"reference_tpot_ms": round(ref.tpot_ms, 3),
                      "b200_tpot_ms": round(b200.tpot_ms, 3),
                      "b200_tpl_us": round(b200.tpl_us, 2),
                      "b200_price_per_mtok": round(b200.price_per_mtok, 4)}
    return out


def run_b200_ep(args):
    """N>1: the expert-parallel layer behind the C ABI (scmoe_ep_*; Python
    caller paper_2509_01322_b200.ep): experts block-partitioned over the
    ranks, tokens sharded (8192 per GPU: weak scaling), the count exchange,
    dispatch (peer stores over NVLink) and return (GEMM2 epilogue stores)
    all device-side, no host synchronisation per layer."""
    import torch
    ws, rank, local = dist_init()
    import paper_2509_01322_b200 as P
    from paper_2509_01322_b200.ep import ExpertParallelLayer, broadcast_unique_id
    from paper_2509_01322_b200.layer import LONGCAT

    cfg = CONFIGS[args.config]
    T = args.tokens or cfg["tokens"]
    Td = args.config_d_tokens // ws
    ctx = P.Context(local)
    uid = broadcast_unique_id()
    ep = ExpertParallelLayer(ctx, LONGCAT, rank, ws, SEED_W, uid,
                             max_tokens=max(T, Td, args.tpot_batch))
    a1_h = P.fill_normal(P.stream_seed(SEED_X, rank), T * D, threads=os.cpu_count() or 8)
    a3_h = P.fill_normal(P.stream_seed(SEED_X + 1, rank), T * D, threads=os.cpu_count() or 8)
    a1 = torch.from_numpy(a1_h).cuda()
    a3 = torch.from_numpy(a3_h).cuda()
    for _ in range(args.warmup):
        out, idx, gates, cnt = ep.forward(a1, a3, None, T)
    torch.cuda.synchronize()
    # untimed warm-up continues until the step time is steady on every rank
    hist = []
    for _ in range(30):
        w0 = torch.cuda.Event(enable_timing=True)
        w1 = torch.cuda.Event(enable_timing=True)
        w0.record()
        out, idx, gates, cnt = ep.forward(a1, a3, None, T)
        w1.record()
        w1.synchronize()
        hist.append(max_over_ranks(w0.elapsed_time(w1), ws))
        if len(hist) >= 3 and max(hist[-3:]) <= 1.05 * min(hist[-3:]):
            break
    log(f"[rank {rank}] extra warm-up steps {len(hist)}: {[round(h, 2) for h in hist]}")
    idx_h = idx.cpu().numpy().view(np.uint32)
    ffn = idx_h[idx_h < N_FFN]
    M = ep.count_matrix()  # [src][dst] slots of the last call
    n_send, n_recv, self_rows = int(M[rank].sum()), int(M[:, rank].sum()), int(M[rank, rank])

    def timed_ep(fn, n=None):
        n = n or args.steps
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        barrier(ws)
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        torch.cuda.synchronize()
        barrier(ws)
        return e0.elapsed_time(e1) / n

    # serial steps (per-batch latency), with the per-stage profile
    ctx.profile(True)
    ctx.profile_flush()
    ms_serial = timed_ep(lambda: [ep.forward(a1, a3, None, T) for _ in range(args.steps)])
    stages = ctx.profile_flush()
    ctx.profile(False)
    ms_serial_max = max_over_ranks(ms_serial, ws)
    # headline: the pipelined batch stream
    pipelined = args.schedule == "pipelined"
    run = ((lambda: ep.forward_batches([a1] * args.steps, [a3] * args.steps, None, T,
                                       corun_router=args.ep_corun)) if pipelined else
           (lambda: [ep.forward(a1, a3, None, T) for _ in range(args.steps)]))
    run()  # untimed block of the timed block's shape
    torch.cuda.synchronize()
    l0 = ep.kernel_launches()
    nv0 = nvlink_bytes(local)
    with ClockSampler(local) as clk:
        ms = timed_ep(run)
    nv1 = nvlink_bytes(local)
    launches = ep.kernel_launches() - l0
    ms_max = max_over_ranks(ms, ws)
    value = T * ws / (ms_max / 1e3)
    # energy per step on this rank's GPU over ~1.5 s of the same schedule (every
    # rank runs the same number of coupled steps); rank 0's is reported
    energy = None
    if args.energy:
        def run_n(n):
            if pipelined:
                ep.forward_batches([a1] * n, [a3] * n, None, T, corun_router=args.ep_corun)
            else:
                for _ in range(n):
                    ep.forward(a1, a3, None, T)
        energy = energy_block(local, run_n, ms_max)
    # NVLink cross-check: hardware tx bytes per step vs the payload this rank
    # stores to peers (dispatch rows + ids to the owners, returned rows to the sources)
    payload = ((n_send - self_rows) * (D * 2 + 4) + (n_recv - self_rows) * D * 2)
    nvlink = None
    if nv0 and nv1:
        tx = (nv1[0] - nv0[0]) / args.steps
        nvlink = {"tx_bytes_per_step": tx, "rx_bytes_per_step": (nv1[1] - nv0[1]) / args.steps,
                  "payload_bytes_per_step": payload, "tx_over_payload": tx / payload if payload
                  else None, "tx_gbs": tx / (ms / 1e3) / 1e9,
                  "source": "NVML NVLINK_THROUGHPUT_DATA_TX/RX counters over the timed block "
                            "(nsys is not installed in this image)"}
    # e2e: every step's H2D of its inputs and D2H of its output inside the region
    a1_p = torch.from_numpy(a1_h).pin_memory()
    a3_p = torch.from_numpy(a3_h).pin_memory()
    outs_p = [torch.empty(T, D, dtype=torch.float32).pin_memory() for _ in range(2)]
    e_steps = max(4, args.steps)
    host_run = lambda: ep.forward_host_batches(  # noqa: E731
        [a1_p] * e_steps, [a3_p] * e_steps, [outs_p[i % 2] for i in range(e_steps)], None, T)
    host_run()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(timed_ep(host_run, e_steps), ws)

    # ---- SURVEY config D: fixed 32k tokens over the ranks, with the dense
    # shortcut FFN (dense_inter) overlapping the dispatch/return; exposed
    # communication = (t_layer - t_layer with the row transfers replaced by
    # no-ops) / t_layer -------------------------------------------------------
    config_d = None
    if args.dense_inter > 0:
        ep.enable_dense(args.dense_inter, seed=SEED_W + 1)
        a1d = torch.from_numpy(P.fill_normal(P.stream_seed(SEED_X + 5, rank), Td * D,
                                             threads=os.cpu_count() or 8)).cuda()

        def timed_d(dense, comm):
            ep.set_comm(comm)
            for _ in range(2):
                ep.forward(a1d, None, None, Td, dense=dense)
            t = max_over_ranks(timed_ep(lambda: [ep.forward(a1d, None, None, Td, dense=dense)
                                                 for _ in range(args.steps)]), ws)
            ep.set_comm(True)
            return t

        t_moe, t_moe_nc = timed_d(False, True), timed_d(False, False)
        t_full, t_full_nc = timed_d(True, True), timed_d(True, False)
        Md = ep.count_matrix()
        config_d = {
            "workload": "SURVEY config D: ScMoE layer = MoE branch + dense shortcut SiLU-MLP "
                        "(rmsnorm, d x dense_inter x d, residual) overlapping dispatch/return",
            "tokens_total": Td * ws, "tokens_per_gpu": Td, "dense_inter": args.dense_inter,
            "ms_moe_branch": t_moe, "ms_moe_branch_comm_noop": t_moe_nc,
            "ms_layer": t_full, "ms_layer_comm_noop": t_full_nc,
            "exposed_comm_frac_layer": (t_full - t_full_nc) / t_full,
            "exposed_comm_frac_moe_only": (t_moe - t_moe_nc) / t_moe,
            "layer_tokens_per_s": Td * ws / (t_full / 1e3),
            "dense_tflop_per_gpu": 4.0 * Td * D * args.dense_inter / 1e12,
            "a2a_bytes_each_way_rank0": int(Md[rank].sum() - Md[rank, rank]) * D * 2,
            "dense_gemm_sms": "all but 16 (left to the dispatch / barrier kernels)",
        }

    # ---- TPOT from measured module latencies (decode batch of
    # `tpot_batch` tokens per device, the reference row's batch_per_device) ---
    tpot = None
    if args.tpot_batch > 0:
        Tb = args.tpot_batch
        a1b = a1[:Tb * D]
        for _ in range(3):
            ep.forward(a1b, None, None, Tb)
        ctx.profile(True)
        ctx.profile_flush()
        ms_b = max_over_ranks(timed_ep(lambda: [ep.forward(a1b, None, None, Tb)
                                                for _ in range(args.steps)]), ws)
        st_b = ctx.profile_flush()
        ctx.profile(False)
        us = lambda *ks: sum(st_b.get(k, (0.0, 1))[0] / max(1, st_b.get(k, (0.0, 1))[1])  # noqa
                             for k in ks) * 1e3
        moe_us = us("permute", "gather", "gemm1_tcgen05", "gemm2_tcgen05", "ep_row_dst")
        disp_us = us("ep_exchange", "ep_put_rows", "ep_dispatch_barrier")
        comb_us = us("ep_return_barrier", "combine")
        # per-stage maxima over the ranks (the slowest rank sets the layer time)
        moe_us, disp_us, comb_us = (max_over_ranks(v, ws) for v in (moe_us, disp_us, comb_us))
        tpot = tpot_block(moe_us, disp_us, comb_us,
                          f"EP x{ws} decode step, {Tb} tokens per GPU ({ms_b:.3f} ms per layer "
                          "call incl. routing); moe = permute + gather + GEMM1 + GEMM2 (return "
                          "fused in GEMM2's epilogue), dispatch = count exchange + peer stores + "
                          "barrier, combine = return barrier + combine kernel")
        tpot["layer_ms_measured"] = ms_b

    if rank != 0:
        ep.close()
        return
    peaks = measured_peaks() or {}
    n_local = N_FFN // ws
    dispatch = None
    put = stages.get("ep_put_rows")
    if put:
        remote = (n_send - self_rows) * D * 2
        put_ms = put[0] / max(1, put[1])
        dispatch = {"kernel": "ep_put_rows (peer stores over NVLink)", "remote_bytes": remote,
                    "ms": put_ms, "gbs": remote / (put_ms / 1e3) / 1e9,
                    "note": "the return is inside GEMM2's epilogue (not separable)"}
    g1 = stages.get("gemm1_tcgen05", (0.0, 1))
    g2 = stages.get("gemm2_tcgen05", (0.0, 1))
    t_gemm = (g1[0] + g2[0]) / max(1, g1[1])
    flops = 4.0 * n_recv * D * INTER
    wbytes = 2 * n_local * D * INTER * 2
    tok_per_expert = n_recv / n_local
    bound = "tensor" if tok_per_expert > 254 else "hbm"
    if bound == "tensor":
        achieved = flops / (t_gemm / 1e3) / 1e12 if t_gemm else None
        peak, unit = peaks.get("bf16_tflops", 1590.0), "TFLOP/s"
    else:
        achieved = (wbytes + n_recv * D * 2 * 2) / (t_gemm / 1e3) / 1e9 if t_gemm else None
        peak, unit = peaks.get("hbm_gbs", 6650.0), "GB/s"
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (CounterRng normal inputs, seeded_init Uniform weights, random-init)",
        "config": {"workload": f"LongCat-Flash ScMoE MoE layer, expert-parallel x{ws} "
                               f"(BASELINE config 4 shape, {T} tokens per GPU)",
                   "tokens_per_gpu": T, "d_model": D, "n_ffn": N_FFN, "n_zero": N_ZERO,
                   "top_k": TOPK, "inter": INTER, "experts_per_gpu": n_local,
                   "parallelism": (f"ep{ws} behind the C ABI (scmoe_ep_layer_forward*): on-device "
                                   "count exchange, dispatch = peer stores into the owners' "
                                   "receive buffers over NVLink, return fused into GEMM2's "
                                   "epilogue, no host sync per layer"),
                   "schedule": ("pipelined batches (scmoe_ep_layer_forward_batches): routing + "
                                "dispatch of batch i+1 on one stream beside the expert GEMMs + "
                                "return + combine of batch i on another") if pipelined
                   else "serial",
                   "serial_ms_per_batch": ms_serial_max,
                   "slot_matrix_rank0_row": M[rank].tolist(),
                   "a2a_bytes_each_way_rank0": (n_send - self_rows) * D * 2,
                   "mean_ffn_per_token": float(ffn.size) / T,
                   "l2": "inputs + weights larger than L2 every step"},
        "e2e": {"value": T * ws / (e2e_ms / 1e3), "unit": "tokens/s",
                "h2d_bytes_per_step": 2 * T * D * 4, "d2h_bytes_per_step": T * D * 4,
                "ms_per_step": e2e_ms, "steps": e_steps,
                "api": "ExpertParallelLayer.forward_host_batches (pinned host tensors; H2D of "
                       "step i+1 and D2H of step i-1 overlap step i)"},
        "gpu_launches": launches,
        "roofline": {"kernel": "grouped_gemm_bf16 (GEMM1+GEMM2, tcgen05), rank 0", "bound": bound,
                     "achieved": achieved, "peak": peak, "unit": unit,
                     "frac": achieved / peak if achieved else None, "traffic": None,
                     "tflops": flops / (t_gemm / 1e3) / 1e12 if t_gemm else None,
                     "weight_stream_gbs": wbytes / (t_gemm / 1e3) / 1e9 if t_gemm else None,
                     "note": "bound = tensor above the bf16/HBM ridge (~254 tokens per expert)",
                     "tokens_per_local_expert": tok_per_expert, "ms_per_step": t_gemm},
        "stages_ms": {k: round(v[0] / v[1], 4) for k, v in stages.items()},
        "dispatch_nvlink": dispatch,
        "nvlink_counters": nvlink,
        "clocks": clk.summary(),
        "energy": energy,
        "cpu_baseline": None,
        "config_d": config_d,
        "tpot": tpot,
    }
    ep.close()
    emit(line)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="prefill", choices=sorted(CONFIGS))
    ap.add_argument("--tokens", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    # N>1: SURVEY config D extra (dense shortcut FFN overlapping the all-to-alls)
    ap.add_argument("--dense-inter", type=int, default=12288)
    # N=1: SURVEY config C extra (decode step of this many tokens; 0 = off)
    ap.add_argument("--decode-tokens", type=int, default=256)
    ap.add_argument("--config-a", type=int, default=1, help="measure SURVEY config A (tiny fp32)")
    ap.add_argument("--config-d-tokens", type=int, default=32768)
    # pipelined = scmoe_layer_forward_batches; measured slower than serial on B200 in round 1
    # (router and GEMM contend for shared-memory bandwidth), so serial is the default
    ap.add_argument("--schedule", default="pipelined", choices=["pipelined", "serial"])
    ap.add_argument("--parallel", default="ep", choices=["ep", "replicated"],
                    help="N>1: expert-parallel (default) or replicated experts")
    ap.add_argument("--ep-corun", action="store_true",
                    help="pipelined EP: small router kernel co-resident with the GEMM")
    ap.add_argument("--tpot-batch", type=int, default=96,
                    help="decode tokens per device for the measured TPOT block (0 = off)")
    ap.add_argument("--energy", type=int, default=1,
                    help="N=1: NVML energy per step of the headline schedule (~2.5 s)")
    ap.add_argument("--full-layer", type=int, default=1,
                    help="N=1: time the full ScMoE layer with the tensor-core MLA")
    ap.add_argument("--e5-steps", type=int, default=100,
                    help="N=1: SURVEY E5 4-layer PID stack steps (0 = off)")
    args = ap.parse_args()
    stdout_to_stderr()
    if args.impl == "reference":
        run_reference_arm(args)
    elif int(os.environ.get("WORLD_SIZE", "1")) > 1 and args.parallel == "ep":
        run_b200_ep(args)
    else:
        run_b200(args)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
