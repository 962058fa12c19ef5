"""Command line: ``python -m paper_2203_13085_b200 {run,validate,compare,plotdata}``
(the SPEC's runner module, on the GPU path).

* ``validate --config C``: resolve defaults, list EVERY violation, print the resolved
  config; exit 0 iff valid (2 otherwise).
* ``run --config C --out DIR``: a real run on this process's GPU — one process per
  GPU under torchrun (P = WORLD_SIZE), LASGD through ``LASGDWorker`` or SGD-AR
  through ``SGDARWorker`` — writing ``trace.csv`` (RunTrace), ``summary.json`` and
  ``config.resolved.json``, each carrying the resolved config's SHA-256.  Exit 3 on
  a numerical failure (non-finite model or loss).
* ``compare S1 S2 ...``: final loss, wall time and speedup relative to the first
  summary (SGD-AR by convention, Table 4); refuses summaries of different problems.
* ``plotdata T1 T2 ... --out F``: long-format CSV (run, algo, x_kind, x, loss) for
  loss-vs-epoch and loss-vs-time curves (Figs. 4-5).

Config (YAML or JSON, schema 1; unknown keys are errors):

    schema: 1
    problem: {kind: mlp, n: 4096, d: 784, hidden: [128], noise: 0.1, data_seed: 0, batch: 32}
    algo: lasgd                     # lasgd | sgd_ar
    lasgd: {tau_max: 4, adaptive: false, alpha: 1.0, mode: pull, pipeline: overlap, nvls: false}
    sgd_ar: {bucketed: false, bucket_mb: 25}   # bucketed: the all-reduce overlapped with backward
    # lasgd.nvls: the side-stream mean reduced inside the NVSwitch (tolerance mode, overlap pipeline)
    sgd: {momentum: 0.0, dampening: 0.0, weight_decay: 0.0, nesterov: false}
    lr: {base_lr: 0.01, scale_nodes: 1, warmup_epochs: 0.0, decay_epochs: [], decay_factor: 10.0}
    steps: 100
    seed: 0
    init_scale: 0.05

``problem.kind`` may also be resnet18 / resnet50 / mobilenet_v2 (synthetic images of
the BASELINE shapes, random init broadcast from rank 0).  Pure orchestration: every
numerical piece lives in the package (CLI tests run without a GPU for validate /
compare / plotdata).
"""

from __future__ import annotations

import argparse
import copy
import hashlib
import json
import os
import sys
from typing import List, Tuple

EXIT_OK, EXIT_CONFIG, EXIT_NUMERIC = 0, 2, 3

DEFAULTS = {
    "schema": 1,
    "problem": {"kind": "mlp", "n": 4096, "d": 784, "hidden": [128], "noise": 0.1, "data_seed": 0, "batch": 32},
    "algo": "lasgd",
    "lasgd": {"tau_max": 4, "adaptive": False, "alpha": 1.0, "mode": "pull", "pipeline": "overlap", "nvls": False},
    "sgd_ar": {"bucketed": False, "bucket_mb": 25},
    "sgd": {"momentum": 0.0, "dampening": 0.0, "weight_decay": 0.0, "nesterov": False},
    "lr": {"base_lr": 0.01, "scale_nodes": 1, "warmup_epochs": 0.0, "decay_epochs": [], "decay_factor": 10.0},
    "steps": 100,
    "seed": 0,
    "init_scale": 0.05,
}
IMAGE_MODELS = {"resnet18": (32, 10), "resnet50": (224, 1000), "mobilenet_v2": (224, 1000)}


class ConfigError(ValueError):
    def __init__(self, errors: List[str]):
        super().__init__("; ".join(errors))
        self.errors = errors


def load_config(path: str) -> dict:
    with open(path) as f:
        text = f.read()
    if path.endswith(".json"):
        return json.loads(text)
    import yaml

    return yaml.safe_load(text) or {}


def resolve(cfg: dict) -> dict:
    """Defaults filled in; raises ConfigError listing every violation."""
    errors: List[str] = []
    out = copy.deepcopy(DEFAULTS)

    def merge(dst, src, prefix):
        for k, v in src.items():
            key = f"{prefix}{k}"
            if k not in dst:
                errors.append(f"unknown key '{key}'")
            elif isinstance(dst[k], dict):
                if not isinstance(v, dict):
                    errors.append(f"'{key}' must be a mapping")
                else:
                    merge(dst[k], v, key + ".")
            else:
                dst[k] = v

    if not isinstance(cfg, dict):
        raise ConfigError(["config must be a mapping"])
    merge(out, cfg, "")
    p, la, sg, lr, sa = out["problem"], out["lasgd"], out["sgd"], out["lr"], out["sgd_ar"]

    def need(cond, msg):
        if not cond:
            errors.append(msg)

    def num(v):
        return isinstance(v, (int, float)) and not isinstance(v, bool)

    def integer(v):
        return isinstance(v, int) and not isinstance(v, bool)

    need(out["schema"] == 1, "schema must be 1")
    need(p["kind"] in ("mlp",) + tuple(IMAGE_MODELS), f"problem.kind must be mlp or one of {sorted(IMAGE_MODELS)}")
    need(integer(p["n"]) and p["n"] >= 1, "problem.n must be a positive integer")
    need(integer(p["d"]) and p["d"] >= 1, "problem.d must be a positive integer")
    need(isinstance(p["hidden"], list) and all(integer(h) and h >= 1 for h in p["hidden"]),
         "problem.hidden must be a list of positive integers")
    need(num(p["noise"]) and p["noise"] >= 0, "problem.noise must be >= 0")
    need(integer(p["data_seed"]), "problem.data_seed must be an integer")
    need(integer(p["batch"]) and p["batch"] >= 1, "problem.batch must be a positive integer")
    need(out["algo"] in ("lasgd", "sgd_ar"), "algo must be lasgd or sgd_ar")
    need(integer(la["tau_max"]) and la["tau_max"] >= 1, "lasgd.tau_max must be an integer >= 1")
    need(isinstance(la["adaptive"], bool), "lasgd.adaptive must be a boolean")
    need(num(la["alpha"]) and 0 < la["alpha"] <= 1, "lasgd.alpha must be in (0, 1]")
    need(la["mode"] in ("pull", "delta"), "lasgd.mode must be pull or delta")
    need(la["pipeline"] in ("overlap", "fused"), "lasgd.pipeline must be overlap or fused")
    if la["mode"] == "delta" and la["alpha"] != 1:
        errors.append("lasgd.mode=delta is the reference LASGD rule, which requires alpha = beta = 1 "
                      "(optimizer.py:71-72); use mode=pull for alpha < 1")
    need(isinstance(la["nvls"], bool), "lasgd.nvls must be a boolean")
    if la["nvls"] is True and la["pipeline"] != "overlap":
        errors.append("lasgd.nvls=true runs the in-switch side-stream mean: it needs pipeline=overlap")
    if la["pipeline"] == "fused" and la["adaptive"]:
        errors.append("lasgd.pipeline=fused implements the deterministic schedule only (adaptive needs overlap)")
    need(isinstance(sa["bucketed"], bool), "sgd_ar.bucketed must be a boolean")
    need(num(sa["bucket_mb"]) and sa["bucket_mb"] > 0, "sgd_ar.bucket_mb must be > 0")
    for k in ("momentum", "dampening", "weight_decay"):
        need(num(sg[k]) and sg[k] >= 0, f"sgd.{k} must be >= 0")
    need(num(sg["dampening"]) and sg["dampening"] <= 1, "sgd.dampening must be <= 1")
    need(isinstance(sg["nesterov"], bool), "sgd.nesterov must be a boolean")
    if sg["nesterov"] is True and not (num(sg["momentum"]) and sg["momentum"] > 0 and sg["dampening"] == 0):
        errors.append("sgd.nesterov requires momentum > 0 and dampening = 0")
    need(num(lr["base_lr"]) and lr["base_lr"] > 0, "lr.base_lr must be > 0")
    need(integer(lr["scale_nodes"]) and lr["scale_nodes"] >= 1, "lr.scale_nodes must be an integer >= 1")
    need(num(lr["warmup_epochs"]) and lr["warmup_epochs"] >= 0, "lr.warmup_epochs must be >= 0")
    need(isinstance(lr["decay_epochs"], list) and all(num(e) for e in lr["decay_epochs"]),
         "lr.decay_epochs must be a list of numbers")
    need(num(lr["decay_factor"]) and lr["decay_factor"] > 0, "lr.decay_factor must be > 0")
    need(integer(out["steps"]) and out["steps"] >= 1, "steps must be a positive integer")
    need(integer(out["seed"]), "seed must be an integer")
    need(num(out["init_scale"]) and out["init_scale"] > 0, "init_scale must be > 0")
    if errors:
        raise ConfigError(errors)
    return out


def config_hash(cfg: dict) -> str:
    return hashlib.sha256(json.dumps(cfg, sort_keys=True).encode()).hexdigest()


def problem_hash(cfg: dict) -> str:
    return hashlib.sha256(json.dumps(cfg["problem"], sort_keys=True).encode()).hexdigest()


# ---------------------------------------------------------------------------- run
def _steps_per_epoch(cfg: dict, P: int) -> int:
    p = cfg["problem"]
    if p["kind"] != "mlp":
        return 1
    per_node = -(-p["n"] // P)
    return max(1, -(-per_node // p["batch"]))


def cmd_run(cfg: dict, out_dir: str) -> int:
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2203_13085_b200 as L
    from . import problems as PR
    from .trace import RunTrace, TraceRecorder, dump_json

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=dev)
    h = config_hash(cfg)
    p, la, sg = cfg["problem"], cfg["lasgd"], cfg["sgd"]
    spe = _steps_per_epoch(cfg, world)
    sched = L.LrSchedule(cfg["lr"]["base_lr"], cfg["lr"]["scale_nodes"], cfg["lr"]["warmup_epochs"],
                         tuple(cfg["lr"]["decay_epochs"]), cfg["lr"]["decay_factor"], spe)
    sgd = L.SgdConfig(sg["momentum"], sg["dampening"], sg["weight_decay"], sg["nesterov"])

    if p["kind"] == "mlp":
        feats, targs = PR.make_synthetic(p["data_seed"], p["n"], p["d"], p["noise"])
        X = torch.from_numpy(feats).to(dev, torch.float32)
        Y = torch.from_numpy(targs).to(dev, torch.float32)
        model = PR.mlp([p["d"]] + list(p["hidden"]) + [1], device=dev)
        flat = L.FlatParams(model)
        x0 = np.random.default_rng(cfg["seed"]).standard_normal(flat.numel) * cfg["init_scale"]
        flat.x.copy_(torch.from_numpy(x0.astype(np.float32)))
        sampler = PR.ShardSampler(p["n"], rank, world, p["batch"], cfg["seed"])

        def batch_loss():
            idx = torch.from_numpy(sampler.next_batch()).to(dev, non_blocking=True)
            return PR.mlp_loss(model, X[idx], Y[idx])

        def warm_loss():  # library initialisation only: no sampler draw, no update
            return PR.mlp_loss(model, X[:p["batch"]], Y[:p["batch"]])

        def full_loss():
            with torch.no_grad():
                return float(PR.mlp_loss(model, X, Y).item())
    else:
        import torchvision

        hw, classes = IMAGE_MODELS[p["kind"]]
        torch.manual_seed(cfg["seed"])
        model = getattr(torchvision.models, p["kind"])(num_classes=classes).to(dev)
        model = model.to(memory_format=torch.channels_last)
        flat = L.FlatParams(model, channels_last=True)
        if world > 1:
            dist.broadcast(flat.x, 0)
        gen = torch.Generator(device=dev)
        gen.manual_seed(1234 + rank)
        images = torch.randn(p["batch"], 3, hw, hw, device=dev, generator=gen).to(memory_format=torch.channels_last)
        labels = torch.randint(0, classes, (p["batch"],), device=dev, generator=gen)
        lossf = torch.nn.CrossEntropyLoss()

        def batch_loss():
            with torch.autocast("cuda", dtype=torch.bfloat16):
                return lossf(model(images), labels)

        def full_loss():
            with torch.no_grad(), torch.autocast("cuda", dtype=torch.bfloat16):
                return float(lossf(model(images), labels).item())

        warm_loss = batch_loss

    nvls = cfg["algo"] == "lasgd" and la["nvls"]
    comm = L.P2PCommunicator(flat.numel, timeout_s=120.0, nvls=nvls) if world > 1 else None
    compute = torch.cuda.Stream(device=dev, priority=-1)
    with torch.cuda.stream(compute):  # untimed: cuBLAS/cuDNN/autograd initialisation
        for _ in range(2):
            warm_loss().backward()
        flat.zero_grad()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with torch.cuda.stream(compute):
        if cfg["algo"] == "sgd_ar" and cfg["sgd_ar"]["bucketed"] and comm is not None:
            # buckets launched from autograd hooks as backward completes them (same bits)
            worker = L.BucketedSGDARWorker(flat, comm, sgd=sgd, schedule=sched, compute_stream=compute,
                                           bucket_bytes=max(16, int(cfg["sgd_ar"]["bucket_mb"] * (1 << 20))))
        elif cfg["algo"] == "sgd_ar":
            worker = L.SGDARWorker(flat.x, comm=comm, sgd=sgd, schedule=sched, compute_stream=compute, flat=flat)
        else:
            worker = L.LASGDWorker(flat.x, flat.g, comm=comm, sync_period=la["tau_max"], alpha=la["alpha"],
                                   mode=la["mode"], sgd=sgd, schedule=sched, adaptive=la["adaptive"],
                                   tau_max=la["tau_max"], compute_stream=compute, pipeline=la["pipeline"])
        rec = TraceRecorder(compute)
        end = torch.cuda.Event(enable_timing=True)
        try:
            for _ in range(cfg["steps"]):
                flat.zero_grad()
                loss = batch_loss()
                loss.backward()
                eta = worker.current_lr()
                closed = worker.step()
                rec.step(True if closed is None else closed, eta, loss)
            if hasattr(worker, "drain"):
                worker.drain()
            end.record(compute)
            torch.cuda.synchronize()
            if hasattr(worker, "state"):
                worker.state.check_finite()
            else:
                worker.check_finite()
        except L.NonFiniteError as e:
            print(f"error: numerical failure: {e}", file=sys.stderr)
            return EXIT_NUMERIC
    wall = rec.start.elapsed_time(end) / 1e3
    # the center model: mean of the replicas' final parameters
    if world > 1:
        t = torch.tensor([wall], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wall = float(t.item())
        dist.all_reduce(flat.x)
        flat.x.div_(world)
    final = full_loss()
    trace = RunTrace.gather(rec, flat.numel, 4)
    trace.validate()
    if rank == 0:
        os.makedirs(out_dir, exist_ok=True)
        trace.to_csv(os.path.join(out_dir, "trace.csv"), h)
        dump_json({"config_sha256": h, "problem_sha256": problem_hash(cfg), **cfg},
                  os.path.join(out_dir, "config.resolved.json"))
        summ = trace.summary(wall, final, algo=cfg["algo"], config_sha256=h, problem_sha256=problem_hash(cfg),
                             batch=p["batch"], steps_per_epoch=spe, n_samples=p["n"] if p["kind"] == "mlp" else None)
        dump_json(summ, os.path.join(out_dir, "summary.json"))
        print(json.dumps(summ))
    if comm is not None:
        if world > 1:
            dist.barrier()
        comm.close()
    if not np.isfinite(final):
        print("error: numerical failure: non-finite final loss", file=sys.stderr)
        return EXIT_NUMERIC
    return EXIT_OK


# ---------------------------------------------------------------------------- compare / plotdata
def compare(summaries: List[Tuple[str, dict]]) -> List[dict]:
    if len(summaries) < 2:
        raise ConfigError(["compare needs at least two summaries"])
    ph = {s.get("problem_sha256") for _, s in summaries}
    if len(ph) != 1:
        raise ConfigError(["summaries are of different problems (problem_sha256 differs)"])
    ref = summaries[0][1]["wall_time_s"]
    return [{"run": name, "algo": s.get("algo"), "final_loss": s["final_loss"], "wall_time_s": s["wall_time_s"],
             "rounds": s["rounds"], "speedup": ref / s["wall_time_s"]} for name, s in summaries]


def plotdata(traces: List[Tuple[str, str, List[dict], dict]]) -> List[dict]:
    """traces: (run name, algo, trace rows, summary) -> long rows (run, algo, x_kind, x, loss)."""
    out = []
    for name, algo, rows, summ in traces:
        n, b = summ.get("n_samples"), summ.get("batch")
        for r in rows:
            if r["loss"] is None:
                continue
            out.append({"run": name, "algo": algo, "x_kind": "time", "x": r["time_s"], "loss": r["loss"]})
            if n and b:
                out.append({"run": name, "algo": algo, "x_kind": "epoch", "x": r["grad_evals"] * b / n,
                            "loss": r["loss"]})
    return out


def _read_summary(path: str) -> dict:
    with open(os.path.join(path, "summary.json") if os.path.isdir(path) else path) as f:
        return json.load(f)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2203_13085_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    v = sub.add_parser("validate")
    v.add_argument("--config", required=True)
    r = sub.add_parser("run")
    r.add_argument("--config", required=True)
    r.add_argument("--out", required=True)
    r.add_argument("--seed", type=int, default=None)
    r.add_argument("--steps", type=int, default=None)
    r.add_argument("--quiet", action="store_true")
    c = sub.add_parser("compare")
    c.add_argument("runs", nargs="+", help="run directories or summary.json files (first = reference)")
    c.add_argument("--csv", default=None)
    pd = sub.add_parser("plotdata")
    pd.add_argument("runs", nargs="+", help="run directories")
    pd.add_argument("--out", required=True)
    a = ap.parse_args(argv)

    try:
        if a.cmd in ("validate", "run"):
            raw = load_config(a.config)
            if a.cmd == "run":
                if a.seed is not None:
                    raw["seed"] = a.seed
                if a.steps is not None:
                    raw["steps"] = a.steps
            cfg = resolve(raw)
            if a.cmd == "validate":
                print(json.dumps(cfg, indent=2, sort_keys=True))
                return EXIT_OK
            return cmd_run(cfg, a.out)
        if a.cmd == "compare":
            table = compare([(p, _read_summary(p)) for p in a.runs])
            for row in table:
                print(f"{row['run']:40s} {str(row['algo']):8s} loss={row['final_loss']!r:>24} "
                      f"wall={row['wall_time_s']:.4f}s speedup={row['speedup']:.3f}")
            if a.csv:
                import csv

                with open(a.csv, "w", newline="") as f:
                    w = csv.DictWriter(f, fieldnames=list(table[0]))
                    w.writeheader()
                    w.writerows(table)
            return EXIT_OK
        if a.cmd == "plotdata":
            import csv

            from .trace import read_trace_csv

            traces = []
            for p in a.runs:
                s = _read_summary(p)
                traces.append((p, s.get("algo"), read_trace_csv(os.path.join(p, "trace.csv")), s))
            rows = plotdata(traces)
            with open(a.out, "w", newline="") as f:
                w = csv.DictWriter(f, fieldnames=["run", "algo", "x_kind", "x", "loss"])
                w.writeheader()
                w.writerows(rows)
            return EXIT_OK
    except ConfigError as e:
        for msg in e.errors:
            print(f"error: {msg}", file=sys.stderr)
        return EXIT_CONFIG
    except (OSError, ValueError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_CONFIG
    return EXIT_CONFIG
