"""RunTrace: per-round records of a real run (SPEC.md harness ``RunTrace`` and
``bytes_accounting``).

Each rank keeps a ``TraceRecorder`` fed after every worker step; a round closes
when the worker says so.  Per closed round the recorder stores the device time
(a CUDA event on the compute stream, no host sync), the rank's tau (local steps in
the round), the rate and the step's minibatch loss (kept on the device).  At the
end ``RunTrace.gather`` pairs the k-th round of every rank — the k-th launch of
every rank pairs in the collective, exactly like the reference transport's round
ids — and builds the trace:

    round, time_s, node_tau_0..P-1, loss, eta, grad_evals, bytes_sent

* ``time_s``: device time since the start event by which every rank that closed the
  round had closed it (max over ranks, non-decreasing; measured, not simulated: the
  reference SPEC's ``sim_time_s`` column);
* ``loss``: mean over ranks of the minibatch training loss at each rank's closing
  step (free: the forward pass computed it);
* ``grad_evals``: cumulative local steps over all ranks at their k-th close;
* ``bytes_sent``: cumulative per-node bytes of the reference ring all-reduce,
  ``k * bytes_per_node(d, P, bpe)`` (collective.py:206-226), so traces are
  comparable with the reference's accounting whatever NVLink algorithm ran.
"""

from __future__ import annotations

import csv
import json
from dataclasses import asdict, dataclass
from typing import List, Optional

import torch

from .collective import bytes_per_node

CSV_FIELDS = ("round", "time_s", "node_tau", "loss", "eta", "grad_evals", "bytes_sent")


@dataclass
class RoundRecord:
    round: int
    local_clock: int
    tau: int
    eta: float
    time_s: float
    loss: Optional[float]


class TraceRecorder:
    def __init__(self, stream: Optional[torch.cuda.Stream] = None):
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        self.start = torch.cuda.Event(enable_timing=True)
        self.start.record(self.stream)
        self._clock = 0
        self._since = 0
        self._rounds = []  # (event, local_clock, tau, eta, loss tensor or None)

    def step(self, closed: bool, eta: float, loss: Optional[torch.Tensor] = None) -> None:
        """Call after every worker step (``closed`` = the step's return value)."""
        self._clock += 1
        self._since += 1
        if not closed:
            return
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(self.stream)
        lt = None if loss is None else loss.detach().reshape(1).to(torch.float64)
        self._rounds.append((ev, self._clock, self._since, float(eta), lt))
        self._since = 0

    def records(self) -> List[RoundRecord]:
        """Synchronises with the recorded events."""
        out = []
        for i, (ev, clock, tau, eta, lt) in enumerate(self._rounds):
            ev.synchronize()
            out.append(RoundRecord(i + 1, clock, tau, eta, self.start.elapsed_time(ev) / 1e3,
                                   None if lt is None else float(lt.item())))
        return out


class RunTrace:
    def __init__(self, per_rank: List[List[RoundRecord]], n_params: int, bytes_per_element: int = 4):
        self.per_rank = per_rank
        self.P = len(per_rank)
        self.n_params = n_params
        self.bpe = bytes_per_element
        self.bytes_per_round = bytes_per_node(n_params, self.P, bytes_per_element) if self.P > 1 else 0

    @classmethod
    def gather(cls, recorder: TraceRecorder, n_params: int, bytes_per_element: int = 4, group=None) -> "RunTrace":
        """Collective over torch.distributed when initialised (every rank gets the trace)."""
        import torch.distributed as dist

        mine = recorder.records()
        if dist.is_available() and dist.is_initialized():
            allr = [None] * dist.get_world_size(group)
            dist.all_gather_object(allr, [asdict(r) for r in mine], group=group)
            per_rank = [[RoundRecord(**d) for d in rs] for rs in allr]
        else:
            per_rank = [mine]
        return cls(per_rank, n_params, bytes_per_element)

    @property
    def rounds(self) -> int:
        return max((len(r) for r in self.per_rank), default=0)

    def rows(self) -> List[dict]:
        rows = []
        last_clock = [0] * self.P  # a rank that closed fewer rounds keeps its last count
        t_done = 0.0  # round k is complete no earlier than round k-1 (ranks drop out at the end)
        for k in range(self.rounds):
            recs = [rs[k] if k < len(rs) else None for rs in self.per_rank]
            present = [r for r in recs if r is not None]
            losses = [r.loss for r in present if r.loss is not None]
            for i, r in enumerate(recs):
                if r is not None:
                    last_clock[i] = r.local_clock
            t_done = max(t_done, max(r.time_s for r in present))
            rows.append({
                "round": k + 1,
                "time_s": t_done,
                "node_tau": [r.tau if r is not None else None for r in recs],
                "loss": sum(losses) / len(losses) if losses else None,
                "eta": present[0].eta,
                "grad_evals": sum(last_clock),
                "bytes_sent": (k + 1) * self.bytes_per_round,
            })
        return rows

    def validate(self) -> None:
        """RunTrace invariants: rounds strictly increasing, cumulative counters nondecreasing
        (per rank in the raw records, and in the merged rows)."""
        for i, recs in enumerate(self.per_rank):
            for a, b in zip(recs, recs[1:]):
                if b.time_s < a.time_s or b.local_clock <= a.local_clock:
                    raise ValueError(f"rank {i}: time / local clock decreased at round {b.round}")
        prev = None
        for row in self.rows():
            if prev is not None:
                if row["round"] <= prev["round"]:
                    raise ValueError("rounds must strictly increase")
                for key in ("time_s", "grad_evals", "bytes_sent"):
                    if row[key] < prev[key]:
                        raise ValueError(f"{key} decreased at round {row['round']}")
            prev = row

    def bytes_accounting(self) -> dict:
        """SPEC bytes_accounting: R rounds -> R * bytes_per_node per node, exactly."""
        R = self.rounds
        return {"rounds": R, "per_node": R * self.bytes_per_round, "total": R * self.bytes_per_round * self.P,
                "bytes_per_round_per_node": self.bytes_per_round}

    def to_csv(self, path: str, config_hash: Optional[str] = None) -> None:
        with open(path, "w", newline="") as f:
            if config_hash:
                f.write(f"# config_sha256={config_hash}\n")
            w = csv.writer(f)
            w.writerow(["round", "time_s"] + [f"node_tau_{i}" for i in range(self.P)]
                       + ["loss", "eta", "grad_evals", "bytes_sent"])
            for row in self.rows():
                w.writerow([row["round"], f"{row['time_s']:.9f}"]
                           + ["" if t is None else t for t in row["node_tau"]]
                           + ["" if row["loss"] is None else repr(row["loss"]), repr(row["eta"]),
                              row["grad_evals"], row["bytes_sent"]])

    def summary(self, wall_time_s: float, final_loss: Optional[float], **extra) -> dict:
        rows = self.rows()
        return {"rounds": self.rounds, "wall_time_s": wall_time_s, "final_loss": final_loss,
                "grad_evals": rows[-1]["grad_evals"] if rows else 0, "bytes": self.bytes_accounting(),
                "n_params": self.n_params, "nodes": self.P, **extra}


def read_trace_csv(path: str) -> List[dict]:
    """Rows of a trace CSV (comment lines skipped), numeric fields parsed."""
    with open(path) as f:
        lines = [ln for ln in f if not ln.startswith("#")]
    rows = []
    for rec in csv.DictReader(lines):
        row = {"round": int(rec["round"]), "time_s": float(rec["time_s"]),
               "loss": float(rec["loss"]) if rec["loss"] else None, "eta": float(rec["eta"]),
               "grad_evals": int(rec["grad_evals"]), "bytes_sent": int(rec["bytes_sent"]),
               "node_tau": [int(v) if v else None for k, v in rec.items() if k.startswith("node_tau_")]}
        rows.append(row)
    return rows


def dump_json(obj, path: str) -> None:
    with open(path, "w") as f:
        json.dump(obj, f, indent=2, sort_keys=True)
        f.write("\n")
