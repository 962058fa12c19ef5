"""Generate the golden fixtures under tests/golden/ by running the REFERENCE itself.

Run here (the build container, where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every array in the .npz files is produced by the unmodified reference package
(``lasgd`` from /root/reference/pkg/src, f64 numpy).  The GPU box has no
/root/reference, so the tests read these committed fixtures instead.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from lasgd import collective as C  # noqa: E402  (reference)
from lasgd import optimizer as O  # noqa: E402
from lasgd import params as PR  # noqa: E402
from lasgd import problems as PB  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def gen_primitives():
    out = {}
    meta = {}
    # partition_chunks (params.py:130-147) incl. d < P
    parts = {}
    for d, P in [(9, 3), (10, 3), (7, 1), (3, 5), (1, 8), (1000, 7), (1001, 8), (25557032, 8), (100609, 4)]:
        parts[f"{d},{P}"] = [list(b) for b in PR.partition_chunks(d, P).bounds]
    meta["partition"] = parts
    # ring schedule sizes (collective.py:51-83)
    meta["ring_steps"] = {str(P): C.ring_schedule(P).num_steps for P in range(1, 9)}
    meta["ring_schedule_3"] = [
        [[e.send_chunk, e.recv_chunk, e.send_to, e.recv_from, e.phase] for e in step]
        for step in C.ring_schedule(3).steps
    ]
    # bytes_per_node (collective.py:206-226)
    bpn = {}
    for d, P, b in [(100, 4, 8), (25557032, 2, 4), (25557032, 4, 4), (25557032, 8, 4), (1001, 3, 8), (7, 8, 4), (1, 1, 4)]:
        bpn[f"{d},{P},{b}"] = [C.bytes_per_node(d, P, b)] + [C.bytes_per_node(d, P, b, rank=r) for r in range(P)]
    meta["bytes_per_node"] = bpn
    # blend KATs + random
    rng = np.random.default_rng(1)
    u = rng.standard_normal(5003)
    v = rng.standard_normal(5003)
    out["blend_u"], out["blend_v"] = u, v
    for name, (a, b) in {"b1": (1.0, -0.037), "b2": (0.5, 0.5), "b3": (1.0, -1.0), "b4": (0.3, 0.7)}.items():
        out[f"blend_{name}"] = PR.blend(a, PR.ParamVector(u), b, PR.ParamVector(v)).data
        meta[f"blend_{name}"] = [a, b]
    # ring mean via execute_allreduce (collective.py:154-203); each rank's copy must match
    for P in range(1, 9):
        for d in (1, 5, 7, 1000, 1001, 4099):
            vecs = [rng.standard_normal(d) for _ in range(P)]
            res = C.execute_allreduce([v.copy() for v in vecs])
            for r in range(1, P):
                assert np.array_equal(res.per_rank[0], res.per_rank[r])
            out[f"mean_in_{P}_{d}"] = np.stack(vecs)
            out[f"mean_out_{P}_{d}"] = res.per_rank[0]
            meta[f"mean_bytes_{P}_{d}"] = list(res.bytes_sent)
    # lr_at (problems.py:355-365)
    sch = PB.LrSchedule(0.1, 16, 5, (30, 60, 80), 10.0, 10)
    meta["lr_sched"] = [0.1, 16, 5, [30, 60, 80], 10.0, 10]
    meta["lr_vals"] = [[s, PB.lr_at(sch, s)] for s in (0, 1, 7, 25, 49, 50, 51, 299, 300, 310, 600, 800, 1000)]
    sch2 = PB.LrSchedule(0.01, 1, 0)
    meta["lr_vals_flat"] = [[s, PB.lr_at(sch2, s)] for s in (0, 1, 99)]
    # loopback fault injection diagnostic (collective.py:238-242, 271-279)
    tr = C.LoopbackTransport(3, fault_at=(0, 1))
    h = tr.all_reduce([PR.ParamVector(rng.standard_normal(10)) for _ in range(3)], round_id=0)
    meta["fault_status"] = h.status.value
    meta["fault_diag"] = h.diagnostic
    return out, meta


def gen_node_loop(n, P, k, steps, seed):
    """Reference node loop (optimizer.py:136-207) with a fixed gradient sequence."""
    rng = np.random.default_rng(seed)
    x0 = rng.standard_normal(n) * 0.1
    grads = rng.standard_normal((steps, P, n))
    sch = PB.LrSchedule(0.05, P, 1.0, (2.0,), 10.0, max(1, steps // 3))
    etas = np.array([PB.lr_at(sch, t) for t in range(steps)])
    tr = C.LoopbackTransport(P)
    states = [O.NodeState.fresh(r, PR.ParamVector(x0)) for r in range(P)]
    rounds = {"id": 0}
    handles = {}
    for r, st in enumerate(states):
        handles[r] = tr.submit(0, r, st.x_snapshot)
        st.pending = handles[r]
    xs_hist = []
    for t in range(steps):
        for r, st in enumerate(states):
            g = PR.ParamVector(grads[t, r])

            def grad_fn(_x, g=g):
                return g

            O.lasgd_node_tick(st, grad_fn, _ConstSchedule(etas[t]), False, None, k, P)
        if states[0].tau_i == k:
            z = states[0].pending.result
            rid = states[0].global_clock + 1
            for r, st in enumerate(states):
                act = O.lasgd_node_tick(
                    st, None, sch, True, z, k, P, submit=lambda v, r=r, rid=rid: tr.submit(rid, r, v)
                )
                assert act is O.TickAction.FINALIZED
        xs_hist.append(np.stack([st.x_local.data for st in states]))
    return {
        "x0": x0,
        "grads": grads,
        "etas": etas,
        "xs_hist": np.stack(xs_hist),
        "final_snap": np.stack([st.x_snapshot.data for st in states]),
        "final_delta": np.stack([st.delta.data for st in states]),
        "P": np.array(P),
        "k": np.array(k),
    }


class _ConstSchedule:
    """Stand-in schedule so the tick uses the pre-tabulated eta (lr_at is pinned separately)."""

    def __init__(self, eta):
        self.base_lr = eta
        self.scale_nodes = 1
        self.warmup_epochs = 0
        self.decay_epochs = ()
        self.decay_factor = 10.0
        self.steps_per_epoch = 1

    @property
    def peak_lr(self):
        return self.base_lr


def gen_pull_loop(n, P, k, steps, alpha, seed):
    """alpha != 1 pull composed from reference primitives (optimizer.py:145, 256-257;
    collective.py:154-203): x = blend(1, x, -alpha, blend(1, snap, -1, xbar))."""
    rng = np.random.default_rng(seed)
    x0 = rng.standard_normal(n) * 0.1
    grads = rng.standard_normal((steps, P, n))
    etas = np.full(steps, 0.03)
    xs = [PR.ParamVector(x0) for _ in range(P)]
    snaps = list(xs)
    z = PR.ParamVector(C.execute_allreduce([s.data for s in snaps]).per_rank[0])
    tau = 0
    hist = []
    for t in range(steps):
        xs = [PR.blend(1.0, xs[r], -etas[t], PR.ParamVector(grads[t, r])) for r in range(P)]
        tau += 1
        if tau == k:
            if P > 1:
                xs = [PR.blend(1.0, xs[r], -alpha, PR.blend(1.0, snaps[r], -1.0, z)) for r in range(P)]
            snaps = list(xs)
            z = PR.ParamVector(C.execute_allreduce([s.data for s in snaps]).per_rank[0])
            tau = 0
        hist.append(np.stack([x.data for x in xs]))
    return {"x0": x0, "grads": grads, "etas": etas, "xs_hist": np.stack(hist), "alpha": np.array(alpha),
            "P": np.array(P), "k": np.array(k)}


def gen_config1(alpha, steps=100, P=4, k=4, hidden=128, batch=32):
    """Config 1 (BASELINE.json configs[0]): MLP [784,hidden,1] on make_synthetic(0,4096,784,0.1,
    'regression'), P=4 simulated workers, tau=4, LrSchedule(0.01,1,0), 100 local steps each."""
    ds = PB.make_synthetic(0, 4096, 784, 0.1, "regression")
    orc = PB.MlpOracle([784, hidden, 1], ds)
    n = orc.dim
    x0 = np.random.default_rng(0).standard_normal(n) * 0.05
    sch = PB.LrSchedule(0.01, 1, 0)
    samplers = [PB.ShardSampler(ds, r, P, batch, seed=0) for r in range(P)]
    losses = np.zeros((steps, P))
    batches = np.zeros((steps, P, batch), dtype=np.int64)
    if alpha == 1.0:
        tr = C.LoopbackTransport(P)
        states = [O.NodeState.fresh(r, PR.ParamVector(x0)) for r in range(P)]
        for r, st in enumerate(states):
            st.pending = tr.submit(0, r, st.x_snapshot)
        t = 0
        while t < steps:
            for r, st in enumerate(states):
                def grad_fn(x, r=r, t=t):
                    b = samplers[r].next_batch()
                    batches[t, r] = b
                    loss, g = orc.loss_and_grad(x, b)
                    losses[t, r] = loss
                    return g

                act = O.lasgd_node_tick(st, grad_fn, sch, False, None, k, P)
                assert act is O.TickAction.COMPUTED_STEP
            t += 1
            if states[0].tau_i == k:
                z = states[0].pending.result
                rid = states[0].global_clock + 1
                for r, st in enumerate(states):
                    O.lasgd_node_tick(st, None, sch, True, z, k, P, submit=lambda v, r=r, rid=rid: tr.submit(rid, r, v))
        final = np.stack([st.x_local.data for st in states])
    else:
        xs = [PR.ParamVector(x0) for _ in range(P)]
        snaps = list(xs)
        z = PR.ParamVector(C.execute_allreduce([s.data for s in snaps]).per_rank[0])
        tau = 0
        clock = 0
        for t in range(steps):
            eta = PB.lr_at(sch, clock)
            for r in range(P):
                b = samplers[r].next_batch()
                batches[t, r] = b
                loss, g = orc.loss_and_grad(xs[r], b)
                losses[t, r] = loss
                xs[r] = PR.blend(1.0, xs[r], -eta, g)
            clock += 1
            tau += 1
            if tau == k:
                xs = [PR.blend(1.0, xs[r], -alpha, PR.blend(1.0, snaps[r], -1.0, z)) for r in range(P)]
                snaps = list(xs)
                z = PR.ParamVector(C.execute_allreduce([s.data for s in snaps]).per_rank[0])
                tau = 0
        final = np.stack([x.data for x in xs])
    sample_idx = np.random.default_rng(7).choice(n, 4096, replace=False)
    return {
        "losses": losses,
        "batches": batches,
        "final_sample_idx": sample_idx,
        "final_sample": final[:, sample_idx],
        "x0_head": x0[:64],
        "ds_checksum": np.array([ds.features.sum(), ds.targets.sum(), ds.features[17, 300], ds.targets[4095]]),
        "n": np.array(n),
        "alpha": np.array(alpha),
    }


def main():
    prim, meta = gen_primitives()
    np.savez_compressed(os.path.join(HERE, "primitives.npz"), **prim)
    with open(os.path.join(HERE, "primitives.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    loops = {}
    for tag, (n, P, k, steps, seed) in {"a": (1001, 3, 2, 6, 11), "b": (4099, 4, 3, 9, 12), "c": (37, 8, 1, 4, 13),
                                         "d": (513, 1, 3, 7, 14), "e": (2048, 2, 4, 8, 15)}.items():
        for key, val in gen_node_loop(n, P, k, steps, seed).items():
            loops[f"{tag}_{key}"] = val
    np.savez_compressed(os.path.join(HERE, "node_loops.npz"), **loops)
    pulls = {}
    for tag, (n, P, k, steps, alpha, seed) in {"a": (1001, 3, 2, 6, 0.5, 21), "b": (4099, 4, 1, 5, 0.25, 22),
                                                "c": (2050, 2, 3, 6, 1.0, 23)}.items():
        for key, val in gen_pull_loop(n, P, k, steps, alpha, seed).items():
            pulls[f"{tag}_{key}"] = val
    np.savez_compressed(os.path.join(HERE, "pull_loops.npz"), **pulls)
    cfg = {}
    for alpha in (1.0, 0.5):
        for key, val in gen_config1(alpha).items():
            cfg[f"a{int(alpha * 100)}_{key}"] = val
    np.savez_compressed(os.path.join(HERE, "config1.npz"), **cfg)
    print("golden fixtures written to", HERE)


def gen_sgd_ar(n=1001, P=3, rounds=5, seed=31):
    """sync_allreduce_sgd_round (optimizer.py:214-242) with fixed gradients (reference)."""
    rng = np.random.default_rng(seed)
    x0 = rng.standard_normal(n)
    grads = rng.standard_normal((rounds, P, n))
    etas = np.array([0.1, 0.05, 0.2, 0.01, 0.07])[:rounds]
    states = [O.NodeState.fresh(r, PR.ParamVector(x0)) for r in range(P)]
    hist, means = [], []
    for t in range(rounds):
        mg = O.sync_allreduce_sgd_round(states, [PR.ParamVector(g) for g in grads[t]], float(etas[t]), round_id=t)
        means.append(mg.data)
        hist.append(states[0].x_local.data.copy())
    return {"x0": x0, "grads": grads, "etas": etas, "x_hist": np.stack(hist), "mean_hist": np.stack(means)}


def main_sgd_ar():
    np.savez_compressed(os.path.join(HERE, "sgd_ar.npz"), **gen_sgd_ar())
    print("sgd_ar fixture written")


def gen_easgd(n=1003, seed=41):
    """elastic_local_step / elastic_center_step / easgd_round_robin_exchange
    (optimizer.py:113-133, 245-259) and mean_of_vectors (params.py:150-158), reference."""
    rng = np.random.default_rng(seed)
    x, z, g = (rng.standard_normal(n) for _ in range(3))
    xs = rng.standard_normal((5, n))
    out = {"x": x, "z": z, "g": g, "xs": xs}
    for i, (eta, alpha) in enumerate([(0.1, 0.5), (0.03, 0.0), (0.2, 1.0), (0.07, 0.3)]):
        out[f"els_{i}"] = O.elastic_local_step(PR.ParamVector(x), PR.ParamVector(z), PR.ParamVector(g), eta, alpha).data
        out[f"els_{i}_args"] = np.array([eta, alpha])
    for i, beta in enumerate([0.0, 0.25, 0.9, 1.0]):
        out[f"ecs_{i}"] = O.elastic_center_step(PR.ParamVector(z), [PR.ParamVector(v) for v in xs[: 2 + i]], beta).data
        out[f"ecs_{i}_args"] = np.array([beta, 2 + i])
    for i, alpha in enumerate([0.1, 0.5, 0.9]):
        nx, nz = O.easgd_round_robin_exchange(PR.ParamVector(x), PR.ParamVector(z), alpha)
        out[f"rr_{i}_x"], out[f"rr_{i}_z"] = nx.data, nz.data
        out[f"rr_{i}_args"] = np.array([alpha])
    for k in (1, 2, 3, 5):
        out[f"mean_{k}"] = PR.mean_of_vectors([PR.ParamVector(v) for v in xs[:k]]).data
    return out


def main_easgd():
    np.savez_compressed(os.path.join(HERE, "easgd.npz"), **gen_easgd())
    print("easgd fixture written")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "sgd_ar":
        main_sgd_ar()
    elif len(sys.argv) > 1 and sys.argv[1] == "easgd":
        main_easgd()
    else:
        main()
        main_sgd_ar()
        main_easgd()
