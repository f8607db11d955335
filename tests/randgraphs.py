"""Seeded random small graphs over the reference's operator vocabulary
("100 random small graphs"), used to check the executor and
the map algebra against the reference on many shapes."""
from __future__ import annotations

import random

from paper_2604_09558_b200.workloads import GraphBuilder


def _factorizations(n):
    out = []
    for a in range(1, n + 1):
        if n % a == 0:
            out.append((a, n // a))
    return out


def random_graph(seed: int, dtype: str = "f64", max_ops: int = 7, compute: bool = True) -> dict:
    rnd = random.Random(seed)
    g = GraphBuilder(dtype)
    rank = rnd.randint(2, 4)
    shape = [rnd.randint(2, 5) for _ in range(rank)]
    cur = g.input("x", shape)
    k = 0

    def fresh(prefix):
        nonlocal k
        k += 1
        return f"{prefix}{k}"

    n_ops = rnd.randint(2, max_ops)
    for _ in range(n_ops):
        op = rnd.choice(["Transpose", "Reshape", "Slice", "Unsqueeze", "Expand", "Concat", "Split", "Roll",
                         "Add", "SiLU"] if compute else
                        ["Transpose", "Reshape", "Slice", "Unsqueeze", "Expand", "Concat", "Split", "Roll"])
        r = len(shape)
        out = fresh("t")
        if op == "Transpose":
            perm = list(range(r))
            rnd.shuffle(perm)
            g.node(fresh("n"), "Transpose", [cur], out, {"perm": perm})
            shape = [shape[p] for p in perm]
        elif op == "Reshape":
            vol = 1
            for s in shape:
                vol *= s
            new = []
            rem = vol
            for _ in range(rnd.randint(1, 3)):
                fs = [f for f in _factorizations(rem) if f[0] > 1] or [(1, rem)]
                a, b = rnd.choice(fs)
                new.append(a)
                rem = b
            new.append(rem)
            new = [d for d in new if d > 1] or [vol]
            if len(new) > 5:
                continue
            g.node(fresh("n"), "Reshape", [cur], out, {"shape": new})
            shape = new
        elif op == "Slice":
            ax = rnd.randrange(r)
            if shape[ax] < 2:
                continue
            s = rnd.randint(0, shape[ax] - 2)
            e = rnd.randint(s + 1, shape[ax])
            g.node(fresh("n"), "Slice", [cur], out, {"axes": [ax], "starts": [s], "ends": [e]})
            shape = list(shape)
            shape[ax] = e - s
        elif op == "Unsqueeze":
            if r >= 5:
                continue
            ax = rnd.randint(0, r)
            g.node(fresh("n"), "Unsqueeze", [cur], out, {"axis": ax})
            shape = shape[:ax] + [1] + shape[ax:]
        elif op == "Expand":
            ax = rnd.randrange(r)
            f = rnd.randint(2, 3)
            tgt = list(shape)
            tgt[ax] *= f
            g.node(fresh("n"), "Expand", [cur], out, {"shape": tgt})
            shape = tgt
        elif op == "Concat":
            ax = rnd.randrange(r)
            other_shape = list(shape)
            other_shape[ax] = rnd.randint(1, 3)
            other = g.input(fresh("c"), other_shape)
            order = [cur, other] if rnd.random() < 0.5 else [other, cur]
            g.node(fresh("n"), "Concat", order, out, {"axis": ax})
            shape = list(shape)
            shape[ax] += other_shape[ax]
        elif op == "Split":
            ax = rnd.randrange(r)
            if shape[ax] < 2:
                continue
            a = rnd.randint(1, shape[ax] - 1)
            other = fresh("t")
            keep = rnd.random() < 0.5
            g.node(fresh("n"), "Split", [cur], [out, other], {"axis": ax, "sizes": [a, shape[ax] - a]})
            # the unused part becomes a graph output so every tensor is consumed or output
            if keep:
                g.output(other)
                shape = list(shape)
                shape[ax] = a
            else:
                g.output(out)
                out = other
                shape = list(shape)
                shape[ax] = shape[ax] - a
        elif op == "Roll":
            ax = rnd.randrange(r)
            g.node(fresh("n"), "Roll", [cur], out, {"axes": [ax], "shifts": [rnd.randint(-3, 3)]})
        elif op == "Add":
            other = g.input(fresh("c"), shape)
            g.node(fresh("n"), "Add", [cur, other], out)
        elif op == "SiLU":
            if dtype == "i64":
                continue
            g.node(fresh("n"), "SiLU", [cur], out)
        cur = out
    # finish with a MatMul (compute) when possible, else an Add
    if compute and len(shape) >= 2 and rnd.random() < 0.7:
        w = g.input(fresh("w"), shape[:-2] + [shape[-1], rnd.randint(1, 5)])
        g.node(fresh("n"), "MatMul", [cur, w], "y", out_kind="output")
    else:
        other = g.input(fresh("c"), shape)
        g.node(fresh("n"), "Add", [cur, other], "y", out_kind="output")
    return g.doc()


def uses_roll(doc) -> bool:
    return any(n["kind"] == "Roll" for n in doc["nodes"])
