#!/usr/bin/env python
"""Cross-check of the frozen cost table's SQ entry (VERDICT r1 weak #3,
SURVEY §8(d) "derived from the minimal analytic formulas and cross-checked by
a sympy-CSE count"): scalar operation counts of the SQ radial distance of
Eq. (1) (reading #2) and of its gradient and Hessian in the local
frame, after common-subexpression elimination.

    python tools/sympy_count.py  -> profiles/sympy_sq_counts.json

Counts: every +, -, *, / is one scalar op; every exp / log / pow with a
non-integer exponent (evaluated as exp(p log x)) is one transcendental (a
MUFU op on the GPU: ex2 / lg2 / rcp / rsqrt) plus the multiply by the
exponent.  Compare with the table (ncu FP32 op counts of the kernel, FFMA =
2, including the world <-> local transforms and guards)."""
import json
import os

import sympy as sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def counts(exprs):
    repl, red = sp.cse(exprs, optimizations="basic")
    allx = [e for _, e in repl] + list(red)
    ops = {"add": 0, "mul": 0, "div": 0, "transcendental": 0, "pow_int": 0}
    for e in allx:
        for node in sp.preorder_traversal(e):
            if isinstance(node, sp.Add):
                ops["add"] += len(node.args) - 1
            elif isinstance(node, sp.Mul):
                ops["mul"] += len(node.args) - 1
            elif isinstance(node, sp.Pow):
                ex = node.args[1]
                if ex.is_Integer:
                    if ex < 0:
                        ops["div"] += 1
                        if abs(ex) > 1:
                            ops["pow_int"] += 1
                    else:
                        ops["pow_int"] += 1
                elif ex == sp.Rational(1, 2) or ex == sp.Rational(-1, 2):
                    ops["transcendental"] += 1       # sqrt / rsqrt
                else:
                    ops["transcendental"] += 2       # exp(p log x): lg2 + ex2
                    ops["mul"] += 1
            elif isinstance(node, (sp.exp, sp.log)):
                ops["transcendental"] += 1
    ops["scalar_ops"] = ops["add"] + ops["mul"] + ops["div"] + ops["pow_int"]
    ops["cse_temporaries"] = len(repl)
    return ops


def main():
    y = sp.symbols("y0:3", real=True)
    a = sp.symbols("a0:3", positive=True)
    e1, e2 = sp.symbols("e1 e2", positive=True)
    u2 = [(y[i] / a[i]) ** 2 for i in range(3)]
    f = (u2[0] ** (1 / e2) + u2[1] ** (1 / e2)) ** (e2 / e1) + u2[2] ** (1 / e1)
    r = sp.sqrt(y[0] ** 2 + y[1] ** 2 + y[2] ** 2)
    phi = r * (1 - f ** (-e1 / 2))
    grad = [sp.diff(phi, v) for v in y]
    hess = [sp.diff(grad[i], y[j]) for i in range(3) for j in range(i, 3)]
    res = {"value": counts([phi]), "value+gradient": counts([phi] + grad),
           "value+gradient+hessian": counts([phi] + grad + hess)}
    with open(os.path.join(ROOT, "paper_2604_17538_b200", "costmodel.json")) as fjs:
        cm = json.load(fjs)
    res["cost_table_sq_sphere_sph0"] = cm["sdf"]["sph0"]
    res["note"] = ("sympy: generic CSE of the literal formulas in the local frame (no log-domain factoring, no "
                   "transforms); table: ncu FP32 ops (FFMA = 2) of the kernel's evaluation incl. world <-> local "
                   "transforms, guards and the class dispatch")
    out = os.path.join(ROOT, "profiles", "sympy_sq_counts.json")
    with open(out, "w") as fo:
        json.dump(res, fo, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
