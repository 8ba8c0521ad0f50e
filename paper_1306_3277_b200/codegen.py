"""Generic models on the device path: a reference `ModelIr`
lowered to a JSON-able description, then to a CUDA source compiled at run
time (NVRTC, csrc/ssm_gen.cu) -- LibBi's own design.

Lowering (`lower`) walks the IR the reference builds (core/ir.py:83-121,
291-347): for the `initial`, `transition` and `observation` blocks it records
every statement unrolled over its dim loop, with expressions as small trees
resolved to role slots exactly as ir.py:151-193 does:

    ["num", v] | ["T", k] | ["X", k] | ["W", k] | ["U", k] | ["neg", e]
    | ["bin", op, l, r] | ["call", name, [args]]

From the trees:
  * `numpy_source` prints the reference's own expression source
    (ir.py:170-193, e.g. "((X[:, 7] * (X[:, 1] - X[:, 6])) - X[:, 0])"), used
    for host-side evaluation with the reference's semantics;
  * `cuda_source` emits `gen::Model` -- the transition sub-step, the
    observation log-density and the initial block for one particle -- in the
    reference's evaluation order (statement order; every slot of a statement
    evaluated before any is written, simulate.py:62-68; RK4 as
    simulate.py:71-93; log-densities as distributions.py:94-123), with every
    arithmetic op individually rounded under `E` (exact mode).

Limits of the device path: n_state <= 32, n_obs <= 32, n_input <= 16.
"""

from __future__ import annotations

import hashlib
import json
import math
import os

import numpy as np

from .errors import UnsupportedModelError

MAX_STATE, MAX_OBS, MAX_INPUT = 32, 32, 16

# distributions.py:33-46 (canonical argument order and defaults)
DIST_PARAMS = {
    "gaussian": ("mean", "sd"),
    "normal": ("mean", "sd"),
    "truncated_gaussian": ("mean", "sd", "lower", "upper"),
    "gamma": ("shape", "scale"),
    "inverse_gamma": ("shape", "scale"),
    "uniform": ("lower", "upper"),
    "wiener": (),
}
DIST_DEFAULTS = {"truncated_gaussian": {"lower": -math.inf, "upper": math.inf}}
KIND_OF = {"normal": "gaussian"}
ROLE_KEY = {"param": "T", "state": "X", "noise": "W", "input": "U"}
FN_NUMPY = {"exp": "np.exp", "sqrt": "np.sqrt", "sin": "np.sin", "pow": "np.power", "mod": "np.mod"}
LOG_SQRT_2PI = 0.5 * np.log(2.0 * np.pi)  # distributions.py:15


# ---------------------------------------------------------------------------
# lowering (reference IR, duck-typed) -> description
# ---------------------------------------------------------------------------


def _resolve_index(dim, ix, binding):
    """ir.py:124-135"""
    value = ix.offset if ix.var is None else binding[ix.var] + ix.offset
    if dim.boundary == "cyclic":
        return value % dim.size
    if not 0 <= value < dim.size:
        raise UnsupportedModelError(f"index {value} out of range for dim {dim.name}")
    return value


def _resolve_slot(var, indices, binding):
    """ir.py:138-146"""
    flat = 0
    for dim, ix in zip(var.dims, indices):
        flat = flat * dim.size + _resolve_index(dim, ix, binding)
    return var.offset + flat


def _expr(node, consts, vars_, binding):
    kind = type(node).__name__
    if kind == "Num":
        return ["num", float(node.value)]
    if kind == "VarRef":
        if node.name in consts:
            return ["num", float(consts[node.name])]
        var = vars_[node.name]
        return [ROLE_KEY[var.role], _resolve_slot(var, node.indices, binding)]
    if kind == "Unary":
        return ["neg", _expr(node.operand, consts, vars_, binding)]
    if kind == "Binary":
        return ["bin", node.op, _expr(node.left, consts, vars_, binding), _expr(node.right, consts, vars_, binding)]
    if kind == "Call":
        if node.name not in FN_NUMPY:
            raise UnsupportedModelError(f"function {node.name!r}")
        return ["call", node.name, [_expr(a, consts, vars_, binding) for a in node.args]]
    raise UnsupportedModelError(f"expression node {kind}")


def _dist_args(dist):
    """ir.py:226-245: canonical arguments with defaults."""
    name = dist.name
    if name not in DIST_PARAMS:
        raise UnsupportedModelError(f"distribution {name!r}")
    params = DIST_PARAMS[name]
    by_name = dict(zip(params, dist.args))
    by_name.update(dict(dist.named))
    out = []
    for p in params:
        if p in by_name:
            out.append(by_name[p])
        else:
            out.append(("default", DIST_DEFAULTS[name][p]))
    return KIND_OF.get(name, name), out


def _lower_op(op, ir):
    consts, vars_ = ir.consts, ir.vars
    cls = type(op).__name__
    if cls == "SampleStmtOp":
        kind, arg_nodes = _dist_args(op.stmt.dist)
        args = []
        for b in op.bindings:
            row = []
            for a in arg_nodes:
                row.append(["num", float(a[1])] if isinstance(a, tuple) else _expr(a, consts, vars_, b))
            args.append(row)
        return {"op": "sample", "role": op.role, "kind": kind, "slots": list(op.slots), "args": args}
    if cls == "AssignStmtOp":
        return {"op": "assign", "role": op.role, "slots": list(op.slots),
                "exprs": [_expr(op.stmt.expr, consts, vars_, b) for b in op.bindings]}
    if cls == "OdeOp":
        if str(op.alg).upper() != "RK4":
            raise UnsupportedModelError(f"ode alg {op.alg!r}")
        return {"op": "ode", "slots": list(op.slots), "h": float(op.h),
                "exprs": [_expr(eq.expr, consts, vars_, b) for eq, b in op.items]}
    raise UnsupportedModelError(f"statement {cls}")


THETA_BLOCKS = ("parameter", "proposal_parameter", "proposal_initial")


def fingerprint(ir) -> str:
    """Digest of every block of a reference ModelIr, lowered (including the
    theta-level blocks the hand-written specs implement on the host)."""
    d = {"name": ir.name, "counts": {k: int(v) for k, v in ir.counts.items()},
         "delta": None if ir.delta is None else float(ir.delta)}
    for name in ("initial", "transition", "observation") + THETA_BLOCKS:
        blk = ir.block(name)
        d[name] = [] if blk is None else [_lower_op(op, ir) for op in blk.ops]
    return hashlib.sha256(dumps(d).encode()).hexdigest()


ROLES_WITH_SLOTS = ("param", "input", "noise", "state", "obs")


def lower(ir) -> dict:
    """Reference ModelIr -> JSON-able description (the codegen input)."""
    counts = {k: int(v) for k, v in ir.counts.items()}
    if counts["state"] > MAX_STATE or counts["obs"] > MAX_OBS or counts["input"] > MAX_INPUT:
        raise UnsupportedModelError(
            f"{ir.name}: device path limits are n_state <= {MAX_STATE}, n_obs <= {MAX_OBS}, n_input <= {MAX_INPUT}")
    out = {"name": ir.name, "counts": counts, "delta": None if ir.delta is None else float(ir.delta)}
    # variable table (name, role, slot offset, dim sizes) for the data-file layer (timeseries.py)
    out["vars"] = [{"name": v.name, "role": v.role, "offset": int(v.offset), "dims": [int(d.size) for d in v.dims]}
                   for v in ir.vars.values() if getattr(v, "role", None) in ROLES_WITH_SLOTS]
    for name in ("initial", "transition", "observation"):
        blk = ir.block(name)
        out[name] = [] if blk is None else [_lower_op(op, ir) for op in blk.ops]
    for op in out["observation"]:
        if op["op"] != "sample" or op["kind"] == "wiener":
            raise UnsupportedModelError("observation block: distribution statements only")
    # theta-level blocks, evaluated on the host by the PMMH / SMC^2 loops (None = absent)
    for name in THETA_BLOCKS:
        blk = ir.block(name)
        out[name] = None if blk is None else [_lower_op(op, ir) for op in blk.ops]
    return out


# ---------------------------------------------------------------------------
# expression printers
# ---------------------------------------------------------------------------


def numpy_source(e) -> str:
    """The reference's expression source (ir.py:170-193)."""
    t = e[0]
    if t == "num":
        return repr(e[1])
    if t == "U":
        return f"U[{e[1]}]"
    if t in ("T", "X", "W"):
        return f"{t}[:, {e[1]}]"
    if t == "neg":
        return f"(-{numpy_source(e[1])})"
    if t == "bin":
        return f"({numpy_source(e[2])} {e[1]} {numpy_source(e[3])})"
    if t == "call":
        return f"{FN_NUMPY[e[1]]}({', '.join(numpy_source(a) for a in e[2])})"
    raise ValueError(e)


def numpy_fn(e):
    """lambda T, X, W, U evaluating the expression like ir.py:196-198 (the
    `inf` default of truncated bounds is made evaluable)."""
    return eval(f"lambda T, X, W, U: {numpy_source(e)}", {"np": np, "inf": np.inf, "__builtins__": {}})


def _is_const(e):
    t = e[0]
    if t == "num":
        return True
    if t in ("T", "X", "W", "U"):
        return False
    if t == "neg":
        return _is_const(e[1])
    if t == "bin":
        return _is_const(e[2]) and _is_const(e[3])
    return all(_is_const(a) for a in e[2])


def _const_value(e):
    z = np.zeros((1, 1))
    return float(np.asarray(numpy_fn(e)(z, z, z, np.zeros(1))).reshape(-1)[0])


def _lit(v: float) -> str:
    if math.isnan(v):
        return "T(CUDART_NAN)"
    if math.isinf(v):
        return "T(CUDART_INF)" if v > 0 else "T(-CUDART_INF)"
    return f"T({float(v).hex()})"


def _dlit(v: float) -> str:
    if math.isinf(v):
        return "CUDART_INF" if v > 0 else "(-CUDART_INF)"
    return float(v).hex()


_OPS = {"+": "add", "-": "sub", "*": "mul", "/": "div"}


def cuda_expr(e, xname="X") -> str:
    """C++ expression of type T (numpy float64 semantics under E: one rounding per op)."""
    t = e[0]
    if t == "num":
        return _lit(e[1])
    if t == "T":
        return f"T(TH[{e[1]}])"
    if t == "X":
        return f"{xname}[{e[1]}]"
    if t == "W":
        return f"W[{e[1]}]"
    if t == "U":
        return f"T(U[{e[1]}])"
    if t == "neg":
        return f"(-{cuda_expr(e[1], xname)})"
    if t == "bin":
        if e[1] == "/" and e[3][0] == "num" and math.isfinite(e[3][1]) and e[3][1] != 0.0:
            c = e[3][1]  # constant divisor: fast mode multiplies by the reciprocal
            return f"O::divc({cuda_expr(e[2], xname)}, {_lit(c)}, {_lit(1.0 / c)})"
        return f"O::{_OPS[e[1]]}({cuda_expr(e[2], xname)}, {cuda_expr(e[3], xname)})"
    if t == "call":
        args = [cuda_expr(a, xname) for a in e[2]]
        fn = {"exp": "exp", "sqrt": "sqrt", "sin": "sin", "pow": "pow", "mod": "ssm::py_mod"}[e[1]]
        return f"{fn}({', '.join(args)})"
    raise ValueError(e)


# ---------------------------------------------------------------------------
# CUDA source
# ---------------------------------------------------------------------------


class _Emitter:
    def __init__(self):
        self.lines = []
        self.ind = 2

    def __call__(self, s=""):
        self.lines.append(" " * self.ind + s if s else "")

    def block(self, head, comment=None):
        self((head + " {").lstrip() + (f"  // {comment}" if comment else ""))
        self.ind += 2

    def end(self, tail="}"):
        self.ind -= 2
        self(tail)


_NORMAL_KINDS = ("wiener", "gaussian")
_UNIFORM_KINDS = ("uniform", "truncated_gaussian")


def draw_plan(kinds):
    """Device words of each draw of a block (kd = draw index): normals take half
    a Box-Muller pair, uniforms a whole pair (two 32-bit words each); pairs are
    packed two per Philox block.  Returns (per-draw ("z", i) | ("u", i) |
    ("g", kd), normal pairs [(pair, z index)], uniform pairs [(pair, u index)],
    n_blocks)."""
    plan, zpairs, upairs = [], [], []
    q, open_z = 0, None
    for kd, kind in enumerate(kinds):
        if kind in _NORMAL_KINDS:
            if open_z is None:
                zpairs.append((q, 2 * len(zpairs)))
                open_z = zpairs[-1][1]
                q += 1
                plan.append(("z", open_z))
            else:
                plan.append(("z", open_z + 1))
                open_z = None
        elif kind in _UNIFORM_KINDS:
            upairs.append((q, len(upairs)))
            q += 1
            plan.append(("u", upairs[-1][1]))
        else:
            plan.append(("g", kd))
    return plan, zpairs, upairs, (q + 1) // 2


def _emit_draw_words(em, kinds):
    """Take each Philox block once; Box-Muller per normal pair; u53 per uniform."""
    plan, zpairs, upairs, nblk = draw_plan(kinds)
    em(f"float Z_[{max(2 * len(zpairs), 1)}];")
    em(f"double V_[{max(len(upairs), 1)}];")
    em("(void)Z_; (void)V_;")
    if nblk:
        em.block("if constexpr (!INJ)")
        for b in range(nblk):
            em(f"const ssm::U4 R{b} = dr.block({b});")
        for pq, zi in zpairs:
            w = ("x", "y") if pq % 2 == 0 else ("z", "w")
            em(f"ssm::box_muller(R{pq // 2}.{w[0]}, R{pq // 2}.{w[1]}, Z_[{zi}], Z_[{zi + 1}]);")
        for pq, ui in upairs:
            w = ("x", "y") if pq % 2 == 0 else ("z", "w")
            em(f"V_[{ui}] = ssm::u53(R{pq // 2}.{w[0]}, R{pq // 2}.{w[1]});")
        em.end()
    return plan


def _draw(plan, kd):
    what, i = plan[kd]
    return f"dr.template pick<INJ>({kd}, T({'Z_' if what == 'z' else 'V_'}[{i}]))"


def _sample_value(em, kind, args, kd, tmp, dname="d", plan=None):
    """Emit `T tmp = <draw of `kind` with args>` (simulate.py:50-60, distributions.py:73-91)."""
    if kind == "wiener":  # rng.normal(0.0, sqrt(d)): 0.0 + sd z
        em(f"const T {tmp} = O::add(T(0.0), O::mul(T(sqrt({dname})), {_draw(plan, kd)}));")
    elif kind == "gaussian":  # rng.normal(mean, sd): mean + sd z
        em(f"const T {tmp}_m = {args[0]}, {tmp}_s = {args[1]};")
        em(f"if (!({tmp}_s > T(0))) perr = true;")
        em(f"const T {tmp} = O::add({tmp}_m, O::mul({tmp}_s, {_draw(plan, kd)}));")
    elif kind == "uniform":  # rng.uniform(lo, hi): lo + (hi - lo) U
        em(f"const T {tmp}_a = {args[0]}, {tmp}_b = {args[1]};")
        em(f"if (!({tmp}_a < {tmp}_b)) perr = true;")
        em(f"const T {tmp} = O::add({tmp}_a, O::mul(O::sub({tmp}_b, {tmp}_a), {_draw(plan, kd)}));")
    elif kind == "truncated_gaussian":  # mean + sd ndtri(fa + u (fb - fa)), distributions.py:78-84
        em(f"const double {tmp}_m = {args[0]}, {tmp}_s = {args[1]}, {tmp}_lo = {args[2]}, {tmp}_hi = {args[3]};")
        em(f"const double {tmp}_fa = normcdf(({tmp}_lo - {tmp}_m) / {tmp}_s), "
           f"{tmp}_fb = normcdf(({tmp}_hi - {tmp}_m) / {tmp}_s);")
        em(f"if (!({tmp}_s > 0.0) || !({tmp}_lo < {tmp}_hi) || !({tmp}_fb - {tmp}_fa > 0.0)) perr = true;")
        em(f"const T {tmp} = T({tmp}_m + {tmp}_s * normcdfinv({tmp}_fa + double({_draw(plan, kd)}) * "
           f"({tmp}_fb - {tmp}_fa)));")
    elif kind == "gamma":  # rng.gamma(shape, scale) = scale * standard_gamma(shape)
        em(f"const double {tmp}_k = {args[0]}, {tmp}_t = {args[1]};")
        em(f"if (!({tmp}_k > 0.0) || !({tmp}_t > 0.0)) perr = true;")
        em(f"const T {tmp} = T({tmp}_t * dr.std_gamma({kd}, {tmp}_k));")
    elif kind == "inverse_gamma":  # 1 / rng.gamma(shape, 1 / scale)
        em(f"const double {tmp}_k = {args[0]}, {tmp}_t = {args[1]};")
        em(f"if (!({tmp}_k > 0.0) || !({tmp}_t > 0.0)) perr = true;")
        em(f"const T {tmp} = T(1.0 / ((1.0 / {tmp}_t) * dr.std_gamma({kd}, {tmp}_k)));")
    else:
        raise UnsupportedModelError(f"cannot sample {kind}")


def _d(e):
    """double-typed argument (truncated/gamma draws compute in float64)"""
    return f"double({cuda_expr(e)})"


def _has_x(e):
    t = e[0]
    if t == "X":
        return True
    if t in ("num", "T", "W", "U"):
        return False
    if t == "neg":
        return _has_x(e[1])
    if t == "bin":
        return _has_x(e[2]) or _has_x(e[3])
    return any(_has_x(a) for a in e[2])


def _sum_terms(e, sign=1):
    """Top-level additive terms of e as (sign, subtree)."""
    if e[0] == "bin" and e[1] in ("+", "-"):
        return _sum_terms(e[2], sign) + _sum_terms(e[3], sign if e[1] == "+" else -sign)
    if e[0] == "neg":
        return _sum_terms(e[1], -sign)
    return [(sign, e)]


def _rebuild(terms):
    out = None
    for sg, t in terms:
        if out is None:
            out = t if sg > 0 else ["neg", t]
        else:
            out = ["bin", "+" if sg > 0 else "-", out, t]
    return out


def _split_invariant(e):
    """(state-dependent part, state-independent part) of an additive expression;
    the second is None when there is nothing to hoist."""
    terms = _sum_terms(e)
    dep = [t for t in terms if _has_x(t[1])]
    inv = [t for t in terms if not _has_x(t[1])]
    if not inv or not dep and len(inv) == 1:
        return None, None
    return _rebuild(dep), _rebuild(inv)


def _emit_statements(em, ops, roles, dname="d"):
    """Statements of a block in order; returns the number of draws used."""
    kinds = [op["kind"] for op in ops if op["op"] == "sample" for _ in op["slots"]]
    plan = _emit_draw_words(em, kinds)
    kd = 0
    for si, op in enumerate(ops):
        if op["op"] == "sample":
            em.block("", f"statement {si}: sample ({op['kind']}) -> {op['role']} {op['slots']}")
            for j, args in enumerate(op["args"]):
                if op["kind"] in ("truncated_gaussian", "gamma", "inverse_gamma"):
                    a = [_d(x) for x in args]
                else:
                    a = [cuda_expr(x) for x in args]
                _sample_value(em, op["kind"], a, kd, f"v{j}", dname, plan)
                kd += 1
            for j, slot in enumerate(op["slots"]):
                em(f"{roles[op['role']]}[{slot}] = v{j};")
            em.end()
        elif op["op"] == "assign":
            em.block("", f"statement {si}: assign -> {op['role']} {op['slots']}")
            for j, ex in enumerate(op["exprs"]):
                em(f"const T v{j} = {cuda_expr(ex)};")
            for j, slot in enumerate(op["slots"]):
                em(f"{roles[op['role']]}[{slot}] = v{j};")
            em.end()
        else:  # ode, simulate.py:71-93
            m = len(op["slots"])
            em.block("", f"statement {si}: ode RK4 h={op['h']!r} over X{op['slots']}")
            em(f"constexpr double H = {_dlit(op['h'])};")
            em(f"const int n_steps = ONE ? 1 : max(1, int(ceil({dname} / H - 1e-9)));")
            # fast mode: the state-independent terms of each derivative (parameters,
            # this sub-step's noise and inputs) summed once per sub-step instead of in
            # every RK4 stage (a reassociation, within the fast path's tolerance)
            split = [_split_invariant(ex) for ex in op["exprs"]]
            for j, (_, inv) in enumerate(split):
                if inv is not None:
                    em(f"T inv{j} = T(0);")
                    em(f"if constexpr (!E) inv{j} = {cuda_expr(inv)};")
            em("auto deriv = [&](const T (&stg)[%d], T (&out)[%d]) {" % (m, m))
            em("  T Xs[NX];")
            em("  for (int i = 0; i < NX; ++i) Xs[i] = X[i];")
            for j, slot in enumerate(op["slots"]):
                em(f"  Xs[{slot}] = stg[{j}];")
            for j, ex in enumerate(op["exprs"]):
                dep, inv = split[j]
                if inv is None:
                    em(f"  out[{j}] = {cuda_expr(ex, 'Xs')};")
                else:
                    em(f"  if constexpr (E) out[{j}] = {cuda_expr(ex, 'Xs')};")
                    fast = f"inv{j}" if dep is None else f"O::add({cuda_expr(dep, 'Xs')}, inv{j})"
                    em(f"  else out[{j}] = {fast};")
            em("};")
            em.block("for (int kk = 0; kk < n_steps; ++kk)")
            em(f"const double s_ = fmin(H, {dname} - double(kk) * H);")
            em("const T s = T(s_);")
            em("const T hs = O::mul(T(0.5), s);  // `0.5 * s * k` == (0.5*s)*k")
            em(f"T y0[{m}], k[{m}], acc[{m}], st[{m}];")
            for j, slot in enumerate(op["slots"]):
                em(f"y0[{j}] = X[{slot}];")
            # y0 + (s/6)(k1 + 2 k2 + 2 k3 + k4) with the sum accumulated as the
            # stages complete: the same operations in the same order (numpy
            # evaluates ((k1 + 2.0*k2) + 2.0*k3) + k4), fewer live registers
            em("deriv(y0, k);")
            em(f"for (int j = 0; j < {m}; ++j) {{ acc[j] = k[j]; st[j] = O::add(y0[j], O::mul(hs, k[j])); }}")
            em("deriv(st, k);")
            em(f"for (int j = 0; j < {m}; ++j) {{ acc[j] = O::add(acc[j], O::mul(T(2.0), k[j])); "
               f"st[j] = O::add(y0[j], O::mul(hs, k[j])); }}")
            em("deriv(st, k);")
            em(f"for (int j = 0; j < {m}; ++j) {{ acc[j] = O::add(acc[j], O::mul(T(2.0), k[j])); "
               f"st[j] = O::add(y0[j], O::mul(s, k[j])); }}")
            em("deriv(st, k);")
            em(f"const T s6 = O::divc(s, T(6.0), {_lit(1.0 / 6.0)});")
            for j, slot in enumerate(op["slots"]):
                em(f"X[{slot}] = O::add(y0[{j}], O::mul(s6, O::add(acc[{j}], k[{j}])));")
            em.end()
            em.end()
    return kd


def _emit_logpdf(em, kind, args, y, tmp):
    """`T tmp` = log-density (distributions.py:94-123); args are expression trees."""
    if kind == "gaussian":
        m, sd = cuda_expr(args[0]), cuda_expr(args[1])
        logsd = _lit(float(np.log(_const_value(args[1])))) if _is_const(args[1]) else f"T(log(double({tmp}_s)))"
        em(f"const T {tmp}_s = {sd};")
        em(f"if (!({tmp}_s > T(0))) perr = true;")
        em(f"const T {tmp}_z = O::div(O::sub({y}, {m}), {tmp}_s);")
        em(f"const T {tmp} = O::sub(O::sub(O::mul(O::mul(T(-0.5), {tmp}_z), {tmp}_z), {logsd}), "
           f"{_lit(LOG_SQRT_2PI)});")
    elif kind == "truncated_gaussian":
        a = [_d(x) for x in args]
        em(f"const double {tmp}_m = {a[0]}, {tmp}_s = {a[1]}, {tmp}_lo = {a[2]}, {tmp}_hi = {a[3]};")
        em(f"const double {tmp}_fa = normcdf(({tmp}_lo - {tmp}_m) / {tmp}_s), "
           f"{tmp}_fb = normcdf(({tmp}_hi - {tmp}_m) / {tmp}_s);")
        em(f"if (!({tmp}_s > 0.0) || !({tmp}_fb - {tmp}_fa > 0.0)) perr = true;")
        em(f"const double {tmp}_z = (double({y}) - {tmp}_m) / {tmp}_s;")
        em(f"const double {tmp}_c = -0.5 * {tmp}_z * {tmp}_z - log({tmp}_s) - {_dlit(LOG_SQRT_2PI)} "
           f"- log({tmp}_fb - {tmp}_fa);")
        em(f"const T {tmp} = (double({y}) >= {tmp}_lo && double({y}) <= {tmp}_hi) ? T({tmp}_c) : T(-CUDART_INF);")
    elif kind == "gamma":
        a = [_d(x) for x in args]
        em(f"const double {tmp}_k = {a[0]}, {tmp}_t = {a[1]}, {tmp}_x = double({y});")
        em(f"if (!({tmp}_k > 0.0) || !({tmp}_t > 0.0)) perr = true;")
        em(f"const T {tmp} = {tmp}_x > 0.0 ? T(((({tmp}_k - 1.0) * log({tmp}_x)) - ({tmp}_x / {tmp}_t)) "
           f"- ({tmp}_k * log({tmp}_t)) - lgamma({tmp}_k)) : T(-CUDART_INF);")
    elif kind == "inverse_gamma":
        a = [_d(x) for x in args]
        em(f"const double {tmp}_k = {a[0]}, {tmp}_t = {a[1]}, {tmp}_x = double({y});")
        em(f"if (!({tmp}_k > 0.0) || !({tmp}_t > 0.0)) perr = true;")
        em(f"const T {tmp} = {tmp}_x > 0.0 ? T((({tmp}_k * log({tmp}_t)) - lgamma({tmp}_k)) "
           f"- (({tmp}_k + 1.0) * log({tmp}_x)) - ({tmp}_t / {tmp}_x)) : T(-CUDART_INF);")
    elif kind == "uniform":
        a = [_d(x) for x in args]
        em(f"const double {tmp}_a = {a[0]}, {tmp}_b = {a[1]}, {tmp}_x = double({y});")
        em(f"if (!({tmp}_a < {tmp}_b)) perr = true;")
        em(f"const T {tmp} = ({tmp}_x >= {tmp}_a && {tmp}_x <= {tmp}_b) ? T(-log({tmp}_b - {tmp}_a)) "
           f": T(-CUDART_INF);")
    else:
        raise UnsupportedModelError(f"observation density {kind}")


_THETA_KINDS = ("gaussian", "uniform", "truncated_gaussian", "gamma", "inverse_gamma")


def _theta_samples(ops):
    """The sample statements of a theta-level block (the walks skip assigns, simulate.py:283-284)."""
    out = []
    for op in ops or ():
        if op["op"] != "sample":
            continue
        out.append(op)
    return out


def theta_supported(desc):
    """True when every theta-level statement samples a kind the device walk has."""
    blocks = theta_walk_blocks(desc) + ("parameter", "initial")
    return all(op["kind"] in _THETA_KINDS for b in blocks for op in _theta_samples(desc.get(b)))


def theta_walk_blocks(desc):
    """(parameter walk block, initial walk block) names: a proposal block, else its
    prior (simulate._walk_proposal's fallback, simulate.py:264-299)."""
    pw = "proposal_parameter" if desc.get("proposal_parameter") is not None else "parameter"
    iw = "proposal_initial" if desc.get("proposal_initial") is not None else "initial"
    return pw, iw


def theta_draw_counts(desc):
    """(draws of the parameter walk, draws of the initial walk): one per sampled slot."""
    pw, iw = theta_walk_blocks(desc)
    return (sum(len(op["slots"]) for op in _theta_samples(desc.get(pw))),
            sum(len(op["slots"]) for op in _theta_samples(desc.get(iw))))


def _emit_theta_walk(em, ops, env, kd0):
    """Sequential-overwrite walk (simulate.py:264-299): every binding's arguments
    are evaluated before the statement writes; then per slot draw (or take
    `to`), add the log-density, write `out` and the environment."""
    kd = kd0
    for si, op in enumerate(_theta_samples(ops)):
        em.block("", f"statement {si}: {op['kind']} -> {op['role']} {op['slots']}")
        for j, args in enumerate(op["args"]):
            em(f"const double a{j}[{len(args)}] = {{{', '.join(cuda_expr(a) for a in args)}}};")
        for j, slot in enumerate(op["slots"]):
            em(f"const double v{j} = to ? to[{slot}] : ssm::th_sample_{op['kind']}(dr, {kd}, a{j}, perr);")
            em(f"logq = __dadd_rn(logq, ssm::th_lp_{op['kind']}(v{j}, a{j}, perr));")
            em(f"out[{slot}] = v{j};")
            em(f"{env}[{slot}] = v{j};")
            kd += 1
        em.end()
    return kd


def _emit_theta_logpdf(em, ops, target):
    """Sum of the block's sample-statement log-densities at `target`
    (parameter_logpdf / initial_logpdf, simulate.py:219-233)."""
    em("double total = 0.0;")
    for si, op in enumerate(_theta_samples(ops)):
        em.block("", f"statement {si}: {op['kind']} {op['slots']}")
        for j, (slot, args) in enumerate(zip(op["slots"], op["args"])):
            em(f"const double a{j}[{len(args)}] = {{{', '.join(cuda_expr(a) for a in args)}}};")
            em(f"total = __dadd_rn(total, ssm::th_lp_{op['kind']}({target}[{slot}], a{j}, perr));")
        em.end()
    em("return total;")


def _emit_theta(em, desc):
    """`struct Theta` of the generated model: the theta-level blocks on the device
    (gen_theta_propose_kernel, ssm_gen_rt.cuh)."""
    c = desc["counts"]
    npar, nx = c["param"], c["state"]
    pw, iw = theta_walk_blocks(desc)
    if not theta_supported(desc):  # stubs: the host keeps these blocks (generic.py)
        em.block("struct Theta")
        em(f"static constexpr int NP = {npar}, NPB = {max(npar, 1)}, NX = {nx}, NXB = {max(nx, 1)}, KP = 0, KI = 0;")
        em("__device__ static void param_walk(const double*, const double*, double*, const ssm::ThetaDraws&, "
           "double&, bool& perr) { perr = true; }")
        em("__device__ static double param_logpdf(const double*, bool& perr) { perr = true; return 0.0; }")
        em("__device__ static void init_walk(const double*, const double*, const double*, double*, "
           "const ssm::ThetaDraws&, double&, bool& perr) { perr = true; }")
        em("__device__ static double init_logpdf(const double*, const double*, bool& perr) { perr = true; return 0.0; }")
        em("__device__ static void init_assign(const double*, double*) {}")
        em.end("};")
        return
    kp, ki = theta_draw_counts(desc)
    init_assigns = [op for op in desc["initial"] if op["op"] == "assign"]
    pre = ["using T = double;", "using O = ssm::Ar<double, true>;", "const double W[1] = {0.0};",
           "const double U[NU] = {};", "(void)W; (void)U;"]
    em.block("struct Theta")
    em(f"static constexpr int NP = {npar}, NPB = {max(npar, 1)}, NX = {nx}, NXB = {max(nx, 1)}, NU = {max(c['input'], 1)}, "
       f"KP = {kp}, KI = {ki};")
    # parameter walk: environment = theta (X zeros)
    em.block("__device__ static void param_walk(const double* from, const double* to, double* out, "
             "const ssm::ThetaDraws& dr, double& logq, bool& perr)", f"walk of `{pw}`")
    em.lines.extend(" " * em.ind + ln for ln in pre)
    em("double TH[NPB];")
    em("const double X[NXB] = {};")
    em("for (int i = 0; i < NP; ++i) TH[i] = out[i] = from[i];")
    em("(void)X; (void)TH; (void)dr; (void)to; (void)logq; (void)perr;")
    _emit_theta_walk(em, desc.get(pw), "TH", 0)
    em.end()
    em.block("__device__ static double param_logpdf(const double* TH, bool& perr)", "parameter_logpdf")
    em.lines.extend(" " * em.ind + ln for ln in pre)
    em("const double X[NXB] = {};")
    em("(void)X; (void)TH; (void)perr;")
    _emit_theta_logpdf(em, desc.get("parameter"), "TH")
    em.end()
    # initial walk: environment = the state (theta = the walk's theta)
    em.block("__device__ static void init_walk(const double* TH, const double* from, const double* to, double* out, "
             "const ssm::ThetaDraws& dr, double& logq, bool& perr)", f"walk of `{iw}`")
    em.lines.extend(" " * em.ind + ln for ln in pre)
    em("double X[NXB];")
    em("for (int i = 0; i < NX; ++i) X[i] = out[i] = from[i];")
    em("(void)TH; (void)X; (void)dr; (void)to; (void)logq; (void)perr;")
    _emit_theta_walk(em, desc.get(iw), "X", kp)
    em.end()
    em.block("__device__ static double init_logpdf(const double* TH, const double* X, bool& perr)", "initial_logpdf")
    em.lines.extend(" " * em.ind + ln for ln in pre)
    em("(void)TH; (void)X; (void)perr;")
    _emit_theta_logpdf(em, desc["initial"], "X")
    em.end()
    em.block("__device__ static void init_assign(const double* TH, double* X)",
             "the initial block's assigns after an x0 proposal")
    em.lines.extend(" " * em.ind + ln for ln in pre)
    em("(void)TH; (void)X;")
    for si, op in enumerate(init_assigns):
        em.block("", f"assign -> {op['slots']}")
        for j, ex in enumerate(op["exprs"]):
            em(f"const double v{j} = {cuda_expr(ex)};")
        for j, slot in enumerate(op["slots"]):
            em(f"X[{slot}] = v{j};")
        em.end()
    em.end()
    em.end("};")


def transition_draws(desc):
    """Per transition sub-step: the draw kinds in kernel order (kd = index)."""
    return [op["kind"] for op in desc["transition"] if op["op"] == "sample" for _ in op["slots"]]


def cuda_source(desc: dict) -> str:
    c = desc["counts"]
    nx, nw = c["state"], c["noise"]
    roles = {"state": "X", "noise": "W", "param": "TH_", "input": "U_"}
    em = _Emitter()
    em.ind = 0
    em(f"// generated by paper_1306_3277_b200/codegen.py from model {desc['name']!r}")
    em('#include "ssm_gen_rt.cuh"')
    em("namespace gen {")
    em("struct Model {")
    em.ind = 2
    kdraw = len(transition_draws(desc))
    em(f"static constexpr int NX = {nx}, NW = {nw}, NWB = {max(nw, 1)}, NU = {max(c['input'], 1)}, "
       f"KDRAW = {max(kdraw, 1)};")
    # transition sub-step
    # ONE: the host guarantees one RK4 step per ode statement (SSM_HINT_SINGLE_SUBSTEP)
    em("template <typename T, bool E, bool INJ, bool ONE = false>")
    em.block("__device__ static void substep(T (&X)[NX], T (&W)[NWB], const double* TH, const double* U, "
             "double d, const ssm::GenDraws<T>& dr, bool& perr)")
    em("using O = ssm::Ar<T, E>;")
    em("(void)W; (void)TH; (void)U; (void)d; (void)dr; (void)perr;")
    for op in desc["transition"]:
        if op["op"] != "ode" and op["role"] not in ("state", "noise"):
            raise UnsupportedModelError(f"transition statement writing a {op['role']} variable")
    _emit_statements(em, desc["transition"], roles)
    em.end()
    # observation
    em("template <typename T, bool E>")
    em.block("__device__ static T obs_logpdf(const T (&X)[NX], const T (&W)[NWB], const double* TH, "
             "const double* U, const double* Y, unsigned mask, bool& perr)")
    em("using O = ssm::Ar<T, E>;")
    em("(void)X; (void)W; (void)TH; (void)U; (void)Y; (void)perr;")
    em("T total = T(0);")
    # fast mode (!E): Gaussian slots with a constant sd accumulate sum(z^2) and the
    # constant terms separately, -z^2/2 folded into one FMA chain (within the fast
    # path's tolerance of the reference order; exact mode keeps the reference order)
    em("T q_fast = T(0), c_fast = T(0);")
    em("(void)q_fast; (void)c_fast;")
    for si, op in enumerate(desc["observation"]):
        for j, (slot, args) in enumerate(zip(op["slots"], op["args"])):
            em.block(f"if (mask & (1u << {slot}))")
            if op["kind"] == "gaussian" and _is_const(args[1]) and _const_value(args[1]) > 0:
                sd = _const_value(args[1])
                em.block("if constexpr (!E)")
                em(f"const T z = (T(Y[{slot}]) - {cuda_expr(args[0])}) * {_lit(1.0 / sd)};")
                em("q_fast = fma(z, z, q_fast);")
                em(f"c_fast += {_lit(float(np.log(sd)) + LOG_SQRT_2PI)};")
                em.end()
                em.block("else")
                _emit_logpdf(em, op["kind"], args, f"T(Y[{slot}])", f"g{si}_{j}")
                em(f"total = O::add(total, g{si}_{j});")
                em.end()
            else:
                _emit_logpdf(em, op["kind"], args, f"T(Y[{slot}])", f"g{si}_{j}")
                em(f"total = O::add(total, g{si}_{j});")
            em.end()
    em("if constexpr (!E) total += fma(T(-0.5), q_fast, -c_fast);")
    em("return total;")
    em.end()
    # initial block
    em("template <typename T, bool E, bool INJ>")
    em.block("__device__ static void initial(T (&X)[NX], const double* TH, const ssm::GenDraws<T>& dr, bool& perr)")
    em("using O = ssm::Ar<T, E>;")
    em("(void)TH; (void)dr; (void)perr;")
    em("T W[NWB] = {};")
    em("const double U[NU] = {};")
    em("(void)W; (void)U;")
    for op in desc["initial"]:
        if op["op"] == "ode" or op["role"] != "state":
            raise UnsupportedModelError("initial block: state sample/assign statements only")
    _emit_statements(em, desc["initial"], roles)
    em.end()
    _emit_theta(em, desc)
    em.ind = 0
    em("};")
    em("}  // namespace gen")
    kp, ki = theta_draw_counts(desc)
    em(f'extern "C" __device__ int ssm_gen_model_info[4] = {{{nx}, {max(kdraw, 1)}, {kp}, {ki}}};')
    return "\n".join(em.lines) + "\n"


def include_dir() -> str:
    return os.path.join(os.path.dirname(os.path.abspath(__file__)), "csrc")


def source_digest(src: str) -> str:
    return hashlib.sha256(src.encode()).hexdigest()[:16]


def dumps(desc) -> str:
    return json.dumps(desc, sort_keys=True)
