"""Expression language of the dynamics / predicates, plus CUDA lowering.

The grammar and evaluation semantics follow pkg/src/impact/expr.py (EBNF at
:9-24, tokenizer :55-81, parser :396-525, function table :40-53): `^` binds
tighter than unary minus, which binds tighter than `*`/`/`, then `+`/`-`;
`^` is right-associative.  Host evaluation uses the same numpy ufuncs in the
same tree order, so x-free subtrees folded on the host are bitwise the
reference's values.

What is new here is `lower_dynamics()`: it splits every dynamics expression
into x-free subtrees (evaluated on the host per (input, disturbance) pair, with
numpy, exactly as the reference would) and an x-dependent residual that is
emitted as CUDA C in the same association order.  The construction kernels
are JIT-compiled (NVRTC, --fmad=false) around that residual.

AST nodes are plain tuples:
  ("num", v) ("var", name) ("neg", a) ("bin", op, a, b) ("call", f, args)
  ("cmp", op, a, b) ("and", a, b) ("or", a, b) ("not", a)
"""

import re
from dataclasses import dataclass

import numpy as np

from .errors import EvalError, ParseError

__all__ = ["Expr", "PredicateExpr", "DynamicsSpec", "parse_expression",
           "parse_predicate", "parse_density", "lower_dynamics"]

_UNARY = {"sin": np.sin, "cos": np.cos, "tan": np.tan, "atan": np.arctan,
          "asin": np.arcsin, "acos": np.arccos, "sqrt": np.sqrt,
          "exp": np.exp, "log": np.log, "abs": np.abs}
_BINARY = {"min": np.minimum, "max": np.maximum}
_ARITY = {**{k: 1 for k in _UNARY}, **{k: 2 for k in _BINARY}}
_ARITH = {"+": np.add, "-": np.subtract, "*": np.multiply,
          "/": np.true_divide, "^": np.power}
_COMPARE = {"<=": np.less_equal, ">=": np.greater_equal, "<": np.less,
            ">": np.greater, "==": np.equal}

_LEX = re.compile(r"\s*(?:(?P<num>(?:\d+\.\d*|\.\d+|\d+)(?:[eE][+-]?\d+)?)"
                  r"|(?P<name>[A-Za-z_]\w*)|(?P<cmp><=|>=|==|<|>)"
                  r"|(?P<sym>[-+*/^&|!(),]))")


def _lex(text):
    out, pos = [], 0
    while pos < len(text):
        if text[pos].isspace():
            pos += 1
            continue
        m = _LEX.match(text, pos)
        if m is None or m.lastgroup is None:
            raise ParseError(f"unexpected character {text[pos]!r}", offset=pos)
        kind = m.lastgroup
        val = m.group(kind)
        start = m.start(kind)
        out.append((kind if kind != "sym" else val, val, start))
        pos = m.end()
    out.append(("end", "", len(text)))
    return out


class _Parser:
    """Recursive descent over the token list; one method per grammar rule."""

    def __init__(self, text, names):
        self.toks = _lex(text)
        self.pos = 0
        self.names = names

    @property
    def tok(self):
        return self.toks[self.pos]

    def take(self, kind=None):
        t = self.toks[self.pos]
        if kind is not None and t[0] != kind:
            raise ParseError(f"expected {kind!r}, found {t[1]!r}", offset=t[2])
        self.pos += 1
        return t

    def error(self, what):
        t = self.tok
        found = repr(t[1]) if t[1] else "end of input"
        raise ParseError(f"{what}, found {found}", offset=t[2])

    def finish(self, node):
        if self.tok[0] != "end":
            self.error("trailing input")
        return node

    # arithmetic
    def sum(self):
        node = self.product()
        while self.tok[0] in ("+", "-"):
            op = self.take()[0]
            node = ("bin", op, node, self.product())
        return node

    def product(self):
        node = self.unary()
        while self.tok[0] in ("*", "/"):
            op = self.take()[0]
            node = ("bin", op, node, self.unary())
        return node

    def unary(self):
        if self.tok[0] == "-":
            self.take()
            return ("neg", self.unary())
        node = self.atom()
        if self.tok[0] == "^":
            self.take()
            node = ("bin", "^", node, self.unary())
        return node

    def atom(self):
        kind, val, off = self.tok
        if kind == "num":
            self.take()
            return ("num", float(val))
        if kind == "name":
            self.take()
            if val in _ARITY:
                self.take("(")
                args = [self.sum()]
                while self.tok[0] == ",":
                    self.take()
                    args.append(self.sum())
                self.take(")")
                if len(args) != _ARITY[val]:
                    raise ParseError(f"{val} takes {_ARITY[val]} argument(s), "
                                     f"got {len(args)}", offset=off)
                return ("call", val, tuple(args))
            if val not in self.names:
                raise ParseError(f"unknown identifier {val!r}", offset=off)
            return ("var", val)
        if kind == "(":
            self.take()
            node = self.sum()
            self.take(")")
            return node
        self.error("expected a number, identifier or '('")

    # boolean layer
    def disj(self):
        node = self.conj()
        while self.tok[0] == "|":
            self.take()
            node = ("or", node, self.conj())
        return node

    def conj(self):
        node = self.neg()
        while self.tok[0] == "&":
            self.take()
            node = ("and", node, self.neg())
        return node

    def neg(self):
        if self.tok[0] == "!":
            self.take()
            return ("not", self.neg())
        if self.tok[0] == "(":
            # '(' may open a boolean group or arithmetic; try boolean first
            mark = self.pos
            try:
                self.take()
                node = self.disj()
                self.take(")")
                if self.tok[0] not in ("cmp", "+", "-", "*", "/", "^"):
                    return node
            except ParseError:
                pass
            self.pos = mark
        left = self.sum()
        if self.tok[0] != "cmp":
            self.error("expected a comparison operator")
        op = self.take()[1]
        return ("cmp", op, left, self.sum())


def _names(**limits):
    return {f"{p}{i + 1}" for p, n in limits.items() for i in range(n)}


def _eval(node, env):
    tag = node[0]
    if tag == "num":
        return node[1]
    if tag == "var":
        return env[node[1]]
    if tag == "neg":
        return -_eval(node[1], env)
    if tag == "bin":
        return _ARITH[node[1]](_eval(node[2], env), _eval(node[3], env))
    if tag == "call":
        args = [_eval(a, env) for a in node[2]]
        fn = _UNARY.get(node[1]) or _BINARY[node[1]]
        return fn(*args)
    if tag == "cmp":
        return _COMPARE[node[1]](_eval(node[2], env), _eval(node[3], env))
    if tag == "and":
        return np.logical_and(_eval(node[1], env), _eval(node[2], env))
    if tag == "or":
        return np.logical_or(_eval(node[1], env), _eval(node[2], env))
    if tag == "not":
        return np.logical_not(_eval(node[1], env))
    raise ValueError(tag)


def _vars(node, out):
    tag = node[0]
    if tag == "var":
        out.add(node[1])
    elif tag == "call":
        for a in node[2]:
            _vars(a, out)
    elif tag in ("neg", "not"):
        _vars(node[1], out)
    elif tag in ("bin", "cmp"):
        _vars(node[2], out)
        _vars(node[3], out)
    elif tag in ("and", "or"):
        _vars(node[1], out)
        _vars(node[2], out)
    return out


def _text(node):
    tag = node[0]
    if tag == "num":
        return repr(node[1])
    if tag == "var":
        return node[1]
    if tag == "neg":
        return f"(-{_text(node[1])})"
    if tag == "not":
        return f"(!{_text(node[1])})"
    if tag == "call":
        return f"{node[1]}({', '.join(_text(a) for a in node[2])})"
    if tag in ("bin", "cmp"):
        return f"({_text(node[2])} {node[1]} {_text(node[3])})"
    return f"({_text(node[1])} {'&' if tag == 'and' else '|'} {_text(node[2])})"


class Expr:
    """Parsed arithmetic expression, numpy-vectorized evaluation."""

    def __init__(self, node, allowed):
        self.node = node
        self.allowed = frozenset(allowed)

    def evaluate_env(self, env):
        with np.errstate(all="ignore"):
            return _eval(self.node, env)

    def evaluate(self, env):
        out = self.evaluate_env(env)
        if not np.all(np.isfinite(out)):
            raise EvalError(f"domain error evaluating {self.unparse()!r}")
        return out

    def variables(self):
        return _vars(self.node, set())

    def unparse(self):
        return _text(self.node)

    def __eq__(self, other):
        return isinstance(other, Expr) and self.node == other.node

    def __hash__(self):
        return hash(self.node)

    def __repr__(self):
        return f"Expr({self.unparse()})"


class PredicateExpr(Expr):
    """Boolean expression over x1..xn."""

    def evaluate(self, x):
        x = np.asarray(x, dtype=float)
        env = {f"x{d + 1}": x[d] for d in range(len(x))}
        try:
            return bool(self.evaluate_env(env))
        except KeyError as exc:
            raise EvalError(f"unbound variable {exc} at point {x.tolist()}")

    def __repr__(self):
        return f"PredicateExpr({self.unparse()})"


def parse_expression(text, dims) -> Expr:
    n, m, p = dims
    names = _names(x=n, u=m, w=p)
    par = _Parser(text, names)
    return Expr(par.finish(par.sum()), names)


def parse_density(text, n) -> Expr:
    names = _names(y=n, m=n)
    par = _Parser(text, names)
    return Expr(par.finish(par.sum()), names)


def parse_predicate(text, n) -> PredicateExpr:
    names = _names(x=n)
    par = _Parser(text, names)
    return PredicateExpr(par.finish(par.disj()), names)


@dataclass(frozen=True)
class DynamicsSpec:
    """Next-state mean f(x, u, w), one expression per state coordinate."""

    exprs: tuple
    dims: tuple  # (n, m, p)

    def __post_init__(self):
        if len(self.exprs) != self.dims[0]:
            raise ParseError(f"need {self.dims[0]} dynamics expressions, "
                             f"got {len(self.exprs)}")

    def _env(self, x, u, w):
        n, m, p = self.dims
        x, u, w = (np.asarray(v, dtype=float) for v in (x, u, w))
        if (len(x), len(u), len(w)) != (n, m, p):
            raise EvalError(f"dimension mismatch: expected {self.dims}, "
                            f"got ({len(x)}, {len(u)}, {len(w)})")
        env = {f"x{d + 1}": x[d] for d in range(n)}
        env.update({f"u{d + 1}": u[d] for d in range(m)})
        env.update({f"w{d + 1}": w[d] for d in range(p)})
        return env

    def eval(self, x, u=(), w=()):
        env = self._env(x, u, w)
        return np.array([float(e.evaluate(env)) for e in self.exprs])

    def eval_env(self, env):
        return [e.evaluate_env(env) for e in self.exprs]

    def state_dependencies(self, d):
        return {int(v[1:]) - 1 for v in self.exprs[d].variables()
                if v.startswith("x")}

    def is_separable(self):
        return all(self.state_dependencies(d) <= {d}
                   for d in range(self.dims[0]))


# --- CUDA lowering ------------------------------------------------------

_CUDA_FN = {"sin": "sin", "cos": "cos", "tan": "tan", "atan": "atan",
            "asin": "asin", "acos": "acos", "sqrt": "sqrt", "exp": "exp",
            "log": "log", "abs": "fabs", "min": "imp_min", "max": "imp_max"}


@dataclass
class LoweredDynamics:
    """Output of lower_dynamics().

    source     CUDA C device functions `imp_f<d>(const double* x, const double* k)`
               and `imp_f_all(x, k, out)`; k = folded constants of one row.
    n_consts   folded constants per (input, disturbance) pair
    consts     (n_u * n_w, n_consts) float64 table, row-major (j, i)
    deps       per-dimension sorted state dependencies
    """
    source: str
    n_consts: int
    consts: np.ndarray
    deps: list


def lower_dynamics(dyn: DynamicsSpec, input_reps, disturb_reps):
    """Fold every x-free subtree on the host (numpy, reference evaluation
    order) and emit the x-dependent residual as CUDA C."""
    folded = []          # list of subtree nodes, index = constant slot
    slot_of = {}

    def fold(node):
        if node not in slot_of:
            slot_of[node] = len(folded)
            folded.append(node)
        return f"k[{slot_of[node]}]"

    def xfree(node):
        return not any(v.startswith("x") for v in _vars(node, set()))

    def emit(node):
        if xfree(node):
            return fold(node)
        tag = node[0]
        if tag == "var":
            return f"x[{int(node[1][1:]) - 1}]"
        if tag == "neg":
            return f"(-{emit(node[1])})"
        if tag == "bin":
            a, b = emit(node[2]), emit(node[3])
            if node[1] == "^":
                return f"pow({a}, {b})"
            if node[1] == "/":
                return _emit_div(a, b, node[3], fold, xfree)
            return f"({a} {node[1]} {b})"
        if tag == "call":
            return f"{_CUDA_FN[node[1]]}({', '.join(emit(a) for a in node[2])})"
        raise ValueError(f"cannot lower {tag}")

    bodies = [emit(e.node) for e in dyn.exprs]
    n = dyn.dims[0]
    lines = []
    for d, body in enumerate(bodies):
        lines.append(f"__device__ __forceinline__ double imp_f{d}("
                     f"const double* x, const double* k) {{ return {body}; }}")
    lines.append("__device__ __forceinline__ double imp_fd(int d, "
                 "const double* x, const double* k) {")
    lines.append("  switch (d) {")
    for d in range(n):
        lines.append(f"    case {d}: return imp_f{d}(x, k);")
    lines.append("  }\n  return 0.0;\n}")
    lines += _emit_all(dyn, fold, xfree)
    src = "\n".join(lines) + "\n"

    n_u, n_w = len(input_reps), len(disturb_reps)
    consts = np.zeros((n_u * n_w, max(len(folded), 1)))
    _, m, p = dyn.dims
    for j in range(n_u):
        for i in range(n_w):
            env = {f"u{q + 1}": input_reps[j][q] for q in range(m)}
            env.update({f"w{q + 1}": disturb_reps[i][q] for q in range(p)})
            with np.errstate(all="ignore"):
                for c, node in enumerate(folded):
                    if node[0] == "rcp":
                        consts[j * n_w + i, c] = _rcp(float(_eval(node[1], env)))
                    else:
                        consts[j * n_w + i, c] = float(_eval(node, env))
    deps = [sorted(dyn.state_dependencies(d)) for d in range(n)]
    return LoweredDynamics(source=src, n_consts=len(folded), consts=consts,
                           deps=deps)


def lower_density(expr, n):
    """CUDA C of a custom noise density (noise.py:76-95, CustomNoise.density)
    over one integration point y[0..n) and the mean m[0..n):
    `__device__ double imp_density(const double* y, const double* m)`.
    Same AST order as numpy's elementwise evaluation; number literals as
    exact hex floats; exp is the glibc restatement (imp_exp)."""
    fns = dict(_CUDA_FN, exp="imp_exp")

    def emit(node):
        tag = node[0]
        if tag == "num":
            return f"({float(node[1]).hex()})"
        if tag == "var":
            name = node[1]
            return f"{'y' if name[0] == 'y' else 'm'}[{int(name[1:]) - 1}]"
        if tag == "neg":
            return f"(-{emit(node[1])})"
        if tag == "bin":
            a, b = emit(node[2]), emit(node[3])
            if node[1] == "^":
                return f"pow({a}, {b})"
            if node[1] == "/":
                return f"imp_div({a}, {b})"
            return f"({a} {node[1]} {b})"
        if tag == "call":
            return f"{fns[node[1]]}({', '.join(emit(a) for a in node[2])})"
        raise ValueError(f"cannot lower {tag}")

    del n
    return ("__device__ __forceinline__ double imp_density(const double* y, "
            f"const double* m) {{ return {emit(expr.node)}; }}\n")


def _rcp(v):
    """RN(1/v) for imp_div_rcp; NaN outside 2^+-100 (device then divides)."""
    return 1.0 / v if 2.0 ** -100 <= abs(v) <= 2.0 ** 100 else float("nan")


def _emit_div(a, b, bnode, fold, xfree):
    """a / b as CUDA C, IEEE-exact: by a folded reciprocal when the divisor
    is x-free (imp_div_rcp, no divide), else imp_div (ndtr.h)."""
    if xfree(bnode):
        return f"imp_div_rcp({a}, {b}, {fold(('rcp', bnode))})"
    return f"imp_div({a}, {b})"


def _emit_all(dyn, fold, xfree):
    """imp_f_all(x, k, f): every f_d at once, identical x-dependent
    subtrees computed once (common-subexpression elimination) and sin/cos
    of one argument fused into sincos().  Evaluation order and rounding of
    each subtree are unchanged, so values equal imp_f<d>'s."""
    from collections import Counter
    seen = Counter()

    def count(node):
        if xfree(node) or node[0] == "var":
            return
        seen[node] += 1
        if seen[node] > 1:
            return
        kids = {"neg": lambda n: [n[1]], "bin": lambda n: [n[2], n[3]],
                "call": lambda n: list(n[2])}[node[0]](node)
        for c in kids:
            count(c)

    for e in dyn.exprs:
        count(e.node)
    trig_args = {}
    for node in seen:
        if node[0] == "call" and node[1] in ("sin", "cos"):
            trig_args.setdefault(node[2][0], set()).add(node[1])
    paired = {a for a, fns in trig_args.items() if fns == {"sin", "cos"}}
    body, memo, sc = [], {}, {}

    def gen(node):
        if xfree(node):
            return fold(node)
        if node in memo:
            return memo[node]
        tag = node[0]
        if tag == "var":
            return f"x[{int(node[1][1:]) - 1}]"
        if tag == "call" and node[1] in ("sin", "cos") and node[2][0] in paired:
            arg = node[2][0]
            if arg not in sc:
                a = gen(arg)
                q = len(sc)
                body.append(f"  double s{q}, c{q};\n  sincos({a}, &s{q}, &c{q});")
                sc[arg] = q
            name = f"{'s' if node[1] == 'sin' else 'c'}{sc[arg]}"
            memo[node] = name
            return name
        if tag == "neg":
            s = f"(-{gen(node[1])})"
        elif tag == "bin":
            a, b = gen(node[2]), gen(node[3])
            if node[1] == "^":
                s = f"pow({a}, {b})"
            elif node[1] == "/":
                s = _emit_div(a, b, node[3], fold, xfree)
            else:
                s = f"({a} {node[1]} {b})"
        else:
            s = f"{_CUDA_FN[node[1]]}({', '.join(gen(a) for a in node[2])})"
        if seen[node] > 1 or tag == "call":
            t = f"t{len(memo)}"
            body.append(f"  const double {t} = {s};")
            memo[node] = t
            return t
        return s

    outs = [gen(e.node) for e in dyn.exprs]
    lines = ["__device__ __forceinline__ void imp_f_all(const double* x, "
             "const double* k, double* f) {"]
    lines += body
    lines += [f"  f[{d}] = {o};" for d, o in enumerate(outs)]
    lines.append("}")
    return lines


def has_x_transcendental(dyn: DynamicsSpec) -> bool:
    """True when some f_d applies a library function (sin, exp, ...) or a
    power to an x-dependent argument.  Those calls are CUDA's on the device
    and numpy's (SIMD) in the reference, so construction parity for such
    dynamics is tolerance-level instead of bitwise (parity)."""
    def walk(node):
        tag = node[0]
        if tag == "call":
            if any(v.startswith("x") for v in _vars(node, set())):
                return True
            return any(walk(a) for a in node[2])
        if tag == "bin":
            if node[1] == "^" and any(v.startswith("x")
                                      for v in _vars(node, set())):
                return True
            return walk(node[2]) or walk(node[3])
        if tag == "neg":
            return walk(node[1])
        return False
    return any(walk(e.node) for e in dyn.exprs)
