"""ktune-compatible configuration spaces (the autotuner-config API the north star keeps).

Same file format, value semantics, enumeration order and SHA-256 digests as the reference's
``ktune.configspace`` / ``ktune.expr`` (ref/pkg/src/ktune/configspace.py:39-45 canonical JSON +
digest; :58-205 the five domain kinds; :244-274 the space digest over
{name, params, canonical constraint texts}; :293-331 KernelConfig / ShapeKey digests; :375-396 lazy
enumeration in declared order; :408-440 validation) and constraint language
(ref/pkg/src/ktune/expr.py:1-19: ``+ - * / %`` with C truncating division, comparisons,
``&& || !`` short-circuit, booleans never coerce; canonical printing fully parenthesised,
ref/pkg/src/ktune/expr.py:196-203).  Digest equality with the reference is pinned by
tests/test_configspace.py against committed digests of the shipped fixtures.

Implementation is independent: a binding-power (Pratt) parser over tuple ASTs, and constraints
compiled once into Python closures so enumerating the 1600-point flash-attention grid is cheap.
"""

from __future__ import annotations

import hashlib
import itertools
import json
import re
from dataclasses import dataclass, field
from typing import Callable, Iterator

KINDS = ("int-list", "int-range", "pow2-range", "categorical", "boolean")
_IDENT = re.compile(r"[A-Za-z_][A-Za-z0-9_]*\Z")


class SpaceError(ValueError):
    """Malformed space document / constraint (with a location)."""

    def __init__(self, message: str, where: str = ""):
        self.message, self.where = message, where
        super().__init__(f"{where}: {message}" if where else message)


class ConstraintEvalError(ValueError):
    """Runtime failure inside a constraint (division by zero, type mix)."""


def canonical_json(obj) -> str:
    return json.dumps(obj, sort_keys=True, separators=(",", ":"))


def digest_of(obj) -> str:
    return hashlib.sha256(canonical_json(obj).encode("utf-8")).hexdigest()


def _strict_int(v) -> bool:
    return isinstance(v, int) and not isinstance(v, bool)


# ----------------------------------------------------------------------------- expressions
_TOK = re.compile(r"\s*(?:(\d+)|([A-Za-z_][A-Za-z0-9_]*)|(\|\||&&|==|!=|<=|>=|[-+*/%<>!()]))")
# binary operator -> binding power (all six comparisons share one level, left-assoc)
_BP = {"||": 1, "&&": 2, "==": 3, "!=": 3, "<": 3, "<=": 3, ">": 3, ">=": 3, "+": 4, "-": 4, "*": 5, "/": 5,
       "%": 5}
_PREFIX_BP = 6


def _lex(text: str):
    out, i, n = [], 0, len(text)
    while True:
        while i < n and text[i].isspace():
            i += 1
        if i >= n:
            out.append(("end", "", n))
            return out
        m = _TOK.match(text, i)
        if not m or m.end() == i:
            raise SpaceError(f"unexpected character {text[i]!r} at {i}")
        start = m.start(m.lastindex)
        kind = ("int", "name", "op")[m.lastindex - 1]
        out.append((kind, m.group(m.lastindex), start))
        i = m.end()


def parse_expr(text: str):
    """Constraint text -> AST: ('lit', int) | ('ref', name) | ('un', op, x) | ('bin', op, a, b)."""
    toks = _lex(text)
    pos = [0]

    def peek():
        return toks[pos[0]]

    def take():
        t = toks[pos[0]]
        pos[0] += 1
        return t

    def nud():
        kind, txt, at = take()
        if kind == "int":
            return ("lit", int(txt))
        if kind == "name":
            return ("ref", txt)
        if kind == "op" and txt in ("!", "-"):
            return ("un", txt, expr(_PREFIX_BP))
        if kind == "op" and txt == "(":
            inner = expr(0)
            k2, t2, a2 = take()
            if t2 != ")":
                raise SpaceError(f"expected ')' at {a2}, found {t2 or 'end of input'!r}")
            return inner
        raise SpaceError(f"expected a value at {at}, found {txt or 'end of input'!r}")

    def expr(min_bp):
        lhs = nud()
        while True:
            kind, txt, _ = peek()
            bp = _BP.get(txt) if kind == "op" else None
            if bp is None or bp <= min_bp:
                return lhs
            take()
            lhs = ("bin", txt, lhs, expr(bp))

    tree = expr(0)
    kind, txt, at = peek()
    if kind != "end":
        raise SpaceError(f"unexpected trailing input {txt!r} at {at}")
    return tree


def canonical_text(node) -> str:
    tag = node[0]
    if tag == "lit":
        return str(node[1])
    if tag == "ref":
        return node[1]
    if tag == "un":
        return f"({node[1]}{canonical_text(node[2])})"
    return f"({canonical_text(node[2])} {node[1]} {canonical_text(node[3])})"


def names_in(node) -> set:
    tag = node[0]
    if tag == "lit":
        return set()
    if tag == "ref":
        return {node[1]}
    if tag == "un":
        return names_in(node[2])
    return names_in(node[2]) | names_in(node[3])


def type_of(node, types: dict) -> str:
    """Static type ('int' | 'bool' | 'str') under parameter types; raises SpaceError."""
    tag = node[0]
    if tag == "lit":
        return "int"
    if tag == "ref":
        if node[1] not in types:
            raise SpaceError(f"unknown parameter {node[1]!r}")
        return types[node[1]]
    if tag == "un":
        t = type_of(node[2], types)
        want = "bool" if node[1] == "!" else "int"
        if t != want:
            raise SpaceError(f"{node[1]!r} needs a {want} operand, got {t}")
        return want
    op, a, b = node[1], type_of(node[2], types), type_of(node[3], types)
    if op in ("+", "-", "*", "/", "%", "<", "<=", ">", ">="):
        if a != "int" or b != "int":
            raise SpaceError(f"{op!r} needs integer operands, got {a} and {b}")
        return "int" if op in "+-*/%" else "bool"
    if op in ("==", "!="):
        if a != b:
            raise SpaceError(f"{op!r} needs operands of one type, got {a} and {b}")
        return "bool"
    if a != "bool" or b != "bool":
        raise SpaceError(f"{op!r} needs boolean operands, got {a} and {b}")
    return "bool"


def _cdiv(a: int, b: int) -> int:
    if b == 0:
        raise ConstraintEvalError(f"division by zero: {a} / 0")
    q = abs(a) // abs(b)
    return q if (a < 0) == (b < 0) else -q


def _cmod(a: int, b: int) -> int:
    if b == 0:
        raise ConstraintEvalError(f"modulo by zero: {a} % 0")
    return a - b * _cdiv(a, b)


def _need_int(v):
    if not _strict_int(v):
        raise ConstraintEvalError(f"expected an integer, got {v!r}")
    return v


def _need_bool(v):
    if not isinstance(v, bool):
        raise ConstraintEvalError(f"expected a boolean, got {v!r}")
    return v


_ARITH = {"+": lambda a, b: a + b, "-": lambda a, b: a - b, "*": lambda a, b: a * b, "/": _cdiv, "%": _cmod}
_CMP = {"<": lambda a, b: a < b, "<=": lambda a, b: a <= b, ">": lambda a, b: a > b, ">=": lambda a, b: a >= b}


def compile_expr(node) -> Callable[[dict], object]:
    tag = node[0]
    if tag == "lit":
        v = node[1]
        return lambda env: v
    if tag == "ref":
        name = node[1]

        def ref(env):
            try:
                return env[name]
            except KeyError:
                raise ConstraintEvalError(f"unknown name {name!r}") from None

        return ref
    if tag == "un":
        f = compile_expr(node[2])
        if node[1] == "!":
            return lambda env: not _need_bool(f(env))
        return lambda env: -_need_int(f(env))
    op, fa, fb = node[1], compile_expr(node[2]), compile_expr(node[3])
    if op == "&&":
        return lambda env: _need_bool(fa(env)) and _need_bool(fb(env))
    if op == "||":
        return lambda env: _need_bool(fa(env)) or _need_bool(fb(env))
    if op in _ARITH:
        g = _ARITH[op]
        return lambda env: g(_need_int(fa(env)), _need_int(fb(env)))
    if op in _CMP:
        g = _CMP[op]
        return lambda env: g(_need_int(fa(env)), _need_int(fb(env)))

    def eq(env):
        a, b = fa(env), fb(env)
        if type(a) is not type(b):
            raise ConstraintEvalError(f"{op!r} needs operands of one type, got {a!r} and {b!r}")
        return (a == b) if op == "==" else (a != b)

    return eq


# ----------------------------------------------------------------------------- domain types
@dataclass(frozen=True)
class ParamDomain:
    name: str
    kind: str
    values: tuple = ()
    lo: int | None = None
    hi: int | None = None
    step: int = 1

    def __post_init__(self):
        where = f"param {self.name!r}"
        if not isinstance(self.name, str) or not _IDENT.match(self.name):
            raise SpaceError(f"invalid parameter name {self.name!r}", "param")
        if self.kind not in KINDS:
            raise SpaceError(f"unknown kind {self.kind!r}", where)
        if self.kind in ("int-list", "categorical"):
            ok = _strict_int if self.kind == "int-list" else (lambda v: isinstance(v, str))
            if not self.values:
                raise SpaceError("empty domain", where)
            bad = [v for v in self.values if not ok(v)]
            if bad:
                raise SpaceError(f"bad domain value {bad[0]!r}", where)
            if len(set(self.values)) != len(self.values):
                raise SpaceError("duplicate values in domain", where)
        elif self.kind in ("int-range", "pow2-range"):
            if not (_strict_int(self.lo) and _strict_int(self.hi)):
                raise SpaceError(f"lo/hi must be integers, got {self.lo!r}, {self.hi!r}", where)
            if self.lo > self.hi:
                raise SpaceError(f"lo {self.lo} > hi {self.hi}", where)
            if self.kind == "int-range" and (not _strict_int(self.step) or self.step < 1):
                raise SpaceError(f"step must be >= 1, got {self.step!r}", where)
            if self.kind == "pow2-range" and not all(x > 0 and x & (x - 1) == 0 for x in (self.lo, self.hi)):
                raise SpaceError(f"lo and hi must be powers of two, got {self.lo}, {self.hi}", where)

    def domain_values(self) -> tuple:
        if self.kind in ("int-list", "categorical"):
            return tuple(self.values)
        if self.kind == "int-range":
            return tuple(range(self.lo, self.hi + 1, self.step))
        if self.kind == "pow2-range":
            return tuple(1 << e for e in range(self.lo.bit_length() - 1, self.hi.bit_length()))
        return (False, True)

    def value_type(self) -> str:
        return {"boolean": "bool", "categorical": "str"}.get(self.kind, "int")

    def contains(self, v) -> bool:
        t = self.value_type()
        typed = isinstance(v, bool) if t == "bool" else (isinstance(v, str) if t == "str" else _strict_int(v))
        return typed and v in self.domain_values()

    def to_json_dict(self) -> dict:
        d = {"name": self.name, "kind": self.kind}
        if self.kind in ("int-list", "categorical"):
            d["values"] = list(self.values)
        elif self.kind == "int-range":
            d.update(lo=self.lo, hi=self.hi, step=self.step)
        elif self.kind == "pow2-range":
            d.update(lo=self.lo, hi=self.hi)
        return d

    @classmethod
    def from_json_dict(cls, d, where: str) -> "ParamDomain":
        if not isinstance(d, dict):
            raise SpaceError(f"expected an object, got {d!r}", where)
        extra = set(d) - {"name", "kind", "values", "lo", "hi", "step"}
        if extra:
            raise SpaceError(f"unknown keys {sorted(extra)}", where)
        kind = d.get("kind")
        if kind in ("int-list", "categorical") and not isinstance(d.get("values"), list):
            raise SpaceError("missing 'values' array", where)
        return cls(d.get("name"), kind, values=tuple(d.get("values", ())), lo=d.get("lo"), hi=d.get("hi"),
                   step=d.get("step", 1))


@dataclass(frozen=True)
class Constraint:
    text: str
    tree: tuple = field(compare=False)
    canonical: str = ""
    fn: Callable = field(compare=False, default=None, repr=False)

    @classmethod
    def parse(cls, text: str) -> "Constraint":
        tree = parse_expr(text)
        return cls(text, tree, canonical_text(tree), compile_expr(tree))

    def holds(self, env: dict) -> bool:
        return bool(self.fn(env))


@dataclass(frozen=True)
class ConfigSpace:
    name: str
    params: tuple
    constraints: tuple
    digest: str

    @classmethod
    def build(cls, name: str, params, constraints=()) -> "ConfigSpace":
        params, constraints = tuple(params), tuple(constraints)
        if not isinstance(name, str) or not _IDENT.match(name):
            raise SpaceError(f"invalid space name {name!r}", "name")
        names = [p.name for p in params]
        dup = [n for n in names if names.count(n) > 1]
        if dup:
            raise SpaceError(f"duplicate parameter name {dup[0]!r}", "params")
        types = {p.name: p.value_type() for p in params}
        for i, c in enumerate(constraints):
            where = f"constraints[{i}] ({c.text!r})"
            unknown = sorted(names_in(c.tree) - set(names))
            if unknown:
                raise SpaceError(f"unknown parameter {unknown[0]!r}", where)
            try:
                t = type_of(c.tree, types)
            except SpaceError as e:
                raise SpaceError(e.message, where) from None
            if t != "bool":
                raise SpaceError(f"expression has type {t}, expected bool", where)
        doc = {"name": name, "params": [p.to_json_dict() for p in params],
               "constraints": [c.canonical for c in constraints]}
        return cls(name, params, constraints, digest_of(doc))

    def param_names(self) -> tuple:
        return tuple(p.name for p in self.params)


@dataclass(frozen=True)
class KernelConfig:
    assignments: dict
    digest: str

    @classmethod
    def from_assignments(cls, assignments: dict) -> "KernelConfig":
        a = dict(assignments)
        return cls(a, digest_of(a))


@dataclass(frozen=True)
class ShapeKey:
    dims: dict
    digest: str

    @classmethod
    def from_dims(cls, dims: dict) -> "ShapeKey":
        if not dims:
            raise SpaceError("shape must have at least one dimension", "shape")
        for k, v in dims.items():
            if not isinstance(k, str) or not k or not isinstance(v, (int, float, str, bool)):
                raise SpaceError(f"invalid dimension {k!r}={v!r}", "shape")
        return cls(dict(dims), digest_of(dims))


def parse_space(text: str) -> ConfigSpace:
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise SpaceError(f"invalid JSON: {e}", "document") from None
    if not isinstance(doc, dict) or not isinstance(doc.get("name"), str):
        raise SpaceError("expected an object with a string 'name'", "document")
    raw = doc.get("params")
    if not isinstance(raw, list) or not raw:
        raise SpaceError("'params' must be a nonempty array", "document")
    params = [ParamDomain.from_json_dict(p, f"params[{i}]") for i, p in enumerate(raw)]
    cons = doc.get("constraints", [])
    if not isinstance(cons, list) or not all(isinstance(c, str) for c in cons):
        raise SpaceError("'constraints' must be an array of strings", "document")
    parsed = []
    for i, c in enumerate(cons):
        try:
            parsed.append(Constraint.parse(c))
        except SpaceError as e:
            raise SpaceError(f"malformed expression: {e.message}", f"constraints[{i}]") from None
    return ConfigSpace.build(doc["name"], params, parsed)


def parse_space_file(path) -> ConfigSpace:
    with open(path, encoding="utf-8") as fh:
        return parse_space(fh.read())


def _violated(space: ConfigSpace, env: dict):
    for c in space.constraints:
        try:
            if not c.holds(env):
                return c
        except ConstraintEvalError as e:
            raise ConstraintEvalError(f"constraint {c.text!r} failed on config {env!r}: {e}") from None
    return None


def enumerate_configs(space: ConfigSpace) -> Iterator[KernelConfig]:
    names = space.param_names()
    for combo in itertools.product(*(p.domain_values() for p in space.params)):
        env = dict(zip(names, combo))
        if _violated(space, env) is None:
            yield KernelConfig.from_assignments(env)


def cardinality(space: ConfigSpace) -> tuple:
    raw = 1
    for p in space.params:
        raw *= len(p.domain_values())
    return raw, sum(1 for _ in enumerate_configs(space))


def validate_config(space: ConfigSpace, config) -> tuple:
    a = config.assignments if isinstance(config, KernelConfig) else dict(config)
    expected, got = set(space.param_names()), set(a)
    if expected != got:
        raise SpaceError(f"missing {sorted(expected - got)} / unknown {sorted(got - expected)} parameters", "config")
    bad = [f"{p.name}: value {a[p.name]!r} not in domain" for p in space.params if not p.contains(a[p.name])]
    for c in space.constraints:
        try:
            if not c.holds(a):
                bad.append(c.text)
        except ConstraintEvalError as e:
            raise ConstraintEvalError(f"constraint {c.text!r} failed on config {a!r}: {e}") from None
    return (not bad), bad
