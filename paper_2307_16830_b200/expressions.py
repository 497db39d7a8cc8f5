"""Instruction language of the SIMD abstraction (host side, structure only).

An instruction is a scalar expression over variable slots ``var(i)`` and
parameter slots ``param(k)``; one instruction is shared by every record of
a pattern block (reference src/gridnlp/expressions.py:1-18).  The tree is
flattened once into a single-assignment tape whose entries are
``(op, a, b)`` triples with the reference's opcode numbering
(expressions.py:23-37) so that tapes are interchangeable with the
reference's.

Evaluation and differentiation never run here: the tape is uploaded to
HBM and interpreted (or matched to a specialised pattern kernel) by the
CUDA AD evaluator in ``csrc/ad.cu``.  This module only provides

* the operator-overloading front end (``var/param/const/sin/...``),
* tape flattening with node sharing (expressions.py:147-170), and
* the structural template: the slots of the first derivative and the
  slot pairs of the second derivative (expressions.py:173-219).
"""
from __future__ import annotations

import numpy as np

VAR, PAR, CONST = 0, 1, 2
ADD, SUB, MUL, DIV, POW = 3, 4, 5, 6, 7
NEG, SIN, COS, LOG, SQRT, EXP = 8, 9, 10, 11, 12, 13

UNARY = frozenset((NEG, SIN, COS, LOG, SQRT, EXP))
BINARY = frozenset((ADD, SUB, MUL, DIV))
# unary operators whose second derivative is nonzero
_CURVED_UNARY = frozenset((SIN, COS, LOG, SQRT, EXP))

MAX_TAPE = 64   # device interpreter limit; longer tapes run on the generated pattern kernels


class Expr:
    """Node of an instruction tree; arithmetic operators build new nodes."""

    __slots__ = ("op", "a", "b", "value")

    def __init__(self, op, a=None, b=None, value=None):
        self.op = op
        self.a = a
        self.b = b
        self.value = value

    def _bin(self, op, other, swap=False):
        other = as_expr(other)
        return Expr(op, other, self) if swap else Expr(op, self, other)

    def __add__(self, o):
        return self._bin(ADD, o)

    def __radd__(self, o):
        return self._bin(ADD, o, True)

    def __sub__(self, o):
        return self._bin(SUB, o)

    def __rsub__(self, o):
        return self._bin(SUB, o, True)

    def __mul__(self, o):
        return self._bin(MUL, o)

    def __rmul__(self, o):
        return self._bin(MUL, o, True)

    def __truediv__(self, o):
        return self._bin(DIV, o)

    def __rtruediv__(self, o):
        return self._bin(DIV, o, True)

    def __pow__(self, exponent):
        if not isinstance(exponent, (int, float)):
            raise TypeError("only constant exponents are supported")
        return Expr(POW, self, value=float(exponent))

    def __neg__(self):
        return Expr(NEG, self)


def as_expr(x) -> Expr:
    return x if isinstance(x, Expr) else const(x)


def var(slot: int) -> Expr:
    return Expr(VAR, value=int(slot))


def param(slot: int) -> Expr:
    return Expr(PAR, value=int(slot))


def const(c: float) -> Expr:
    return Expr(CONST, value=float(c))


def sin(x) -> Expr:
    return Expr(SIN, as_expr(x))


def cos(x) -> Expr:
    return Expr(COS, as_expr(x))


def log(x) -> Expr:
    return Expr(LOG, as_expr(x))


def sqrt(x) -> Expr:
    return Expr(SQRT, as_expr(x))


def exp(x) -> Expr:
    return Expr(EXP, as_expr(x))


class Tape:
    """Flattened instruction plus its structural sparsity template."""

    def __init__(self, root: Expr):
        self.ops: list[tuple[int, int, int]] = []
        self.consts: list[float] = []
        seen: dict[int, int] = {}
        self.out = self._flatten(root, seen)
        vslots = [a for (op, a, _) in self.ops if op == VAR]
        pslots = [a for (op, a, _) in self.ops if op == PAR]
        self.n_var_slots = max(vslots) + 1 if vslots else 0
        self.n_param_slots = max(pslots) + 1 if pslots else 0
        self.first_slots, self.second_pairs = self._template()

    def _flatten(self, root: Expr, seen) -> int:
        """Post-order emission with node sharing, iterative (deep trees)."""
        stack = [(root, False)]
        while stack:
            node, expanded = stack.pop()
            if id(node) in seen:
                continue
            op = node.op
            kids = []
            if op in BINARY:
                kids = [node.a, node.b]
            elif op in UNARY or op == POW:
                kids = [node.a]
            if not expanded and any(id(k) not in seen for k in kids):
                stack.append((node, True))
                for k in reversed(kids):
                    if id(k) not in seen:
                        stack.append((k, False))
                continue
            if op in (VAR, PAR):
                entry = (op, int(node.value), -1)
            elif op == CONST:
                self.consts.append(float(node.value))
                entry = (op, -1, len(self.consts) - 1)
            elif op == POW:
                self.consts.append(float(node.value))
                entry = (op, seen[id(node.a)], len(self.consts) - 1)
            elif op in UNARY:
                entry = (op, seen[id(node.a)], -1)
            else:
                entry = (op, seen[id(node.a)], seen[id(node.b)])
            self.ops.append(entry)
            seen[id(node)] = len(self.ops) - 1
        return seen[id(root)]

    def _template(self):
        """First-derivative slots and (max, min) second-derivative pairs.

        Dependence sets propagate forward; every nonlinear interaction
        (product, quotient, power != 0/1, curved unary) records the cross
        product of its operands' sets.  Only pairs whose slots both reach
        the output are kept (reference expressions.py:216-219).
        """
        deps: list[frozenset] = []
        pairs: set[tuple[int, int]] = set()

        def cross(u, w):
            pairs.update((max(i, j), min(i, j)) for i in u for j in w)

        for op, a, b in self.ops:
            if op == VAR:
                d = frozenset((a,))
            elif op in (PAR, CONST):
                d = frozenset()
            elif op in (ADD, SUB):
                d = deps[a] | deps[b]
            elif op == NEG:
                d = deps[a]
            elif op == MUL:
                cross(deps[a], deps[b])
                d = deps[a] | deps[b]
            elif op == DIV:
                cross(deps[a], deps[b])
                cross(deps[b], deps[b])
                d = deps[a] | deps[b]
            elif op == POW:
                c = self.consts[b]
                if c == 0.0:
                    d = frozenset()
                else:
                    if c != 1.0:
                        cross(deps[a], deps[a])
                    d = deps[a]
            else:
                cross(deps[a], deps[a])
                d = deps[a]
            deps.append(d)
        live = deps[self.out]
        kept = sorted(p for p in pairs if p[0] in live and p[1] in live)
        return sorted(live), kept

    # -- device encoding ---------------------------------------------------
    def encode(self):
        """(ops int32[T,3], consts float64[C]) as uploaded to the device."""
        ops = np.asarray(self.ops, dtype=np.int32).reshape(-1, 3)
        consts = np.asarray(self.consts, dtype=np.float64)
        return ops, consts

    def signature(self) -> tuple:
        """Structural identity used to match specialised pattern kernels."""
        return (tuple(self.ops), tuple(self.consts), self.out)
