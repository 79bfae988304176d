"""Expression stencil oracle (NEXT #4: "offset list + expression", SURVEY.md §8(f);
reading R24 of DESIGN.md).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py); shares nothing with the CUDA path.

A Fortran loop body the discovery pass turns into a stencil.apply region
(Listing 3; RHS accesses) is an
arithmetic expression over accesses at constant offsets. Here it is written with
a(dy, dx) for the access at row offset dy, column offset dx, numeric literals
(binary64), + - * /, unary minus and parentheses, with C/Fortran/Python
precedence and left associativity. Each sweep evaluates the expression with NumPy
float64 arrays (elementwise, one IEEE rounding per operation, in parse order,
never contracted) on the shifted views of the previous iterate (value semantics,
PAPER.md:126). Halo R = max |offset|: the R-wide ring is fixed.
"""
from __future__ import annotations

import ast
import re

import numpy as np

_ACCESS = re.compile(r"a\(\s*(-?\d+)\s*,\s*(-?\d+)\s*\)")
_ACCESS3 = re.compile(r"a\(\s*(-?\d+)\s*,\s*(-?\d+)\s*,\s*(-?\d+)\s*\)")
_ALLOWED = re.compile(r"^[\sa0-9.eE+\-*/(),]*$")


def offsets(expr: str) -> list[tuple[int, int]]:
    """The (dy, dx) accesses of the expression, in order of appearance."""
    return [(int(dy), int(dx)) for dy, dx in _ACCESS.findall(expr)]


def offsets3(expr: str) -> list[tuple[int, int, int]]:
    """The (dz, dy, dx) accesses of a 3-D expression, in order of appearance."""
    return [(int(dz), int(dy), int(dx)) for dz, dy, dx in _ACCESS3.findall(expr)]


def halo3(expr: str) -> int:
    offs = offsets3(expr)
    if not offs:
        raise ValueError("expression has no a(dz, dy, dx) access")
    return max(max(abs(v) for v in o) for o in offs)


def halo(expr: str) -> int:
    offs = offsets(expr)
    if not offs:
        raise ValueError("expression has no a(dy, dx) access")
    return max(max(abs(dy), abs(dx)) for dy, dx in offs)


def check(expr: str) -> None:
    """Accept only accesses, literals, + - * /, unary minus and parentheses."""
    if not _ALLOWED.match(expr):
        raise ValueError(f"expression has characters outside a(), digits, . e E + - * / ( ) ,: {expr!r}")
    tree = ast.parse(expr, mode="eval")
    for node in ast.walk(tree):
        if isinstance(node, ast.Call):
            if not (isinstance(node.func, ast.Name) and node.func.id == "a" and len(node.args) in (2, 3)):
                raise ValueError("only a(dy, dx) / a(dz, dy, dx) calls are allowed")
        elif isinstance(node, ast.BinOp):
            if not isinstance(node.op, (ast.Add, ast.Sub, ast.Mult, ast.Div)):
                raise ValueError("only + - * / are allowed")
        elif isinstance(node, ast.UnaryOp):
            if not isinstance(node.op, (ast.USub, ast.UAdd)):
                raise ValueError("only unary +/- are allowed")
        elif isinstance(node, ast.Constant):
            if not isinstance(node.value, (int, float)) or isinstance(node.value, bool):
                raise ValueError("only numeric literals are allowed")
        elif not isinstance(node, (ast.Expression, ast.Name, ast.Load, ast.Add, ast.Sub, ast.Mult, ast.Div,
                                   ast.USub, ast.UAdd)):
            raise ValueError(f"unsupported syntax: {type(node).__name__}")


class _FloatLiterals(ast.NodeTransformer):
    """Every numeric literal outside an access is a binary64 value (as in the CUDA path,
    where the generated source spells it as a double literal)."""

    def visit_Call(self, node):
        return node  # a(dy, dx) / f<i>(dz, dy, dx): the offsets stay integers

    def visit_Constant(self, node):
        return ast.copy_location(ast.Constant(float(node.value)), node)


def _compile(expr: str):
    tree = ast.fix_missing_locations(_FloatLiterals().visit(ast.parse(expr, mode="eval")))
    return compile(tree, "<stencil>", "eval")


def stencil2d_expr(a0: np.ndarray, expr: str, iters: int, nx: int | None = None) -> np.ndarray:
    """`iters` sweeps of the expression stencil on the padded field a0 ((ny + 2R) x ld)."""
    check(expr)
    R = halo(expr)
    ny = a0.shape[0] - 2 * R
    nx = a0.shape[1] - 2 * R if nx is None else nx
    if ny < 1 or nx < 1:
        raise ValueError("no interior")
    code = _compile(expr)
    cur = a0.copy()
    for _ in range(iters):
        def a(dy, dx, _c=cur):
            return _c[R + dy:R + dy + ny, R + dx:R + dx + nx]
        out = eval(code, {"__builtins__": {}}, {"a": a})
        nxt = cur.copy()
        nxt[R:R + ny, R:R + nx] = out
        cur = nxt
    return cur


def stencil3d_expr(a0: np.ndarray, expr: str, iters: int, nx: int | None = None) -> np.ndarray:
    """`iters` sweeps of a 3-D expression stencil over a(dz, dy, dx) on the padded field
    a0 ((nz + 2R) x (ny + 2R) x ldx, x fastest)."""
    check(expr)
    R = halo3(expr)
    nz, ny = a0.shape[0] - 2 * R, a0.shape[1] - 2 * R
    nx = a0.shape[2] - 2 * R if nx is None else nx
    if min(nx, ny, nz) < 1:
        raise ValueError("no interior")
    code = _compile(expr)
    cur = a0.copy()
    for _ in range(iters):
        def a(dz, dy, dx, _c=cur):
            return _c[R + dz:R + dz + nz, R + dy:R + dy + ny, R + dx:R + dx + nx]
        out = eval(code, {"__builtins__": {}}, {"a": a})
        nxt = cur.copy()
        nxt[R:R + nz, R:R + ny, R:R + nx] = out
        cur = nxt
    return cur


def eval_exact(expr: str, a_of):
    """Evaluate the expression with a user access function (e.g. returning Fractions)."""
    check(expr)
    return eval(compile(ast.parse(expr, mode="eval"), "<stencil>", "eval"), {"__builtins__": {}}, {"a": a_of})


# ----------------------------------------------------------------- fused multi-field regions
_FIELD = re.compile(r"^f([0-7])$")
_COEF = re.compile(r"^k([0-7])$")
_ALLOWED_FUSED = re.compile(r"^[\sfk0-9.eE+\-*/(),]*$")


def check_fused(expr: str) -> None:
    """Fused-region grammar: field accesses f0..f7(dz, dy, dx), per-plane coefficients k0..k7
    (their value at the output point's plane), literals, + - * /, unary signs, parentheses."""
    if not _ALLOWED_FUSED.match(expr):
        raise ValueError(f"expression has characters outside f(), k, digits, . e E + - * / ( ) ,: {expr!r}")
    tree = ast.parse(expr, mode="eval")
    for node in ast.walk(tree):
        if isinstance(node, ast.Call):
            if not (isinstance(node.func, ast.Name) and _FIELD.match(node.func.id) and len(node.args) == 3):
                raise ValueError("only f<i>(dz, dy, dx) calls are allowed")
        elif isinstance(node, ast.Name):
            if not (_FIELD.match(node.id) or _COEF.match(node.id)):
                raise ValueError(f"unknown name {node.id}")
        elif isinstance(node, ast.BinOp):
            if not isinstance(node.op, (ast.Add, ast.Sub, ast.Mult, ast.Div)):
                raise ValueError("only + - * / are allowed")
        elif isinstance(node, ast.UnaryOp):
            if not isinstance(node.op, (ast.USub, ast.UAdd)):
                raise ValueError("only unary +/- are allowed")
        elif isinstance(node, ast.Constant):
            if not isinstance(node.value, (int, float)) or isinstance(node.value, bool):
                raise ValueError("only numeric literals are allowed")
        elif not isinstance(node, (ast.Expression, ast.Load, ast.Add, ast.Sub, ast.Mult, ast.Div, ast.USub,
                                   ast.UAdd)):
            raise ValueError(f"unsupported syntax: {type(node).__name__}")


def fused_halo(exprs) -> int:
    offs = [tuple(int(v) for v in m) for e in exprs
            for m in re.findall(r"f[0-7]\(\s*(-?\d+)\s*,\s*(-?\d+)\s*,\s*(-?\d+)\s*\)", e)]
    if not offs:
        raise ValueError("no field access")
    return max(max(abs(v) for v in o) for o in offs)


def fused3d_expr(inputs, exprs, plane_coefs=(), nx: int | None = None, out=None):
    """One application of a fused region (several stencils over several fields
    computed in one pass): output j = exprs[j] evaluated at every interior point of the
    (nz + 2R) x (ny + 2R) x ldx fields, R = max |offset|; k<j> is plane_coefs[j][z]. Output
    halos are left as they are (zeros unless `out` is given)."""
    for e in exprs:
        check_fused(e)
    R = fused_halo(exprs)
    a0 = inputs[0]
    nz, ny = a0.shape[0] - 2 * R, a0.shape[1] - 2 * R
    nx = a0.shape[2] - 2 * R if nx is None else nx
    env = {}
    for i, f in enumerate(inputs):
        env[f"f{i}"] = (lambda _f: lambda dz, dy, dx: _f[R + dz:R + dz + nz, R + dy:R + dy + ny,
                                                           R + dx:R + dx + nx])(f)
    for j, c in enumerate(plane_coefs):
        env[f"k{j}"] = np.asarray(c, dtype=np.float64)[R:R + nz, None, None]
    outs = out if out is not None else [np.zeros_like(a0) for _ in exprs]
    for o, e in zip(outs, exprs):
        o[R:R + nz, R:R + ny, R:R + nx] = eval(_compile(e), {"__builtins__": {}}, env)
    return outs
