"""Host-side validation of expression stencils (st_stencil2d_expr_halo, reading
R24): the C translator accepts exactly the grammar the oracle evaluates and
reports the halo; no GPU needed."""
import pytest

from oracle import expr as ox

GOOD = [
    "(a(-1,0) + a(1,0) + a(0,-1) + a(0,1)) * 0.25",
    "a(0,1)*a(0,-1) - a(1,0)",
    "-(a(3,0) - 2*a(0,0)) / 3",
    ".5*a(0, 0) + 1e-3 - 2.5E+2*a( -8 , 8 )",
    "--a(0,0)",
    "+a(2,-1)",
]
BAD = ["a(0,0)**2", "b(0,0)", "a(0,0) + ", "a(0,9)", "a(0,0) % 2", "a(0)", "(a(0,0)", "a(0,0))", "abs(a(0,0))",
       "a(0,0); x", "1 + 2", "a(0,0) a(0,1)", "3a(0,0)"]


@pytest.fixture(scope="module")
def lib():
    import paper_2310_01882_b200 as st
    return st


@pytest.mark.parametrize("e", GOOD)
def test_accepts_and_reports_halo(lib, e):
    assert lib.st_stencil2d_expr_halo(e) == ox.halo(e)


@pytest.mark.parametrize("e", BAD)
def test_rejects(lib, e):
    with pytest.raises(lib.StencilError):
        lib.st_stencil2d_expr_halo(e)


@pytest.mark.parametrize("e,want", [("(a(-1,0,0)+a(1,0,0)+a(0,-1,0)+a(0,1,0)+a(0,0,-1)+a(0,0,1))/6", (1, 3)),
                                    ("a(0,2)", (2, 2)), ("a(3,-1,0)*a(0,0,0)", (3, 3))])
def test_info_reports_halo_and_arity(lib, e, want):
    assert lib.st_stencil_expr_info(e) == want


@pytest.mark.parametrize("e", ["a(0,0) + a(0,0,0)", "a(1,2,3,4)"])
def test_rejects_mixed_or_wrong_arity(lib, e):
    with pytest.raises(lib.StencilError):
        lib.st_stencil_expr_info(e)
