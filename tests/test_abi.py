"""CPU checks of the C ABI: the in-tree library loads, exports every function
include/mdot.h declares, and the ctypes structs match the C layout.  No
compute call is made (no GPU here)."""
import ctypes as ct
import os
import re
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "mdot.h")


def _declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(mdot_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def L():
    from paper_2307_08507_b200 import build
    build.build()
    import paper_2307_08507_b200 as M
    return M.lib()


def test_library_exports_every_declared_symbol(L):
    names = _declared_functions()
    assert len(names) >= 13, names
    for nm in names:
        assert hasattr(L, nm), f"{nm} declared in include/mdot.h but not exported"
    out = subprocess.check_output(["nm", "-D", "--defined-only", L._name]).decode()
    exported = set(re.findall(r" T (mdot_\w+)", out))
    assert set(names) <= exported


def test_struct_layouts_match_header(L):
    import paper_2307_08507_b200._binding as B
    prog = r'''
#include <stdio.h>
#include <stddef.h>
#include "mdot.h"
int main(void){
  printf("%zu %zu %zu %zu\n", sizeof(mdot_problem), sizeof(mdot_schedule), sizeof(mdot_options), sizeof(mdot_result));
  printf("%zu %zu %zu %zu\n", offsetof(mdot_options, stream), offsetof(mdot_result, status),
         offsetof(mdot_result, rho0), offsetof(mdot_problem, c));
  return 0;
}
'''
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "t.c")
        exe = os.path.join(d, "t")
        open(src, "w").write(prog)
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", exe])
        lines = subprocess.check_output([exe]).decode().split("\n")
    sizes = list(map(int, lines[0].split()))
    offs = list(map(int, lines[1].split()))
    assert sizes == [ct.sizeof(B.Problem), ct.sizeof(B.Schedule), ct.sizeof(B.Options), ct.sizeof(B.Result)]
    assert offs == [B.Options.stream.offset, B.Result.status.offset, B.Result.rho0.offset, B.Problem.c.offset]


def test_defaults_and_host_side_validation(L):
    import paper_2307_08507_b200 as M
    o = M.options()
    assert o.eps == 1e-6 and o.c1 == 0.1 and o.c2 == 0.4 and o.projector == M.MDOT_PROJ_PNCG
    s = M.schedule()
    assert s.kind == M.MDOT_SCHED_FIXED and s.gamma_bar == 4096.0 and s.step_max == 256.0
    import paper_2307_08507_b200._binding as B
    res = B.Result()
    # NULL problem is rejected before any CUDA call
    st = L.mdot_solve(None, ct.byref(s), ct.byref(o), None, None, None, ct.byref(res))
    assert st == 1 and "NULL" in M.mdot_last_error()
    assert L.mdot_abi_version() == 3


def test_binding_rejects_wrong_dtypes_before_any_call(L):
    """The C side reads r, c, U, V, A, B as fp64 and writes u/v/lr/lc as fp64
    and P as fp32 (include/mdot.h): the binding refuses other element types
    and mixed host/device buffers instead of letting the library over-read or
    overwrite them."""
    import numpy as np
    import paper_2307_08507_b200 as M
    C = np.zeros((4, 4), dtype=np.float32)
    r = np.full(4, 0.25)
    with pytest.raises(TypeError, match="r: dtype float32"):
        M.mdot_solve(C, r.astype(np.float32), r)
    with pytest.raises(TypeError, match="C: dtype int32"):
        M.mdot_solve(C.astype(np.int32), r, r)
    with pytest.raises(TypeError, match="u_out: dtype float32"):
        M.mdot_solve(C, r, r, u_out=np.zeros(4, dtype=np.float32))
    with pytest.raises(TypeError, match="P_out: dtype float64"):
        M.mdot_solve(C, r, r, P_out=np.zeros((4, 4)))
    with pytest.raises(TypeError, match="lr: dtype float32"):
        M.mdot_marginals(r, r, 1.0, C, r, r, lr=np.zeros(4, dtype=np.float32))
    with pytest.raises(TypeError, match="X: dtype float64"):
        M.mdot_solve(X=np.zeros((4, 2)), Y=np.zeros((4, 2), dtype=np.float32), r=r, c=r)
    with pytest.raises(TypeError, match="V: dtype float32"):
        M.mdot_round(r, r.astype(np.float32), 1.0, C, r, r)
