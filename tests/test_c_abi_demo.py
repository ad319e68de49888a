"""The C-ABI driven from a compiled C host (examples/c_abi_demo.c): plan from
LDU addressing, caller-owned device arena, per-source pinned uploads,
Jacobi-PCG synchronously and stream-ordered.  Its results must equal the
Python drop-in's on the same 2-rank cavity bit for bit (iterations, residual,
x[0]) — the boundary is the same library either way."""

import json
import math
import os
import shutil
import subprocess

import numpy as np
import pytest

import paper_2510_08536_b200 as lrb
from helpers_b200 import cavity_case

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "examples", "c_abi_demo.c")
BIN = os.path.join(ROOT, "examples", "c_abi_demo")
N = 32


def build_demo():
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    cmd = [shutil.which("gcc") or "gcc", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(cuda, "include"), SRC, "-o", BIN,
           "-L", os.path.join(ROOT, "paper_2510_08536_b200"), "-lldurepart_b200",
           "-L", os.path.join(cuda, "lib64"), "-lcudart",
           "-Wl,-rpath," + os.path.join(ROOT, "paper_2510_08536_b200")]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_c_demo_compiles_against_the_header():
    build_demo()
    assert os.access(BIN, os.X_OK)


@pytest.mark.gpu
def test_c_demo_matches_python_drop_in():
    build_demo()
    out = subprocess.run([BIN, str(N)], check=True, capture_output=True, text=True, timeout=300)
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    _, asm, pm = cavity_case((N, N, N), 2, 2)

    def program(ctx):
        s = lrb.repartition(*asm[ctx.rank], pm, ctx)
        res = []
        for step in (2, 3, 4):
            lrb.update(s, *lrb.perturb_coefficients(*asm[ctx.rank], step), "direct")
            if s.is_owner:
                x, rep = lrb.cg_solve(s.matrix, s.halo, np.ones(s.matrix.n_owned), 1e-6, 2000,
                                      s.comm, method="pcg")
                res.append((step, rep, x))
        return res

    py = lrb.run_world(2, program)[0]
    sync = [d for d in lines if d["mode"] == "sync"]
    assert [d["step"] for d in sync] == [2, 3, 4]
    for d, (step, rep, x) in zip(sync, py):
        assert d["converged"] == 1 and d["iterations"] == rep.iterations
        assert d["residual"] == rep.residual and d["x0"] == x[0]
        s = 0.0
        for v in x.tolist():   # the C program's sequential sum
            s += v
        assert d["x_sum"] == s
    a = [d for d in lines if d["mode"] == "async"][0]
    assert a["iterations"] == sync[-1]["iterations"] and a["x_sum"] == sync[-1]["x_sum"]
    assert a["residual"] == sync[-1]["residual"] and math.isfinite(a["x0"])
