"""CHECKED-library runs: the stand-in for compute-sanitizer, which the GPU pool
refuses (profiles/r02_sanitizer/).  `make rg-checked` builds lib/librg_checked.so with device-side
bounds and invariant checks on the hand-computed indexing (RG_CHK, csrc/common.cuh): every TMA / bulk
copy's basis columns and rows, DCGS2 / CGS2 pass widths against their shared-memory rings and
reduction buffers, least-squares state indices, sparse column indices (CSR, SELL, BSR block
columns), the persistent kernel's neighbour ranges and per-step column indices, the operator build's
recycle dimension.  A failing check makes the call return RG_E_CHECK with the source location.

Here the seeded fuzz (every execution path: persistent single/multi-CTA, CUDA graph + DCGS2,
classical CGS2, SELL, SSOR, x0, all variants) and the parity suite run in a subprocess against the
checked library; any check failure fails them."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1807_09467_b200", "lib", "librg_checked.so")


def _run(files, timeout):
    if not os.path.exists(LIB):
        pytest.fail(f"{LIB} missing: build it with `make rg-checked` (__graft_entry__.build() does)")
    mark = os.path.join(ROOT, "gpurun_out", f"checked_maps_{os.getpid()}.txt")
    os.makedirs(os.path.dirname(mark), exist_ok=True)
    env = dict(os.environ, RG_TEST_CHECKED_LIB=LIB, RG_TEST_CHECKED_MARK=mark)
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", "-m", "gpu", *files],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
    libs = open(mark).read().split()
    os.remove(mark)
    assert any(p.endswith("librg_checked.so") for p in libs), libs   # the runs went through the checked library


def test_checked_library_is_checked():
    """The checked library carries the device check (rg_chk_fail) and the product library does not."""
    def elf(path):
        return subprocess.run(["cuobjdump", "-elf", path], capture_output=True, text=True).stdout
    assert "rg_chk_fail" in elf(LIB)
    assert "rg_chk_fail" not in elf(os.path.join(ROOT, "paper_1807_09467_b200", "lib", "librg.so"))


def test_fuzz_under_checks():
    _run(["tests/test_gpu_fuzz.py"], 1500)


def test_parity_and_sequences_under_checks():
    _run(["tests/test_gpu_parity.py", "tests/test_gpu_precond.py", "tests/test_gpu_basis.py"], 1500)
