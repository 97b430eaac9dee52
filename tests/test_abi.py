"""The C-ABI library loads, exports every symbol include/pcpm.h declares, and
rejects invalid arguments before touching a GPU (CPU-only tests)."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pcpm.h")


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(pcpm_[a-z_]+)\s*\(", txt)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for f in ("pcpm_build", "pcpm_pagerank", "pcpm_spmv", "pcpm_destroy"):
        assert f in names


def test_library_exports_every_declared_symbol():
    from paper_1709_07122_b200 import build_ext
    lib = build_ext.build()
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib]).decode()
    exported = set(re.findall(r"\bT (pcpm_\w+)", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, f"declared but not exported: {missing}"
    from paper_1709_07122_b200 import pcpm
    for f in declared_functions():
        assert f in pcpm.EXPORTED, f"binding lacks {f}"


def test_library_is_sm100a():
    from paper_1709_07122_b200 import build_ext
    lib = build_ext.build()
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "-lelf", lib]).decode()
    assert "sm_100a" in out


def test_invalid_arguments_rejected_without_gpu():
    from paper_1709_07122_b200 import pcpm
    rp = np.array([0, 1, 2], dtype=np.int64)
    col = np.array([1, 0], dtype=np.uint32)
    csr = pcpm.make_csr(2, 2, rp, col)
    for bits in (0, 17, -3):
        with pytest.raises(pcpm.PcpmError) as e:
            pcpm.pcpm_build(csr, bits)
        assert e.value.code == pcpm.PCPM_EINVAL
    big = pcpm.pcpm_csr(1 << 31, 4, 0, csr.row_ptr, csr.col_idx, None)
    with pytest.raises(pcpm.PcpmError) as e:
        pcpm.pcpm_build(big, 8)
    assert e.value.code == pcpm.PCPM_ETOOBIG
    kk = pcpm.pcpm_csr(1 << 30, 1 << 30, 0, csr.row_ptr, csr.col_idx, None)
    with pytest.raises(pcpm.PcpmError) as e:
        pcpm.pcpm_build(kk, 1)
    assert e.value.code == pcpm.PCPM_ETOOBIG
    with pytest.raises(pcpm.PcpmError) as e:
        pcpm.pcpm_pagerank(None, 0.85, 1, np.zeros(2, np.float32))
    assert e.value.code == pcpm.PCPM_EINVAL
    with pytest.raises(pcpm.PcpmError) as e:
        pcpm.pcpm_pool_reserve(-1)
    assert e.value.code == pcpm.PCPM_EINVAL
    assert pcpm.pcpm_pool_reserve(0) == pcpm.PCPM_OK      # nothing to map: no CUDA call


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1709_07122_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "pcpm_oracle" not in txt, f


def _build_c_example(tmp_path):
    import subprocess
    exe = tmp_path / "pagerank_c"
    libdir = os.path.join(ROOT, "paper_1709_07122_b200")
    subprocess.run(["gcc", "-O2", "-Wall", "-Werror", "-std=c99", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "pagerank_c.c"), "-L", libdir, "-lpcpm",
                    "-Wl,-rpath," + libdir, "-o", str(exe)], check=True)
    return exe


def test_c_example_compiles_against_the_header(tmp_path):
    """include/pcpm.h is plain C99 and libpcpm.so links from C (no CUDA or Python)."""
    assert _build_c_example(tmp_path).exists()


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    import subprocess
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([str(_build_c_example(tmp_path)), "200000"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "sum_pr=" in r.stdout
