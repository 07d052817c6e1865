"""The drop-in boundary from C: a caller written against the reference's
header (proj/include/bitsort/bitsort.h, same entry points as include/bitsort/
bitsort.h here) compiles with gcc and links against libbitsort.so.1 unchanged
(INTEGRATION.md). On a machine without a GPU the call reports the missing
device (no CPU fallback); on a B200 it sorts.
"""
from __future__ import annotations

import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_1312_0138_b200" / "lib"

CALLER = r"""
#include <bitsort/bitsort.h>
#include <stdio.h>

int main(void) {
    /* test_capi.cpp:78-82's vector, widened to uint32 */
    uint32_t keys[] = {200, 3, 255, 0};
    bws_algorithm alg;
    if (bws_algorithm_from_name("bitwise", &alg) != BWS_OK) return 3;
    bws_status st = bws_sort(keys, 4, 32, 1, alg);
    if (st != BWS_OK) {
        printf("status %d: %s\n", (int)st, bws_last_error());
        return 2;
    }
    printf("%u %u %u %u (%s)\n", keys[0], keys[1], keys[2], keys[3], bws_version());
    return 0;
}
"""


@pytest.fixture(scope="module")
def caller(tmp_path_factory):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    d = tmp_path_factory.mktemp("c_caller")
    src = d / "caller.c"
    src.write_text(CALLER)
    exe = d / "caller"
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-I", str(ROOT / "include"), str(src),
                    "-L", str(LIB), "-lbitsort", f"-Wl,-rpath,{LIB}", "-o", str(exe)], check=True)
    return exe


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU behaviour")
def test_c_caller_links_and_reports_no_device(caller):
    r = subprocess.run([str(caller)], capture_output=True, text=True)
    assert r.returncode == 2, r.stdout + r.stderr
    assert "status 5" in r.stdout and "no CPU fallback" in r.stdout


@pytest.mark.gpu
def test_c_caller_sorts_on_gpu(caller):
    r = subprocess.run([str(caller)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("0 3 200 255 (1.0.0)")
