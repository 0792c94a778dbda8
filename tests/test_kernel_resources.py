"""Static resource guards on the built sm_100a kernels (CPU: cuobjdump on libgdx.so).

The hot aggregation kernels are occupancy-sensitive: a 40 -> 48 register change cost
5-14% of the L2/HBM-bound gather (48 -> 40 resident warps per SM), and they are built
for 8 blocks per SM (<= 32 registers) with a small spill area outside the gather loop.
The tensor-core GEMMs must not touch local memory."""
import functools
import os
import re
import shutil
import subprocess

import pytest

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2311_06837_b200", "libgdx.so")

pytestmark = pytest.mark.skipif(not (os.path.exists(LIB) and shutil.which("cuobjdump")),
                                reason="libgdx.so or cuobjdump missing")

# the instantiations the benchmarks run: 64-wide warp-per-row, 48-wide and 64-wide
# lane-group-per-row (Reddit last layer, cooperative batches)
HOT = ["aggregate_vec4ILi16ELi1ELb1ELi4E", "aggregate_rowsILi12ELi1ELb1ELi4E",
       "aggregate_rowsILi16ELi1ELb1ELi4E"]


@functools.lru_cache(maxsize=None)
def _usage():
    out = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True).stdout
    res, name = {}, None
    for line in out.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            name = m.group(1)
            continue
        m = re.search(r"REG:(\d+) STACK:(\d+)", line)
        if m and name:
            res[name] = (int(m.group(1)), int(m.group(2)))
    return res


@functools.lru_cache(maxsize=None)
def _sass_all():
    return subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout


def _sass(fragment):
    out = _sass_all()
    keep, lines = False, []
    for line in out.splitlines():
        if "Function :" in line:
            keep = fragment in line
        elif keep:
            lines.append(line)
    return lines


@pytest.mark.parametrize("frag", HOT)
def test_hot_aggregation_registers(frag):
    use = [v for k, v in _usage().items() if frag in k]
    assert use and max(r for r, _ in use) <= 32 and max(st for _, st in use) <= 64, (frag, use)


@pytest.mark.parametrize("frag", ["gemm_bf16x3ILi128ELi3ELb0ELb0ELi8E", "gemm_bf16x3ILi64ELi4ELb0ELb1ELi16E"])
def test_gemm_no_local_memory(frag):
    n = sum(1 for line in _sass(frag) if re.search(r"\b(LDL|STL)\b", line))
    assert n <= 2, (frag, n)
