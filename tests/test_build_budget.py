"""Build-time guard for the hot kernels (CPU; reads the ptxas log `make lib` leaves under build/obj).

The streaming CG kernel runs one 512-thread block per SM at up to 128 registers per thread.  A
feature added to a shared helper once pushed the m = 4 instance over that budget: ptxas moved the
kernel parameters to a 736-byte local copy and configs[3] went from 1119 to 1779 us per iteration
with every parity test still green.  This test fails the build check instead."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LOG = os.path.join(ROOT, "build", "obj", "cg_stream.o.ptxas.log")


def entries(path):
    out = {}
    name = None
    for line in open(path, errors="replace"):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            name = m.group(1)
            out[name] = {}
            continue
        if name is None:
            continue
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m:
            out[name].update(stack=int(m.group(1)), spill_st=int(m.group(2)), spill_ld=int(m.group(3)))
        m = re.search(r"Used (\d+) registers", line)
        if m:
            out[name]["regs"] = int(m.group(1))
    return out


@pytest.mark.skipif(not os.path.exists(LOG), reason="no ptxas log (library not built in this tree)")
@pytest.mark.parametrize("inst", ["cg_streamILi480ELi4ELb0ELb0E", "cg_streamILi480ELi1ELb0ELb0E"])
def test_stream_kernel_keeps_its_parameters_in_registers(inst):
    hits = {k: v for k, v in entries(LOG).items() if inst in k}
    assert hits, f"{inst} not found in {LOG}"
    for k, v in hits.items():
        assert v["regs"] <= 128, (k, v)
        assert v["spill_st"] == 0 and v["spill_ld"] == 0, (k, v)
        # a local copy of StreamParams shows up as a stack frame of several hundred bytes
        assert v["stack"] <= 128, (k, v)
