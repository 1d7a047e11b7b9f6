"""The shared-memory transposition layouts of fam_tensor_apply
(kernels.cuh:PatchLayout) under the wavefront model of tools/smem_layouts.py:
A and B at the ideal (2 wavefronts per fp64 warp access, 1 per fp32 access,
over the 4 warps of a 5-family block), N within the stated excess, and every
layout injective on the 5^3 patch and inside its slot.  The constants are read
from the header, so the test fails if the kernel's layouts drift from the
search."""
import importlib.util
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_tool():
    spec = importlib.util.spec_from_file_location("smem_layouts_cost", os.path.join(ROOT, "tools", "smem_layouts.py"))
    src = open(os.path.join(ROOT, "tools", "smem_layouts.py")).read().split("lays = []")[0]
    mod = importlib.util.module_from_spec(spec)
    exec(compile(src, "smem_layouts.py", "exec"), mod.__dict__)
    return mod


def header_layouts():
    s = open(os.path.join(ROOT, "paper_1904_03317_b200", "csrc", "kernels.cuh")).read()
    out = {}
    for t in ("double", "float"):
        m = re.search(r"struct PatchLayout<2, %s> \{(.*?)\};" % t, s, re.S)
        body = m.group(1)
        kv = dict((k, int(v)) for k, v in re.findall(r"(\w+) = (\d+)", body))
        out[t] = kv
    return out


@pytest.mark.parametrize("t", ["double", "float"])
def test_patch_layouts_reach_the_stated_wavefronts(t):
    tool = load_tool()
    L = header_layouts()[t]
    wf = tool.wf64 if t == "double" else tool.wf32
    ideal = 40 if t == "double" else 20                 # per pass and array, 5 families (4 warps)
    A, B, N = (L["ax"], L["ay"], L["az"]), (L["bx"], L["by"], L["bz"]), (L["nx"], L["ny"], L["nz"])
    R = range(5)
    for lay, stride in ((A, L["sab"]), (B, L["sab"]), (N, L["sn"])):
        idx = [lay[0] * x + lay[1] * y + lay[2] * z for x in R for y in R for z in R]
        assert len(set(idx)) == 125 and max(idx) < stride        # injective, inside the slot
    assert tool.cost(wf, A, L["sab"], "z") == ideal and tool.cost(wf, A, L["sab"], "y") == ideal
    assert tool.cost(wf, B, L["sab"], "y") == ideal and tool.cost(wf, B, L["sab"], "x") == ideal
    n_cost = tool.cost(wf, N, L["sn"], "x") + tool.cost(wf, N, L["sn"], "z")
    assert n_cost <= (100 if t == "double" else 55)        # 25 % / 38 % above 2 x ideal (odd cycle)
