"""Host-side checks of the C-ABI library (no GPU needed).

The library must load, export every function include/noc_sim.h declares,
agree with the Python binding on struct layouts, validate configurations
before touching a device, and fail loudly (NOC_ECUDA) when there is no GPU.
"""
import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

import paper_1508_03235_b200 as nb
from paper_1508_03235_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "noc_sim.h")


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|uint32_t|const char \*)\s*\*?\s*(noc_sim_\w+)\s*\(",
                                 src, re.M)))


def test_library_exports_every_declared_symbol():
    L = nb.lib()
    names = declared_functions()
    assert len(names) >= 10
    for name in names:
        assert hasattr(L, name), name
    hdr = open(HEADER).read()
    assert L.noc_sim_abi_version() == int(re.search(r"#define NOC_SIM_ABI_VERSION (\d+)u", hdr).group(1))


def test_struct_layouts_match_header():
    """sizeof/offsetof from the C compiler vs the ctypes mirrors."""
    fields = {
        "noc_sim_config": [f for f, _ in nb.noc_sim_config._fields_],
        "noc_sim_counters": [f for f, _ in nb.noc_sim_counters._fields_],
        "noc_sim_info": [f for f, _ in nb.noc_sim_info._fields_],
        "noc_sim_event": [f for f, _ in nb.noc_sim_event._fields_],
    }
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "noc_sim.h"', "int main(void){"]
    for st, fs in fields.items():
        lines.append('printf("%s %%zu\\n", sizeof(%s));' % (st, st))
        for f in fs:
            lines.append('printf("%s.%s %%zu\\n", offsetof(%s, %s));' % (st, f, st, f))
    lines.append("return 0;}")
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "l.c")
        exe = os.path.join(d, "l")
        open(c, "w").write("\n".join(lines))
        subprocess.check_call(["gcc", "-I" + os.path.join(ROOT, "include"), c, "-o", exe])
        out = subprocess.check_output([exe]).decode().split("\n")
    want = {}
    for line in out:
        if line:
            k, v = line.split()
            want[k] = int(v)
    for st, fs in fields.items():
        cls = getattr(nb, st)
        assert C.sizeof(cls) == want[st], st
        for f in fs:
            assert getattr(cls, f).offset == want["%s.%s" % (st, f)], (st, f)


@pytest.mark.parametrize("bad", [
    dict(mesh_w=1), dict(mesh_h=4096), dict(sendq_cap=3), dict(hist_bins=0), dict(nfl_ra=9),
    dict(mode=W.MODE_LSPD, priv_tags=128), dict(mode=W.MODE_LSPD, l2_ways=17),
    dict(mode=W.MODE_LSPD, mem_lat=0), dict(mode=2), dict(age_base=65536), dict(band_streams=1),
    dict(band_streams=2),
])
def test_invalid_configs_rejected_before_device(bad):
    cfg = W.make(**bad)
    with pytest.raises(nb.NocSimError) as e:
        nb.noc_sim_create(cfg)
    assert e.value.code == nb.NOC_EINVAL


def test_invalid_script_rejected():
    with pytest.raises(nb.NocSimError) as e:
        nb.noc_sim_create(W.c1a(), script=[(0, 3, 3)])        # probe to itself
    assert e.value.code == nb.NOC_EINVAL
    with pytest.raises(nb.NocSimError) as e:
        nb.noc_sim_create(W.c1b(), script=[(0, 3, 16 * 128)])  # tag out of range
    assert e.value.code == nb.NOC_EINVAL


def test_no_silent_cpu_fallback_without_gpu(has_gpu):
    if has_gpu:
        pytest.skip("GPU present")
    with pytest.raises(nb.NocSimError) as e:
        nb.noc_sim_create(W.c1a())
    assert e.value.code == nb.NOC_ECUDA


def test_sass_is_sm100a():
    """The kernels in the library are compiled for sm_100a."""
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", nb.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
