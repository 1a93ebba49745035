"""The boundary is a real C ABI: a plain-C program (tests/c/abi_host.c) compiled with gcc
against include/daso.h and linked with libdaso.so drives the host-only entry points; its
schedule records must equal the oracle's (CPU only)."""
import os
import shutil
import subprocess

import pytest

from oracle.schedule import SchedConfig, plateau_arg, run_schedule
from paper_2104_05588_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_plain_c_client(tmp_path):
    exe = str(tmp_path / "abi_host")
    libdir = os.path.dirname(L.LIB_PATH)
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c", "abi_host.c"), "-L", libdir, "-l:libdaso.so",
                    f"-Wl,-rpath,{libdir}", "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stderr
    got = [tuple(int(v) for v in line.split(",")) for line in r.stdout.strip().splitlines()]
    cfg = SchedConfig(B_init=4, S_init=1, warmup_epochs=1, cooldown_epochs=1, total_epochs=5, steps_per_epoch=8,
                      gpus_per_node=2)
    flags = [0, 1, 1, 0, 0]          # plateau args 1 at k = 16 and k = 24 (ends of epochs 1 and 2)
    recs = run_schedule(cfg, 40, flags)
    want = [(r.step, r.phase, r.B, r.S, r.batch_in_cycle, r.send, r.blocking, r.send_group, r.merge, r.merge_S,
             r.merge_group, r.pending, r.due) for r in recs]
    assert [plateau_arg(k, flags, 8) for k in (16, 24)] == [1, 1]
    assert got == want


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_binding_structs_match_the_header_layout(tmp_path):
    """The ctypes mirrors of the header's structs (argument marshalling at the boundary) have the C
    compiler's size and field offsets, so no field is read from the wrong place (e.g. daso_trace's
    kernel_nvl_bytes appended in round 2)."""
    structs = {"daso_sched_config": L.SchedConfig, "daso_record": L.Record, "daso_config": L.Config,
               "daso_trace": L.Trace}
    src = ["#include <stddef.h>", "#include <stdio.h>", '#include "daso.h"', "int main(void) {"]
    for cname, cls in structs.items():
        src.append(f'  printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for f, _ in cls._fields_:
            src.append(f'  printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    src += ["  return 0;", "}"]
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src) + "\n")
    exe = str(tmp_path / "layout")
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), str(c), "-o", exe],
                   check=True)
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {tuple(line.split()[:2]): int(line.split()[2]) for line in out if line}
    import ctypes
    for cname, cls in structs.items():
        assert got[(cname, "sizeof")] == ctypes.sizeof(cls), cname
        for f, _ in cls._fields_:
            assert got[(cname, f)] == getattr(cls, f).offset, (cname, f)
