"""The ctypes mirrors of include/hetplan_b200.h (engine.py, capi.py) have the
C layout: a tiny C program compiled against the header prints every struct's
size and field offsets, which must equal ctypes'. CPU only (gcc)."""
import ctypes as C
import os
import shutil
import subprocess

import pytest

from paper_2512_20953_b200 import capi, engine

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STRUCTS = [engine.hpk_grouping_problem, engine.hpk_grouping_result, engine.hpk_search_config,
           engine.hpk_timing, engine.hpk_plan_candidate, engine.hpk_plan_result,
           engine.hpk_affinity_problem, engine.hpk_pipeline, capi.hp_plan_options,
           capi.hp_sim_options]


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_ctypes_mirrors_match_the_header(tmp_path):
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "hetplan_b200.h"',
             "int main(void) {"]
    for st in STRUCTS:
        name = st.__name__
        lines.append(f'  printf("{name} size %zu\\n", sizeof({name}));')
        for f in st._fields_:
            lines.append(f'  printf("{name}.{f[0]} %zu\\n", offsetof({name}, {f[0]}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o",
                    str(exe)], check=True, capture_output=True)
    got = dict(line.rsplit(" ", 1) for line in
               subprocess.run([str(exe)], check=True, capture_output=True, text=True)
               .stdout.splitlines())
    want = {}
    for st in STRUCTS:
        name = st.__name__
        want[f"{name} size"] = str(C.sizeof(st))
        for f in st._fields_:
            want[f"{name}.{f[0]}"] = str(getattr(st, f[0]).offset)
    bad = {k: (got.get(k), v) for k, v in want.items() if got.get(k) != v}
    assert not bad, bad
