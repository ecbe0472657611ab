"""The Python binding's ctypes structures match the C ABI of include/flmisr.h field by field: a small C
program compiled with gcc against the header prints sizeof and offsetof of every field of
flmisr_config and flmisr_report, and the ctypes layouts must agree (an appended or reordered config
field, e.g. x0_mode / det_rows, would otherwise be read from the wrong offset without any error)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CONFIG_FIELDS = ["k", "lr_h", "lr_w", "shifts", "psf", "psf_h", "psf_w", "mag", "p_norm", "l1_eps", "lambda",
                 "btv_alpha", "btv_window", "n_iter", "scg_sigma0", "scg_lambda0", "rank", "world",
                 "nccl_unique_id", "device", "btv_offsets", "curv_mode", "scg_rules", "x0_mode", "det_rows"]
REPORT_FIELDS = ["iters_run", "accepted", "converged_at", "failed_stage", "failed_iter", "f_trace"]
PY_NAME = {"lambda": "lam"}   # a Python keyword in the binding


def _c_layout(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "flmisr.h"', "int main(void) {",
             '  printf("config %zu\\n", sizeof(flmisr_config));', '  printf("report %zu\\n", sizeof(flmisr_report));']
    for f in CONFIG_FIELDS:
        lines.append(f'  printf("config.{f} %zu\\n", offsetof(flmisr_config, {f}));')
    for f in REPORT_FIELDS:
        lines.append(f'  printf("report.{f} %zu\\n", offsetof(flmisr_report, {f}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = subprocess.check_output([str(exe)], text=True)
    return dict((k, int(v)) for k, v in (line.split() for line in out.splitlines()))


def test_ctypes_structs_match_the_c_header(tmp_path):
    import sys
    sys.path.insert(0, ROOT)
    from paper_2108_04315_b200.flmisr import Config, Report   # no GPU needed: ctypes declarations only
    import ctypes as C
    lay = _c_layout(tmp_path)
    assert [n if n != "lam" else "lambda" for n, _ in Config._fields_] == CONFIG_FIELDS
    assert [n for n, _ in Report._fields_] == REPORT_FIELDS
    assert C.sizeof(Config) == lay["config"]
    assert C.sizeof(Report) == lay["report"]
    for f in CONFIG_FIELDS:
        assert getattr(Config, PY_NAME.get(f, f)).offset == lay[f"config.{f}"], f
    for f in REPORT_FIELDS:
        assert getattr(Report, f).offset == lay[f"report.{f}"], f
