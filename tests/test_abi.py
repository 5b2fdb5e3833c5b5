"""CPU-only checks of the drop-in boundary: the C-ABI library loads, exports
every entry point include/biscale_gpu.h declares, its ctypes mirror has the
C compiler's struct layouts, and with no GPU it fails loudly (no fallback)."""
from __future__ import annotations

import ctypes as C
import re
import subprocess
import tempfile
from pathlib import Path

import pytest

from paper_2602_18755_b200 import _abi as A
from paper_2602_18755_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "biscale_gpu.h"

STRUCTS = ["bs_grid", "bs_idle_entry", "bs_model_set", "bs_features", "bs_scheduler_policy", "bs_mpc_config",
           "bs_waiting", "bs_snapshot", "bs_mpc_problem", "bs_level_stats", "bs_mpc_result", "bs_projected_batch",
           "bs_decode_config", "bs_decode_query", "bs_decode_result", "bs_request", "bs_trace", "bs_length_dist",
           "bs_slo", "bs_goodput_search", "bs_instance_config", "bs_table_entry", "bs_sim_summary",
           "bs_cluster_instance", "bs_replay_config", "bs_scenario", "bs_replay_summary", "bs_replay_request",
           "bs_batch_record", "bs_idle_record", "bs_decision_record", "bs_replay_logs"]


def declared_functions() -> set:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(bs_[a-z0-9_]+)\s*\(", text))


def test_header_and_prototypes_agree():
    assert declared_functions() == set(_lib.exported_symbols())


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (bs_[a-z0-9_]+)", out))
    assert declared_functions() <= exported


def test_struct_layouts_match_c_compiler():
    src = "#include <stdio.h>\n#include <stddef.h>\n#include \"biscale_gpu.h\"\nint main(void){\n"
    for s in STRUCTS:
        src += f'printf("{s} %zu\\n", sizeof({s}));\n'
    src += 'printf("snap_waiting %zu\\n", offsetof(bs_snapshot, waiting));\n'
    src += 'printf("result_levels %zu\\n", offsetof(bs_mpc_result, levels));\nreturn 0;}\n'
    with tempfile.TemporaryDirectory() as d:
        cpath = Path(d) / "l.c"
        cpath.write_text(src)
        exe = Path(d) / "l"
        subprocess.run(["gcc", "-I", str(ROOT / "include"), str(cpath), "-o", str(exe)], check=True)
        sizes = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True,
                                                             text=True).stdout.splitlines())
    for s in STRUCTS:
        assert int(sizes[s]) == C.sizeof(getattr(A, s)), s
    assert int(sizes["snap_waiting"]) == A.bs_snapshot.waiting.offset
    assert int(sizes["result_levels"]) == A.bs_mpc_result.levels.offset


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2602_18755_b200 import pdsim as P
    with pytest.raises(P.CudaError):
        P.Device(0)


def test_kernels_are_sm100a_fp64_without_fma():
    """The shipped library carries sm_100a SASS, its kernels compute with
    DADD/DMUL, and no kernel contracts a multiply-add: every DFMA belongs to
    an IEEE double division -- the inline reciprocal refinement that follows
    its MUFU.RCP64H (7 DFMA) or the division's slow-path subroutine (its own
    MUFU.RCP64H) -- i.e. lies within 64 instructions after a MUFU.RCP64H, and
    each kernel has at most 7 DFMA per reciprocal plus 10 per slow path."""
    import re

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "DADD" in sass and "DMUL" in sass
    funcs, cur = {}, None
    for ln in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", ln)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur and re.search(r"/\*[0-9a-f]{4}\*/", ln):
            funcs[cur].append(ln)
    assert len(funcs) > 20
    for name, body in funcs.items():
        rcp = [i for i, ln in enumerate(body) if "MUFU.RCP64H" in ln]
        fma = [i for i, ln in enumerate(body) if re.search(r"\bDFMA\b", ln)]
        calls = sum(1 for ln in body if "RET.REL" in ln)
        for i in fma:
            assert any(0 < i - p <= 64 for p in rcp), f"{name}: DFMA outside a division at instruction {i}"
        assert len(fma) <= 7 * len(rcp) + 10 * max(1, calls), name


def test_pdsim_shim_compiles_against_reference():
    """include/biscale_gpu_pdsim.hpp compiles against the unmodified reference
    headers (the C++ drop-in a pdsim maintainer would include)."""
    import oracle
    if not (oracle.REFERENCE_ROOT / "proj" / "include").is_dir():
        pytest.skip("/root/reference absent")
    res = subprocess.run(["make", "-C", str(oracle.HERE), "replay"], capture_output=True, text=True)
    assert res.returncode == 0, res.stdout + res.stderr
    assert oracle.REPLAY_BIN.exists() and oracle.PLACEMENT_BIN.exists() and oracle.EXPERIMENT_BIN.exists() and \
        oracle.CSV_BIN.exists()
