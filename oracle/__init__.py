"""TEST INFRASTRUCTURE ONLY -- CPU checkers for the sm_100a path.

* ``load_oracle()``: the plain-C restatement (``oracle/biscale_oracle.c``).
* ``load_ref()``: the unmodified reference headers compiled by
  ``oracle/Makefile`` into ``oracle/_ref/libpdsim_ref.so``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

from paper_2602_18755_b200 import _abi as A

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libpdsim_ref.so"
REPLAY_BIN = HERE / "_ref" / "replay_parity"
PLACEMENT_BIN = HERE / "_ref" / "placement_parity"
EXPERIMENT_BIN = HERE / "_ref" / "experiment_parity"
CSV_BIN = HERE / "_ref" / "csv_parity"
REFERENCE_ROOT = Path("/root/reference")

_P = C.POINTER
_dp = A.dp

_COMMON = {
    "interpolate": None,
    "predict_batch": (C.c_int, [_P(A.bs_model_set), C.c_int, _P(A.bs_features), _P(C.c_int32), _dp, C.c_int, _dp,
                                _P(C.c_int32)]),
    "synth_model_set": (C.c_int, [C.c_int, _dp, C.c_int, _P(C.c_int32), C.c_int, _dp, _dp, _dp, _dp, _dp, _dp,
                                  _dp]),
    "project": (C.c_int, [_P(A.bs_mpc_config), _P(A.bs_scheduler_policy), _P(A.bs_snapshot),
                          _P(A.bs_projected_batch), _P(C.c_int32)]),
    "greedy": (C.c_int, [_P(A.bs_model_set), _P(A.bs_mpc_config), _P(A.bs_scheduler_policy), _P(A.bs_snapshot),
                         _P(A.bs_mpc_result)]),
    "exhaustive": (C.c_int, [_P(A.bs_model_set), _P(A.bs_mpc_config), _P(A.bs_scheduler_policy),
                             _P(A.bs_snapshot), _P(A.bs_mpc_result)]),
    "eval_codes": (C.c_int, [_P(A.bs_model_set), _P(A.bs_mpc_config), _P(A.bs_scheduler_policy),
                             _P(A.bs_snapshot), _P(C.c_uint64), C.c_int, _P(C.c_int32), _dp]),
    "decode_pick": (C.c_int, [_P(A.bs_model_set), _P(A.bs_decode_config), _P(A.bs_decode_query), C.c_int,
                              _P(A.bs_decode_result)]),
}


def build(quiet: bool = True) -> None:
    """Compile liboracle.so, and _ref/libpdsim_ref.so when /root/reference exists."""
    targets = ["oracle"]
    if (REFERENCE_ROOT / "proj" / "include").is_dir():
        targets.append("ref")
        if (HERE.parent / "paper_2602_18755_b200" / "libbiscale_gpu.so").exists():
            targets.append("replay")
    res = subprocess.run(["make", "-C", str(HERE), *targets], capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + res.stdout + res.stderr)


def _bind(path: Path, prefix: str, extra: dict) -> C.CDLL:
    if not path.exists():
        raise FileNotFoundError(f"{path} not built (run oracle.build() where /root/reference is present)")
    lib = C.CDLL(str(path))
    for name, proto in {**_COMMON, **extra}.items():
        if proto is None:
            continue
        fn = getattr(lib, prefix + name, None)
        if fn is None:
            continue
        fn.restype, fn.argtypes = proto
    lib.last_error = getattr(lib, prefix + "last_error")
    lib.last_error.restype = C.c_char_p
    return lib


_oracle = None
_ref = None


def load_oracle() -> C.CDLL:
    global _oracle
    if _oracle is None:
        _oracle = _bind(ORACLE_SO, "orc_", {
            "interpolate_one": None,
        })
        _oracle.orc_interpolate.restype = C.c_int
        _oracle.orc_interpolate.argtypes = [_P(A.bs_grid), _dp, _dp, _P(C.c_uint32)]
        _oracle.orc_ladder_select.restype = C.c_int
        _oracle.orc_ladder_select.argtypes = [_dp, C.c_int, C.c_int, _dp]
    return _oracle


class ref_runner_config(C.Structure):
    """RunnerConfig as a POD (ref_driver.h)."""
    _fields_ = [("slo", A.bs_slo), ("total_gpus", C.c_int32), ("n_tp", C.c_int32), ("tp_options", _P(C.c_int32)),
                ("ladder", _dp), ("n_ladder", C.c_int32), ("mpc_k", C.c_int32), ("scheduler", A.bs_scheduler_policy),
                ("alpha", C.c_double), ("peak_subwindow_s", C.c_double), ("search", A.bs_goodput_search),
                ("plan_policy", A.bs_scheduler_policy), ("rampup_s", C.c_double),
                ("switch_latency_ms", C.c_double), ("mpc_n", C.c_int32), ("_pad", C.c_int32),
                ("mpc_margin", C.c_double), ("kv_threshold", C.c_double), ("decode_margin", C.c_double)]


class ref_window_run(C.Structure):
    _fields_ = [("window", C.c_int32), ("policy", C.c_int32), ("gpus_used", C.c_int32), ("slo_pass", C.c_int32),
                ("objective_w", C.c_double), ("target_rps", C.c_double), ("report", A.bs_replay_summary)]


def load_ref() -> C.CDLL:
    global _ref
    if _ref is None:
        _ref = _bind(REF_SO, "ref_", {
            "predict": (C.c_int, [_P(A.bs_model_set), C.c_int, _P(A.bs_features), _P(C.c_int32), _dp, C.c_int, _dp,
                                  _P(C.c_int32)]),
            "greedy_batch": (C.c_int, [_P(A.bs_model_set), _P(A.bs_mpc_config), _P(A.bs_scheduler_policy),
                                       _P(A.bs_mpc_problem), C.c_int, _P(A.bs_mpc_result), C.c_int]),
            "exhaustive_batch": (C.c_int, [_P(A.bs_model_set), _P(A.bs_mpc_config), _P(A.bs_scheduler_policy),
                                           _P(A.bs_mpc_problem), C.c_int, _P(A.bs_mpc_result), C.c_int]),
            "tables": (C.c_int, [_P(A.bs_model_set), _P(A.bs_mpc_config), _P(A.bs_scheduler_policy),
                                 _P(A.bs_snapshot), _P(C.c_int32), _P(C.c_int32), _dp, _dp, _dp]),
            "gen_gamma_trace": (C.c_int, [C.c_double, C.c_double, C.c_double, _P(A.bs_length_dist), C.c_uint64,
                                          _P(A.bs_request), C.c_int64, _P(C.c_int64)]),
            "downsample_keep": (C.c_int, [_P(A.bs_trace), _P(A.bs_goodput_search), C.c_int64, C.c_int,
                                          _P(C.c_int32), _P(C.c_int64)]),
            "config_table": (C.c_int, [_P(A.bs_model_set), _P(A.bs_trace), _P(A.bs_slo), _P(A.bs_scheduler_policy),
                                       _P(A.bs_goodput_search), _P(A.bs_instance_config), C.c_int,
                                       _P(A.bs_table_entry)]),
            "simulate": (C.c_int, [_P(A.bs_model_set), _P(A.bs_trace), C.c_int, _P(A.bs_instance_config),
                                   _P(A.bs_scheduler_policy), _P(A.bs_slo), _P(A.bs_sim_summary)]),
            "solve_placement": (C.c_int, [_P(A.bs_table_entry), C.c_int, C.c_int, C.c_double, C.c_double,
                                          _P(C.c_int64), _dp, _P(C.c_int32)]),
            "solve_max_throughput": (C.c_int, [_P(A.bs_table_entry), C.c_int, C.c_int, C.c_double, C.c_double,
                                               C.c_double, _P(C.c_int64), _dp, _P(C.c_int32)]),
            "run_experiment": (C.c_int, [_P(A.bs_model_set), _P(A.bs_trace), C.c_double, _P(C.c_int32), C.c_int,
                                         _P(ref_runner_config), _P(ref_window_run), C.c_int, _P(C.c_int),
                                         _P(C.c_int32)]),
            "replay": (C.c_int, [_P(A.bs_model_set), _P(A.bs_model_set), _P(A.bs_replay_config), _P(A.bs_scenario),
                                 C.c_int, _P(A.bs_replay_summary), _P(A.bs_replay_request), _P(A.bs_replay_logs),
                                 C.c_int]),
        })
        _ref.ref_interpolate.restype = C.c_int
        _ref.ref_interpolate.argtypes = [_P(A.bs_grid), _dp, C.c_int, _dp, _P(C.c_uint32)]
        # the reference's predict has the batch signature under the name ref_predict
        _ref.ref_predict_batch = _ref.ref_predict
    return _ref


def ref_available() -> bool:
    return REF_SO.exists()
