"""Drop-in proof at the controller boundary: the reference's own, unmodified
simulate_cluster (simulator.hpp:758-893) driven by the GPU controllers of
include/biscale_gpu_pdsim.hpp must produce the same decision log, batch
records and request records, bit for bit, as with the reference's
TwoTierFactory (dvfs.hpp:370-390).  The binary is oracle/_ref/replay_parity
(built where /root/reference exists; it travels with the repo snapshot)."""
from __future__ import annotations

import json
import subprocess

import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("args", [
    ["--seed", "7", "--duration-s", "60", "--rps", "6"],
    ["--seed", "11", "--duration-s", "60", "--rps", "10", "--shape", "0.5", "--ttft", "400"],
    ["--seed", "3", "--duration-s", "40", "--rps", "12", "--prefill", "2", "--decode", "2", "--mpc-n", "5"],
])
def test_reference_simulator_with_gpu_controllers(args):
    if not oracle.REPLAY_BIN.exists():
        pytest.skip("replay_parity not built (needs /root/reference at build time)")
    res = subprocess.run([str(oracle.REPLAY_BIN), *args], capture_output=True, text=True, timeout=600)
    line = json.loads(res.stdout.strip().splitlines()[-1])
    assert line["checked"] and line["decisions"] > 100
    assert line["match"], line
    assert res.returncode == 0


@pytest.mark.parametrize("args", [
    ["--seed", "7", "--duration-s", "600", "--rps", "12", "--levels", "8"],
    ["--seed", "9", "--duration-s", "300", "--rps", "20", "--levels", "16", "--gpus", "8"],
    ["--seed", "5", "--duration-s", "300", "--rps", "6", "--levels", "5", "--ttft", "300", "--tpot", "60"],
])
def test_reference_planner_with_gpu_config_table(args):
    """build_config_table / solve_placement / solve_max_throughput through the
    C++ shim (pdsim_gpu::*) against the reference's own functions."""
    if not oracle.PLACEMENT_BIN.exists():
        pytest.skip("placement_parity not built (needs /root/reference at build time)")
    res = subprocess.run([str(oracle.PLACEMENT_BIN), *args], capture_output=True, text=True, timeout=900)
    line = json.loads(res.stdout.strip().splitlines()[-1])
    assert line["table_mismatch"] == 0, line
    assert line["match"], line
    assert res.returncode == 0


@pytest.mark.parametrize("args", [
    ["--seed", "7", "--minutes", "6", "--window-s", "120", "--rps", "8"],
    ["--seed", "12", "--minutes", "4", "--window-s", "60", "--rps", "14", "--shape", "0.5", "--gpus", "16"],
])
def test_reference_experiment_vs_gpu_experiment(args):
    """run_experiment (runner.hpp:155-172) vs pdsim_gpu::run_experiment (GPU
    plans + batched replay) through the C++ shim: plans, SimResult counters,
    MetricsReports and SLO verdicts run by run."""
    if not oracle.EXPERIMENT_BIN.exists():
        pytest.skip("experiment_parity not built (needs /root/reference at build time)")
    res = subprocess.run([str(oracle.EXPERIMENT_BIN), *args], capture_output=True, text=True, timeout=900)
    line = json.loads(res.stdout.strip().splitlines()[-1])
    assert line["runs"] > 0 and line["mismatch"] == 0, line
    assert line["match"], line
    assert res.returncode == 0


@pytest.mark.parametrize("args", [
    ["--seed", "7", "--minutes", "4", "--window-s", "120", "--rps", "8"],
    ["--seed", "21", "--minutes", "3", "--window-s", "60", "--rps", "12"],
])
def test_cli_output_files_identical(args, tmp_path):
    """The CLI run's files (plan JSON, requests / batches / decisions CSVs,
    report.csv; cli.hpp:371-378) written by the reference's own writers from
    the reference's run_experiment and from pdsim_gpu::run_experiment with
    records: byte-identical."""
    if not oracle.CSV_BIN.exists():
        pytest.skip("csv_parity not built (needs /root/reference at build time)")
    res = subprocess.run([str(oracle.CSV_BIN), *args, str(tmp_path)], capture_output=True, text=True, timeout=900)
    line = json.loads(res.stdout.strip().splitlines()[-1])
    assert line["files"] > 10 and line["bytes"] > 10000, line
    assert line["differ"] == 0 and line["match"], line
    assert res.returncode == 0
