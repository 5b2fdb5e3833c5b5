"""Host-side mirror of the reference's ``pdsim`` interface for the decision path.

Names, argument meanings and error behaviour follow
``/root/reference/proj/include/pdsim/*.hpp`` so code (and tests) written
against the reference read the same here.  The value types (ladders, grids,
snapshots, configs) are plain Python; every computation on the decision path
(prediction, projection, greedy/exhaustive MPC, decode pick) runs on the
B200 through the C ABI of ``libbiscale_gpu.so`` -- there is no CPU fallback.

Pure-Python pieces, which are input construction rather than decisions:
``FrequencyLadder.select`` (host-side, as in the reference's controller
constructor), ``BatchFeatures.from_lengths``, and ``synth_model`` /
``synth_model_set`` (grid generation; bit-identical to the reference, see
``tests/test_pdsim_host.py``).
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import threading
from dataclasses import dataclass, field
from typing import Optional, Sequence

from . import _abi
from ._lib import lib

# ---------------------------------------------------------------------------
# errors.hpp:10-56
# ---------------------------------------------------------------------------


class PdsimError(Exception):
    pass


class ParameterError(PdsimError, ValueError):
    pass


class ModelError(PdsimError, RuntimeError):
    pass


class SimulationError(PdsimError, RuntimeError):
    pass


class ConfigError(PdsimError, RuntimeError):
    pass


class AccountingError(PdsimError, RuntimeError):
    pass


class IoError(PdsimError, RuntimeError):
    pass


class InfeasibleError(PdsimError, RuntimeError):
    def __init__(self, constraint: str, what: str):
        super().__init__(what)
        self.constraint = constraint

    def binding_constraint(self) -> str:
        return self.constraint


class CudaError(PdsimError, RuntimeError):
    pass


_STATUS_EXC = {
    _abi.BS_PARAMETER_ERROR: ParameterError,
    _abi.BS_MODEL_ERROR: ModelError,
    _abi.BS_SIMULATION_ERROR: SimulationError,
    _abi.BS_CONFIG_ERROR: ConfigError,
    _abi.BS_ACCOUNTING_ERROR: AccountingError,
    _abi.BS_IO_ERROR: IoError,
    _abi.BS_CUDA_ERROR: CudaError,
}


def raise_status(code: int, message: str) -> None:
    if code == _abi.BS_OK:
        return
    if code == _abi.BS_INFEASIBLE_ERROR:
        constraint, _, what = message.partition("|")
        raise InfeasibleError(constraint, what)
    raise _STATUS_EXC.get(code, PdsimError)(message)


# ---------------------------------------------------------------------------
# perfmodel.hpp
# ---------------------------------------------------------------------------


class Phase(enum.IntEnum):
    prefill = 0
    decode = 1


@dataclass
class BatchFeatures:
    """perfmodel.hpp:30-51."""

    n_requests: int = 0
    sum_len: int = 0
    mean_len: float = 0.0
    std_len: float = 0.0

    @staticmethod
    def from_lengths(lengths: Sequence[int]) -> "BatchFeatures":
        f = BatchFeatures()
        f.n_requests = len(lengths)
        f.sum_len = int(sum(int(x) for x in lengths))
        if f.n_requests > 0:
            f.mean_len = float(f.sum_len) / float(f.n_requests)
            ss = 0.0
            for x in lengths:
                d = float(x) - f.mean_len
                ss += d * d
            f.std_len = math.sqrt(ss / float(f.n_requests))
        return f


@dataclass
class FrequencyLadder:
    """perfmodel.hpp:53-92."""

    freqs_mhz: list = field(default_factory=list)

    def validate(self) -> None:
        if not self.freqs_mhz:
            raise ParameterError("frequency ladder: empty")
        prev = 0.0
        for f in self.freqs_mhz:
            if not (f > prev):
                raise ParameterError("frequency ladder: must be strictly increasing and > 0")
            prev = f

    def min_mhz(self) -> float:
        return self.freqs_mhz[0]

    def max_mhz(self) -> float:
        return self.freqs_mhz[-1]

    def contains(self, f: float) -> bool:
        return any(g == f for g in self.freqs_mhz)

    def select(self, n: int) -> "FrequencyLadder":
        self.validate()
        if n == 0:
            raise ParameterError("frequency ladder: select(0)")
        size = len(self.freqs_mhz)
        if n >= size:
            return FrequencyLadder(list(self.freqs_mhz))
        if n == 1:
            return FrequencyLadder([self.freqs_mhz[-1]])
        out: list = []
        for i in range(n):
            idx = (i * (size - 1)) // (n - 1)
            if not out or out[-1] != self.freqs_mhz[idx]:
                out.append(self.freqs_mhz[idx])
        return FrequencyLadder(out)


kAxisSumLen = "sum_len"
kAxisNumRequests = "n_requests"
kAxisTp = "tp"
kAxisFreq = "freq_mhz"


@dataclass
class Axis:
    name: str
    knots: list


@dataclass
class NdGrid:
    """perfmodel.hpp:116-201 (values row-major, last axis fastest)."""

    axes: list = field(default_factory=list)
    values: list = field(default_factory=list)

    def expected_size(self) -> int:
        n = 1
        for a in self.axes:
            n *= len(a.knots)
        return n

    def validate_structure(self) -> None:
        if not self.axes:
            raise ModelError("grid: no axes")
        for a in self.axes:
            if not a.knots:
                raise ModelError(f"grid: axis '{a.name}' has no knots")
            for i in range(1, len(a.knots)):
                if a.knots[i] <= a.knots[i - 1]:
                    raise ModelError(f"grid: axis '{a.name}' knots not strictly increasing")
        if len(self.values) != self.expected_size():
            raise ModelError("grid: value count does not match axes")

    def interpolate(self, coords: Sequence[float], device: "Device | None" = None) -> float:
        """NdGrid::interpolate on the GPU (bs_grid_interpolate)."""
        if len(coords) != len(self.axes):
            raise ModelError("grid: coordinate rank mismatch")
        return (device or default_device()).interpolate(self, [list(coords)])[0][0]


@dataclass
class LatencyTable:
    phase: Phase = Phase.prefill
    grid: NdGrid = field(default_factory=NdGrid)
    synth: Optional[dict] = None


@dataclass
class PowerTable:
    phase: Phase = Phase.prefill
    grid: NdGrid = field(default_factory=NdGrid)
    synth: Optional[dict] = None


@dataclass
class TpEntry:
    tp: int = 1
    freqs_mhz: list = field(default_factory=list)
    idle_w: list = field(default_factory=list)


@dataclass
class IdlePowerModel:
    entries: list = field(default_factory=list)


@dataclass
class ModelSet:
    """perfmodel.hpp:494-503."""

    latency_prefill: LatencyTable = field(default_factory=LatencyTable)
    latency_decode: LatencyTable = field(default_factory=lambda: LatencyTable(Phase.decode))
    power_prefill: PowerTable = field(default_factory=PowerTable)
    power_decode: PowerTable = field(default_factory=lambda: PowerTable(Phase.decode))
    idle: IdlePowerModel = field(default_factory=IdlePowerModel)

    def latency(self, p: Phase) -> LatencyTable:
        return self.latency_prefill if p == Phase.prefill else self.latency_decode

    def power(self, p: Phase) -> PowerTable:
        return self.power_prefill if p == Phase.prefill else self.power_decode


class SynthFamily(enum.IntEnum):
    compute_bound = 0
    memory_bound = 1


@dataclass
class SynthOptions:
    """perfmodel.hpp:379-387."""

    lat_coef: float = 40.0
    power_a: float = 1e-7
    power_b: float = 10.0
    mem_knee_mhz: float = 1200.0
    idle_frac: float = 0.35
    sum_len_knots: list = field(default_factory=lambda: [16.0, 64.0, 256.0, 1024.0, 4096.0, 16384.0])
    n_request_knots: list = field(default_factory=lambda: [1.0, 2.0, 4.0, 8.0, 16.0, 32.0, 64.0, 128.0, 256.0])

    def as_array(self) -> list:
        return [self.lat_coef, self.power_a, self.power_b, self.mem_knee_mhz, self.idle_frac]


def _synth_latency_ms(family, opt, sum_len, tp, freq):  # perfmodel.hpp:397-405
    per_shard = sum_len / tp
    if family == SynthFamily.compute_bound:
        return opt.lat_coef * per_shard / freq
    eff = min(freq, opt.mem_knee_mhz)
    return opt.lat_coef * per_shard / eff


def _synth_power_w(family, opt, tp, freq):  # perfmodel.hpp:407-412
    if family == SynthFamily.compute_bound:
        per_gpu = opt.power_a * freq * freq * freq + opt.power_b
    else:
        per_gpu = opt.power_a * freq + opt.power_b
    return per_gpu * tp


def synth_model(family: SynthFamily, phase: Phase, ladder: FrequencyLadder, tp_list: Sequence[int],
                opt: SynthOptions | None = None) -> tuple:
    """perfmodel.hpp:418-491; returns (latency, power, idle)."""
    opt = opt or SynthOptions()
    ladder.validate()
    if not tp_list:
        raise ParameterError("synth_model: tp_list empty")
    for tp in tp_list:
        if tp < 1:
            raise ParameterError("synth_model: tp must be >= 1")
    tpk = sorted(set(float(t) for t in tp_list))
    meta = {"family": "compute-bound" if family == SynthFamily.compute_bound else "memory-bound",
            "lat_coef": opt.lat_coef, "power_a": opt.power_a, "power_b": opt.power_b,
            "mem_knee_mhz": opt.mem_knee_mhz if family == SynthFamily.memory_bound else 0.0,
            "idle_frac": opt.idle_frac}
    lat = LatencyTable(phase, NdGrid([Axis(kAxisSumLen, list(opt.sum_len_knots)),
                                      Axis(kAxisNumRequests, list(opt.n_request_knots)),
                                      Axis(kAxisTp, list(tpk)), Axis(kAxisFreq, list(ladder.freqs_mhz))], []), meta)
    for s in opt.sum_len_knots:
        for _ in opt.n_request_knots:
            for tp in tpk:
                for f in ladder.freqs_mhz:
                    lat.grid.values.append(_synth_latency_ms(family, opt, s, tp, f))
    if phase == Phase.prefill:
        pw = PowerTable(phase, NdGrid([Axis(kAxisSumLen, list(opt.sum_len_knots)), Axis(kAxisTp, list(tpk)),
                                       Axis(kAxisFreq, list(ladder.freqs_mhz))], []), meta)
        for _ in opt.sum_len_knots:
            for tp in tpk:
                for f in ladder.freqs_mhz:
                    pw.grid.values.append(_synth_power_w(family, opt, tp, f))
    else:
        pw = PowerTable(phase, NdGrid([Axis(kAxisSumLen, list(opt.sum_len_knots)),
                                       Axis(kAxisNumRequests, list(opt.n_request_knots)), Axis(kAxisTp, list(tpk)),
                                       Axis(kAxisFreq, list(ladder.freqs_mhz))], []), meta)
        for _ in opt.sum_len_knots:
            for _ in opt.n_request_knots:
                for tp in tpk:
                    for f in ladder.freqs_mhz:
                        pw.grid.values.append(_synth_power_w(family, opt, tp, f))
    idle = IdlePowerModel([TpEntry(int(tp), list(ladder.freqs_mhz),
                                   [opt.idle_frac * _synth_power_w(family, opt, tp, f) for f in ladder.freqs_mhz])
                           for tp in tpk])
    lat.grid.validate_structure()
    pw.grid.validate_structure()
    return lat, pw, idle


def synth_model_set(family: SynthFamily, ladder: FrequencyLadder, tp_list: Sequence[int],
                    prefill_opt: SynthOptions | None = None, decode_opt: SynthOptions | None = None) -> ModelSet:
    """perfmodel.hpp:505-516."""
    pl, pp, pi = synth_model(family, Phase.prefill, ladder, tp_list, prefill_opt)
    dl, dpw, _ = synth_model(family, Phase.decode, ladder, tp_list, decode_opt)
    return ModelSet(pl, dl, pp, dpw, pi)


# ---------------------------------------------------------------------------
# slo.hpp, scheduler.hpp, controller.hpp, dvfs.hpp value types
# ---------------------------------------------------------------------------


@dataclass
class SLOSpec:
    ttft_ms: float = 600.0
    tpot_ms: float = 100.0
    percentile: float = 0.99

    def validate(self) -> None:
        if self.ttft_ms <= 0.0 or self.tpot_ms <= 0.0:
            raise ParameterError("slo: bounds must be > 0")
        if self.percentile <= 0.0 or self.percentile > 1.0:
            raise ParameterError("slo: percentile must be in (0,1]")


@dataclass
class SchedulerPolicy:
    max_batch_tokens: int = 8192
    max_batch_requests: int = 256
    chunking: bool = True
    kv_capacity_tokens: int = 1000000

    def validate(self) -> None:
        if self.max_batch_tokens < 1:
            raise ParameterError("scheduler: max_batch_tokens must be >= 1")
        if self.max_batch_requests < 1:
            raise ParameterError("scheduler: max_batch_requests must be >= 1")
        if self.kv_capacity_tokens < 1:
            raise ParameterError("scheduler: kv_capacity_tokens must be >= 1")


@dataclass
class MpcConfig:
    horizon_K: int = 8
    ladder_N: int = 7
    ladder: FrequencyLadder = field(default_factory=FrequencyLadder)
    slo: SLOSpec = field(default_factory=SLOSpec)
    switch_latency_ms: float = 30.0
    margin: float = 0.05

    def validate(self) -> None:
        if self.horizon_K < 1:
            raise ParameterError("mpc: horizon_K must be >= 1")
        if self.ladder_N < 1:
            raise ParameterError("mpc: ladder_N must be >= 1")
        self.ladder.validate()
        self.slo.validate()
        if self.margin < 0.0:
            raise ParameterError("mpc: margin must be >= 0")

    def candidates(self) -> FrequencyLadder:
        return self.ladder.select(self.ladder_N)


@dataclass
class DecodePolicyConfig:
    tbt_slo_ms: float = 100.0
    kv_threshold: float = 0.9
    ladder: FrequencyLadder = field(default_factory=FrequencyLadder)
    margin: float = 0.0

    def validate(self) -> None:
        if self.tbt_slo_ms <= 0.0:
            raise ParameterError("decode policy: tbt_slo_ms must be > 0")
        if self.kv_threshold <= 0.0 or self.kv_threshold >= 1.0:
            raise ParameterError("decode policy: kv_threshold in (0,1)")
        self.ladder.validate()
        if self.margin < 0.0:
            raise ParameterError("decode policy: margin must be >= 0")


@dataclass
class KVCacheState:
    capacity_tokens: int = 0
    used_tokens: int = 0
    threshold: float = 0.9

    def utilization(self) -> float:
        return float(self.used_tokens) / float(self.capacity_tokens) if self.capacity_tokens > 0 else 0.0


@dataclass
class SnapshotWaiting:
    id: int = -1
    arrival_ms: float = 0.0
    total_len: int = 0
    remaining_len: int = 0


@dataclass
class SnapshotRunning:
    active: bool = False
    ids: list = field(default_factory=list)
    chunk_lens: list = field(default_factory=list)
    completes: list = field(default_factory=list)
    arrivals_ms: list = field(default_factory=list)
    work_remaining: float = 0.0
    elapsed_ms: float = 0.0
    features: BatchFeatures = field(default_factory=BatchFeatures)


@dataclass
class QueueSnapshot:
    now_ms: float = 0.0
    phase: Phase = Phase.prefill
    tp: int = 1
    current_freq_mhz: float = 0.0
    target_freq_mhz: float = 0.0
    waiting: list = field(default_factory=list)
    running: SnapshotRunning = field(default_factory=SnapshotRunning)
    decode_batch: BatchFeatures = field(default_factory=BatchFeatures)
    kv: KVCacheState = field(default_factory=KVCacheState)


@dataclass
class FreqDecision:
    freq_mhz: float = 0.0
    feasible: bool = True
    eval_count: int = 0


@dataclass
class ProjectedBatch:
    features: BatchFeatures
    work_fraction: float
    n_completing: int
    min_completing_arrival_ms: float


@dataclass
class FrequencyAssignment:
    freqs: list = field(default_factory=list)


@dataclass
class GreedyLevelStats:
    level: int = 0
    replaced_mhz: float = 0.0
    k_prime: int = 0
    mutations: int = 0
    feasible_mutations: int = 0
    accepted: bool = False


@dataclass
class GreedyResult:
    assignment: FrequencyAssignment = field(default_factory=FrequencyAssignment)
    feasible: bool = True
    eval_count: int = 0
    objective_w: float = 0.0
    levels: list = field(default_factory=list)
    # exhaustive-only extras
    feasible_count: int = 0
    trajectories: int = 0
    best_code: int = 0
    decision_freq_mhz: float = 0.0
    freq_index: list = field(default_factory=list)


@dataclass
class DecodeDecision:
    freq_mhz: float = 0.0
    eval_count: int = 0
    kv_override: bool = False


# ---------------------------------------------------------------------------
# marshalling into the C ABI
# ---------------------------------------------------------------------------


def _darr(vals) -> C.Array:
    return (C.c_double * max(1, len(vals)))(*[float(v) for v in vals])


def c_grid(grid: NdGrid, keep: list) -> _abi.bs_grid:
    g = _abi.bs_grid()
    if len(grid.axes) > _abi.BS_MAX_RANK:
        raise ParameterError(f"grid: rank {len(grid.axes)} exceeds {_abi.BS_MAX_RANK}")
    g.rank = len(grid.axes)
    for d, a in enumerate(grid.axes):
        g.role[d] = _abi.AXIS_ROLE.get(a.name, _abi.BS_AXIS_UNKNOWN)
        g.n_knots[d] = len(a.knots)
        arr = _darr(a.knots)
        keep.append(arr)
        g.knots[d] = C.cast(arr, _abi.dp)
    vals = _darr(grid.values)
    keep.append(vals)
    g.values = C.cast(vals, _abi.dp)
    return g


def c_model_set(m: ModelSet, keep: list) -> _abi.bs_model_set:
    for t in (m.latency_prefill, m.latency_decode, m.power_prefill, m.power_decode):
        t.grid.validate_structure()
    s = _abi.bs_model_set()
    s.latency_prefill = c_grid(m.latency_prefill.grid, keep)
    s.latency_decode = c_grid(m.latency_decode.grid, keep)
    s.power_prefill = c_grid(m.power_prefill.grid, keep)
    s.power_decode = c_grid(m.power_decode.grid, keep)
    n = len(m.idle.entries)
    ents = (_abi.bs_idle_entry * max(1, n))()
    for i, e in enumerate(m.idle.entries):
        fa, wa = _darr(e.freqs_mhz), _darr(e.idle_w)
        keep += [fa, wa]
        ents[i].tp = e.tp
        ents[i].n = len(e.freqs_mhz)
        ents[i].freqs_mhz = C.cast(fa, _abi.dp)
        ents[i].idle_w = C.cast(wa, _abi.dp)
    keep.append(ents)
    s.n_idle = n
    s.idle = C.cast(ents, C.POINTER(_abi.bs_idle_entry))
    return s


def c_policy(p: SchedulerPolicy) -> _abi.bs_scheduler_policy:
    c = _abi.bs_scheduler_policy()
    c.max_batch_tokens = p.max_batch_tokens
    c.max_batch_requests = p.max_batch_requests
    c.kv_capacity_tokens = p.kv_capacity_tokens
    c.chunking = 1 if p.chunking else 0
    return c


def c_mpc_config(cfg: MpcConfig, keep: list) -> _abi.bs_mpc_config:
    c = _abi.bs_mpc_config()
    c.horizon_K = cfg.horizon_K
    c.ladder_N = cfg.ladder_N
    lad = _darr(cfg.ladder.freqs_mhz)
    keep.append(lad)
    c.n_ladder = len(cfg.ladder.freqs_mhz)
    c.ladder_mhz = C.cast(lad, _abi.dp)
    c.ttft_ms = cfg.slo.ttft_ms
    c.tpot_ms = cfg.slo.tpot_ms
    c.percentile = cfg.slo.percentile
    c.switch_latency_ms = cfg.switch_latency_ms
    c.margin = cfg.margin
    return c


def c_decode_config(cfg: DecodePolicyConfig, keep: list) -> _abi.bs_decode_config:
    c = _abi.bs_decode_config()
    c.tbt_slo_ms = cfg.tbt_slo_ms
    c.kv_threshold = cfg.kv_threshold
    c.margin = cfg.margin
    lad = _darr(cfg.ladder.freqs_mhz)
    keep.append(lad)
    c.n_ladder = len(cfg.ladder.freqs_mhz)
    c.ladder_mhz = C.cast(lad, _abi.dp)
    return c


def c_snapshot(q: QueueSnapshot, keep: list) -> _abi.bs_snapshot:
    s = _abi.bs_snapshot()
    s.now_ms = q.now_ms
    s.current_freq_mhz = q.current_freq_mhz
    s.target_freq_mhz = q.target_freq_mhz
    s.tp = q.tp
    n = len(q.waiting)
    w = (_abi.bs_waiting * max(1, n))()
    for i, e in enumerate(q.waiting):
        w[i].id = e.id
        w[i].arrival_ms = e.arrival_ms
        w[i].total_len = e.total_len
        w[i].remaining_len = e.remaining_len
    keep.append(w)
    s.n_waiting = n
    s.waiting = C.cast(w, C.POINTER(_abi.bs_waiting))
    r = q.running
    s.running_active = 1 if r.active else 0
    if r.active:
        nr = len(r.completes)
        comp = (C.c_uint8 * max(1, nr))(*[1 if x else 0 for x in r.completes])
        arr = _darr(r.arrivals_ms)
        keep += [comp, arr]
        s.n_running = nr
        s.running_completes = C.cast(comp, C.POINTER(C.c_uint8))
        s.running_arrivals_ms = C.cast(arr, _abi.dp)
        s.running_work_remaining = r.work_remaining
        s.running_features.n_requests = r.features.n_requests
        s.running_features.sum_len = r.features.sum_len
    return s


def c_problems(snaps: Sequence[QueueSnapshot], cfg_index: Sequence[int] | None, keep: list):
    n = len(snaps)
    arr = (_abi.bs_mpc_problem * max(1, n))()
    for i, q in enumerate(snaps):
        arr[i].snap = c_snapshot(q, keep)
        arr[i].cfg_index = 0 if cfg_index is None else cfg_index[i]
    keep.append(arr)
    return arr


def greedy_from_c(r: _abi.bs_mpc_result) -> GreedyResult:
    g = GreedyResult()
    g.assignment = FrequencyAssignment([r.freqs_mhz[k] for k in range(r.K)])
    g.freq_index = [r.freq_index[k] for k in range(r.K)]
    g.feasible = bool(r.feasible)
    g.eval_count = r.eval_count
    g.objective_w = r.objective_w
    g.levels = [GreedyLevelStats(r.levels[i].level, r.levels[i].replaced_mhz, r.levels[i].k_prime,
                                 r.levels[i].mutations, r.levels[i].feasible_mutations, bool(r.levels[i].accepted))
                for i in range(max(0, r.n_levels))]
    g.feasible_count = r.feasible_count
    g.trajectories = r.trajectories
    g.best_code = r.best_code
    g.decision_freq_mhz = r.decision_freq_mhz
    return g


# ---------------------------------------------------------------------------
# device context
# ---------------------------------------------------------------------------


class Device:
    """One C-ABI context (one CUDA stream) on one GPU.  Not thread-safe."""

    def __init__(self, device: int = 0):
        self._lib = lib()
        h = _abi.ctx_t()
        rc = self._lib.bs_ctx_create(device, C.byref(h))
        if rc != _abi.BS_OK:
            raise CudaError(f"bs_ctx_create(device={device}) failed with status {rc}: no usable CUDA device "
                            "(the decision path has no CPU fallback)")
        self.handle = h
        self.device = device
        self._models: dict = {}

    def close(self) -> None:
        if self.handle:
            for mh, _ in self._models.values():
                self._lib.bs_models_free(self.handle, mh)
            self._models.clear()
            self._lib.bs_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def error(self) -> str:
        return (self._lib.bs_last_error(self.handle) or b"").decode()

    def check(self, rc: int) -> None:
        if rc != _abi.BS_OK:
            raise_status(rc, self.error())

    def kernel_launches(self) -> int:
        return int(self._lib.bs_ctx_kernel_launches(self.handle))

    def sm_count(self) -> int:
        d, s = C.c_int(), C.c_int()
        self.check(self._lib.bs_ctx_info(self.handle, C.byref(d), C.byref(s)))
        return s.value

    def models(self, m: ModelSet) -> C.c_void_p:
        """Device copy of a ModelSet (uploaded once per object, immutable)."""
        key = id(m)
        hit = self._models.get(key)
        if hit is not None and hit[1] is m:
            return hit[0]
        keep: list = []
        cm = c_model_set(m, keep)
        mh = _abi.models_t()
        self.check(self._lib.bs_models_upload(self.handle, C.byref(cm), C.byref(mh)))
        self._models[key] = (mh, m)
        return mh

    def set_exhaustive_limits(self, sweep3_min_prefixes: float = 0.0, level_cap: int = 0, final_cap: int = 0) -> None:
        """Exhaustive-MPC limits of this context (0 restores a default): the
        prefixes at depth K - 2 above which the sweep walks three levels
        (2^24), and the frontier capacities in entries (2.5e8 per BFS list,
        2e9 final).  Batches that exceed them are split; results never
        depend on them."""
        self.check(self._lib.bs_ctx_set_exhaustive_limits(self.handle, float(sweep3_min_prefixes), int(level_cap),
                                                          int(final_cap)))

    def interpolate(self, grid: NdGrid, coords: Sequence[Sequence[float]]) -> tuple:
        grid.validate_structure()
        keep: list = []
        g = c_grid(grid, keep)
        n = len(coords)
        flat = _darr([x for c in coords for x in c])
        out = (C.c_double * max(1, n))()
        cl = (C.c_uint32 * max(1, n))()
        self.check(self._lib.bs_grid_interpolate(self.handle, C.byref(g), flat, n, out, cl))
        return list(out[:n]), list(cl[:n])


_default_lock = threading.Lock()
_default: Device | None = None


def default_device() -> Device:
    global _default
    with _default_lock:
        if _default is None:
            _default = Device(0)
        return _default


# ---------------------------------------------------------------------------
# decision-path entry points (GPU)
# ---------------------------------------------------------------------------

_WHICH = {("latency", Phase.prefill): 0, ("latency", Phase.decode): 1,
          ("power", Phase.prefill): 2, ("power", Phase.decode): 3}


def _predict(kind: str, table, f: BatchFeatures, tp: int, freq_mhz: float, models: ModelSet,
             device: Device | None) -> float:
    dev = device or default_device()
    which = _WHICH[(kind, table.phase)]
    feats = (_abi.bs_features * 1)()
    feats[0].n_requests = f.n_requests
    feats[0].sum_len = f.sum_len
    tpa = (C.c_int32 * 1)(tp)
    fr = (C.c_double * 1)(freq_mhz)
    out = (C.c_double * 1)()
    st = (C.c_int32 * 1)()
    dev.check(dev._lib.bs_predict(dev.handle, dev.models(models), which, feats, tpa, fr, 1, out, st, None))
    if st[0] != _abi.BS_OK:
        raise ModelError(f"{kind} model returned non-positive value")
    return out[0]


def predict_latency(models: ModelSet, phase: Phase, f: BatchFeatures, tp: int, freq_mhz: float,
                    device: Device | None = None) -> float:
    """predict_latency (perfmodel.hpp:262-266) on the GPU."""
    return _predict("latency", models.latency(phase), f, tp, freq_mhz, models, device)


def predict_power(models: ModelSet, phase: Phase, f: BatchFeatures, tp: int, freq_mhz: float,
                  device: Device | None = None) -> float:
    """predict_power (perfmodel.hpp:268-272) on the GPU."""
    return _predict("power", models.power(phase), f, tp, freq_mhz, models, device)


def project_batches(q: QueueSnapshot, policy: SchedulerPolicy, horizon_K: int,
                    device: Device | None = None) -> list:
    """project_batches (dvfs.hpp:63-100) on the GPU; ProjectedBatch summaries."""
    if horizon_K < 1:
        raise ParameterError("project_batches: horizon_K must be >= 1")
    dev = device or default_device()
    keep: list = []
    cfg = MpcConfig(horizon_K=horizon_K, ladder_N=1, ladder=FrequencyLadder([1.0]))
    cc = c_mpc_config(cfg, keep)
    pc = c_policy(policy)
    probs = c_problems([q], None, keep)
    out = (_abi.bs_projected_batch * _abi.BS_MAX_K)()
    K = (C.c_int32 * 1)()
    st = (C.c_int32 * 1)()
    dev.check(dev._lib.bs_project_batches(dev.handle, C.byref(cc), C.byref(pc), 1, probs, 1, out, K, st))
    if st[0] != _abi.BS_OK:
        raise_status(st[0], "scheduler: queued request with no remaining tokens")
    res = []
    for k in range(K[0]):
        b = out[k]
        res.append(ProjectedBatch(BatchFeatures(b.features.n_requests, b.features.sum_len), b.work_fraction,
                                  b.n_completing, b.min_completing_arrival_ms))
    return res


def _mpc_batch(fn_name: str, snaps: Sequence[QueueSnapshot], cfgs: Sequence[MpcConfig],
               policies: Sequence[SchedulerPolicy], cfg_index: Sequence[int] | None, models: ModelSet,
               device: Device | None, code_slice: tuple | None = None) -> list:
    dev = device or default_device()
    for c in cfgs:
        c.validate()
    keep: list = []
    carr = (_abi.bs_mpc_config * len(cfgs))(*[c_mpc_config(c, keep) for c in cfgs])
    parr = (_abi.bs_scheduler_policy * len(policies))(*[c_policy(p) for p in policies])
    probs = c_problems(snaps, cfg_index, keep)
    n = len(snaps)
    out = (_abi.bs_mpc_result * max(1, n))()
    fn = getattr(dev._lib, fn_name)
    if code_slice is None:
        dev.check(fn(dev.handle, dev.models(models), carr, parr, len(cfgs), probs, n, out))
    else:
        digits, lo, hi = code_slice
        sl = _abi.bs_slice(int(digits), 0, int(lo), int(hi))
        dev.check(dev._lib.bs_mpc_exhaustive_slice(dev.handle, dev.models(models), carr, parr, len(cfgs), probs, n,
                                                   C.byref(sl), out))
    return [greedy_from_c(out[i]) for i in range(n)]


def greedy_freq_select(q: QueueSnapshot, cfg: MpcConfig, models: ModelSet, policy: SchedulerPolicy,
                       device: Device | None = None) -> GreedyResult:
    """greedy_freq_select (dvfs.hpp:185-259), one warp on the GPU."""
    return _mpc_batch("bs_mpc_greedy", [q], [cfg], [policy], None, models, device)[0]


def greedy_freq_select_batch(snaps: Sequence[QueueSnapshot], cfg: MpcConfig, models: ModelSet,
                             policy: SchedulerPolicy, device: Device | None = None) -> list:
    return _mpc_batch("bs_mpc_greedy", snaps, [cfg], [policy], None, models, device)


def exhaustive_freq_select(q: QueueSnapshot, cfg: MpcConfig, models: ModelSet, policy: SchedulerPolicy,
                           device: Device | None = None) -> GreedyResult:
    """Exhaustive MPC (the reference's oracle loop, tests/test_dvfs.cpp:74-94),
    argmin over (objective, lexicographic frequency vector)."""
    return _mpc_batch("bs_mpc_exhaustive", [q], [cfg], [policy], None, models, device)[0]


def exhaustive_freq_select_batch(snaps: Sequence[QueueSnapshot], cfg: MpcConfig, models: ModelSet,
                                 policy: SchedulerPolicy, device: Device | None = None,
                                 code_slice: tuple | None = None) -> list:
    """Exhaustive MPC of many decisions in one launch.  code_slice = (digits,
    lo, hi) restricts every decision to the assignments whose first `digits`
    digits (batch 0 most significant) lie in [lo, hi) (bs_mpc_exhaustive_slice);
    the decision is then the minimum over a partition's slices
    (sharding.argmin_over_ranks) and the feasible counts add up."""
    return _mpc_batch("bs_mpc_exhaustive", snaps, [cfg], [policy], None, models, device, code_slice)


def mpc_tables(q: QueueSnapshot, cfg: MpcConfig, models: ModelSet, policy: SchedulerPolicy,
               device: Device | None = None) -> tuple:
    """(lat, pow, energy) K x N tables of MpcEvaluator::eval (dvfs.hpp:150-160)."""
    dev = device or default_device()
    cfg.validate()
    keep: list = []
    cc = c_mpc_config(cfg, keep)
    pc = c_policy(policy)
    probs = c_problems([q], None, keep)
    K, nc = C.c_int32(), C.c_int32()
    size = _abi.BS_MAX_K * _abi.BS_MAX_CAND
    lat, pw, en = (C.c_double * size)(), (C.c_double * size)(), (C.c_double * size)()
    dev.check(dev._lib.bs_mpc_tables(dev.handle, dev.models(models), C.byref(cc), C.byref(pc), probs, C.byref(K),
                                     C.byref(nc), lat, pw, en))
    k, n = K.value, nc.value
    rows = lambda a: [[a[i * n + j] for j in range(n)] for i in range(k)]  # noqa: E731
    return rows(lat), rows(pw), rows(en)


def mpc_eval_codes(q: QueueSnapshot, cfg: MpcConfig, models: ModelSet, policy: SchedulerPolicy,
                   codes: Sequence[int], device: Device | None = None) -> tuple:
    """meets_slo + time_weighted_power of given assignments (batch 0 most significant)."""
    dev = device or default_device()
    cfg.validate()
    keep: list = []
    cc = c_mpc_config(cfg, keep)
    pc = c_policy(policy)
    probs = c_problems([q], None, keep)
    n = len(codes)
    ca = (C.c_uint64 * max(1, n))(*codes)
    feas = (C.c_int32 * max(1, n))()
    obj = (C.c_double * max(1, n))()
    dev.check(dev._lib.bs_mpc_eval_codes(dev.handle, dev.models(models), C.byref(cc), C.byref(pc), probs, ca, n,
                                         feas, obj))
    return [bool(x) for x in feas[:n]], list(obj[:n])


def select_decode_freq_ex(batch: BatchFeatures, kv: KVCacheState, cfg: DecodePolicyConfig, models: ModelSet,
                          tp: int, device: Device | None = None) -> DecodeDecision:
    """select_decode_freq_ex (dvfs.hpp:274-293), one warp on the GPU."""
    return select_decode_freq_batch([(batch, kv, tp)], cfg, models, device)[0]


def select_decode_freq(batch: BatchFeatures, kv: KVCacheState, cfg: DecodePolicyConfig, models: ModelSet, tp: int,
                       device: Device | None = None) -> float:
    return select_decode_freq_ex(batch, kv, cfg, models, tp, device).freq_mhz


def select_decode_freq_batch(queries: Sequence[tuple], cfg: DecodePolicyConfig, models: ModelSet,
                             device: Device | None = None) -> list:
    dev = device or default_device()
    cfg.validate()
    keep: list = []
    cc = c_decode_config(cfg, keep)
    n = len(queries)
    qa = (_abi.bs_decode_query * max(1, n))()
    for i, (b, kv, tp) in enumerate(queries):
        qa[i].batch.n_requests = b.n_requests
        qa[i].batch.sum_len = b.sum_len
        qa[i].kv_capacity_tokens = kv.capacity_tokens
        qa[i].kv_used_tokens = kv.used_tokens
        qa[i].tp = tp
        qa[i].cfg_index = 0
    out = (_abi.bs_decode_result * max(1, n))()
    dev.check(dev._lib.bs_decode_pick(dev.handle, dev.models(models), C.byref(cc), 1, qa, n, out))
    return [DecodeDecision(out[i].freq_mhz, out[i].eval_count, bool(out[i].kv_override)) for i in range(n)]


# ---------------------------------------------------------------------------
# controllers (dvfs.hpp:302-390): the FreqController / ControllerFactory shape
# ---------------------------------------------------------------------------


class FreqController:
    def decide(self, q: QueueSnapshot) -> FreqDecision:
        raise NotImplementedError

    def reacts_to_arrivals(self) -> bool:
        return False

    def on_arrival(self, q: QueueSnapshot) -> Optional[FreqDecision]:
        return None

    def predicted_latency_ms(self, f: BatchFeatures, phase: Phase, tp: int, freq_mhz: float) -> float:
        raise NotImplementedError

    def safety_margin(self) -> float:
        return 0.05

    def max_freq_mhz(self) -> float:
        raise NotImplementedError


class PrefillMpcController(FreqController):
    """PrefillMpcController (dvfs.hpp:302-339) backed by bs_mpc_greedy."""

    def __init__(self, cfg: MpcConfig, models: ModelSet, policy: SchedulerPolicy, device: Device | None = None):
        cfg.validate()
        policy.validate()
        self.cfg, self.models, self.policy = cfg, models, policy
        self.device = device or default_device()
        self._max = cfg.candidates().max_mhz()

    def decide(self, q: QueueSnapshot) -> FreqDecision:
        return self._run(q)

    def reacts_to_arrivals(self) -> bool:
        return True

    def on_arrival(self, q: QueueSnapshot) -> Optional[FreqDecision]:
        return self._run(q)

    def predicted_latency_ms(self, f, phase, tp, freq_mhz):
        return predict_latency(self.models, phase, f, tp, freq_mhz, self.device)

    def safety_margin(self) -> float:
        return self.cfg.margin

    def max_freq_mhz(self) -> float:
        return self._max

    def _run(self, q: QueueSnapshot) -> FreqDecision:
        g = greedy_freq_select(q, self.cfg, self.models, self.policy, self.device)
        return FreqDecision(g.decision_freq_mhz, g.feasible, g.eval_count)


class DecodePolicyController(FreqController):
    """DecodePolicyController (dvfs.hpp:341-365) backed by bs_decode_pick."""

    def __init__(self, cfg: DecodePolicyConfig, models: ModelSet, device: Device | None = None):
        cfg.validate()
        self.cfg, self.models = cfg, models
        self.device = device or default_device()
        self._safety = 0.05

    def decide(self, q: QueueSnapshot) -> FreqDecision:
        d = select_decode_freq_ex(q.decode_batch, q.kv, self.cfg, self.models, q.tp, self.device)
        return FreqDecision(d.freq_mhz, True, d.eval_count)

    def predicted_latency_ms(self, f, phase, tp, freq_mhz):
        return predict_latency(self.models, phase, f, tp, freq_mhz, self.device)

    def safety_margin(self) -> float:
        return self._safety

    def set_safety_margin(self, m: float) -> None:
        self._safety = m

    def max_freq_mhz(self) -> float:
        return self.cfg.ladder.max_mhz()


class TwoTierFactory:
    """TwoTierFactory (dvfs.hpp:370-390): MPC on prefill, TBT policy on decode."""

    def __init__(self, mpc: MpcConfig, decode: DecodePolicyConfig, controller_models: ModelSet,
                 policy: SchedulerPolicy, device: Device | None = None):
        self.mpc, self.decode, self.models, self.policy = mpc, decode, controller_models, policy
        self.device = device

    def make(self, phase: Phase, tp: int, base_freq_mhz: float) -> FreqController:
        if phase == Phase.prefill:
            return PrefillMpcController(self.mpc, self.models, self.policy, self.device)
        ctl = DecodePolicyController(self.decode, self.models, self.device)
        ctl.set_safety_margin(self.decode.margin if self.decode.margin > 0.0 else 0.05)
        return ctl


# ---------------------------------------------------------------------------
# workload.hpp: requests, traces, windows
# ---------------------------------------------------------------------------


@dataclass
class Request:
    id: int = 0
    arrival_ms: float = 0.0
    input_len: int = 1
    output_len: int = 1


@dataclass
class Trace:
    """workload.hpp:26-50."""

    requests: list = field(default_factory=list)
    duration_ms: float = 0.0
    seed: Optional[int] = None

    def duration_s(self) -> float:
        return self.duration_ms / 1000.0

    def mean_rps(self) -> float:
        if self.duration_ms <= 0.0:
            return 0.0
        return float(len(self.requests)) / self.duration_s()

    def validate(self) -> None:
        prev = 0.0
        for r in self.requests:
            if r.arrival_ms < 0.0:
                raise ParameterError("trace: negative arrival")
            if r.input_len < 1 or r.output_len < 1:
                raise ParameterError("trace: lengths must be >= 1")
            if r.arrival_ms < prev:
                raise ParameterError("trace: arrivals not sorted")
            prev = r.arrival_ms
        if self.requests and self.duration_ms < self.requests[-1].arrival_ms:
            raise ParameterError("trace: duration shorter than last arrival")


@dataclass
class Lognormal:
    input_mu: float = 6.0
    input_sigma: float = 0.5
    output_mu: float = 4.5
    output_sigma: float = 0.5


@dataclass
class LengthDistribution:
    """workload.hpp:54-85."""

    samples: list = field(default_factory=list)
    lognormal: Optional[Lognormal] = None

    @staticmethod
    def fixed(input_len: int, output_len: int) -> "LengthDistribution":
        return LengthDistribution([(input_len, output_len)])


def c_trace(t: Trace, keep: list) -> _abi.bs_trace:
    n = len(t.requests)
    arr = (_abi.bs_request * max(1, n))()
    for i, r in enumerate(t.requests):
        arr[i].id, arr[i].arrival_ms, arr[i].input_len, arr[i].output_len = r.id, r.arrival_ms, r.input_len, r.output_len
    keep.append(arr)
    ct = _abi.bs_trace()
    ct.n = n
    ct.requests = C.cast(arr, C.POINTER(_abi.bs_request))
    ct.duration_ms = t.duration_ms
    return ct


def c_lengths(d: LengthDistribution, keep: list) -> _abi.bs_length_dist:
    c = _abi.bs_length_dist()
    if d.samples:
        ins = (C.c_int64 * len(d.samples))(*[a for a, _ in d.samples])
        outs = (C.c_int64 * len(d.samples))(*[b for _, b in d.samples])
        keep += [ins, outs]
        c.n_samples = len(d.samples)
        c.sample_input = C.cast(ins, C.POINTER(C.c_int64))
        c.sample_output = C.cast(outs, C.POINTER(C.c_int64))
    elif d.lognormal is not None:
        c.lognormal = 1
        ln = d.lognormal
        c.input_mu, c.input_sigma, c.output_mu, c.output_sigma = ln.input_mu, ln.input_sigma, ln.output_mu, ln.output_sigma
    else:
        raise ParameterError("length distribution: no samples and no parametric form")
    return c


def gen_gamma_trace(mean_rps: float, shape: float, duration_ms: float, lengths: LengthDistribution,
                    seed: int) -> Trace:
    """gen_gamma_trace (workload.hpp:95-116): native host synthesis with the
    reference's own samplers (bit-identical)."""
    if mean_rps <= 0.0:
        raise ParameterError("gen_gamma_trace: mean_rps must be > 0")
    if shape <= 0.0:
        raise ParameterError("gen_gamma_trace: shape must be > 0")
    if duration_ms <= 0.0:
        raise ParameterError("gen_gamma_trace: duration_ms must be > 0")
    L = lib()
    keep: list = []
    cl = c_lengths(lengths, keep)
    n = C.c_int64()
    rc = L.bs_gen_gamma_trace(mean_rps, shape, duration_ms, C.byref(cl), seed, None, 0, C.byref(n))
    raise_status(rc, "gen_gamma_trace failed")
    out = (_abi.bs_request * max(1, n.value))()
    rc = L.bs_gen_gamma_trace(mean_rps, shape, duration_ms, C.byref(cl), seed, out, n.value, C.byref(n))
    raise_status(rc, "gen_gamma_trace failed")
    return Trace([Request(out[i].id, out[i].arrival_ms, out[i].input_len, out[i].output_len) for i in range(n.value)],
                 duration_ms, seed)


def split_windows(t: Trace, window_ms: float) -> list:
    """split_windows (workload.hpp:184-201)."""
    if window_ms <= 0.0:
        raise ParameterError("split_windows: window_ms must be > 0")
    n = max(1, int(math.ceil(t.duration_ms / window_ms)))
    wins = [Trace([], min(window_ms, t.duration_ms - float(i) * window_ms), t.seed) for i in range(n)]
    for r in t.requests:
        idx = int(r.arrival_ms / window_ms)
        if idx >= n:
            idx = n - 1
        wins[idx].requests.append(Request(r.id, r.arrival_ms - float(idx) * window_ms, r.input_len, r.output_len))
    return wins


def predict_next_window(history: Trace) -> Trace:
    """predict_next_window (workload.hpp:205-208): identity."""
    if not history.requests:
        raise ParameterError("predict_next_window: empty history")
    return history


# ---------------------------------------------------------------------------
# placement.hpp: config table, goodput search, ILP, window planning
# ---------------------------------------------------------------------------


@dataclass
class InstanceConfig:
    phase: Phase = Phase.prefill
    tp: int = 1
    base_freq_mhz: float = 0.0


@dataclass
class ConfigTableEntry:
    """placement.hpp:25-34."""

    config: InstanceConfig = field(default_factory=InstanceConfig)
    r_c: float = 0.0
    e_c: Optional[float] = None
    g_c: int = 0
    saturated: bool = False
    error: str = ""
    k_star: int = 0

    def usable(self) -> bool:
        return not self.error and self.r_c > 0.0 and self.e_c is not None


@dataclass
class GoodputSearch:
    tolerance_rps: float = 0.25
    probe_count: int = 1
    seed: int = 0x9e3779b97f4a7c15


@dataclass
class GoodputResult:
    r_c: float = 0.0
    k_star: int = 0
    saturated: bool = False


@dataclass
class ClusterInstance:
    config: InstanceConfig = field(default_factory=InstanceConfig)
    weight: float = 0.0


@dataclass
class PlacementProblem:
    table: list = field(default_factory=list)
    total_gpus: int = 0
    target_rps: float = 0.0
    alpha: float = 0.05


@dataclass
class PlacementPlan:
    counts: list = field(default_factory=list)
    table: list = field(default_factory=list)
    objective_w: float = 0.0
    target_rps: float = 0.0
    alpha: float = 0.0
    total_gpus: int = 0
    gpus_used: int = 0
    instances: list = field(default_factory=list)


def c_slo(s: SLOSpec) -> _abi.bs_slo:
    c = _abi.bs_slo()
    c.ttft_ms, c.tpot_ms, c.percentile = s.ttft_ms, s.tpot_ms, s.percentile
    return c


def c_search(s: GoodputSearch) -> _abi.bs_goodput_search:
    c = _abi.bs_goodput_search()
    c.tolerance_rps, c.probe_count, c.seed = s.tolerance_rps, s.probe_count, s.seed
    return c


def c_candidates(cands) -> C.Array:
    arr = (_abi.bs_instance_config * max(1, len(cands)))()
    for i, c in enumerate(cands):
        arr[i].phase, arr[i].tp, arr[i].base_freq_mhz = int(c.phase), c.tp, c.base_freq_mhz
    return arr


def entry_from_c(e: _abi.bs_table_entry) -> ConfigTableEntry:
    return ConfigTableEntry(InstanceConfig(Phase(e.config.phase), e.config.tp, e.config.base_freq_mhz), e.r_c,
                            e.e_c if e.has_e_c else None, e.g_c, bool(e.saturated),
                            e.error.decode() if e.error_code else "", e.k_star)


def c_table(table) -> C.Array:
    arr = (_abi.bs_table_entry * max(1, len(table)))()
    for i, e in enumerate(table):
        arr[i].config.phase, arr[i].config.tp, arr[i].config.base_freq_mhz = int(e.config.phase), e.config.tp, \
            e.config.base_freq_mhz
        arr[i].r_c = e.r_c
        arr[i].has_e_c = 1 if e.e_c is not None else 0
        arr[i].e_c = e.e_c if e.e_c is not None else 0.0
        arr[i].g_c = e.g_c
        arr[i].saturated = 1 if e.saturated else 0
        arr[i].error_code = 2 if e.error else 0
        arr[i].error = e.error.encode()[:95]
        arr[i].k_star = e.k_star
    return arr


def enumerate_candidates(ladder: FrequencyLadder, tp_options) -> list:
    """enumerate_candidates (placement.hpp:535-548): phase x tp x ladder."""
    ladder.validate()
    if not tp_options:
        raise ParameterError("candidates: tp_options empty")
    return [InstanceConfig(ph, tp, f) for ph in (Phase.prefill, Phase.decode) for tp in tp_options
            for f in ladder.freqs_mhz]


def build_config_table(candidates, base: Trace, slo: SLOSpec, models: ModelSet, policy: SchedulerPolicy,
                       search: GoodputSearch, parallel: bool = True, device: Device | None = None) -> list:
    """build_config_table (placement.hpp:240-260) on the GPU: every candidate's
    goodput probes in one grid, then the E_c runs."""
    if not candidates:
        raise ParameterError("config table: no candidates")
    dev = device or default_device()
    keep: list = []
    ct = c_trace(base, keep)
    cs, cp, cg = c_slo(slo), c_policy(policy), c_search(search)
    cands = c_candidates(candidates)
    out = (_abi.bs_table_entry * len(candidates))()
    dev.check(dev._lib.bs_goodput_table(dev.handle, dev.models(models), C.byref(ct), C.byref(cs), C.byref(cp),
                                        C.byref(cg), cands, len(candidates), out))
    return [entry_from_c(out[i]) for i in range(len(candidates))]


def evaluate_candidate(cfg: InstanceConfig, base: Trace, slo: SLOSpec, models: ModelSet, policy: SchedulerPolicy,
                       search: GoodputSearch, device: Device | None = None) -> ConfigTableEntry:
    """evaluate_candidate (placement.hpp:217-238)."""
    return build_config_table([cfg], base, slo, models, policy, search, device=device)[0]


def max_goodput(cfg: InstanceConfig, base: Trace, slo: SLOSpec, models: ModelSet, policy: SchedulerPolicy,
                search: GoodputSearch, device: Device | None = None) -> GoodputResult:
    """max_goodput (placement.hpp:154-199); ModelError propagates."""
    e = evaluate_candidate(cfg, base, slo, models, policy, search, device)
    if e.error and e.error != "no completed request at R_c":
        raise ModelError(e.error)
    return GoodputResult(e.r_c, e.k_star, e.saturated)


def downsample_keep(base: Trace, search: GoodputSearch, k: int, replicate: int = 0,
                    device: Device | None = None) -> list:
    """Indices kept by goodput_probe_trace (placement.hpp:145-149) on the GPU."""
    dev = device or default_device()
    keep: list = []
    ct = c_trace(base, keep)
    cg = c_search(search)
    idx = (C.c_int32 * max(1, len(base.requests)))()
    n = C.c_int64()
    dev.check(dev._lib.bs_downsample_keep(dev.handle, C.byref(ct), C.byref(cg), k, replicate, idx, C.byref(n)))
    return list(idx[:n.value])


def goodput_probe_trace(base: Trace, search: GoodputSearch, k: int, replicate: int = 0,
                        device: Device | None = None) -> Trace:
    idx = downsample_keep(base, search, k, replicate, device)
    return Trace([base.requests[i] for i in idx], base.duration_ms, None)


def derive_routing_weights(counts, table) -> list:
    """derive_routing_weights (placement.hpp:264-280)."""
    if len(counts) != len(table):
        raise ParameterError("weights: count/table size mismatch")
    phase_r = [0.0, 0.0]
    for n, e in zip(counts, table):
        phase_r[0 if e.config.phase == Phase.prefill else 1] += float(n) * e.r_c
    out = []
    for n, e in zip(counts, table):
        p = 0 if e.config.phase == Phase.prefill else 1
        for _ in range(n):
            out.append(ClusterInstance(e.config, e.r_c / phase_r[p]))
    return out


def _solve(fn_name: str, p: PlacementProblem, extra: tuple, device: Device | None) -> PlacementPlan:
    dev = device or default_device()
    n = len(p.table)
    tab = c_table(p.table)
    counts = (C.c_int64 * max(1, n))()
    obj = C.c_double()
    used = C.c_int32()
    rc = getattr(dev._lib, fn_name)(dev.handle, tab, n, p.total_gpus, p.target_rps, p.alpha, *extra, counts,
                                    C.byref(obj), C.byref(used))
    if rc != _abi.BS_OK:
        raise_status(rc, dev.error())
    plan = PlacementPlan(list(counts[:n]), list(p.table), obj.value, p.target_rps, p.alpha, p.total_gpus, used.value)
    if fn_name == "bs_placement_max_throughput":
        # the baseline plan carries the restricted table (placement.hpp:423-430, 486)
        restricted = []
        for e in p.table:
            if e.config.base_freq_mhz != extra[0]:
                e = ConfigTableEntry(e.config, 0.0, None, e.g_c, e.saturated, "below maximum frequency", e.k_star)
            restricted.append(e)
        plan.table = restricted
    plan.instances = derive_routing_weights(plan.counts, plan.table)
    return plan


def solve_placement_batch(problems: Sequence[tuple], device: Device | None = None) -> list:
    """Many placement problems in one device call (bs_placement_solve_batch):
    problems = [(PlacementProblem, max_freq_mhz or None)], None selecting
    solve_placement and a frequency solve_max_throughput.  Returns, per
    problem, its PlacementPlan or the exception the single call would raise."""
    dev = device or default_device()
    n = len(problems)
    arr = (_abi.bs_placement_problem * max(1, n))()
    keep: list = []
    for k, (p, mf) in enumerate(problems):
        tab = c_table(p.table)
        cnt = (C.c_int64 * max(1, len(p.table)))()
        keep += [tab, cnt]
        arr[k].table = C.cast(tab, C.c_void_p)
        arr[k].n = len(p.table)
        arr[k].total_gpus = p.total_gpus
        arr[k].target_rps = p.target_rps
        arr[k].alpha = p.alpha
        arr[k].max_throughput = 0 if mf is None else 1
        arr[k].max_freq_mhz = 0.0 if mf is None else mf
        arr[k].counts = cnt
    out = (_abi.bs_placement_solution * max(1, n))()
    dev.check(dev._lib.bs_placement_solve_batch(dev.handle, arr, n, out))
    res = []
    for k, (p, mf) in enumerate(problems):
        o = out[k]
        if o.status != _abi.BS_OK:
            try:
                raise_status(o.status, o.error.decode())
            except PdsimError as e:
                res.append(e)
            continue
        counts = [arr[k].counts[i] for i in range(len(p.table))]
        plan = PlacementPlan(counts, list(p.table), o.objective_w, p.target_rps, p.alpha, p.total_gpus, o.gpus_used)
        if mf is not None:
            plan.table = [e if e.config.base_freq_mhz == mf else
                          ConfigTableEntry(e.config, 0.0, None, e.g_c, e.saturated, "below maximum frequency", e.k_star)
                          for e in p.table]
        plan.instances = derive_routing_weights(plan.counts, plan.table)
        res.append(plan)
    return res


def solve_placement(p: PlacementProblem, device: Device | None = None) -> PlacementPlan:
    """solve_placement (placement.hpp:357-416): exact branch and bound."""
    return _solve("bs_placement_solve", p, (), device)


def solve_max_throughput(p: PlacementProblem, max_freq_mhz: float, device: Device | None = None) -> PlacementPlan:
    """solve_max_throughput (placement.hpp:421-499)."""
    return _solve("bs_placement_max_throughput", p, (max_freq_mhz,), device)


@dataclass
class PlanOptions:
    alpha: float = 0.05
    peak_subwindow_s: float = 10.0
    search: GoodputSearch = field(default_factory=GoodputSearch)
    policy: SchedulerPolicy = field(default_factory=SchedulerPolicy)
    probe_trace: Optional[Trace] = None
    parallel_table: bool = True


@dataclass
class WindowPlanResult:
    plan: PlacementPlan = field(default_factory=PlacementPlan)
    predicted_peak_rps: float = 0.0
    table: list = field(default_factory=list)


def peak_rps(t: Trace, subwindow_s: float) -> float:
    """peak_rps (placement.hpp:513-527)."""
    if not t.requests:
        raise ParameterError("peak_rps: empty trace")
    if subwindow_s <= 0.0:
        raise ParameterError("peak_rps: subwindow must be > 0")
    w_ms = subwindow_s * 1000.0
    n_windows = int(t.duration_ms / w_ms)
    if n_windows < 1:
        return t.mean_rps()
    counts = [0] * n_windows
    for r in t.requests:
        idx = int(r.arrival_ms / w_ms)
        if idx >= n_windows:
            continue
        counts[idx] += 1
    return float(max(counts)) / subwindow_s


def plan_window(history: Trace, total_gpus: int, slo: SLOSpec, models: ModelSet, ladder: FrequencyLadder,
                tp_options, opts: PlanOptions | None = None, device: Device | None = None) -> WindowPlanResult:
    """plan_window (placement.hpp:558-582) without the table cache file."""
    opts = opts or PlanOptions()
    history.validate()
    if not history.requests:
        raise ParameterError("plan_window: empty history")
    predicted = predict_next_window(history)
    res = WindowPlanResult()
    res.predicted_peak_rps = peak_rps(predicted, opts.peak_subwindow_s)
    probe = opts.probe_trace if opts.probe_trace is not None else predicted
    candidates = enumerate_candidates(ladder, tp_options)
    res.table = build_config_table(candidates, probe, slo, models, opts.policy, opts.search, opts.parallel_table, device)
    res.plan = solve_placement(PlacementProblem(res.table, total_gpus, res.predicted_peak_rps, opts.alpha), device)
    return res


# ---------------------------------------------------------------------------
# simulator.hpp:741-893 + metrics.hpp:71-156: cluster replay on the device
# ---------------------------------------------------------------------------


@dataclass
class ClusterSpec:
    """ClusterSpec (simulator.hpp:746-756): index = instance id."""

    instances: list = field(default_factory=list)


@dataclass
class SimOptions:
    """SimOptions (simulator.hpp:126-130)."""

    switch_latency_ms: float = 30.0
    horizon_ms: float = -1.0


@dataclass
class MetricsReport:
    """MetricsReport (metrics.hpp:104-119); absent optionals are None."""

    p99_ttft_ms: Optional[float] = None
    p99_mean_tpot_ms: Optional[float] = None
    energy_per_first_token_j: Optional[float] = None
    energy_per_output_token_j: Optional[float] = None
    avg_power_prefill_w: float = 0.0
    avg_power_decode_w: float = 0.0
    prefill_energy_j: float = 0.0
    decode_energy_j: float = 0.0
    span_ms: float = 0.0
    completed_requests: int = 0
    generated_tokens: int = 0
    ttft_violations: int = 0
    tpot_violations: int = 0
    window_id: str = ""
    system: str = ""


@dataclass
class ReplayScenario:
    """One simulate_cluster call (run_policy, runner.hpp:112-122) followed by
    make_report(trim_steady_state(sim, rampup_s), slo)."""

    trace: Trace
    cluster: ClusterSpec
    policy: SchedulerPolicy = field(default_factory=SchedulerPolicy)
    controllers: Optional[TwoTierFactory] = None  # None: fixed base frequencies
    opts: SimOptions = field(default_factory=SimOptions)
    slo: SLOSpec = field(default_factory=SLOSpec)
    rampup_s: float = 30.0


@dataclass
class ReplayResult:
    status: int = 0
    horizon_ms: float = 0.0
    completed_requests: int = 0
    generated_tokens: int = 0
    n_batches: int = 0
    n_idles: int = 0
    n_decisions: int = 0
    decisions_by_trigger: tuple = (0, 0, 0)
    report: MetricsReport = field(default_factory=MetricsReport)
    requests: Optional[list] = None   # bs_replay_request per trace request (trace order)
    batches: Optional[list] = None    # bs_batch_record, SimResult order
    idles: Optional[list] = None
    decisions: Optional[list] = None


def _opt(has: int, v: float) -> Optional[float]:
    return float(v) if has else None


def c_replay_config(s: ReplayScenario, keep: list) -> _abi.bs_replay_config:
    c = _abi.bs_replay_config()
    f = s.controllers
    if f is not None:
        c.mpc = c_mpc_config(f.mpc, keep)
        c.decode = c_decode_config(f.decode, keep)
        c.controlled = 1
    c.policy = c_policy(s.policy)
    c.slo = c_slo(s.slo)
    c.switch_latency_ms = s.opts.switch_latency_ms
    c.horizon_ms = s.opts.horizon_ms
    c.rampup_s = s.rampup_s
    return c


def summary_from_c(o: _abi.bs_replay_summary) -> ReplayResult:
    rep = MetricsReport(_opt(o.has_p99_ttft, o.p99_ttft_ms), _opt(o.has_p99_tpot, o.p99_mean_tpot_ms),
                        _opt(o.has_e_first, o.energy_per_first_token_j),
                        _opt(o.has_e_output, o.energy_per_output_token_j), o.avg_power_prefill_w,
                        o.avg_power_decode_w, o.prefill_energy_j, o.decode_energy_j, o.span_ms, o.report_completed,
                        o.report_generated, o.ttft_violations, o.tpot_violations)
    return ReplayResult(o.status, o.horizon_ms, o.completed_requests, o.generated_tokens, o.n_batches, o.n_idles,
                        o.n_decisions, tuple(o.decisions_by_trigger), rep)


def c_replay_inputs(scenarios: Sequence[ReplayScenario], keep: list) -> tuple:
    """(bs_replay_config[n], bs_scenario[n], total requests): one configuration per scenario."""
    n = len(scenarios)
    cfgs = (_abi.bs_replay_config * n)()
    scs = (_abi.bs_scenario * n)()
    total = 0
    for i, s in enumerate(scenarios):
        cfgs[i] = c_replay_config(s, keep)
        scs[i].trace = c_trace(s.trace, keep)
        inst = (_abi.bs_cluster_instance * max(1, len(s.cluster.instances)))()
        for j, ci in enumerate(s.cluster.instances):
            inst[j].config.phase, inst[j].config.tp = int(ci.config.phase), ci.config.tp
            inst[j].config.base_freq_mhz, inst[j].weight = ci.config.base_freq_mhz, ci.weight
        keep.append(inst)
        scs[i].instances = C.cast(inst, C.POINTER(_abi.bs_cluster_instance))
        scs[i].n_instances = len(s.cluster.instances)
        scs[i].config = i
        total += len(s.trace.requests)
    return cfgs, scs, total


def c_replay_logs(scenarios: Sequence[ReplayScenario], keep: list) -> C.Array:
    lg = (_abi.bs_replay_logs * len(scenarios))()
    for i, s in enumerate(scenarios):
        cap = sum(r.output_len for r in s.trace.requests) + 4 * len(s.trace.requests) + 1024
        for name, typ, cap_name in (("batches", _abi.bs_batch_record, "batch_cap"),
                                    ("idles", _abi.bs_idle_record, "idle_cap"),
                                    ("decisions", _abi.bs_decision_record, "decision_cap")):
            arr = (typ * cap)()
            keep.append(arr)
            setattr(lg[i], name, C.cast(arr, C.POINTER(typ)))
            setattr(lg[i], cap_name, cap)
    return lg


def replay(scenarios: Sequence[ReplayScenario], models: ModelSet, device: Device | None = None,
           requests: bool = False, logs: bool = False, raise_errors: bool = True) -> list:
    """simulate_cluster + trim_steady_state + make_report for every scenario
    in one device call (bs_replay).  All scenarios share the simulator's
    ModelSet and the controllers' ModelSet (TwoTierFactory.models)."""
    dev = device or default_device()
    n = len(scenarios)
    if n == 0:
        return []
    ctl = None
    for s in scenarios:
        if s.controllers is not None:
            if ctl is not None and s.controllers.models is not ctl:
                raise ParameterError("replay: one controller ModelSet per call")
            ctl = s.controllers.models
    keep: list = []
    cfgs, scs, total = c_replay_inputs(scenarios, keep)
    out = (_abi.bs_replay_summary * n)()
    reqs = (_abi.bs_replay_request * max(1, total))() if requests else None
    lg = c_replay_logs(scenarios, keep) if logs else None
    mh = dev.models(models)
    ch = dev.models(ctl) if ctl is not None else mh
    rc = dev._lib.bs_replay(dev.handle, mh, ch, cfgs, n, scs, n, out, reqs, lg)
    if rc != _abi.BS_OK and (raise_errors or rc == _abi.BS_CUDA_ERROR):
        raise_status(rc, dev.error())
    res = [summary_from_c(out[i]) for i in range(n)]
    q = 0
    for i, s in enumerate(scenarios):
        if requests:
            res[i].requests = [reqs[q + k] for k in range(len(s.trace.requests))]
            q += len(s.trace.requests)
        if logs:
            L = lg[i]
            if L.n_batches > L.batch_cap or L.n_idles > L.idle_cap or L.n_decisions > L.decision_cap:
                raise SimulationError("replay: log capacity exceeded")
            res[i].batches = [L.batches[k] for k in range(L.n_batches)]
            res[i].idles = [L.idles[k] for k in range(L.n_idles)]
            res[i].decisions = [L.decisions[k] for k in range(L.n_decisions)]
    return res


def simulate_cluster_report(trace: Trace, cluster: ClusterSpec, policy: SchedulerPolicy, models: ModelSet,
                            controllers: Optional[TwoTierFactory] = None, opts: SimOptions | None = None,
                            slo: SLOSpec | None = None, rampup_s: float = 30.0,
                            device: Device | None = None) -> ReplayResult:
    """One scenario of replay(): run_policy (runner.hpp:112-122) + the
    window report (runner.hpp:131-133)."""
    return replay([ReplayScenario(trace, cluster, policy, controllers, opts or SimOptions(), slo or SLOSpec(),
                                  rampup_s)], models, device, requests=True)[0]


# ---------------------------------------------------------------------------
# runner.hpp: policies, window plans, run_experiment
# ---------------------------------------------------------------------------


class Policy(enum.IntEnum):
    maxfreq_distserve = 0
    place_only = 1
    two_tier = 2


POLICY_NAMES = {Policy.maxfreq_distserve: "maxfreq-distserve", Policy.place_only: "place-only",
                Policy.two_tier: "two-tier"}


@dataclass
class RunnerConfig:
    """RunnerConfig (runner.hpp:39-86)."""

    slo: SLOSpec = field(default_factory=SLOSpec)
    total_gpus: int = 8
    tp_options: list = field(default_factory=lambda: [1])
    ladder: FrequencyLadder = field(default_factory=FrequencyLadder)
    scheduler: SchedulerPolicy = field(default_factory=SchedulerPolicy)
    plan: PlanOptions = field(default_factory=PlanOptions)
    rampup_s: float = 30.0
    switch_latency_ms: float = 30.0
    mpc_horizon_k: int = 8
    mpc_ladder_n: int = 7
    mpc_margin: float = 0.05
    kv_threshold: float = 0.9
    decode_margin: float = 0.05

    def mpc_config(self) -> MpcConfig:
        return MpcConfig(self.mpc_horizon_k, self.mpc_ladder_n, self.ladder, self.slo, self.switch_latency_ms,
                         self.mpc_margin)

    def decode_config(self) -> DecodePolicyConfig:
        return DecodePolicyConfig(self.slo.tpot_ms, self.kv_threshold, self.ladder, self.decode_margin)

    def validate(self) -> None:
        self.slo.validate()
        self.ladder.validate()
        self.scheduler.validate()
        if self.total_gpus <= 0:
            raise ParameterError("total_gpus must be positive")
        if not self.tp_options:
            raise ParameterError("tp_options must not be empty")
        if any(tp <= 0 for tp in self.tp_options):
            raise ParameterError("tp options must be positive")
        if self.rampup_s < 0.0:
            raise ParameterError("rampup_s must be >= 0")
        self.mpc_config().validate()
        self.decode_config().validate()


@dataclass
class WindowPlans:
    target_rps: float = 0.0
    table: list = field(default_factory=list)
    ilp: PlacementPlan = field(default_factory=PlacementPlan)
    maxfreq: PlacementPlan = field(default_factory=PlacementPlan)


@dataclass
class WindowRun:
    window_index: int = 0
    policy: Policy = Policy.maxfreq_distserve
    plan: PlacementPlan = field(default_factory=PlacementPlan)
    result: ReplayResult = field(default_factory=ReplayResult)
    report: MetricsReport = field(default_factory=MetricsReport)
    slo_pass: bool = False


@dataclass
class ExperimentResult:
    runs: list = field(default_factory=list)
    reports: list = field(default_factory=list)
    two_tier_slo_pass: bool = True
    seconds: dict = field(default_factory=dict)  # wall time of the planning and replay phases


def plan_window_policies(history: Trace, cfg: RunnerConfig, models: ModelSet,
                         device: Device | None = None) -> WindowPlans:
    """plan_window_policies (runner.hpp:98-110): one GPU config table shared
    by the ILP plan and the max-frequency baseline."""
    cfg.validate()
    wp = plan_window(history, cfg.total_gpus, cfg.slo, models, cfg.ladder, cfg.tp_options, cfg.plan, device)
    out = WindowPlans(wp.predicted_peak_rps, wp.table, wp.plan)
    out.maxfreq = solve_max_throughput(PlacementProblem(out.table, cfg.total_gpus, out.target_rps, cfg.plan.alpha),
                                       cfg.ladder.max_mhz(), device)
    return out


def _scenario_for(window: Trace, plan: PlacementPlan, policy: Policy, cfg: RunnerConfig,
                  models: ModelSet) -> ReplayScenario:
    """run_policy (runner.hpp:112-122) as a replay scenario."""
    fac = None
    if policy == Policy.two_tier:
        fac = TwoTierFactory(cfg.mpc_config(), cfg.decode_config(), models, cfg.scheduler)
    return ReplayScenario(window, ClusterSpec(list(plan.instances)), cfg.scheduler, fac,
                          SimOptions(cfg.switch_latency_ms), cfg.slo, cfg.rampup_s)


_ctx_pools: dict = {}


def _context_pool(device: int, n: int) -> list:
    """n library contexts on one GPU (each its own stream), reused across calls."""
    with _default_lock:
        pool = _ctx_pools.setdefault(device, [])
        while len(pool) < n:
            pool.append(Device(device))
        return pool[:n]


def build_config_tables(bases, candidates, slo: SLOSpec, models: ModelSet, policy: SchedulerPolicy,
                        search: GoodputSearch, device: Device | None = None) -> list:
    """build_config_table for several probe traces (e.g. consecutive windows)
    in one device call (bs_goodput_tables): every table's probes share one
    grid, long probes first, so a stream of tables is bound by the device's
    throughput rather than by each table's longest probe in turn."""
    bases = list(bases)
    if not candidates:
        raise ParameterError("config table: no candidates")
    if not bases:
        return []
    dev = device or default_device()
    keep: list = []
    trs = (_abi.bs_trace * len(bases))()
    for i, b in enumerate(bases):
        trs[i] = c_trace(b, keep)
    cs, cp, cg = c_slo(slo), c_policy(policy), c_search(search)
    cands = c_candidates(candidates)
    n = len(candidates)
    out = (_abi.bs_table_entry * (n * len(bases)))()
    dev.check(dev._lib.bs_goodput_tables(dev.handle, dev.models(models), trs, len(bases), C.byref(cs), C.byref(cp),
                                         C.byref(cg), cands, n, out))
    return [[entry_from_c(out[t * n + i]) for i in range(n)] for t in range(len(bases))]


def run_experiment(trace: Trace, window_ms: float, policies, cfg: RunnerConfig, models: ModelSet,
                   device: Device | None = None) -> ExperimentResult:
    """run_experiment (runner.hpp:155-172): window w is planned from window
    w-1 (the first from itself): every window's config table in ONE
    bs_goodput_tables call, every window's ILP and max-throughput baseline in
    ONE bs_placement_solve_batch call, then every (window, policy) replay in
    ONE bs_replay call (windows are independent once planned).  Reports, SLO verdicts and their order follow
    the reference."""
    dev = device or default_device()
    cfg.validate()
    policies = list(policies)
    if not policies:
        raise ParameterError("no policies selected")
    windows = split_windows(trace, window_ms)
    # windows are planned independently (window w from window w - 1): one
    # context (own CUDA stream) per worker thread, so the config tables'
    # kernels overlap on the GPU and the critical path is the longest table,
    # not their sum (the reference parallelises inside build_config_table)
    import time as _time

    t0 = _time.perf_counter()
    histories = [windows[0] if w == 0 else windows[w - 1] for w in range(len(windows))]
    # plan_window (placement.hpp:558-582) for every window, with all the
    # windows' config tables in ONE device call
    for h in histories:
        h.validate()
        if not h.requests:
            raise ParameterError("plan_window: empty history")
    opts = cfg.plan
    predicted = [predict_next_window(h) for h in histories]
    probes = [opts.probe_trace if opts.probe_trace is not None else p for p in predicted]
    candidates = enumerate_candidates(cfg.ladder, cfg.tp_options)
    tables = build_config_tables(probes, candidates, cfg.slo, models, opts.policy, opts.search, dev)
    # every window's ILP and max-throughput baseline in ONE device call
    # (bs_placement_solve_batch); errors surface in the reference's order
    # (window by window, solve_placement before solve_max_throughput)
    targets = [peak_rps(p, opts.peak_subwindow_s) for p in predicted]
    probs = []
    for table, target in zip(tables, targets):
        probs.append((PlacementProblem(table, cfg.total_gpus, target, opts.alpha), None))
        probs.append((PlacementProblem(table, cfg.total_gpus, target, opts.alpha), cfg.ladder.max_mhz()))
    solved = solve_placement_batch(probs, dev)
    for x in solved:
        if isinstance(x, Exception):
            raise x
    plans = [WindowPlans(targets[w], tables[w], solved[2 * w], solved[2 * w + 1]) for w in range(len(tables))]
    scs, keys = [], []
    for w, win in enumerate(windows):
        for pol in policies:
            plan = plans[w].maxfreq if pol == Policy.maxfreq_distserve else plans[w].ilp
            scs.append(_scenario_for(win, plan, pol, cfg, models))
            keys.append((w, pol, plan))
    t1 = _time.perf_counter()
    results = replay(scs, models, dev)
    out = ExperimentResult()
    out.seconds = {"plan": t1 - t0, "replay": _time.perf_counter() - t1}
    for (w, pol, plan), res in zip(keys, results):
        rep = res.report
        rep.window_id, rep.system = f"w{w}", POLICY_NAMES[pol]
        ok = (rep.p99_ttft_ms is None or rep.p99_ttft_ms <= cfg.slo.ttft_ms) and \
             (rep.p99_mean_tpot_ms is None or rep.p99_mean_tpot_ms <= cfg.slo.tpot_ms)
        if pol == Policy.two_tier and not ok:
            out.two_tier_slo_pass = False
        out.reports.append(rep)
        out.runs.append(WindowRun(w, pol, plan, res, rep, ok))
    return out
