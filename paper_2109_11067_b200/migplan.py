"""Python mirror of the reference's `migplan` API for the optimizer hot path.

Names, argument meaning and error behaviour follow the reference headers
(`proj/include/migplan/{core,mig_rules,config_enum,greedy,mcts,ga,bench}.hpp`); every
call that does work goes through the C-ABI (`include/migplan_b200.h`) of a
*backend* library.  The default backend is the product —
`_native/libmigplan_b200.so`, CUDA sm_100a — and there is no fallback: if the
library is missing or no CUDA device is usable, creating a context raises.

Tests pass `backend=Backend.load(<oracle or reference .so>)` to run the very same
calls on the CPU checkers.
"""
from __future__ import annotations

import ctypes as C
import json
import math
import os
import threading
from dataclasses import dataclass, field
from typing import Callable, Iterable, Sequence

from . import abi

# ---------------------------------------------------------------- errors (util.hpp:12-25)


class SchemaError(RuntimeError):
    """Malformed input (util.hpp:12-15; CLI exit 2)."""


class PlanningError(RuntimeError):
    """Infeasible workload / planning failure (util.hpp:17-20; CLI exit 1)."""


class ExecutionError(RuntimeError):
    """Simulator precondition failure (util.hpp:22-25)."""


class DeviceError(RuntimeError):
    """CUDA failure inside the product library."""


kSatisfyEps = 1e-9  # core.hpp:18
kInstanceSlices = (1, 2, 3, 4, 7)  # core.hpp:21


def valid_slices(s: int) -> bool:
    return s in kInstanceSlices


# ---------------------------------------------------------------- backend


class Backend:
    """A loaded implementation of include/migplan_b200.h."""

    _lock = threading.Lock()
    _product: "Backend | None" = None

    def __init__(self, lib: C.CDLL, path: str):
        self.lib = lib
        self.path = path
        self.name = lib.mig_impl_name().decode()

    @classmethod
    def load(cls, path: str, extras: dict | None = None) -> "Backend":
        return cls(abi.bind(path, extras), path)

    @classmethod
    def product(cls) -> "Backend":
        with cls._lock:
            if cls._product is None:
                from . import native_library_path

                cls._product = cls.load(native_library_path())
            return cls._product

    def check(self, rc: int) -> None:
        if rc == abi.MIG_OK:
            return
        msg = (self.lib.mig_last_error() or b"").decode(errors="replace")
        if rc == abi.MIG_ERR_PLANNING:
            raise PlanningError(msg)
        if rc == abi.MIG_ERR_SCHEMA:
            raise SchemaError(msg)
        if rc == abi.MIG_ERR_DEVICE:
            raise DeviceError(msg)
        raise ValueError(msg)


def _backend(b: Backend | None) -> Backend:
    return b if b is not None else Backend.product()


# ---------------------------------------------------------------- domain types (core.hpp)


@dataclass(frozen=True, order=True)
class Placement:  # core.hpp:41-46
    slices: int = 1
    start_slot: int = 0


def make_placement(slices: int, start_slot: int) -> Placement:  # core.hpp:48-54
    if not valid_slices(slices):
        raise PlanningError(f"instance size {slices}/7 does not exist")
    if start_slot < 0 or start_slot + slices > 7:
        raise PlanningError(f"placement {slices}@{start_slot} exceeds the 7-slot budget")
    return Placement(slices, start_slot)


@dataclass(frozen=True)
class ProfileEntry:  # core.hpp:57-61
    batch: int = 1
    throughput_rps: float = 0.0
    p90_ms: float = 0.0


@dataclass
class ModelProfile:  # core.hpp:64-76
    model_name: str
    entries: dict = field(default_factory=dict)  # size -> [ProfileEntry] sorted by batch

    def find(self, size: int, batch: int) -> ProfileEntry | None:
        for e in self.entries.get(size, []):
            if e.batch == batch:
                return e
        return None


@dataclass(frozen=True)
class ServiceSpec:  # core.hpp:113-118
    service_id: str
    model_name: str
    required_rps: float = 0.0
    max_p90_ms: float = 0.0


@dataclass(frozen=True, order=True)
class AssignedInstance:  # core.hpp:174-180
    placement: Placement
    service_id: str
    batch: int = 1


@dataclass(frozen=True, order=True)
class GpuConfig:  # core.hpp:184-200; instances sorted by placement
    instances: tuple = ()

    def partition(self) -> list[Placement]:
        return [i.placement for i in self.instances]

    def empty(self) -> bool:
        return not self.instances


@dataclass
class Candidate:  # config_enum.hpp:13-18
    config: GpuConfig
    util: list  # [(service index, fraction)] ascending index
    util_sum: float


@dataclass
class DeployedGpu:
    id: str
    config: GpuConfig


@dataclass
class Deployment:  # core.hpp:284-287
    gpus: list


def zero_completion(n: int) -> list[float]:
    return [0.0] * n


def is_satisfied(comp: Sequence[float]) -> bool:  # core.hpp:217-221
    return all(not (c < 1.0 - kSatisfyEps) for c in comp)


def slack_of(comp: Sequence[float]) -> float:  # core.hpp:232-236
    s = 0.0
    for c in comp:
        s += max(0.0, c - 1.0)
    return s


def _config_sort_key(c: GpuConfig) -> tuple:
    """The GpuConfig order (core.hpp:174-200) as plain tuples: the same lexicographic order as
    the dataclass comparison (instances by placement, service id, batch), without its cost."""
    return tuple((i.placement.slices, i.placement.start_slot, i.service_id, i.batch) for i in c.instances)


def make_deployment(configs: Iterable[GpuConfig], prefix: str = "gpu-") -> Deployment:  # core.hpp:305-312
    cfgs = sorted(configs, key=_config_sort_key)
    return Deployment([DeployedGpu(f"{prefix}{i}", c) for i, c in enumerate(cfgs)])


def service_index(services: Sequence[ServiceSpec], sid: str) -> int:  # core.hpp:142-148
    lo, hi = 0, len(services)
    while lo < hi:
        mid = (lo + hi) // 2
        if services[mid].service_id < sid:
            lo = mid + 1
        else:
            hi = mid
    return lo if lo < len(services) and services[lo].service_id == sid else -1


def select_batch(service: ServiceSpec, profile: ModelProfile, size: int) -> int | None:  # core.hpp:122-129
    best = None
    for e in profile.entries.get(size, []):
        if e.p90_ms <= service.max_p90_ms:
            best = e.batch
    return best


def select_entry(service: ServiceSpec, profile: ModelProfile, size: int):  # core.hpp:132-138
    b = select_batch(service, profile, size)
    if b is None:
        return None
    return b, profile.find(size, b).throughput_rps


def profile_for(profiles: dict, model: str) -> ModelProfile:
    if model not in profiles:
        raise PlanningError(f"no profile for model '{model}'")
    return profiles[model]


def _sum_rates(configs: Iterable[GpuConfig], services, profiles) -> list[float]:
    """detail::sum_rates, core.hpp:245-269 (count-based, key order, one division)."""
    counts: dict = {}
    for cfg in configs:
        for inst in cfg.instances:
            idx = service_index(services, inst.service_id)
            if idx < 0:
                raise PlanningError(f"unknown service '{inst.service_id}' in configuration")
            k = (idx, inst.placement.slices, inst.batch)
            counts[k] = counts.get(k, 0) + 1
    total = [0.0] * len(services)
    for (idx, size, batch) in sorted(counts):
        e = profile_for(profiles, services[idx].model_name).find(size, batch)
        if e is None:
            raise PlanningError(f"profile '{services[idx].model_name}' has no entry for size {size} batch {batch}")
        total[idx] += float(counts[(idx, size, batch)]) * e.throughput_rps
    return [total[i] / services[i].required_rps for i in range(len(services))]


def utility_of(config: GpuConfig, services, profiles) -> list[float]:  # core.hpp:271-276
    return _sum_rates([config], services, profiles)


def completion_of(configs, services, profiles) -> list[float]:  # core.hpp:291-302
    if isinstance(configs, Deployment):
        configs = [g.config for g in configs.gpus]
    return _sum_rates(configs, services, profiles)


def apply_utility(comp: Sequence[float], u: Sequence[float]) -> list[float]:  # core.hpp:223-230
    if len(comp) != len(u):
        raise PlanningError(f"completion/utility dimension mismatch: {len(comp)} vs {len(u)}")
    return [c + x for c, x in zip(comp, u)]


# ---------------------------------------------------------------- rules (mig_rules.hpp)


@dataclass
class PartitionRuleSet:  # mig_rules.hpp:15-34
    slot_positions: dict = field(default_factory=dict)
    memory_weight: dict = field(default_factory=dict)
    hard_exclusions: set = field(default_factory=set)
    memory_budget: int = 8

    @staticmethod
    def defaults() -> "PartitionRuleSet":
        return PartitionRuleSet(
            slot_positions={1: [0, 1, 2, 3, 4, 5, 6], 2: [0, 2, 4], 3: [0, 4], 4: [0], 7: [0]},
            memory_weight={1: 1, 2: 2, 3: 4, 4: 4, 7: 8},
            hard_exclusions={(3, 4)},
            memory_budget=8,
        )

    def to_c(self) -> abi.RulesC:
        r = abi.RulesC()
        if len(self.slot_positions) > 8 or len(self.memory_weight) > 8 or len(self.hard_exclusions) > 16:
            raise SchemaError("partition rules exceed the C-ABI limits")
        for i, (size, slots) in enumerate(sorted(self.slot_positions.items())):
            if len(slots) > 16:
                raise SchemaError("too many slot positions")
            r.size[i] = size
            r.n_slots[i] = len(slots)
            for k, s in enumerate(sorted(slots)):
                r.slots[i][k] = s
        r.n_sizes = len(self.slot_positions)
        for i, (size, w) in enumerate(sorted(self.memory_weight.items())):
            r.weight_size[i] = size
            r.weight[i] = w
        r.n_weights = len(self.memory_weight)
        for i, (a, b) in enumerate(sorted(self.hard_exclusions)):
            r.exclusion[i][0], r.exclusion[i][1] = min(a, b), max(a, b)
        r.n_exclusions = len(self.hard_exclusions)
        r.memory_budget = self.memory_budget
        return r


@dataclass
class LegalPartition:
    placements: list
    maximal: bool = True


def is_legal_partition(placements: Sequence[Placement], rules: PartitionRuleSet, backend=None) -> bool:
    b = _backend(backend)
    n = len(placements)
    sl = (C.c_int32 * max(n, 1))(*[p.slices for p in placements])
    st = (C.c_int32 * max(n, 1))(*[p.start_slot for p in placements])
    out = C.c_int32()
    rc = rules.to_c()
    b.check(b.lib.mig_is_legal_partition(C.byref(rc), sl, st, n, C.byref(out)))
    return bool(out.value)


def enumerate_maximal_partitions(rules: PartitionRuleSet, backend=None) -> list[LegalPartition]:
    b = _backend(backend)
    cap = 4096
    buf = (abi.PartitionC * cap)()
    n = C.c_int32()
    rc = rules.to_c()
    b.check(b.lib.mig_enumerate_maximal_partitions(C.byref(rc), buf, cap, C.byref(n)))
    return [LegalPartition([Placement(buf[i].slices[k], buf[i].slot[k]) for k in range(buf[i].n)], True)
            for i in range(n.value)]


# ---------------------------------------------------------------- I/O (io.hpp:85-151, format plumbing)


def _expect_keys(j, allowed, required, where):
    if not isinstance(j, dict):
        raise SchemaError(f"{where}: expected an object")
    for k in j:
        if k not in allowed:
            raise SchemaError(f"{where}: unknown field '{k}'")
    for k in required:
        if k not in j:
            raise SchemaError(f"{where}: missing field '{k}'")


def _load_json(path):
    try:
        with open(path, "rb") as f:
            return json.loads(f.read())
    except OSError:
        raise SchemaError(f"cannot open '{path}'")
    except json.JSONDecodeError as e:
        raise SchemaError(f"'{path}': {e}")


def validate_profile(p: ModelProfile) -> None:  # core.hpp:81-104
    if not p.model_name:
        raise SchemaError("profile with empty model name")
    for size, lst in sorted(p.entries.items()):
        if not valid_slices(size):
            raise SchemaError(f"profile {p.model_name}: invalid instance size {size}")
        prev_p90, prev_batch = 0.0, 0
        for e in lst:
            if e.batch <= 0:
                raise SchemaError(f"profile {p.model_name}: non-positive batch")
            if e.batch <= prev_batch:
                raise SchemaError(f"profile {p.model_name}: duplicate or unsorted batch {e.batch} for size {size}")
            if e.throughput_rps <= 0.0 or e.p90_ms <= 0.0:
                raise SchemaError(f"profile {p.model_name}: non-positive measurement at size {size} batch {e.batch}")
            if e.p90_ms < prev_p90:
                raise SchemaError(f"profile {p.model_name}: p90 decreases with batch at size {size}")
            prev_p90, prev_batch = e.p90_ms, e.batch


def load_profiles(path: str) -> dict:  # io.hpp:85-114
    j = _load_json(path)
    _expect_keys(j, {"models"}, {"models"}, path)
    store: dict = {}
    for mi, m in enumerate(j["models"]):
        where = f"{path}:models[{mi}]"
        _expect_keys(m, {"name", "entries"}, {"name", "entries"}, where)
        prof = ModelProfile(str(m["name"]))
        for e in m["entries"]:
            _expect_keys(e, {"size", "batch", "throughput_rps", "p90_ms"}, {"size", "batch", "throughput_rps", "p90_ms"},
                         where)
            if not isinstance(e["size"], int) or not valid_slices(e["size"]):
                raise SchemaError(f"{where}: invalid instance size {e['size']}")
            prof.entries.setdefault(e["size"], []).append(
                ProfileEntry(int(e["batch"]), float(e["throughput_rps"]), float(e["p90_ms"])))
        for size in prof.entries:
            prof.entries[size].sort(key=lambda x: x.batch)
        prof.entries = dict(sorted(prof.entries.items()))
        validate_profile(prof)
        if prof.model_name in store:
            raise SchemaError(f"{path}: duplicate model '{prof.model_name}'")
        store[prof.model_name] = prof
    return dict(sorted(store.items()))


def validate_services(services: list, profiles: dict) -> list:  # core.hpp:151-171
    services.sort(key=lambda s: s.service_id)
    for a, b in zip(services, services[1:]):
        if a.service_id == b.service_id:
            raise SchemaError(f"duplicate service id '{a.service_id}'")
    for s in services:
        if not s.service_id:
            raise SchemaError("service with empty id")
        if s.required_rps <= 0.0:
            raise PlanningError(f"service '{s.service_id}': required throughput must be positive")
        if s.max_p90_ms <= 0.0:
            raise PlanningError(f"service '{s.service_id}': latency ceiling must be positive")
        p = profile_for(profiles, s.model_name)
        if not any(select_batch(s, p, size) is not None for size in kInstanceSlices):
            raise PlanningError(f"service '{s.service_id}' is unschedulable: no (size, batch) of model "
                                f"'{s.model_name}' meets p90 <= {s.max_p90_ms:f} ms")
    return services


def load_services(path: str, profiles: dict) -> list:  # io.hpp:133-151
    j = _load_json(path)
    _expect_keys(j, {"services"}, {"services"}, path)
    out = []
    for si, s in enumerate(j["services"]):
        where = f"{path}:services[{si}]"
        _expect_keys(s, {"id", "model", "required_rps", "max_p90_ms"}, {"id", "model", "required_rps", "max_p90_ms"},
                     where)
        out.append(ServiceSpec(str(s["id"]), str(s["model"]), float(s["required_rps"]), float(s["max_p90_ms"])))
    return validate_services(out, profiles)


def deployment_to_json(dep: Deployment) -> dict:  # io.hpp:196-208
    return {"gpus": [{"id": g.id, "instances": [{"size": i.placement.slices, "slot": i.placement.start_slot,
                                                 "service": i.service_id, "batch": i.batch}
                                                for i in g.config.instances]} for g in dep.gpus]}


# ---------------------------------------------------------------- RNG (util.hpp:27-51)


class Rng:
    """std::mt19937_64 stream living in the backend library."""

    def __init__(self, seed: int = 5489, backend=None):
        self._b = _backend(backend)
        p = C.c_void_p()
        self._b.check(self._b.lib.mig_rng_create(C.c_uint64(seed & (2**64 - 1)), C.byref(p)))
        self._p = p

    def __call__(self) -> int:
        return self._b.lib.mig_rng_next(self._p)

    def __del__(self):
        if getattr(self, "_p", None):
            self._b.lib.mig_rng_destroy(self._p)
            self._p = None


def mix_seed(a: int, b: int) -> int:  # util.hpp:30-35 (pure integer; restated for host use)
    M = 2**64 - 1
    z = (a + 0x9E3779B97F4A7C15 * (b + 1)) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def pick_index(rng: Rng, n: int) -> int:  # util.hpp:39-47
    return rng._b.lib.mig_pick_index(rng._p, n)


def uniform01(rng: Rng) -> float:  # util.hpp:49-51
    return float(rng() >> 11) * 2.0 ** -53


def normal_sample(rng: Rng, mu: float, sigma: float) -> float:  # util.hpp:55-60
    u1 = uniform01(rng)
    u2 = uniform01(rng)
    if u1 <= 0.0:
        u1 = 2.0 ** -53
    return mu + sigma * math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)


def lognormal_sample(rng: Rng, mu: float, sigma: float) -> float:  # util.hpp:62-64
    return math.exp(normal_sample(rng, mu, sigma))


def gen_workload(n: int, lognormal: bool, mu: float, sigma: float, latency_ms: float, seed: int, profiles: dict,
                 backend=None) -> list:
    """gen_workload, bench.hpp:125-156 (Normal when lognormal=False)."""
    if n < 1:
        raise PlanningError("gen_workload: n must be >= 1")
    if not profiles:
        raise PlanningError("gen_workload: no model profiles loaded")
    models = sorted(profiles)
    rng = Rng(mix_seed(seed, 0x776B6C64), backend)
    out = []
    for i in range(n):
        model = models[pick_index(rng, len(models))]
        while True:
            draw = lognormal_sample(rng, mu, sigma) if lognormal else normal_sample(rng, mu, sigma)
            if draw > 0.0:
                break
        out.append(ServiceSpec(f"svc-{i:03d}", model, draw, latency_ms))
    return validate_services(out, profiles)


# ---------------------------------------------------------------- plan context (greedy.hpp:16-31)


def _profiles_to_c(profiles: dict):
    keep = []
    arr = (abi.ModelProfileC * max(len(profiles), 1))()
    for i, (name, prof) in enumerate(sorted(profiles.items())):
        ents = [(size, e) for size, lst in sorted(prof.entries.items()) for e in lst]
        earr = (abi.ProfileEntryC * max(len(ents), 1))()
        for k, (size, e) in enumerate(ents):
            earr[k] = abi.ProfileEntryC(size, e.batch, e.throughput_rps, e.p90_ms)
        nb = name.encode()
        keep += [earr, nb]
        arr[i] = abi.ModelProfileC(nb, earr, len(ents))
    keep.append(arr)
    return arr, len(profiles), keep


def _services_to_c(services):
    keep = []
    arr = (abi.ServiceC * max(len(services), 1))()
    for i, s in enumerate(services):
        a, b = s.service_id.encode(), s.model_name.encode()
        keep += [a, b]
        arr[i] = abi.ServiceC(a, b, s.required_rps, s.max_p90_ms)
    keep.append(arr)
    return arr, keep


class CandidatePool:
    """View of the context's base pool (config_enum.hpp:20-32)."""

    def __init__(self, ctx: "PlanContext"):
        self._ctx = ctx
        self._cache: dict = {}

    def __len__(self):
        n = C.c_int64()
        self._ctx.backend.check(self._ctx.backend.lib.mig_pool_size(self._ctx._p, C.byref(n)))
        return n.value

    @property
    def items(self):
        return self

    def __getitem__(self, idx: int) -> Candidate:
        if idx < 0:
            idx += len(self)
        c = self._cache.get(idx)
        if c is None:
            out = abi.CandidateC()
            self._ctx.backend.check(self._ctx.backend.lib.mig_pool_candidate(self._ctx._p, idx, C.byref(out)))
            c = self._ctx._cand_from_c(out)
            self._cache[idx] = c
        return c

    def __iter__(self):
        for i in range(len(self)):
            yield self[i]

    @property
    def best_single_util(self) -> list[float]:
        n = self._ctx.n
        buf = (C.c_double * max(n, 1))()
        self._ctx.backend.check(self._ctx.backend.lib.mig_pool_best_single_util(self._ctx._p, buf))
        return list(buf[:n])

    @property
    def n_services(self) -> int:
        return self._ctx.n


class PlanContext:
    """PlanContext (greedy.hpp:16-21): services, profiles, rules and the device-resident pool."""

    def __init__(self, services, profiles, rules, max_mix=2, backend=None, device=0):
        self.backend = _backend(backend)
        self.services = list(services)
        self.profiles = profiles
        self.rules = rules
        self.max_mix = max_mix
        self.device = device
        self.n = len(self.services)
        self._ids = {s.service_id: i for i, s in enumerate(self.services)}
        prof_c, n_models, k1 = _profiles_to_c(profiles)
        svc_c, k2 = _services_to_c(self.services)
        rc = rules.to_c()
        p = C.c_void_p()
        self.backend.check(self.backend.lib.mig_ctx_create(C.byref(rc), prof_c, n_models, svc_c, self.n, max_mix,
                                                          device, C.byref(p)))
        self._p = p
        self.pool = CandidatePool(self)

    def close(self):
        if getattr(self, "_p", None):
            self.backend.lib.mig_ctx_destroy(self._p)
            self._p = None

    def __del__(self):
        self.close()

    # ---- conversions
    def _config_from_c(self, c: abi.ConfigC) -> GpuConfig:
        return GpuConfig(tuple(AssignedInstance(Placement(c.inst[k].slices, c.inst[k].slot),
                                                self.services[c.inst[k].service].service_id, c.inst[k].batch)
                               for k in range(c.n_instances)))

    def _configs_from_buf(self, buf, n: int) -> list[GpuConfig]:
        """n ConfigC records at once: one unpack of the raw ints; within the call, repeated
        instances and configurations share one immutable object (plans repeat configurations)."""
        if n <= 0:
            return []
        w = C.sizeof(abi.ConfigC) // 4
        ints = memoryview(buf).cast("B")[: n * w * 4].cast("i").tolist()
        icache, ccache = {}, {}
        ids = [sv.service_id for sv in self.services]
        out = []
        for i in range(n):
            b = i * w
            k = ints[b]
            key = tuple(ints[b + 1: b + 1 + 4 * k])
            g = ccache.get(key)
            if g is None:
                insts = []
                for j in range(k):
                    o = b + 1 + 4 * j
                    ik = (ints[o], ints[o + 1], ints[o + 2], ints[o + 3])
                    inst = icache.get(ik)
                    if inst is None:
                        inst = icache[ik] = AssignedInstance(Placement(ik[0], ik[1]), ids[ik[2]], ik[3])
                    insts.append(inst)
                g = ccache[key] = GpuConfig(tuple(insts))
            out.append(g)
        return out

    def _config_to_c(self, g: GpuConfig, out: abi.ConfigC) -> None:
        if len(g.instances) > abi.MAX_INST:
            raise PlanningError("config has more than 7 instances")
        out.n_instances = len(g.instances)
        for k, inst in enumerate(g.instances):
            idx = self._ids.get(inst.service_id, -1)
            if idx < 0:
                raise PlanningError(f"unknown service '{inst.service_id}' in configuration")
            out.inst[k] = abi.InstanceC(inst.placement.slices, inst.placement.start_slot, idx, inst.batch)

    def _configs_to_c(self, cfgs):
        arr = (abi.ConfigC * max(len(cfgs), 1))()
        for i, g in enumerate(cfgs):
            self._config_to_c(g, arr[i])
        return arr

    def _cand_from_c(self, c: abi.CandidateC) -> Candidate:
        return Candidate(self._config_from_c(c.config), [(c.util_idx[k], c.util_val[k]) for k in range(c.nnz)],
                         c.util_sum)

    def _comp(self, comp):
        vals = list(comp)
        return (C.c_double * max(len(vals), 1))(*vals), len(vals)

    def stats(self) -> dict:
        s = abi.StatsC()
        self.backend.check(self.backend.lib.mig_ctx_stats(self._p, C.byref(s)))
        return {k: getattr(s, k) for k, _ in abi.StatsC._fields_}

    def reset_stats(self):
        self.backend.lib.mig_ctx_reset_stats(self._p)


def make_plan_context(services, profiles, rules, max_mix: int = 2, backend=None, device: int = 0) -> PlanContext:
    return PlanContext(services, profiles, rules, max_mix, backend, device)


def release_device_cache(device: int = 0, backend=None) -> None:
    """Free the process-wide pooled per-call device resources (mig_device_cache_release)."""
    b = _backend(backend)
    b.check(b.lib.mig_device_cache_release(device))


def _run_plan(ctx: PlanContext, call) -> list[GpuConfig]:
    cap = 4096
    buf = (abi.ConfigC * cap)()
    n = C.c_int32()
    rc = call(buf, cap, n)
    if rc == abi.MIG_ERR_ARGUMENT and n.value > cap:
        # a longer plan: the library kept it (mig_last_plan), so the call is not re-run (a
        # re-run would consume an Rng's draws or a time budget a second time)
        cap = n.value
        buf = (abi.ConfigC * cap)()
        rc = ctx.backend.lib.mig_last_plan(buf, cap, C.byref(n))
    ctx.backend.check(rc)
    return ctx._configs_from_buf(buf, n.value)


# ---------------------------------------------------------------- greedy (greedy.hpp)


def score(cand, comp, ctx: PlanContext | None = None) -> float:
    """score(Candidate|Utility, comp), greedy.hpp:36-54, evaluated in plain Python doubles.
    `cand` may be a Candidate, a dense utility list, or a pool index (with ctx: device call)."""
    if isinstance(cand, int) and ctx is not None:
        buf, n = ctx._comp(comp)
        out = C.c_double()
        ctx.backend.check(ctx.backend.lib.mig_score(ctx._p, cand, buf, n, C.byref(out)))
        return out.value
    if isinstance(cand, Candidate):
        s = 0.0
        for idx, u in cand.util:
            need = 1.0 - comp[idx]
            if need > 0.0:
                s += need * u
        return s
    if len(cand) != len(comp):
        raise PlanningError("score: utility/completion dimension mismatch")
    s = 0.0
    for u, c in zip(cand, comp):
        need = 1.0 - c
        if need > 0.0:
            s += need * u
    return s


def candidate_preferred(a: Candidate, sa: float, b: Candidate, sb: float) -> bool:  # greedy.hpp:63-67
    if sa != sb:
        return sa > sb
    if a.util_sum != b.util_sum:
        return a.util_sum > b.util_sum
    return a.config < b.config


def fast_algo(comp, ctx: PlanContext, trace: Callable | None = None) -> list[GpuConfig]:
    """fast_algo, greedy.hpp:95-145.  trace(iter, Candidate, score, comp_after)."""
    buf, n = ctx._comp(comp)
    cb = abi.GREEDY_TRACE()
    if trace is not None:
        def _tr(_u, it, cand, s, cp, nn):
            trace(it, ctx._cand_from_c(cand.contents), s, list(cp[:nn]))
        cb = abi.GREEDY_TRACE(_tr)
    return _run_plan(ctx, lambda out, cap, nout: ctx.backend.lib.mig_fast_algo(ctx._p, buf, n, out, cap,
                                                                              C.byref(nout), cb, None))


class OptimizerProcedure:  # greedy.hpp:155-158 — the plugin interface
    def solve(self, comp, ctx: PlanContext, rng: Rng) -> list[GpuConfig]:
        raise NotImplementedError


class FastProcedure(OptimizerProcedure):  # greedy.hpp:160-164
    kind = 0

    def solve(self, comp, ctx, rng):
        return fast_algo(comp, ctx)


# ---------------------------------------------------------------- MCTS (mcts.hpp)


@dataclass
class MctsParams:  # mcts.hpp:13-18
    budget_iters: int = 200
    topk: int = 10
    pick_services: int = 5
    ucb_c: float = 1.4142135623730951

    def to_c(self) -> abi.MctsParamsC:
        return abi.MctsParamsC(self.budget_iters, self.topk, self.pick_services, self.ucb_c)


def topk_candidates(ctx: PlanContext, comp, k: int, from_: Sequence[int] | None = None) -> list[int]:
    """detail::topk_candidates, mcts.hpp:56-76 (indices into ctx.pool)."""
    buf, n = ctx._comp(comp)
    out = (C.c_int64 * max(k, 1))()
    nout = C.c_int32()
    if from_ is None:
        ctx.backend.check(ctx.backend.lib.mig_topk_candidates(ctx._p, buf, n, k, None, -1, out, C.byref(nout)))
    else:
        f = (C.c_int64 * max(len(from_), 1))(*from_)
        ctx.backend.check(ctx.backend.lib.mig_topk_candidates(ctx._p, buf, n, k, f, len(from_), out, C.byref(nout)))
    return list(out[:nout.value])


class SearchNode:  # mcts.hpp:22-35 (only what expand() exposes)
    def __init__(self, comp):
        self.comp = list(comp)
        self.leaf = is_satisfied(self.comp)
        self.expanded = False
        self.children: list = []  # [(cand index, SearchNode)]


def expand(node: SearchNode, ctx: PlanContext, params: MctsParams, rng: Rng) -> list[int]:  # mcts.hpp:89-116
    if node.leaf:
        raise PlanningError("expand: node is already satisfied")
    buf, n = ctx._comp(node.comp)
    cap = max(params.topk, 1)
    out = (C.c_int64 * cap)()
    nout = C.c_int32()
    pc = params.to_c()
    ctx.backend.check(ctx.backend.lib.mig_expand(ctx._p, buf, n, C.byref(pc), rng._p, out, cap, C.byref(nout)))
    top = list(out[:nout.value])
    node.children = []
    for idx in top:
        child = list(node.comp)
        for svc, u in ctx.pool[idx].util:
            child[svc] += u
        node.children.append((idx, SearchNode(child)))
    node.expanded = True
    return top


class RolloutCache:  # mcts.hpp:47-50
    def __init__(self, backend=None):
        self._b = _backend(backend)
        p = C.c_void_p()
        self._b.check(self._b.lib.mig_rollout_cache_create(C.byref(p)))
        self._p = p

    @property
    def builds(self) -> int:
        return self._b.lib.mig_rollout_cache_builds(self._p)

    def __del__(self):
        if getattr(self, "_p", None):
            self._b.lib.mig_rollout_cache_destroy(self._p)
            self._p = None


def rollout(comp, ctx: PlanContext, params: MctsParams, cache: RolloutCache, rng: Rng, max_depth: int,
            picked: list | None = None) -> int:  # mcts.hpp:122-143
    buf, n = ctx._comp(comp)
    cap = max(max_depth, 1)
    out = (C.c_int64 * cap)()
    steps = C.c_int32()
    pc = params.to_c()
    ctx.backend.check(ctx.backend.lib.mig_rollout(ctx._p, buf, n, C.byref(pc), cache._p, rng._p, max_depth,
                                                  out if picked is not None else None, cap, C.byref(steps)))
    if picked is not None:
        picked.extend(out[:min(steps.value, cap)])
    return steps.value


def mcts_solve(comp, ctx: PlanContext, params: MctsParams, seed: int, trace: Callable | None = None):
    """mcts_solve, mcts.hpp:148-252.  trace(iter, depth, estimate, best_len)."""
    buf, n = ctx._comp(comp)
    pc = params.to_c()
    cb = abi.MCTS_TRACE()
    if trace is not None:
        cb = abi.MCTS_TRACE(lambda _u, a, b, c, d: trace(a, b, c, d))
    return _run_plan(ctx, lambda out, cap, nout: ctx.backend.lib.mig_mcts_solve(
        ctx._p, buf, n, C.byref(pc), C.c_uint64(seed & (2**64 - 1)), out, cap, C.byref(nout), cb, None))


class MctsProcedure(OptimizerProcedure):  # mcts.hpp:254-260
    kind = 1

    def __init__(self, params: MctsParams | None = None):
        self.params = params or MctsParams()

    def solve(self, comp, ctx, rng):
        return mcts_solve(comp, ctx, self.params, rng())


# ---------------------------------------------------------------- MCTS throughput mode (rollout.cu)


@dataclass
class RolloutParams:
    """Root-parallel rollouts (include/migplan_b200.h, mig_rollouts): Philox draws, lock-step
    rounds, one shared key cache per call.  max_depth < 0: 2 * |fast_algo(comp)|."""
    n_rollouts: int = 1 << 16
    topk: int = 10
    max_depth: int = -1
    seed: int = 0
    id_offset: int = 0
    batch: int = 0
    table_log2: int = 0

    def to_c(self) -> abi.RolloutParamsC:
        return abi.RolloutParamsC(self.n_rollouts, self.topk, self.max_depth, self.seed & (2**64 - 1),
                                  self.id_offset, self.batch, self.table_log2)


@dataclass
class RolloutResult:
    best_len: int
    max_depth: int
    best_id: int
    completed: int
    capped: int
    failed: int
    steps: int
    keys: int
    rounds: int
    device_ms: float
    path: list = field(default_factory=list)  # pool indices of the best rollout
    lengths: list | None = None


def _rollout_result(r: abi.RolloutResultC, path, lengths) -> RolloutResult:
    return RolloutResult(r.best_len, r.max_depth, r.best_id, r.completed, r.capped, r.failed, r.steps, r.keys,
                         r.rounds, r.device_ms, path, lengths)


def rollouts(comp, ctx: PlanContext, params: RolloutParams, lengths: bool = False) -> RolloutResult:
    """params.n_rollouts root-parallel rollouts from `comp` (rollout, mcts.hpp:122-143, run
    concurrently with Philox draws); returns the shortest completed one."""
    buf, n = ctx._comp(comp)
    pc = params.to_c()
    res = abi.RolloutResultC()
    lbuf = (C.c_int32 * max(params.n_rollouts, 1))() if lengths else None
    cap = 1 << 16
    path = (C.c_int64 * cap)()
    ctx.backend.check(ctx.backend.lib.mig_rollouts(ctx._p, buf, n, C.byref(pc), lbuf, path, cap, C.byref(res)))
    return _rollout_result(res, list(path[:res.path_len]), list(lbuf[:params.n_rollouts]) if lengths else None)


def mcts_solve_parallel(comp, ctx: PlanContext, params: RolloutParams) -> tuple[list[GpuConfig], RolloutResult]:
    """Throughput-mode mcts_solve: the shorter of fast_algo(comp) and the best root-parallel
    rollout (fast_ref wins ties, mcts.hpp:245-251)."""
    buf, n = ctx._comp(comp)
    pc = params.to_c()
    res = abi.RolloutResultC()
    plan = _run_plan(ctx, lambda out, cap, nout: ctx.backend.lib.mig_mcts_solve_parallel(
        ctx._p, buf, n, C.byref(pc), out, cap, C.byref(nout), C.byref(res)))
    return plan, _rollout_result(res, [], None)


# ---------------------------------------------------------------- GA (ga.hpp)


@dataclass
class GaParams:  # ga.hpp:24-36
    population: int = 16
    erase_fraction: float = 0.10
    mutation_pairs: int = 2
    stall_rounds: int = 10
    time_budget_s: float = 0.0
    seed: int = 0
    max_rounds: int = 1 << 30
    workers: int = 1
    slow: MctsParams = field(default_factory=lambda: MctsParams(budget_iters=48))

    def to_c(self) -> abi.GaParamsC:
        return abi.GaParamsC(self.population, self.erase_fraction, self.mutation_pairs, self.stall_rounds,
                             self.time_budget_s, self.seed & (2**64 - 1), self.max_rounds, self.workers,
                             self.slow.to_c())


@dataclass
class Chromosome:  # ga.hpp:13-17
    gpus: list = field(default_factory=list)
    gpu_count: int = 0
    slack: float = 0.0


@dataclass
class GaRoundLog:  # ga.hpp:115-121
    round: int
    best_gpus: int
    best_slack: float
    improved: bool
    elapsed_s: float


def fitter(a: Chromosome, b: Chromosome) -> bool:  # ga.hpp:19-22
    if a.gpu_count != b.gpu_count:
        return a.gpu_count < b.gpu_count
    return a.slack < b.slack


def ctx_completion_of(ctx: PlanContext, gpus) -> list[float]:
    arr = ctx._configs_to_c(gpus)
    out = (C.c_double * max(ctx.n, 1))()
    ctx.backend.check(ctx.backend.lib.mig_completion_of(ctx._p, arr, len(gpus), out))
    return list(out[:ctx.n])


def evaluate_chromosome(gpus, ctx: PlanContext) -> Chromosome:  # ga.hpp:38-46
    comp = ctx_completion_of(ctx, gpus)
    if not is_satisfied(comp):
        raise PlanningError("chromosome violates the deployment validity invariant")
    return Chromosome(list(gpus), len(gpus), slack_of(comp))


def mutate(parent: Chromosome, params: GaParams, rng: Rng, ctx: PlanContext) -> Chromosome:  # ga.hpp:83-113
    arr = ctx._configs_to_c(parent.gpus)
    out = (abi.ConfigC * max(len(parent.gpus), 1))()
    gp = params.to_c()
    ctx.backend.check(ctx.backend.lib.mig_mutate(ctx._p, arr, len(parent.gpus), C.byref(gp), rng._p, out))
    return Chromosome([ctx._config_from_c(out[i]) for i in range(len(parent.gpus))], parent.gpu_count, parent.slack)


def crossover(parent: Chromosome, slow: OptimizerProcedure, ctx: PlanContext, params: GaParams,
              rng: Rng) -> Chromosome:  # ga.hpp:51-77
    kind = getattr(slow, "kind", None)
    if kind is None:
        return _crossover_py(parent, slow, ctx, params, rng)
    arr = ctx._configs_to_c(parent.gpus)
    gp = params.to_c()
    if isinstance(slow, MctsProcedure):
        gp.slow = slow.params.to_c()
    gpus = _run_plan(ctx, lambda out, cap, nout: ctx.backend.lib.mig_crossover(
        ctx._p, arr, len(parent.gpus), kind, C.byref(gp), rng._p, out, cap, C.byref(nout)))
    if not gpus:
        return Chromosome([], 0, 0.0)
    return evaluate_chromosome(gpus, ctx)


def _crossover_py(parent, slow, ctx, params, rng):
    """crossover for a user-supplied Python OptimizerProcedure (same RNG consumption as ga.hpp:51-77)."""
    n = len(parent.gpus)
    erase = 0 if n == 0 else int(math.ceil(params.erase_fraction * float(n)))
    if erase == 0:
        return parent
    order = list(range(n))
    for i in range(erase):
        j = i + pick_index(rng, n - i)
        order[i], order[j] = order[j], order[i]
    erased = set(order[:erase])
    survivors = [g for i, g in enumerate(parent.gpus) if i not in erased]
    try:
        residual = ctx_completion_of(ctx, survivors) if survivors else zero_completion(ctx.n)
        refill = slow.solve(residual, ctx, rng)
        return evaluate_chromosome(survivors + list(refill), ctx)
    except PlanningError:
        return parent


def two_phase(services, profiles, rules, params: GaParams, log: Callable | None = None, backend=None,
              ctx: PlanContext | None = None) -> Deployment:
    """two_phase, ga.hpp:126-179 (builds its own max_mix-2 context unless one is passed)."""
    own = ctx is None
    if own:
        ctx = make_plan_context(services, profiles, rules, 2, backend)
    gp = params.to_c()
    cb = abi.GA_LOG()
    if log is not None:
        cb = abi.GA_LOG(lambda _u, r, g, s, imp, el: log(GaRoundLog(r, g, s, bool(imp), el)))
    cfgs = _run_plan(ctx, lambda out, cap, nout: ctx.backend.lib.mig_two_phase(ctx._p, C.byref(gp), out, cap,
                                                                              C.byref(nout), cb, None))
    return make_deployment(cfgs)


def two_phase_parallel(services, profiles, rules, params: GaParams, log: Callable | None = None, backend=None,
                       ctx: PlanContext | None = None, slow: RolloutParams | None = None) -> Deployment:
    """Throughput-mode two_phase (include/migplan_b200.h): device-resident population, every
    generation's mutation / crossover / fitness on the B200, Philox draws.  Same rounds,
    elitism and stop rules as two_phase.  slow=None: FastProcedure refill
    (mig_two_phase_parallel); slow=RolloutParams: the throughput mcts_solve refill — the
    shorter of the greedy refill and the best of slow.n_rollouts root-parallel rollouts
    (mig_two_phase_parallel_mcts)."""
    own = ctx is None
    if own:
        ctx = make_plan_context(services, profiles, rules, 2, backend)
    gp = params.to_c()
    cb = abi.GA_LOG()
    if log is not None:
        cb = abi.GA_LOG(lambda _u, r, g, s, imp, el: log(GaRoundLog(r, g, s, bool(imp), el)))
    if slow is None:
        cfgs = _run_plan(ctx, lambda out, cap, nout: ctx.backend.lib.mig_two_phase_parallel(
            ctx._p, C.byref(gp), out, cap, C.byref(nout), cb, None))
    else:
        rp = slow.to_c()
        cfgs = _run_plan(ctx, lambda out, cap, nout: ctx.backend.lib.mig_two_phase_parallel_mcts(
            ctx._p, C.byref(gp), C.byref(rp), out, cap, C.byref(nout), cb, None))
    return make_deployment(cfgs)


# ---------------------------------------------------------------- bench helpers (bench.hpp)


def lower_bound(services, profiles) -> int:  # bench.hpp:93-108 (host arithmetic)
    if not services:
        return 0
    total = 0.0
    for svc in services:
        prof = profile_for(profiles, svc.model_name)
        best = 0.0
        for size in kInstanceSlices:
            e = select_entry(svc, prof, size)
            if e is not None:
                best = max(best, e[1] / size)
        if best <= 0.0:
            raise PlanningError(f"service '{svc.service_id}' has no feasible instance size")
        total += svc.required_rps / best
    return int(math.ceil(total / 7.0 - 1e-9))


BASELINE_KINDS = {"7of7": 0, "7x1": 1, "mix": 2}  # A100-7/7, A100-7x1/7, A100-MIX (bench.hpp:13-22)
BASELINE_NAMES = {0: "A100-7/7", 1: "A100-7x1/7", 2: "A100-MIX"}


def baseline(kind, services, profiles, backend=None) -> Deployment:
    """baseline(kind, services, profiles), bench.hpp:42-90 — static-partition deployments.
    kind: 0/"7of7" whole GPUs, 1/"7x1" 1/7 instances packed seven per GPU, 2/"mix" 4+2+1."""
    k = BASELINE_KINDS[kind] if isinstance(kind, str) else int(kind)
    services = list(services)
    if not services:
        return make_deployment([])
    ctx = PlanContext(services, profiles, PartitionRuleSet.defaults(), 1, backend)
    plan = _run_plan(ctx, lambda out, cp, nout: ctx.backend.lib.mig_baseline(ctx._p, k, out, cp, C.byref(nout)))
    return make_deployment(plan)


def brute_force_optimum(services, profiles, rules, cap: int, node_budget: int = 20_000_000,
                        backend=None, device: int = 0) -> Deployment | None:
    """brute_force_optimum, bench.hpp:160-219 — the exhaustive minimum-GPU oracle for small
    instances; None when the optimum exceeds cap.  The search builds its own max_mix =
    min(n, 7) pool (bench.hpp:164-165), so the context only carries the model (max_mix 1);
    the device search takes n <= 16 services."""
    services = list(services)
    if not services:  # bench.hpp:163
        return make_deployment([])
    ctx = PlanContext(services, profiles, rules, 1, backend, device)
    found = C.c_int32()
    plan = _run_plan(ctx, lambda out, cp, nout: ctx.backend.lib.mig_brute_force_optimum(
        ctx._p, cap, node_budget, out, cp, C.byref(nout), C.byref(found)))
    return make_deployment(plan) if found.value else None


def validate_deployment(dep: Deployment, services, profiles, rules, backend=None) -> None:  # mig_rules.hpp:155-177
    ids = set()
    for gpu in dep.gpus:
        if gpu.id in ids:
            raise PlanningError(f"duplicate gpu id '{gpu.id}'")
        ids.add(gpu.id)
        if not is_legal_partition(gpu.config.partition(), rules, backend):
            raise PlanningError(f"gpu '{gpu.id}' is not a legal partition")
        for inst in gpu.config.instances:
            idx = service_index(services, inst.service_id)
            if idx < 0:
                raise PlanningError(f"gpu '{gpu.id}' assigns unknown service '{inst.service_id}'")
            svc = services[idx]
            e = profile_for(profiles, svc.model_name).find(inst.placement.slices, inst.batch)
            if e is None:
                raise PlanningError(f"gpu '{gpu.id}': no profile entry for '{svc.model_name}' size "
                                    f"{inst.placement.slices} batch {inst.batch}")
            if e.p90_ms > svc.max_p90_ms:
                raise PlanningError(f"gpu '{gpu.id}': service '{svc.service_id}' batch {inst.batch} violates "
                                    f"its latency ceiling")
