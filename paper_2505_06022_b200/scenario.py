"""Scenario documents and the runs the ``clusterq`` CLI makes of them, on the
B200 executor.

Same JSON format as the reference (pkg/src/clusterq/scenario.py:1-7,
docs/formats.md): buffers, an ordered task list with kernel bodies as text,
optionally the machine shape (nodes, device models, link), a queue-wide
energy target and expected buffer values.  Parsing is strict -- unknown
keys, wrong types, bad shapes and kernel grammar errors raise
``ScenarioError`` naming the JSON path of the offending field, so documents
the reference rejects are rejected here too.

The difference is the run: ``run_scenario`` plans with the same
``generate_commands`` and executes on the GPUs (``executor.run``), with
measured CUDA-event times in the trace and, with ``energy=True``, NVML joules
per device and per task (``measured_energy``).
"""

import json
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .energy import DeviceModel, EnergyTarget, account_energy
from .errors import ClusterqError, ScenarioError
from .graph import TaskGraph
from .kernel import format_kernel, parse_kernel
from .model import Accessor, AccessMode, All, Buffer, BufferInit, Fixed, Neighborhood, OneToOne, Slice, Task
from .region import Box, Region

EXAMPLES = os.path.join(os.path.dirname(os.path.abspath(__file__)), "scenarios")


@dataclass
class Scenario:
    buffers: list = field(default_factory=list)
    tasks: list = field(default_factory=list)
    nodes: Optional[int] = None
    devices: Optional[list] = None
    link: Optional[object] = None          # executor.LinkModel (accepted, not modelled)
    queue_target: Optional[EnergyTarget] = None
    expectations: list = field(default_factory=list)   # (buffer name, values)


# ------------------------------------------------------------- JSON cursor

class _Node:
    """A JSON value plus the path it was found at; typed accessors raise
    ScenarioError with that path."""

    __slots__ = ("v", "path")

    def __init__(self, value, path):
        self.v, self.path = value, path

    def fail(self, message):
        raise ScenarioError(f"{self.path}: {message}")

    def _kind(self, ok, want):
        if not ok:
            self.fail(f"expected {want}, got {type(self.v).__name__}")
        return self.v

    def int(self):
        return self._kind(isinstance(self.v, int) and not isinstance(self.v, bool), "an integer")

    def num(self):
        return self._kind(isinstance(self.v, (int, float)) and not isinstance(self.v, bool), "a number")

    def str(self):
        return self._kind(isinstance(self.v, str), "a string")

    def list(self):
        return [_Node(x, f"{self.path}[{i}]") for i, x in enumerate(self._kind(isinstance(self.v, list), "a list"))]

    def dict(self):
        self._kind(isinstance(self.v, dict), "an object")
        return self

    def obj(self, allowed):
        d = self._kind(isinstance(self.v, dict), "an object")
        for k in d:
            if k not in allowed:
                raise ScenarioError(f"{self.path}.{k}: unknown field")
        return self

    def has(self, key):
        return key in self.v and self.v[key] is not None

    def at(self, key, default=None):
        return _Node(self.v.get(key, default), f"{self.path}.{key}")

    def need(self, key):
        if key not in self.v:
            self.fail(f"missing required field '{key}'")
        return self.at(key)

    def items(self):
        return [(k, _Node(x, f"{self.path}.{k}")) for k, x in self._kind(isinstance(self.v, dict), "an object").items()]

    def wrap(self, fn, *args, **kw):
        """Call a model constructor; its own errors are re-raised at this path."""
        try:
            return fn(*args, **kw)
        except ClusterqError as exc:
            raise ScenarioError(f"{self.path}: {exc}") from exc


def _shape(node):
    sizes = [x.int() for x in node.list()]
    if not 1 <= len(sizes) <= 3:
        node.fail(f"expected 1 to 3 sizes, got {len(sizes)}")
    if min(sizes) < 1:
        node.fail(f"sizes must be positive, got {sizes}")
    return Box.from_shape(tuple(sizes))


_INIT_SHORT = {"zeros": BufferInit.zeros, "iota": BufferInit.iota, "uninitialized": BufferInit.uninitialized}


def _init(node):
    if node.v is None:
        return BufferInit.zeros()
    if isinstance(node.v, str):
        if node.v not in _INIT_SHORT:
            node.fail(f"unknown init shorthand '{node.v}' (expected one of {sorted(_INIT_SHORT)})")
        return _INIT_SHORT[node.v]()
    node.dict()   # its keys are checked per kind
    kind = node.need("kind").str()
    extra = {"constant": {"value"}, "values": {"values"}}
    if kind not in _INIT_SHORT and kind not in extra:
        node.at("kind").fail(f"unknown init kind '{kind}'")
    node.obj({"kind"} | extra.get(kind, set()))
    if kind in _INIT_SHORT:
        return _INIT_SHORT[kind]()
    if kind == "constant":
        return BufferInit.constant(node.need("value").num())
    return BufferInit.explicit([x.num() for x in node.need("values").list()])


def _buffer(node):
    node.obj({"name", "extent", "element_kind", "init"})
    name = node.need("name").str()
    extent = _shape(node.need("extent"))
    kind = node.at("element_kind", "float64").str()
    return node.wrap(Buffer, name=name, extent=extent, element_kind=kind, init=_init(node.at("init")))


def _region(node):
    boxes = []
    for b in node.list():
        b.obj({"min", "max"})
        lo = tuple(x.int() for x in b.need("min").list())
        hi = tuple(x.int() for x in b.need("max").list())
        boxes.append(b.wrap(Box, lo, hi))
    if not boxes:
        node.fail("fixed region needs at least one box")
    return node.wrap(Region, boxes[0].dims, boxes)


def _mapper(node):
    if node.v is None:
        return OneToOne()
    if isinstance(node.v, str):
        short = {"one_to_one": OneToOne, "all": All}
        if node.v not in short:
            node.fail(f"unknown mapper '{node.v}' (shorthand accepts 'one_to_one' or 'all'; others need an "
                      f"object with 'kind')")
        return short[node.v]()
    node.dict()   # its keys are checked per kind
    kind = node.need("kind").str()
    fields = {"one_to_one": set(), "all": set(), "neighborhood": {"radius", "radii"}, "fixed": {"region"},
              "slice": {"dim"}}
    if kind not in fields:
        node.at("kind").fail(f"unknown mapper kind '{kind}'")
    node.obj({"kind"} | fields[kind])
    if kind == "one_to_one":
        return OneToOne()
    if kind == "all":
        return All()
    if kind == "neighborhood":
        if node.has("radii"):
            radii = tuple(x.int() for x in node.at("radii").list())
        elif node.has("radius"):
            radii = (node.at("radius").int(),)
        else:
            node.fail("neighborhood needs 'radius' or 'radii'")
        return node.wrap(Neighborhood, radii)
    if kind == "fixed":
        return Fixed(_region(node.need("region")))
    return node.wrap(Slice, node.need("dim").int())


def _accessor(node, mode):
    if isinstance(node.v, str):
        return Accessor(buffer=node.v, mode=mode)
    node.obj({"buffer", "name", "mapper"})
    buf = node.need("buffer").str()
    name = node.at("name").str() if node.has("name") else None
    return Accessor(buffer=buf, mode=mode, mapper=_mapper(node.at("mapper")), name=name or buf)


def _target(node):
    name = node.str()
    try:
        return EnergyTarget(name)
    except ValueError:
        node.fail(f"unknown target '{name}' (expected one of {[t.value for t in EnergyTarget]})")


def _task(node, buffers):
    node.obj({"name", "range", "reads", "writes", "body", "params", "beta", "target"})
    name = node.need("name").str()
    rng = _shape(node.need("range"))
    reads = [_accessor(x, AccessMode.READ) for x in node.at("reads", []).list()]
    writes = [_accessor(x, AccessMode.WRITE) for x in node.need("writes").list()]
    params = {k: v.num() for k, v in node.at("params", {}).items()}
    beta = node.at("beta", 0.0).num()
    target = _target(node.at("target")) if node.has("target") else None
    body_node = node.need("body")
    if isinstance(body_node.v, str):
        if len(writes) != 1:
            body_node.fail(f"a bare expression string needs exactly one write accessor, task has {len(writes)}")
        body_node = _Node({writes[0].name: body_node.v}, body_node.path)
    arity = {}
    for kind, accs in (("reads", reads), ("writes", writes)):
        for a in accs:
            if a.buffer not in buffers:
                node.at(kind).fail(f"unknown buffer '{a.buffer}'")
            if kind == "reads":
                arity[a.name] = buffers[a.buffer].dims
    body = {w: n.wrap(parse_kernel, n.str(), arity, set(params), rng.dims) for w, n in body_node.items()}
    return Task(name=name, global_range=rng, accessors=reads + writes, body=body, params=params, beta=beta,
                target=target)


_DEVICE_KEYS = ("f_ref_ghz", "p_static_w", "p_dyn_ref_w", "alpha_exp", "throughput_ref")


def _device(node):
    node.obj({"levels_ghz", *_DEVICE_KEYS})
    kw = {k: node.at(k).num() for k in _DEVICE_KEYS if k in node.v}
    if "levels_ghz" in node.v:
        kw["levels_ghz"] = tuple(x.num() for x in node.at("levels_ghz").list())
    return node.wrap(DeviceModel, **kw)


def scenario_from_dict(data, path: str = "scenario") -> Scenario:
    """A ``Scenario`` from the parsed JSON document (strict)."""
    from .executor import LinkModel
    doc = _Node(data, path).obj({"nodes", "device", "devices", "link", "target", "queue_target", "buffers",
                                 "tasks", "expectations"})
    sc = Scenario()
    if doc.has("nodes"):
        sc.nodes = doc.at("nodes").int()
        if sc.nodes < 1:
            doc.at("nodes").fail(f"must be at least 1, got {sc.nodes}")
    for a, b in (("device", "devices"), ("target", "queue_target")):
        if a in doc.v and b in doc.v:
            doc.fail(f"give either '{a}' or '{b}', not both")
    if doc.has("device"):
        sc.devices = [_device(doc.at("device"))]
    elif doc.has("devices"):
        items = doc.at("devices").list()
        if not items:
            doc.at("devices").fail("must not be empty")
        sc.devices = [_device(x) for x in items]
    if doc.has("link"):
        ln = doc.at("link").obj({"latency_s", "bandwidth_bytes_per_s"})
        sc.link = ln.wrap(LinkModel, latency_s=ln.at("latency_s", 1e-6).num(),
                          bandwidth_bytes_per_s=ln.at("bandwidth_bytes_per_s", 1e9).num())
    tkey = "target" if "target" in doc.v else "queue_target"
    if doc.has(tkey):
        sc.queue_target = _target(_Node(doc.v[tkey], f"{path}.target"))
    buffers = {}
    for node in doc.at("buffers", []).list():
        buf = _buffer(node)
        if buf.name in buffers:
            node.fail(f"duplicate buffer name '{buf.name}'")
        buffers[buf.name] = buf
    sc.buffers = list(buffers.values())
    sc.tasks = [_task(x, buffers) for x in doc.at("tasks", []).list()]
    for node in doc.at("expectations", []).list():
        node.obj({"buffer", "values"})
        name = node.need("buffer").str()
        if name not in buffers:
            node.at("buffer").fail(f"unknown buffer '{name}'")
        vals = [x.num() for x in node.need("values").list()]
        want = buffers[name].extent.volume()
        if len(vals) != want:
            node.at("values").fail(f"expected {want} values for buffer '{name}', got {len(vals)}")
        sc.expectations.append((name, vals))
    return sc


def load_scenario(path) -> Scenario:
    with open(path, "r", encoding="utf-8") as fh:
        text = fh.read()
    try:
        data = json.loads(text)
    except json.JSONDecodeError as exc:
        raise ScenarioError(f"{path}: invalid JSON: {exc}") from exc
    return scenario_from_dict(data, path=str(path))


# ------------------------------------------------------------- writing

def _mapper_json(m):
    if isinstance(m, OneToOne):
        return "one_to_one"
    if isinstance(m, All):
        return "all"
    if isinstance(m, Neighborhood):
        return {"kind": "neighborhood", "radii": list(m.radii)}
    if isinstance(m, Slice):
        return {"kind": "slice", "dim": m.axis}
    if isinstance(m, Fixed):
        return {"kind": "fixed", "region": [{"min": list(b.mins), "max": list(b.maxs)} for b in m.region.boxes]}
    raise ScenarioError(f"cannot serialize mapper {type(m).__name__}")


def _accessor_json(a):
    plain = a.name == a.buffer and isinstance(a.mapper, OneToOne)
    if plain:
        return a.buffer
    out = {"buffer": a.buffer}
    if a.name != a.buffer:
        out["name"] = a.name
    if not isinstance(a.mapper, OneToOne):
        out["mapper"] = _mapper_json(a.mapper)
    return out


def _init_json(init):
    if init.kind in _INIT_SHORT:
        return init.kind
    if init.kind == "constant":
        return {"kind": "constant", "value": init.value}
    if init.kind == "array":
        return {"kind": "values", "values": np.asarray(init.data).reshape(-1).tolist()}
    return {"kind": "values", "values": list(init.values)}


def scenario_to_dict(sc: Scenario) -> dict:
    out = {}
    if sc.nodes is not None:
        out["nodes"] = sc.nodes
    if sc.devices is not None:
        out["devices"] = [{"levels_ghz": list(d.levels_ghz), **{k: getattr(d, k) for k in _DEVICE_KEYS}}
                          for d in sc.devices]
    if sc.link is not None:
        out["link"] = {"latency_s": sc.link.latency_s, "bandwidth_bytes_per_s": sc.link.bandwidth_bytes_per_s}
    if sc.queue_target is not None:
        out["target"] = sc.queue_target.value
    out["buffers"] = [{"name": b.name, "extent": list(b.extent.shape), "element_kind": b.element_kind,
                       "init": _init_json(b.init)} for b in sc.buffers]
    out["tasks"] = []
    for t in sc.tasks:
        d = {"name": t.name, "range": list(t.global_range.shape), "reads": [_accessor_json(a) for a in t.reads()],
             "writes": [_accessor_json(a) for a in t.writes()],
             "body": {k: format_kernel(e) for k, e in t.body.items()}}
        if t.params:
            d["params"] = dict(t.params)
        if t.beta:
            d["beta"] = t.beta
        if t.target is not None:
            d["target"] = t.target.value
        out["tasks"].append(d)
    if sc.expectations:
        out["expectations"] = [{"buffer": n, "values": list(v)} for n, v in sc.expectations]
    return out


def save_scenario(sc: Scenario, path):
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(scenario_to_dict(sc), fh, indent=2)
        fh.write("\n")


def bundled_scenario_path(name: str):
    """An example scenario shipped with this package (scenarios/), or None."""
    path = os.path.join(EXAMPLES, name if name.endswith(".json") else name + ".json")
    return path if os.path.isfile(path) else None


# ------------------------------------------------------------- running

@dataclass
class RunBundle:
    scenario: Scenario
    plan: object
    result: object
    energy: object            # EnergyReport (the reference model over measured durations)
    nodes: int
    target: EnergyTarget
    measured: object = None   # EnergyReport from NVML joules (run with energy=True)


def build_graph(sc: Scenario) -> TaskGraph:
    g = TaskGraph({b.name: b for b in sc.buffers})
    for t in sc.tasks:
        g.submit(t)
    return g


def run_scenario(sc: Scenario, nodes: Optional[int] = None, target: Optional[EnergyTarget] = None,
                 energy: bool = False, placement=None) -> RunBundle:
    """Plan and run on the GPUs.  CLI flag > scenario field > default
    (1 node, MAX_PERF), as the reference (scenario.py:559-580)."""
    from .executor import run
    from .measure import measured_energy
    from .scheduler import generate_commands
    n = nodes if nodes is not None else (sc.nodes or 1)
    tgt = target if target is not None else (sc.queue_target or EnergyTarget.MAX_PERF)
    plan = generate_commands(build_graph(sc), n, devices=sc.devices, queue_target=tgt)
    result = run(plan, link=sc.link, energy=energy, placement=placement)
    model = account_energy(result.trace, plan.devices, result.makespan)
    meas = measured_energy(result) if energy else None
    return RunBundle(sc, plan, result, model, n, tgt, meas)


def _bits(a):
    return a.view(np.uint64) if a.dtype == np.float64 else a.view(np.uint32) if a.dtype == np.float32 else a


def _first_diff(a, b):
    return tuple(int(x[0]) for x in np.nonzero(_bits(a) != _bits(b)))


def check_expectations(sc: Scenario, buffers: dict) -> list:
    """Declared expected values vs the gathered buffers, bit for bit."""
    out = []
    kinds = {b.name: b for b in sc.buffers}
    for name, values in sc.expectations:
        b = kinds[name]
        want = np.array(values, dtype=b.dtype).reshape(b.extent.shape)
        got = buffers[name]
        if not np.array_equal(_bits(want), _bits(got)):
            at = _first_diff(want, got)
            out.append(f"buffer '{name}' differs from expectation at index {at}: expected {want[at]}, got {got[at]}")
    return out


def validate_against_serial(sc: Scenario, nodes: int, target: Optional[EnergyTarget] = None,
                            placement=None) -> list:
    """The distributed run against a 1-node run, every buffer bit for bit."""
    one = run_scenario(sc, nodes=1, target=target, placement=placement).result.buffers
    many = run_scenario(sc, nodes=nodes, target=target, placement=placement).result.buffers
    out = []
    for b in sc.buffers:
        x, y = one[b.name], many[b.name]
        if not np.array_equal(_bits(x), _bits(y)):
            at = _first_diff(x, y)
            out.append(f"buffer '{b.name}' diverges at index {at} with {nodes} nodes: serial {x[at]}, "
                       f"distributed {y[at]}")
    return out
