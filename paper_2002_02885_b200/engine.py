"""Model description and optimizer state for the pack path.

Mirrors the parts of the reference's `packtrain.engine` that the pack API
exposes (engine.py:14-177): constants, error types, the flat node-list graph
a handle carries, Xavier initialisation (bit-identical seeding) and the
optimizer state object.  The arithmetic itself (forward, backward, update)
runs on the GPU inside `pk_pack_step` — see csrc/pk_kernels.cuh — so this
module has no numpy forward/backward: there is no CPU path.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

LEAKY_SLOPE = 0.01
MOMENTUM_COEF = 0.9
ADAM_BETA1 = 0.9
ADAM_BETA2 = 0.999
ADAM_EPS = 1e-8
ADAGRAD_EPS = 1e-10

ACTIVATIONS = ("sigmoid", "leaky_relu", "tanh", "relu")
OPTIMIZERS = ("sgd", "momentum", "adam", "adagrad")
SLOT_NAMES = {"sgd": (), "momentum": ("velocity",), "adagrad": ("accum",),
              "adam": ("m", "v")}


class EngineError(Exception):
    pass


class ShapeMismatch(EngineError):
    def __init__(self, port: str, expected, got):
        self.port, self.expected, self.got = port, expected, got
        super().__init__(f"port {port!r}: expected shape {expected}, got {got}")

    def __reduce__(self):  # pickles across the Hyperband pool's gather
        return (type(self), (self.port, self.expected, self.got))


class NonFiniteGradient(EngineError):
    def __init__(self, param: str):
        self.param = param
        super().__init__(f"non-finite gradient for parameter {param!r}")

    def __reduce__(self):
        return (type(self), (self.param,))


@dataclass(frozen=True)
class Node:
    name: str
    op: str
    inputs: tuple = ()
    port: str | None = None
    weight: str | None = None
    bias: str | None = None
    label_port: str | None = None
    member: str = ""
    layer_index: int = -1


@dataclass
class ComputationGraph:
    """Same fields as the reference graph (engine.py:56-72); here it is a
    description (names, ports, shapes) — execution is the device's."""
    model_id: str
    nodes: list
    input_ports: dict
    label_ports: dict
    output_ports: dict
    loss_heads: dict
    param_shapes: dict
    port_alias: dict = field(default_factory=dict)

    def resolve(self, port: str) -> str:
        return self.port_alias.get(port, port)

    def physical_ports(self):
        return sorted({self.resolve(p) for p in self.input_ports})


def build_mlp(model_id, input_dim, hidden, classes, activation="relu",
              dataset_binding="default") -> ComputationGraph:
    """Affine stack + softmax-xent head; node/param names as engine.py:108-143."""
    if activation not in ACTIVATIONS:
        raise EngineError(f"unknown activation {activation!r}")
    dims = [input_dim, *hidden, classes]
    nodes = [Node(f"{model_id}/in", "input", port=f"{model_id}/x", member=model_id)]
    shapes = {}
    prev = nodes[0].name
    n_aff = len(dims) - 1
    for i in range(n_aff):
        w, b = f"{model_id}/L{i}/W", f"{model_id}/L{i}/b"
        shapes[w] = (dims[i], dims[i + 1])
        shapes[b] = (dims[i + 1],)
        nodes.append(Node(f"{model_id}/aff{i}", "affine", (prev,), weight=w, bias=b,
                          member=model_id, layer_index=i))
        prev = nodes[-1].name
        if i + 1 < n_aff:
            nodes.append(Node(f"{model_id}/act{i}", activation, (prev,),
                              member=model_id, layer_index=i))
            prev = nodes[-1].name
    nodes.append(Node(f"{model_id}/loss", "softmax_xent", (prev,),
                      label_port=f"{model_id}/y", member=model_id))
    return ComputationGraph(model_id, nodes, {f"{model_id}/x": (input_dim, dataset_binding)},
                            {f"{model_id}/y": classes}, {model_id: prev},
                            {model_id: nodes[-1].name}, shapes)


def _param_rng(member: str, layer_index: int, seed: int) -> np.random.Generator:
    h = hashlib.sha256(f"{member}|{layer_index}|{seed}".encode()).digest()
    return np.random.default_rng(int.from_bytes(h[:8], "little"))


def init_parameters(graph: ComputationGraph, seed: int) -> dict:
    """Xavier-uniform W, zero b (engine.py:162-177).  Done on the host with
    the reference's exact numpy draws, then uploaded: the device starts from
    float32(reference init) bit-exactly."""
    out = {}
    for node in graph.nodes:
        if node.op != "affine":
            continue
        fi, fo = graph.param_shapes[node.weight]
        lim = np.sqrt(6.0 / (fi + fo))
        out[node.weight] = _param_rng(node.member, node.layer_index, seed).uniform(
            -lim, lim, size=(fi, fo))
        out[node.bias] = np.zeros(fo)
    return out


class OptimizerState:
    """kind / learning_rate / step_counter / slots as engine.py:85-96.

    When owned by a device-backed handle, `slots` materialises lazily from the
    device (download on read) and `learning_rate` writes through to the
    member's device control block."""

    def __init__(self, kind: str, learning_rate: float, step_counter: int = 0,
                 slots: dict | None = None):
        self.kind = kind
        self._lr = float(learning_rate)
        self._step = int(step_counter)
        self._slots = {} if slots is None else slots
        self._owner = None  # the ModelHandle that syncs with the device

    @property
    def learning_rate(self):
        return self._lr

    @learning_rate.setter
    def learning_rate(self, v):
        if v <= 0:
            raise EngineError("learning rate must be positive")
        self._lr = float(v)
        if self._owner is not None:
            self._owner._lr_changed()

    @property
    def step_counter(self):
        return self._step

    @step_counter.setter
    def step_counter(self, v):
        if self._owner is not None:
            self._owner._pull()
            self._owner._host_authoritative()
        self._step = int(v)

    @property
    def slots(self):
        if self._owner is not None:
            self._owner._pull()
            self._owner._host_authoritative()
        return self._slots

    @slots.setter
    def slots(self, v):
        if self._owner is not None:
            self._owner._pull()
            self._owner._host_authoritative()
        self._slots = v

    def slot(self, param: str, like: np.ndarray, name: str) -> np.ndarray:
        per = self.slots.setdefault(param, {})
        if name not in per:
            per[name] = np.zeros_like(like)
        return per[name]

    def __repr__(self):
        return (f"OptimizerState(kind={self.kind!r}, learning_rate={self._lr!r}, "
                f"step_counter={self._step!r})")


def make_optimizer(kind: str, learning_rate: float) -> OptimizerState:
    """engine.py:99-105."""
    kind = kind.lower()
    if kind not in OPTIMIZERS:
        raise EngineError(f"unknown optimizer kind {kind!r}")
    if learning_rate <= 0:
        raise EngineError("learning rate must be positive")
    return OptimizerState(kind, learning_rate)
