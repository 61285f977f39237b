"""ctypes wrapper over oracle/liboracle.so — the CPU parity checker.

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs. The product package
(paper_2502_02493_b200) never imports this module.

The C library restates the reference path (proj/src/*.cpp under
/root/reference) with identical fp32 operation order; tests/test_oracle.py
pins it bit-for-bit against fixtures written by the unmodified reference.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

ALGORITHMS = {"vanilla": 0, "sd": 1, "sd_tree": 2, "easyspec": 3}
STATUS_NAMES = {0: "ok", 1: "config", 2: "io", 3: "check", 4: "shape", 5: "structure", 6: "domain"}


class EoConfig(C.Structure):
    _fields_ = [
        ("vocab_size", C.c_int), ("d_model", C.c_int), ("n_layers", C.c_int), ("n_heads", C.c_int),
        ("d_head", C.c_int), ("d_mlp", C.c_int), ("max_positions", C.c_int), ("norm_eps", C.c_float),
        ("seed", C.c_uint64),
    ]


class EoRun(C.Structure):
    _fields_ = [
        ("algorithm", C.c_int), ("n", C.c_int), ("widths", C.POINTER(C.c_int)), ("lp_size", C.c_int),
        ("plan_override", C.c_char_p), ("temperature", C.c_float), ("max_new_tokens", C.c_int),
        ("seed", C.c_uint64), ("calibration", C.c_int),
    ]


def build() -> None:
    """Compile liboracle.so (gcc, no GPU)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        P = C.POINTER
        L.eo_model_init.restype = C.c_void_p
        L.eo_model_init.argtypes = [P(EoConfig), P(C.c_int)]
        L.eo_model_truncated.restype = C.c_void_p
        L.eo_model_truncated.argtypes = [C.c_void_p, C.c_int, P(C.c_int)]
        L.eo_model_free.argtypes = [C.c_void_p]
        L.eo_model_tensor.restype = P(C.c_float)
        L.eo_model_tensor.argtypes = [C.c_void_p, C.c_char_p, C.c_int, P(C.c_int), P(C.c_int)]
        L.eo_prefill.argtypes = [C.c_void_p, C.c_char_p, P(C.c_int), C.c_int] + [P(C.c_float)] * 4
        L.eo_plan_groups.argtypes = [C.c_int, C.c_int, C.c_char_p, C.c_int]
        L.eo_parse_plan.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
        L.eo_generate.restype = C.c_void_p
        L.eo_generate.argtypes = [C.c_void_p, C.c_void_p, P(EoRun), C.c_char_p, C.c_int]
        L.eo_result_status.argtypes = [C.c_void_p]
        L.eo_result_error.restype = C.c_char_p
        L.eo_result_error.argtypes = [C.c_void_p]
        L.eo_result_tokens.restype = P(C.c_int)
        L.eo_result_tokens.argtypes = [C.c_void_p, P(C.c_int)]
        L.eo_result_n_iters.argtypes = [C.c_void_p]
        L.eo_result_iter.argtypes = [C.c_void_p, C.c_int, P(C.c_int)]
        L.eo_result_kvsums.argtypes = [C.c_void_p, C.c_int, C.c_int, P(C.c_double)]
        L.eo_result_cache_len.argtypes = [C.c_void_p, C.c_int]
        L.eo_result_cache_rows.argtypes = [C.c_void_p, C.c_int, C.c_int, P(C.c_float), P(C.c_float)]
        L.eo_result_free.argtypes = [C.c_void_p]
        L.eo_verify_tree.argtypes = [C.c_int, C.c_int, P(C.c_int), P(C.c_int), P(C.c_int), C.c_int,
                                     P(C.c_float), P(C.c_float), C.c_int, P(C.c_int), C.c_float,
                                     C.c_uint64, P(C.c_int), P(C.c_int), P(C.c_int)]
        L.eo_select_children.argtypes = [P(C.c_float), C.c_int, C.c_int, C.c_float, C.c_uint64, P(C.c_int)]
        L.eo_rng_uniforms.argtypes = [C.c_uint64, C.c_int, P(C.c_double)]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.kind = STATUS_NAMES.get(status, str(status))


def _fptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _iptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int))


@dataclass
class ModelConfig:
    """espec::ModelConfig (proj/include/espec/model.hpp:19-33)."""
    vocab_size: int = 258
    d_model: int = 64
    n_layers: int = 4
    n_heads: int = 4
    d_head: int = 16
    d_mlp: int = 128
    max_positions: int = 512
    norm_eps: float = 1e-5
    seed: int = 0

    def to_c(self) -> EoConfig:
        return EoConfig(self.vocab_size, self.d_model, self.n_layers, self.n_heads, self.d_head,
                        self.d_mlp, self.max_positions, self.norm_eps, self.seed)


def tiny_config(n_layers: int, seed: int, d_model=32, n_heads=2, d_head=16, d_mlp=64, max_positions=128):
    """proj/tests/test_support.hpp:44-54."""
    return ModelConfig(d_model=d_model, n_heads=n_heads, d_head=d_head, d_mlp=d_mlp,
                       n_layers=n_layers, max_positions=max_positions, seed=seed)


class Model:
    """A seeded fp32 model (init_model, proj/src/model.cpp:38-84)."""

    def __init__(self, cfg: ModelConfig, _handle=None, _parent=None):
        self.cfg = cfg
        self._parent = _parent
        if _handle is None:
            st = C.c_int(0)
            c = cfg.to_c()
            _handle = lib().eo_model_init(C.byref(c), C.byref(st))
            if not _handle:
                raise OracleError(st.value, "init_model rejected the config")
        self._h = _handle

    def truncated(self, keep: int) -> "Model":
        st = C.c_int(0)
        h = lib().eo_model_truncated(self._h, keep, C.byref(st))
        if not h:
            raise OracleError(st.value, "keep_layers out of range")
        cfg = ModelConfig(**{**self.cfg.__dict__, "n_layers": keep})
        return Model(cfg, _handle=h, _parent=self)

    def tensor(self, name: str, layer: int = -1) -> np.ndarray:
        r, c = C.c_int(0), C.c_int(0)
        p = lib().eo_model_tensor(self._h, name.encode(), layer, C.byref(r), C.byref(c))
        if not p:
            raise KeyError(name)
        return np.ctypeslib.as_array(p, shape=(r.value, c.value)).copy()

    def prefill(self, tokens: Sequence[int], plan: Optional[str] = None):
        """One chain pass on a fresh cache -> (hidden, logits, k, v)."""
        n = len(tokens)
        cfg = self.cfg
        toks = np.asarray(tokens, dtype=np.int32)
        hidden = np.zeros((n, cfg.d_model), np.float32)
        logits = np.zeros((n, cfg.vocab_size), np.float32)
        k = np.zeros((cfg.n_layers, n, cfg.d_model), np.float32)
        v = np.zeros_like(k)
        st = lib().eo_prefill(self._h, (plan or "").encode(), _iptr(toks), n, _fptr(hidden),
                              _fptr(logits), _fptr(k), _fptr(v))
        if st:
            raise OracleError(st)
        return hidden, logits, k, v

    def __del__(self):
        try:
            if self._h and lib is not None:
                lib().eo_model_free(self._h)
        except Exception:
            pass


@dataclass
class RunConfig:
    """espec::RunConfig (proj/include/espec/orchestrator.hpp:23-38)."""
    algorithm: str = "easyspec"
    n: int = 5
    widths: Optional[List[int]] = None
    lp_size: int = 4
    plan_override: Optional[str] = None
    temperature: float = 0.8
    max_new_tokens: int = 64
    seed: int = 1
    calibration: bool = True

    def effective_widths(self) -> List[int]:
        return list(self.widths) if self.widths else [1] * self.n


@dataclass
class Iteration:
    m: int
    n: int
    drafted_nodes: int
    emitted: int
    sequential_forwards: int
    fuzzy_forwards: int
    base_forwards: int
    committed: int
    draft_committed: int
    base_committed: int
    draft_kv: np.ndarray = field(repr=False, default=None)
    base_kv: np.ndarray = field(repr=False, default=None)


@dataclass
class Generation:
    tokens: List[int]
    iterations: List[Iteration]
    draft_cache: List[tuple]  # per layer (k, v) of the final committed rows
    base_cache: List[tuple]

    @property
    def alpha(self) -> float:
        att = sum(it.n for it in self.iterations)
        return sum(it.m for it in self.iterations) / att if att else 0.0


def generate(base: Model, draft: Model, run: RunConfig, prompt: bytes, with_cache: bool = True) -> Generation:
    """espec::generate (proj/src/orchestrator.cpp:488-492)."""
    L = lib()
    widths = np.asarray(run.effective_widths(), dtype=np.int32)
    r = EoRun(ALGORITHMS[run.algorithm], run.n, _iptr(widths), run.lp_size,
              (run.plan_override or "").encode(), run.temperature, run.max_new_tokens, run.seed,
              1 if run.calibration else 0)
    h = L.eo_generate(base._h, draft._h, C.byref(r), prompt, len(prompt))
    try:
        st = L.eo_result_status(h)
        if st:
            raise OracleError(st, L.eo_result_error(h).decode())
        n = C.c_int(0)
        p = L.eo_result_tokens(h, C.byref(n))
        tokens = [p[i] for i in range(n.value)]
        iters = []
        out = (C.c_int * 10)()
        for i in range(L.eo_result_n_iters(h)):
            L.eo_result_iter(h, i, out)
            it = Iteration(*list(out))
            ds = np.zeros((draft.cfg.n_layers, 4), np.float64)
            bs = np.zeros((base.cfg.n_layers, 4), np.float64)
            L.eo_result_kvsums(h, i, 0, ds.ctypes.data_as(C.POINTER(C.c_double)))
            L.eo_result_kvsums(h, i, 1, bs.ctypes.data_as(C.POINTER(C.c_double)))
            it.draft_kv, it.base_kv = ds, bs
            iters.append(it)
        caches = []
        for which, m in ((0, draft), (1, base)):
            rows = L.eo_result_cache_len(h, which)
            layers = []
            if with_cache:
                for layer in range(m.cfg.n_layers):
                    k = np.zeros((rows, m.cfg.d_model), np.float32)
                    v = np.zeros_like(k)
                    L.eo_result_cache_rows(h, which, layer, _fptr(k), _fptr(v))
                    layers.append((k, v))
            caches.append(layers)
        return Generation(tokens, iters, caches[0], caches[1])
    finally:
        L.eo_result_free(h)


def plan_groups(n_layers: int, lp: int) -> str:
    buf = C.create_string_buffer(4096)
    st = lib().eo_plan_groups(n_layers, lp, buf, 4096)
    if st:
        raise OracleError(st)
    return buf.value.decode()


def parse_plan(spec: str) -> str:
    buf = C.create_string_buffer(4096)
    st = lib().eo_parse_plan(spec.encode(), buf, 4096)
    if st:
        raise OracleError(st, spec)
    return buf.value.decode()


def verify_tree(vocab, tokens, parents, prob_index, dists, base_dists, widths, temperature, seed):
    """verify_tree over an explicit tree (proj/src/verifier.cpp:86-177) -> (m, accepted, bonus)."""
    t = np.asarray(tokens, np.int32)
    p = np.asarray(parents, np.int32)
    pi = np.asarray(prob_index, np.int32)
    d = np.ascontiguousarray(dists, np.float32)
    b = np.ascontiguousarray(base_dists, np.float32)
    w = np.asarray(widths, np.int32)
    m, bonus = C.c_int(0), C.c_int(0)
    acc = np.zeros(len(w) + 1, np.int32)
    st = lib().eo_verify_tree(vocab, len(t), _iptr(t), _iptr(p), _iptr(pi), d.shape[0], _fptr(d), _fptr(b),
                              len(w), _iptr(w), temperature, seed, C.byref(m), _iptr(acc), C.byref(bonus))
    if st:
        raise OracleError(st)
    return m.value, list(acc[: m.value]), bonus.value


def select_children(logits, k, temperature, seed) -> List[int]:
    lg = np.ascontiguousarray(logits, np.float32)
    out = np.zeros(k, np.int32)
    n = lib().eo_select_children(_fptr(lg), lg.shape[0], k, temperature, seed, _iptr(out))
    if n < 0:
        raise OracleError(-n)
    return list(out[:n])


def rng_uniforms(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n, np.float64)
    lib().eo_rng_uniforms(seed, n, out.ctypes.data_as(C.POINTER(C.c_double)))
    return out


def tokenize(prompt: bytes) -> List[int]:
    """tokenize_prompt (proj/src/orchestrator.cpp:42-52): BOS + bytes."""
    return [256] + list(prompt)
