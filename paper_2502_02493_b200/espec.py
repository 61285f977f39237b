"""Python binding of the B200 EasySpec engine (ctypes over include/espec_c.h).

Mirrors the reference's public C++ surface (proj/include/espec/*.hpp):
``ModelConfig``/``RunConfig`` (model.hpp:19-33, orchestrator.hpp:23-38),
``Engine.generate`` (= espec::generate, orchestrator.cpp:488-492), the
stage-level ``begin``/``step`` loop (Generation::run, orchestrator.cpp:163-195),
``forward`` (forward_sequential / forward_fuzzy, draft_engine.cpp:35-133),
``cache_view`` (the IterationHook view) and ``plan_groups`` /
``parse_plan_override`` (layer_plan.cpp). Errors surface as ``EspecError``
carrying the reference's exception kind (errors.hpp:11-44).

There is no CPU fallback: importing this module without the compiled
``libespec_b200.so`` raises, and every compute call runs on the GPU.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field, replace
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# ESPEC_LIB: load another in-tree build (A/B of two builds on one box)
LIB_PATH = os.path.join(_HERE, os.environ.get("ESPEC_LIB", "libespec_b200.so"))

F32, BF16 = 0, 1
ALGORITHMS = {"vanilla": 0, "sd": 1, "sd_tree": 2, "easyspec": 3}
STATUS = {0: "ok", 1: "config", 2: "io", 3: "check", 4: "shape", 5: "structure", 6: "domain", 7: "cuda", 8: "nccl"}
BOS, EOS = 256, 257


class EspecError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.kind = STATUS.get(status, str(status))


class _ModelCfg(C.Structure):
    _fields_ = [("vocab_size", C.c_int), ("d_model", C.c_int), ("n_layers", C.c_int), ("n_heads", C.c_int),
                ("n_kv_heads", C.c_int), ("d_head", C.c_int), ("d_mlp", C.c_int), ("max_positions", C.c_int),
                ("norm_eps", C.c_float), ("rope_theta", C.c_float), ("tied_head", C.c_int),
                ("weight_dtype", C.c_int), ("kv_dtype", C.c_int), ("seed", C.c_uint64)]


class _RunCfg(C.Structure):
    _fields_ = [("algorithm", C.c_int), ("n", C.c_int), ("widths", C.POINTER(C.c_int)), ("lp_size", C.c_int),
                ("plan_override", C.c_char_p), ("temperature", C.c_float), ("max_new_tokens", C.c_int),
                ("seed", C.c_uint64), ("calibration", C.c_int), ("strict_greedy_tree", C.c_int)]


MAX_NODES = 64  # ESPEC_MAX_NODES


class _Tree(C.Structure):
    """espec_tree = espec::DraftTree (draft_engine.hpp:63-84)."""
    _fields_ = [("id", C.c_uint64), ("n_nodes", C.c_int), ("root_children", C.c_int), ("n_levels", C.c_int),
                ("n_dists", C.c_int), ("widths", C.c_int32 * MAX_NODES)] + \
               [(n, C.c_int32 * MAX_NODES) for n in ("token", "parent", "depth", "prob_index", "cache_row",
                                                     "first_child", "n_children")] + \
               [("dists", C.POINTER(C.c_float)), ("dist_capacity", C.c_int)]


class _Outcome(C.Structure):
    """espec_outcome = espec::VerificationOutcome (verifier.hpp:14-21)."""
    _fields_ = [("id", C.c_uint64), ("m", C.c_int), ("n", C.c_int), ("bonus", C.c_int32),
                ("accepted_path", C.c_int32 * MAX_NODES), ("accepted_tokens", C.c_int32 * MAX_NODES)]


class _DevMap(C.Structure):
    _fields_ = [("device", C.c_int), ("n_lp_devices", C.c_int), ("lp_devices", C.POINTER(C.c_int)),
                ("tp_size", C.c_int), ("tp_rank", C.c_int)]


class _Iter(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("m", "n", "drafted_nodes", "emitted", "sequential_forwards",
                                       "fuzzy_forwards", "base_forwards", "committed", "draft_committed",
                                       "base_committed", "bonus")] + \
               [(n, C.c_float) for n in ("calibrate_ms", "draft_ms", "verify_ms")] + \
               [(n, C.c_double) for n in ("calibrate_sim", "draft_sim", "verify_sim")]


class _Report(C.Structure):
    """espec_report = RunReport's derived metrics (report.hpp:40-57)."""
    _fields_ = [("n_iterations", C.c_int), ("has_alpha", C.c_int), ("alpha", C.c_double),
                ("tokens_emitted", C.c_int64), ("mean_accept_len", C.c_double), ("tokens_per_s", C.c_double),
                ("draft_per_100_s", C.c_double), ("verify_per_100_s", C.c_double),
                ("calibrate_per_100_s", C.c_double), ("draft_total_per_100_s", C.c_double),
                ("total_s", C.c_double), ("speedup_vs_vanilla", C.c_double),
                ("draft_per_100_sim", C.c_double), ("verify_per_100_sim", C.c_double),
                ("calibrate_per_100_sim", C.c_double), ("draft_total_per_100_sim", C.c_double),
                ("total_sim", C.c_double)]


class _CostParams(C.Structure):
    """espec_cost_params = CostParams (cost_sim.hpp:17-32)."""
    _fields_ = [(n, C.c_double) for n in ("c_fixed", "c_mem", "c_comp", "t_addi", "attn_workload", "mlp_workload",
                                          "base_layer_workload")] + \
               [(n, C.c_int) for n in ("tp_size_base", "tp_size_draft", "devices")]


class _SimRow(C.Structure):
    """espec_similarity_row = SimilarityRow (draft_engine.hpp:124-127)."""
    _fields_ = [("lp_size", C.c_int)] + [(n, C.c_double) for n in ("h", "q", "k", "v", "attn_out")]


_lib = None


def lib():
    """Load libespec_b200.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (make -C "
                              f"paper_2502_02493_b200/csrc) — there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        P, V = C.POINTER, C.c_void_p
        L.espec_engine_create.argtypes = [P(_ModelCfg), P(_ModelCfg), P(_RunCfg), P(_DevMap), P(V)]
        L.espec_engine_destroy.argtypes = [V]
        L.espec_last_error.restype = C.c_char_p
        L.espec_last_error.argtypes = [V]
        L.espec_create_error.restype = C.c_char_p
        L.espec_init_weights_seeded.argtypes = [V, C.c_int, C.c_uint64, C.c_int]
        L.espec_share_truncated_draft.argtypes = [V]
        L.espec_load_tensor.argtypes = [V, C.c_int, C.c_char_p, C.c_int, P(C.c_float), C.c_int64, C.c_int64]
        L.espec_read_tensor.argtypes = [V, C.c_int, C.c_char_p, C.c_int, P(C.c_float), C.c_int64, C.c_int64]
        L.espec_set_run.argtypes = [V, P(_RunCfg)]
        L.espec_generate.argtypes = [V, C.c_char_p, C.c_int, P(C.c_int32), P(C.c_int), P(_Iter), P(C.c_int)]
        L.espec_begin.argtypes = [V, P(C.c_int32), C.c_int]
        L.espec_step.argtypes = [V, P(C.c_int32), P(C.c_int), P(_Iter)]
        L.espec_done.argtypes = [V]
        L.espec_cache_view.argtypes = [V, C.c_int, C.c_int, C.c_int, C.c_int, P(C.c_float), P(C.c_float), P(C.c_int)]
        L.espec_committed.argtypes = [V, P(C.c_int32), C.c_int, P(C.c_int)]
        L.espec_forward.argtypes = [V, C.c_int, P(C.c_int32), C.c_int, C.c_char_p, P(C.c_float), P(C.c_float)]
        L.espec_plan_groups.argtypes = [C.c_int, C.c_int, C.c_char_p, C.c_int]
        L.espec_parse_plan.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
        L.espec_kernel_launches.argtypes = [V]
        L.espec_reset_kernel_launches.argtypes = [V]
        L.espec_sync.argtypes = [V]
        L.espec_generate_tokens.argtypes = [V, P(C.c_int32), C.c_int, P(C.c_int32), P(C.c_int), P(_Iter), P(C.c_int)]
        L.espec_stream.restype = C.c_void_p
        L.espec_stream.argtypes = [V]
        L.espec_time_site.argtypes = [V, C.c_int, C.c_int]
        L.espec_site_stats.argtypes = [V, P(C.c_int), P(C.c_double), P(C.c_double)]
        L.espec_io_bytes.argtypes = [V, P(C.c_int64), P(C.c_int64)]
        L.espec_comm_link.argtypes = [P(V), C.c_int]
        L.espec_comm_export.argtypes = [V, C.c_void_p]
        L.espec_comm_import.argtypes = [V, C.c_void_p, C.c_int]
        L.espec_comm_loopback.argtypes = [V]
        L.espec_prefill.argtypes = [V, P(C.c_int32), C.c_int]
        L.espec_prefix_distribution.argtypes = [V, P(C.c_int32), C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                                P(C.c_int32), P(C.c_int64), C.c_int, P(C.c_int)]
        L.espec_total_variation.restype = C.c_double
        L.espec_total_variation.argtypes = [P(C.c_int32), P(C.c_int64), C.c_int, P(C.c_int32), P(C.c_int64), C.c_int,
                                            C.c_int, C.c_int64, C.c_int64]
        L.espec_forward_tree.argtypes = [V, C.c_int, P(C.c_int32), C.c_int, P(C.c_int32), P(C.c_int32), C.c_int,
                                         C.c_char_p, P(C.c_float), P(C.c_float)]
        L.espec_calibrate.argtypes = [V, P(C.c_float)]
        L.espec_draft.argtypes = [V, P(_Tree)]
        L.espec_verify.argtypes = [V, P(_Tree), P(_Outcome)]
        L.espec_resolve_draft_cache.argtypes = [V, P(_Outcome)]
        L.espec_commit_outcome.argtypes = [V, P(C.c_int32), P(C.c_int), P(_Iter)]
        L.espec_aggregate.argtypes = [P(_Iter), C.c_int, C.c_double, P(_Report)]
        L.espec_cost_defaults.argtypes = [P(_CostParams)]
        L.espec_cost_eval.argtypes = [P(_CostParams), C.c_int, C.c_double, C.c_double, C.c_int, C.c_char_p,
                                      P(C.c_double)]
        L.espec_cost_total_time.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, C.c_double, P(C.c_double)]
        L.espec_set_cost.argtypes = [V, P(_CostParams)]
        L.espec_occupancy_csv.argtypes = [V, C.c_char_p, C.c_int, P(C.c_int)]
        L.espec_report_emit.argtypes = [P(_Report), P(_Iter), C.c_int, C.c_char_p, C.c_int, P(C.c_int), C.c_int,
                                        C.c_int, C.c_int, C.c_char_p, C.c_int, P(C.c_int)]
        L.espec_model_file_config.argtypes = [C.c_char_p, P(_ModelCfg)]
        L.espec_load_model_file.argtypes = [V, C.c_int, C.c_char_p]
        L.espec_save_model_file.argtypes = [V, C.c_int, C.c_char_p]
        L.espec_probe_similarity.argtypes = [V, P(C.c_int), C.c_int, P(C.c_int32), P(C.c_int), C.c_int, P(_SimRow)]
        _lib = L
    return _lib


def _f(a):
    return a.ctypes.data_as(C.POINTER(C.c_float)) if a is not None else None


def _i(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


@dataclass
class ModelConfig:
    """espec::ModelConfig plus GQA / rope base / untied head / storage dtypes."""
    vocab_size: int = 258
    d_model: int = 64
    n_layers: int = 4
    n_heads: int = 4
    d_head: int = 16
    d_mlp: int = 128
    max_positions: int = 512
    norm_eps: float = 1e-5
    seed: int = 0
    n_kv_heads: Optional[int] = None
    rope_theta: float = 10000.0
    tied_head: bool = True
    weight_dtype: int = F32
    kv_dtype: int = F32

    def _c(self) -> _ModelCfg:
        return _ModelCfg(self.vocab_size, self.d_model, self.n_layers, self.n_heads,
                         self.n_kv_heads or self.n_heads, self.d_head, self.d_mlp, self.max_positions,
                         self.norm_eps, self.rope_theta, 1 if self.tied_head else 0, self.weight_dtype,
                         self.kv_dtype, self.seed)


def tiny_config(n_layers: int, seed: int, d_model=32, n_heads=2, d_head=16, d_mlp=64, max_positions=128):
    """proj/tests/test_support.hpp:44-54."""
    return ModelConfig(d_model=d_model, n_heads=n_heads, d_head=d_head, d_mlp=d_mlp, n_layers=n_layers,
                       max_positions=max_positions, seed=seed)


@dataclass
class RunConfig:
    """espec::RunConfig (proj/include/espec/orchestrator.hpp:23-38)."""
    algorithm: str = "easyspec"
    n: int = 5
    widths: Optional[List[int]] = None
    lp_size: int = 4
    plan_override: Optional[str] = None
    temperature: float = 0.0
    max_new_tokens: int = 64
    seed: int = 1
    calibration: bool = True
    # reproduce the reference's greedy multi-sibling CheckError (verifier.cpp:146-158)
    strict_greedy_tree: bool = False

    def effective_widths(self) -> List[int]:
        return list(self.widths) if self.widths else [1] * self.n


@dataclass
class IterationTrace:
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
    bonus: int
    calibrate_ms: float
    draft_ms: float
    verify_ms: float
    calibrate_sim: float = 0.0  # the cost model's units (IterationTrace::*_sim)
    draft_sim: float = 0.0
    verify_sim: float = 0.0


def _trace(t: _Iter) -> IterationTrace:
    return IterationTrace(*(getattr(t, n) for n, _ in _Iter._fields_))


def tokenize(prompt: bytes) -> List[int]:
    """tokenize_prompt (proj/src/orchestrator.cpp:42-52)."""
    return [BOS] + list(prompt)


class Engine:
    """One base/drafter pair with its caches on one B200."""

    DRAFT, BASE = 0, 1

    def __init__(self, base: ModelConfig, draft: ModelConfig, run: RunConfig, device: int = 0, tp_size: int = 1,
                 tp_rank: int = 0, draft_layout: str = "tp"):
        """draft_layout "tp": the drafter is tensor-parallel like the base;
        "lp": the paper's layer-parallel placement (group slot j on rank j,
        full-head attention + its KV on the owner, MLP / head tensor-parallel)."""
        L = lib()
        self.base_cfg, self.draft_cfg = base, draft
        self.tp_size, self.tp_rank = tp_size, tp_rank
        self._h = C.c_void_p()
        self._keep = []
        if draft_layout == "lp":
            if tp_size < 2:  # n_lp_devices <= 1 would silently mean the tensor-parallel drafter
                raise EspecError(1, "layer-parallel placement needs tp_size > 1 (one GPU per group slot)")
            lpd = (C.c_int * tp_size)(*range(tp_size))
            self._lpd = lpd
            dm = _DevMap(device, tp_size, lpd, tp_size, tp_rank)
        elif draft_layout == "tp":
            dm = _DevMap(device, 1, None, tp_size, tp_rank)
        else:
            raise ValueError(f"draft_layout must be 'tp' or 'lp', not {draft_layout!r}")
        st = L.espec_engine_create(C.byref(base._c()), C.byref(draft._c()), C.byref(self._run(run)), C.byref(dm),
                                   C.byref(self._h))
        if st:
            raise EspecError(st, L.espec_create_error().decode())
        self.run = run

    def _run(self, run: RunConfig) -> _RunCfg:
        w = np.asarray(run.effective_widths(), np.int32)
        po = (run.plan_override or "").encode()
        self._keep = [w, po]
        return _RunCfg(ALGORITHMS[run.algorithm], run.n, _i(w), run.lp_size, po, run.temperature,
                       run.max_new_tokens, run.seed, 1 if run.calibration else 0,
                       1 if run.strict_greedy_tree else 0)

    def _check(self, st: int):
        if st:
            raise EspecError(st, lib().espec_last_error(self._h).decode())

    def close(self):
        if self._h:
            lib().espec_engine_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- tensor-parallel wiring (tp_size > 1)
    @staticmethod
    def link_local(engines: Sequence["Engine"]):
        """All shards of a TP group in this process (rank order)."""
        arr = (C.c_void_p * len(engines))(*[e._h.value for e in engines])
        st = lib().espec_comm_link(arr, len(engines))
        if st:
            raise EspecError(st, lib().espec_last_error(engines[0]._h).decode())

    def ipc_handle(self) -> bytes:
        buf = C.create_string_buffer(64)
        self._check(lib().espec_comm_export(self._h, buf))
        return buf.raw

    def ipc_import(self, handles: Sequence[bytes]):
        blob = b"".join(handles)
        self._check(lib().espec_comm_import(self._h, blob, len(handles)))

    def link_loopback(self):
        """Shard proxy: this rank-0 engine of a TP-N group stands in for all N
        ranks (collectives loop back; timing only, outputs are not the model's)."""
        self._check(lib().espec_comm_loopback(self._h))

    def link_process_group(self, group=None):
        """One process per GPU: all-gather the IPC handles over a
        torch.distributed group (any backend) and import them."""
        self.ipc_import(exchange_ipc_handles(self.ipc_handle(), group))

    # ---- weights
    def init_weights(self, which: int, seed: int, parity: bool = True):
        self._check(lib().espec_init_weights_seeded(self._h, which, seed, 1 if parity else 0))

    def share_truncated_draft(self):
        self._check(lib().espec_share_truncated_draft(self._h))

    def load_tensor(self, which: int, name: str, data: np.ndarray, layer: int = -1):
        a = np.ascontiguousarray(data, np.float32)
        if a.ndim == 1:
            a = a[None, :]
        self._check(lib().espec_load_tensor(self._h, which, name.encode(), layer, _f(a), a.shape[0], a.shape[1]))

    def read_tensor(self, which: int, name: str, rows: int, cols: int, layer: int = -1) -> np.ndarray:
        out = np.zeros((rows, cols), np.float32)
        self._check(lib().espec_read_tensor(self._h, which, name.encode(), layer, _f(out), rows, cols))
        return out

    def set_run(self, run: RunConfig):
        self._check(lib().espec_set_run(self._h, C.byref(self._run(run))))
        self.run = run

    # ---- generation
    def set_cost(self, cost: "CostParams"):
        """RunConfig::cost for the next generation (validated)."""
        c = cost._c()
        self._check(lib().espec_set_cost(self._h, C.byref(c)))

    def occupancy_csv(self) -> str:
        need = C.c_int(0)
        buf = C.create_string_buffer(1 << 16)
        self._check(lib().espec_occupancy_csv(self._h, buf, 1 << 16, C.byref(need)))
        return buf.value.decode()

    def generate(self, prompt: bytes):
        n = self.run.max_new_tokens
        out = np.zeros(n, np.int32)
        traces = (_Iter * max(n, 1))()
        n_out, n_it = C.c_int(0), C.c_int(0)
        self._check(lib().espec_generate(self._h, prompt, len(prompt), _i(out), C.byref(n_out), traces,
                                         C.byref(n_it)))
        return list(out[: n_out.value]), [_trace(traces[i]) for i in range(n_it.value)]

    def generate_tokens(self, tokens: Sequence[int]):
        """generate() over token ids (host buffers in, host buffers out)."""
        n = self.run.max_new_tokens
        t = np.ascontiguousarray(tokens, np.int32)
        out = np.zeros(n, np.int32)
        traces = (_Iter * max(n, 1))()
        n_out, n_it = C.c_int(0), C.c_int(0)
        self._check(lib().espec_generate_tokens(self._h, _i(t), len(t), _i(out), C.byref(n_out), traces,
                                                C.byref(n_it)))
        return list(out[: n_out.value]), [_trace(traces[i]) for i in range(n_it.value)]

    def load_model_file(self, which: int, path: str):
        """load_model (model_io.cpp:106-190) into the drafter (0) or base (1)."""
        self._check(lib().espec_load_model_file(self._h, which, os.fsencode(path)))

    def save_model_file(self, which: int, path: str):
        """save_model (model_io.cpp:76-104) of the drafter (0) or base (1)."""
        self._check(lib().espec_save_model_file(self._h, which, os.fsencode(path)))

    def probe_similarity(self, lp_sizes: Sequence[int], corpus: Sequence[Sequence[int]]) -> List["SimilarityRow"]:
        """probe_similarity (draft_engine.cpp:337-357) on the drafter."""
        lps = np.ascontiguousarray(lp_sizes, np.int32)
        toks = np.ascontiguousarray([t for seq in corpus for t in seq], np.int32)
        offs = np.ascontiguousarray(np.cumsum([0] + [len(s) for s in corpus]), np.int32)
        rows = (_SimRow * max(len(lps), 1))()
        self._check(lib().espec_probe_similarity(self._h, lps.ctypes.data_as(C.POINTER(C.c_int)), len(lps),
                                                 _i(toks), offs.ctypes.data_as(C.POINTER(C.c_int)), len(corpus),
                                                 rows))
        return [SimilarityRow(r.lp_size, r.h, r.q, r.k, r.v, r.attn_out) for r in rows[: len(lps)]]

    def stream(self) -> int:
        """cudaStream_t (as an int) all of this engine's kernels run on."""
        return lib().espec_stream(self._h)

    def time_site(self, which: int, kind: int):
        """Per-launch event timing of one kernel site (kind: 0 qkv, 1 attention,
        2 o-proj, 3 gate/up, 4 down, 5 head); which < 0 disables."""
        self._check(lib().espec_time_site(self._h, which, kind))

    def site_stats(self):
        n, ms, b = C.c_int(0), C.c_double(0), C.c_double(0)
        self._check(lib().espec_site_stats(self._h, C.byref(n), C.byref(ms), C.byref(b)))
        return n.value, ms.value, b.value

    def io_bytes(self):
        a, b = C.c_int64(0), C.c_int64(0)
        self._check(lib().espec_io_bytes(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def begin(self, tokens: Sequence[int]):
        t = np.asarray(tokens, np.int32)
        self._check(lib().espec_begin(self._h, _i(t), len(t)))

    def step(self):
        em = np.zeros(self.run.n + 2, np.int32)
        n = C.c_int(0)
        tr = _Iter()
        self._check(lib().espec_step(self._h, _i(em), C.byref(n), C.byref(tr)))
        return list(em[: n.value]), _trace(tr)

    # ---- stage-level iteration (Generation's stages, orchestrator.cpp:256-428)
    def prefill(self, tokens: Sequence[int]):
        t = np.ascontiguousarray(tokens, np.int32)
        self._check(lib().espec_prefill(self._h, _i(t), len(t)))

    def calibrate(self, want_logits: bool = False):
        """drafter_leading_pass; returns the root logits (vocab floats) on request."""
        out = np.zeros(self.base_cfg.vocab_size, np.float32) if want_logits else None
        self._check(lib().espec_calibrate(self._h, _f(out)))
        return out

    def draft(self, want_dists: bool = False) -> "DraftTree":
        """draft_stage / draft_tree -> the drafted tree."""
        t = _Tree()
        buf = None
        if want_dists:
            buf = np.zeros((MAX_NODES + 1, self.base_cfg.vocab_size), np.float32)
            t.dists = _f(buf)
            t.dist_capacity = MAX_NODES + 1
        self._check(lib().espec_draft(self._h, C.byref(t)))
        return DraftTree._from(t, buf)

    def verify(self, tree: Optional["DraftTree"] = None) -> "Outcome":
        """verify_stage + verify_tree; `tree` (this iteration's, tokens possibly
        edited) or None for the tree as drafted."""
        o = _Outcome()
        ct = tree._c() if tree is not None else None
        self._check(lib().espec_verify(self._h, C.byref(ct) if ct is not None else None, C.byref(o)))
        return Outcome(o.id, o.m, o.n, o.bonus, list(o.accepted_path[: o.m]), list(o.accepted_tokens[: o.m]))

    def resolve_draft_cache(self, outcome: Optional["Outcome"] = None):
        o = None
        if outcome is not None:
            o = _Outcome(outcome.id, outcome.m, outcome.n, outcome.bonus)
            for i, p in enumerate(outcome.path):
                o.accepted_path[i] = p
        self._check(lib().espec_resolve_draft_cache(self._h, C.byref(o) if o is not None else None))

    def commit_outcome(self):
        em = np.zeros(MAX_NODES + 2, np.int32)
        n = C.c_int(0)
        tr = _Iter()
        self._check(lib().espec_commit_outcome(self._h, _i(em), C.byref(n), C.byref(tr)))
        return list(em[: n.value]), _trace(tr)

    def iterate_stages(self, edit=None):
        """One speculative iteration through the five stage calls (what
        espec_step fuses); `edit(tree)` may rewrite the tree's tokens before
        verification. Returns (emitted, trace, tree, outcome)."""
        self.calibrate()
        tree = self.draft()
        if edit is not None:
            edit(tree)
            out = self.verify(tree)
        else:
            out = self.verify()
        self.resolve_draft_cache(out)
        em, tr = self.commit_outcome()
        return em, tr, tree, out

    def done(self) -> bool:
        return bool(lib().espec_done(self._h))

    def committed(self) -> List[int]:
        n = C.c_int(0)
        self._check(lib().espec_committed(self._h, None, 0, C.byref(n)))
        buf = np.zeros(max(n.value, 1), np.int32)
        self._check(lib().espec_committed(self._h, _i(buf), len(buf), C.byref(n)))
        return list(buf[: n.value])

    # ---- probes
    def forward(self, which: int, tokens: Sequence[int], plan: Optional[str] = None):
        cfg = self.base_cfg if which == self.BASE else self.draft_cfg
        t = np.asarray(tokens, np.int32)
        logits = np.zeros((len(t), cfg.vocab_size), np.float32)
        hidden = np.zeros((len(t), cfg.d_model), np.float32)
        self._check(lib().espec_forward(self._h, which, _i(t), len(t), (plan or "").encode(), _f(logits),
                                        _f(hidden)))
        return logits, hidden

    def forward_tree(self, which: int, prompt: Sequence[int], tokens: Sequence[int], parents: Sequence[int],
                     plan: Optional[str] = None):
        """Prefill `prompt`, then one decode-sized pass over a tree of rows
        (parents: -1 = child of the prompt tail, j = an earlier row)."""
        cfg = self.base_cfg if which == self.BASE else self.draft_cfg
        p = np.ascontiguousarray(prompt, np.int32)
        t = np.ascontiguousarray(tokens, np.int32)
        par = np.ascontiguousarray(parents, np.int32)
        logits = np.zeros((len(t), cfg.vocab_size), np.float32)
        hidden = np.zeros((len(t), cfg.d_model), np.float32)
        self._check(lib().espec_forward_tree(self._h, which, _i(p), len(p), _i(t), _i(par), len(t),
                                             (plan or "").encode(), _f(logits), _f(hidden)))
        return logits, hidden

    def prefix_distribution(self, prompt: bytes, runs: int, first: int = 0, stride: int = 1, cap: int = 1 << 16):
        """prefix_distribution (orchestrator.cpp:494-526) over runs first,
        first + stride, ... -> {prefix tuple: count}."""
        t = np.asarray(tokenize(prompt), np.int32)
        L = self.run.max_new_tokens
        pre = np.zeros((cap, L), np.int32)
        cnt = np.zeros(cap, np.int64)
        nd = C.c_int(0)
        self._check(lib().espec_prefix_distribution(self._h, _i(t), len(t), runs, first, stride, _i(pre),
                                                    cnt.ctypes.data_as(C.POINTER(C.c_int64)), cap, C.byref(nd)))
        return {tuple(int(x) for x in pre[i]): int(cnt[i]) for i in range(nd.value)}

    def cache_view(self, which: int, layer: int, row0: int = 0, n: Optional[int] = None):
        cfg = self.base_cfg if which == self.BASE else self.draft_cfg
        committed = C.c_int(0)
        self._check(lib().espec_cache_view(self._h, which, layer, 0, 0, None, None, C.byref(committed)))
        if n is None:
            n = committed.value - row0
        w = (cfg.n_kv_heads or cfg.n_heads) * cfg.d_head
        k = np.zeros((max(n, 0), w), np.float32)
        v = np.zeros_like(k)
        if n > 0:
            self._check(lib().espec_cache_view(self._h, which, layer, row0, n, _f(k), _f(v), C.byref(committed)))
        return k, v, committed.value

    def kernel_launches(self) -> int:
        return lib().espec_kernel_launches(self._h)

    def reset_kernel_launches(self):
        lib().espec_reset_kernel_launches(self._h)

    def sync(self):
        self._check(lib().espec_sync(self._h))


@dataclass
class DraftTree:
    """espec::DraftTree (draft_engine.hpp:63-84) as lists."""
    id: int
    root_children: int
    widths: List[int]
    token: List[int]
    parent: List[int]
    depth: List[int]
    prob_index: List[int]
    cache_row: List[int]
    first_child: List[int]
    n_children: List[int]
    n_dists: int
    dists: Optional[np.ndarray] = None

    @staticmethod
    def _from(t: _Tree, buf) -> "DraftTree":
        n = t.n_nodes
        g = lambda k: list(getattr(t, k)[:n])  # noqa: E731
        return DraftTree(t.id, t.root_children, list(t.widths[: t.n_levels]), g("token"), g("parent"), g("depth"),
                         g("prob_index"), g("cache_row"), g("first_child"), g("n_children"), t.n_dists,
                         None if buf is None else buf[: t.n_dists].copy())

    def _c(self) -> _Tree:
        t = _Tree()
        t.id = self.id
        t.n_nodes = len(self.token)
        t.root_children = self.root_children
        t.n_levels = len(self.widths)
        for i, w in enumerate(self.widths):
            t.widths[i] = w
        for k in ("token", "parent", "depth", "prob_index", "cache_row", "first_child", "n_children"):
            arr = getattr(t, k)
            for i, v in enumerate(getattr(self, k)):
                arr[i] = v
        return t


@dataclass
class Outcome:
    """espec::VerificationOutcome (verifier.hpp:14-21)."""
    id: int
    m: int
    n: int
    bonus: int
    path: List[int]
    tokens: List[int]


def exchange_ipc_handles(local: bytes, group=None) -> List[bytes]:
    """All-gather every rank's 64-byte receive-region handle, in rank order."""
    import torch.distributed as dist
    if len(local) != 64:
        raise ValueError("an IPC handle is 64 bytes")
    handles = [None] * dist.get_world_size(group)
    dist.all_gather_object(handles, local, group=group)
    return handles


def tp_group_local(base: ModelConfig, draft: ModelConfig, run: RunConfig, tp: int, device: int = 0,
                   parity: bool = True, truncated: int = 0, draft_layout: str = "tp") -> List[Engine]:
    """All tp shards of one tensor-parallel group in this process (testing
    the sharded path on one GPU: the collectives run over plain device
    pointers instead of NVLink-mapped ones)."""
    engines = [Engine(base, draft, run, device=device, tp_size=tp, tp_rank=r, draft_layout=draft_layout)
               for r in range(tp)]
    Engine.link_local(engines)
    for e in engines:
        e.init_weights(Engine.BASE, base.seed, parity=parity)
        if truncated and draft_layout == "tp":
            e.share_truncated_draft()
        else:
            # the layer-parallel drafter cannot alias the head-sharded base
            # blocks; init_model(keep layers, same seed) is the same drafter
            e.init_weights(Engine.DRAFT, base.seed if truncated else draft.seed, parity=parity)
    return engines


def tp_generate(engines: Sequence[Engine], prompt: bytes = None, tokens: Sequence[int] = None):
    """Run one generation on every shard concurrently (one host thread per
    shard, as one process per GPU would); returns each shard's result."""
    import threading
    out = [None] * len(engines)
    err = []

    def work(i):
        try:
            out[i] = engines[i].generate(prompt) if prompt is not None else engines[i].generate_tokens(tokens)
        except Exception as ex:  # surfaced below
            err.append(ex)

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(engines))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    return out


def prefix_distribution(engines: Sequence["Engine"], prompt: bytes, runs: int) -> dict:
    """The reference's threaded prefix_distribution (orchestrator.cpp:494-526):
    engine t (one host thread each, its own stream) runs r = t, t + n, ... and
    the partial counts are merged; identical to one engine running them all."""
    import threading
    parts = [None] * len(engines)
    err = []

    def work(t):
        try:
            parts[t] = engines[t].prefix_distribution(prompt, runs, first=t, stride=len(engines))
        except Exception as ex:  # surfaced below
            err.append(ex)

    th = [threading.Thread(target=work, args=(t,)) for t in range(len(engines))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    merged = {}
    for p in parts:
        for k, v in p.items():
            merged[k] = merged.get(k, 0) + v
    return merged


def total_variation(a: dict, b: dict, runs_a: int, runs_b: int) -> float:
    """total_variation (orchestrator.cpp:528-553) through the C ABI."""
    keys_a, keys_b = sorted(a), sorted(b)
    n = len((keys_a or keys_b)[0])
    pa = np.asarray(keys_a, np.int32).reshape(-1, n)
    pb = np.asarray(keys_b, np.int32).reshape(-1, n)
    ca = np.asarray([a[k] for k in keys_a], np.int64)
    cb = np.asarray([b[k] for k in keys_b], np.int64)
    P64 = C.POINTER(C.c_int64)
    return lib().espec_total_variation(_i(pa), ca.ctypes.data_as(P64), len(keys_a), _i(pb), cb.ctypes.data_as(P64),
                                       len(keys_b), n, runs_a, runs_b)


@dataclass
class SimilarityRow:
    """SimilarityRow (draft_engine.hpp:124-127)."""
    lp_size: int
    h: float
    q: float
    k: float
    v: float
    attn_out: float


def similarity_csv(rows: Sequence[SimilarityRow]) -> str:
    """similarity_csv (draft_engine.cpp:359-370)."""
    out = "lp_size,h,q,k,v,attnoutput\n"
    for r in rows:
        out += f"{r.lp_size},{r.h:.6f},{r.q:.6f},{r.k:.6f},{r.v:.6f},{r.attn_out:.6f}\n"
    return out


@dataclass
class RunReport:
    """RunReport's derived metrics (report.hpp:40-57): *_s in measured device
    seconds, *_sim in the cost model's units; speedup_vs_vanilla is the cost
    model's (vanilla_baseline_sim / total_sim, report.cpp:87-90)."""
    n_iterations: int
    has_alpha: bool
    alpha: float
    tokens_emitted: int
    mean_accept_len: float
    tokens_per_s: float
    draft_per_100_s: float
    verify_per_100_s: float
    calibrate_per_100_s: float
    draft_total_per_100_s: float
    total_s: float
    speedup_vs_vanilla: float
    draft_per_100_sim: float = 0.0
    verify_per_100_sim: float = 0.0
    calibrate_per_100_sim: float = 0.0
    draft_total_per_100_sim: float = 0.0
    total_sim: float = 0.0
    _c: object = field(default=None, repr=False, compare=False)


def _iters(traces: Sequence[IterationTrace]):
    arr = (_Iter * max(len(traces), 1))()
    for i, t in enumerate(traces):
        arr[i] = _Iter(*(getattr(t, n) for n, _ in _Iter._fields_))
    return arr


def aggregate(traces: Sequence[IterationTrace], vanilla_baseline_sim: float) -> RunReport:
    """aggregate(traces, vanilla_baseline_sim) (report.cpp:51-95) through the C ABI."""
    r = _Report()
    st = lib().espec_aggregate(_iters(traces), len(traces), vanilla_baseline_sim, C.byref(r))
    if st:
        raise EspecError(st, lib().espec_create_error().decode())
    vals = [getattr(r, n) for n, _ in _Report._fields_]
    vals[1] = bool(vals[1])
    return RunReport(*vals, _c=r)


def emit_report(report: RunReport, traces: Sequence[IterationTrace], algorithm: str, n: int, widths: Sequence[int],
                lp_size: int, fmt: str = "json") -> str:
    """emit_report (report.cpp:97-171): fmt "json" or "csv"."""
    w = np.ascontiguousarray(widths, np.int32)
    need = C.c_int(0)
    cap = 4096 + 512 * len(traces)
    buf = C.create_string_buffer(cap)
    st = lib().espec_report_emit(C.byref(report._c), _iters(traces), len(traces), algorithm.encode(), n,
                                 w.ctypes.data_as(C.POINTER(C.c_int)), len(w), lp_size, 0 if fmt == "json" else 1,
                                 buf, cap, C.byref(need))
    if st:
        raise EspecError(st, lib().espec_create_error().decode())
    return buf.value.decode()


@dataclass
class CostParams:
    """CostParams (proj/include/espec/cost_sim.hpp:17-32), the reference's defaults."""
    c_fixed: float = 0.02
    c_mem: float = 1.0
    c_comp: float = 0.01
    t_addi: float = 0.1
    attn_workload: float = 0.15
    mlp_workload: float = 0.05
    base_layer_workload: float = 2.0
    tp_size_base: int = 8
    tp_size_draft: int = 1
    devices: int = 8

    def _c(self) -> _CostParams:
        return _CostParams(*(getattr(self, n) for n, _ in _CostParams._fields_))


COST_VALIDATE, COST_T_EXE, COST_GROUP_ATTENTION, COST_DRAFT_GROUP, COST_SEQUENTIAL_DRAFT, COST_BASE_FORWARD, \
    COST_VANILLA_BASELINE = range(7)


def _cost(p: CostParams, what: int, a: float = 0.0, b: float = 0.0, n: int = 0, plan: str = None) -> float:
    out = C.c_double(0.0)
    c = p._c()
    st = lib().espec_cost_eval(C.byref(c), what, a, b, n, plan.encode() if plan is not None else None, C.byref(out))
    if st:
        raise EspecError(st, lib().espec_create_error().decode())
    return out.value


def cost_defaults() -> CostParams:
    c = _CostParams()
    lib().espec_cost_defaults(C.byref(c))
    return CostParams(*(getattr(c, n) for n, _ in _CostParams._fields_))


def cost_validate(p: CostParams):
    _cost(p, COST_VALIDATE)


def t_exe(p: CostParams, workload: float, s_tokens: float, tp_size: int) -> float:
    return _cost(p, COST_T_EXE, workload, s_tokens, tp_size)


def group_attention_time(p: CostParams, group_size: int, s_tokens: float) -> float:
    return _cost(p, COST_GROUP_ATTENTION, s_tokens, 0.0, group_size)


def simulate_draft_group(p: CostParams, plan: str, s_tokens: float = 1) -> float:
    return _cost(p, COST_DRAFT_GROUP, s_tokens, 0.0, 0, plan)


def sequential_draft_forward_time(p: CostParams, n_layers: int, s_tokens: float = 1) -> float:
    return _cost(p, COST_SEQUENTIAL_DRAFT, s_tokens, 0.0, n_layers)


def base_forward_time(p: CostParams, n_layers: int, s_tokens: float = 1) -> float:
    return _cost(p, COST_BASE_FORWARD, s_tokens, 0.0, n_layers)


def vanilla_baseline_sim(p: CostParams, base_layers: int, prompt_len: int, tokens: int) -> float:
    return _cost(p, COST_VANILLA_BASELINE, prompt_len, tokens, base_layers)


def total_time_model(n_tokens: float, t_draft: float, t_base: float, n: int, alpha: float) -> float:
    out = C.c_double(0.0)
    st = lib().espec_cost_total_time(n_tokens, t_draft, t_base, n, alpha, C.byref(out))
    if st:
        raise EspecError(st, lib().espec_create_error().decode())
    return out.value


def model_file_config(path: str) -> ModelConfig:
    """Validate an ESPEC1 file (load_model's checks) and return its config."""
    c = _ModelCfg()
    st = lib().espec_model_file_config(os.fsencode(path), C.byref(c))
    if st:
        raise EspecError(st, lib().espec_create_error().decode())
    return ModelConfig(vocab_size=c.vocab_size, d_model=c.d_model, n_layers=c.n_layers, n_heads=c.n_heads,
                       d_head=c.d_head, d_mlp=c.d_mlp, max_positions=c.max_positions, norm_eps=c.norm_eps,
                       seed=c.seed, n_kv_heads=c.n_kv_heads, rope_theta=c.rope_theta, tied_head=True)


def plan_groups(n_layers: int, lp_size: int) -> str:
    buf = C.create_string_buffer(4096)
    st = lib().espec_plan_groups(n_layers, lp_size, buf, 4096)
    if st:
        raise EspecError(st, lib().espec_create_error().decode())
    return buf.value.decode()


def parse_plan_override(spec: str) -> str:
    buf = C.create_string_buffer(4096)
    st = lib().espec_parse_plan(spec.encode(), buf, 4096)
    if st:
        raise EspecError(st, lib().espec_create_error().decode())
    return buf.value.decode()


def truncated_pair(base: ModelConfig, keep: int, run: RunConfig, device: int = 0, parity: bool = True) -> Engine:
    """Base model from init_model(base) + make_truncated_draft(base, keep)."""
    eng = Engine(base, replace(base, n_layers=keep), run, device)
    eng.init_weights(Engine.BASE, base.seed, parity)
    eng.share_truncated_draft()
    return eng
