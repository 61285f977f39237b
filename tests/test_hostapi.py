"""Host-side analysis API through the C ABI, pinned to
fixtures the unmodified reference produced (oracle/ref_dump.cpp ->
tests/golden/ref_hostapi.json, tests/golden/ref_tiny.espec1):

* RunReport aggregation / emission — proj/src/report.cpp:51-173
* the ESPEC1 model file            — proj/src/model_io.cpp:106-190
* the similarity probe             — proj/src/draft_engine.cpp:291-372 (GPU)

CPU tests need no device: aggregation, emission and the file parser are host
code in the library; the GPU tests load/save through an engine and run the
probe's forward passes."""
import json
import os
import struct

import numpy as np
import pytest

from paper_2502_02493_b200 import espec as E

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
HOST = json.load(open(os.path.join(GOLD, "ref_hostapi.json")))
MODEL_FILE = os.path.join(GOLD, "ref_tiny.espec1")


def _traces(rep):
    # the fixture's stage times are k * 2^-10 s: exact as the engine's float ms
    # (wall) and as the simulated units (the fixture sets sim = wall)
    out = []
    for t in rep["traces"]:
        out.append(E.IterationTrace(m=t["m"], n=t["n"], drafted_nodes=t["drafted_nodes"], emitted=t["emitted"],
                                    sequential_forwards=t["sequential_forwards"], fuzzy_forwards=t["fuzzy_forwards"],
                                    base_forwards=t["base_forwards"], committed=0, draft_committed=0,
                                    base_committed=0, bonus=0, calibrate_ms=t["calibrate"] * 1000.0,
                                    draft_ms=t["draft"] * 1000.0, verify_ms=t["verify"] * 1000.0,
                                    calibrate_sim=t["calibrate"], draft_sim=t["draft"], verify_sim=t["verify"]))
    return out


@pytest.mark.parametrize("rep", HOST["reports"], ids=[r["case"] for r in HOST["reports"]])
def test_aggregate_matches_reference_bit_for_bit(rep):
    tr = _traces(rep)
    for t, g in zip(tr, rep["traces"]):  # the float ms carry the seconds exactly
        assert np.float32(t.draft_ms) / 1000.0 == g["draft"]
    r = E.aggregate(tr, rep["vanilla_baseline"])
    assert r.has_alpha == rep["has_alpha"]
    assert r.alpha == rep["alpha"]
    assert r.tokens_emitted == rep["tokens_emitted"]
    assert [r.draft_per_100_s, r.verify_per_100_s, r.calibrate_per_100_s] == rep["per100"]
    assert r.draft_total_per_100_s == rep["draft_total_per100"]
    assert r.total_s == rep["total"]
    assert r.speedup_vs_vanilla == rep["speedup"]
    assert r.tokens_per_s == rep["tokens_per_s_wall"]
    assert r.mean_accept_len == rep["tokens_emitted"] / len(tr)
    csv = E.emit_report(r, tr, rep["algorithm"], rep["n"], rep["widths"], rep["lp_size"], fmt="csv")
    assert csv == rep["csv"]


def test_report_json_has_the_reference_layout():
    rep = HOST["reports"][0]
    tr = _traces(rep)
    r = E.aggregate(tr, rep["vanilla_baseline"])
    j = json.loads(E.emit_report(r, tr, rep["algorithm"], rep["n"], rep["widths"], rep["lp_size"]))
    # emit_report's keys (report.cpp:102-134), in order
    assert list(j) == ["algorithm", "n", "widths", "lp_size", "alpha", "tokens_emitted", "tokens_per_s_wall", "sim",
                       "wall", "config", "iterations"]
    assert list(j["sim"]) == ["draft_per_100", "verify_per_100", "calibrate_per_100", "draft_total_per_100",
                              "total_sim", "total_speedup_vs_vanilla"]
    assert j["alpha"] == rep["alpha"] and j["widths"] == rep["widths"]
    assert j["sim"]["total_speedup_vs_vanilla"] == rep["speedup"]
    assert j["wall"]["verify_per_100"] == rep["per100"][1]
    assert len(j["iterations"]) == len(tr)
    assert j["iterations"][0]["draft_wall"] == rep["traces"][0]["draft"]
    # vanilla drafts nothing: alpha is null (report.cpp:106-110)
    van = next(x for x in HOST["reports"] if x["algorithm"] == "vanilla")
    rv = E.aggregate(_traces(van), van["vanilla_baseline"])
    jv = json.loads(E.emit_report(rv, _traces(van), "vanilla", van["n"], van["widths"], van["lp_size"]))
    assert jv["alpha"] is None


def test_aggregate_errors_match_reference():
    with pytest.raises(E.EspecError) as ex:
        E.aggregate([], 1.0)
    assert ex.value.kind == "config" and HOST["empty_error"] in str(ex.value)
    z = E.IterationTrace(*([0] * 11 + [0.0] * 3))
    with pytest.raises(E.EspecError) as ex:
        E.aggregate([z], 1.0)
    assert ex.value.kind == "config" and HOST["zero_error"] in str(ex.value)


def test_model_file_config_reads_reference_file():
    c = E.model_file_config(MODEL_FILE)
    g = HOST["model_file"]["config"]
    for k in ("vocab_size", "d_model", "n_layers", "n_heads", "d_head", "d_mlp", "max_positions", "seed"):
        assert getattr(c, k) == g[k], k
    assert np.float32(c.norm_eps) == np.float32(g["norm_eps"])
    assert c.n_kv_heads == c.n_heads and c.tied_head


def _corrupt(tmp_path, name, edit):
    raw = bytearray(open(MODEL_FILE, "rb").read())
    raw = edit(raw)
    p = tmp_path / name
    p.write_bytes(bytes(raw))
    with pytest.raises(E.EspecError) as ex:
        E.model_file_config(str(p))
    return ex.value


def _header(raw):
    n = struct.unpack("<Q", raw[7:15])[0]
    return n, json.loads(bytes(raw[15:15 + n]))


def _with_header(raw, hdr):
    text = json.dumps(hdr, separators=(",", ":")).encode()
    n, _ = _header(raw)
    return raw[:7] + struct.pack("<Q", len(text)) + text + raw[15 + n:]


def test_model_file_errors_match_load_model(tmp_path):
    # IoError texts of load_model (proj/src/model_io.cpp:106-190)
    e = _corrupt(tmp_path, "magic.bin", lambda r: b"ESPEC2\n" + r[7:])
    assert e.kind == "io" and "is not a model file (bad magic)" in str(e)
    e = _corrupt(tmp_path, "len.bin", lambda r: r[:7] + struct.pack("<Q", 0) + r[15:])
    assert "corrupt model header length" in str(e)
    e = _corrupt(tmp_path, "hdr.bin", lambda r: r[:40])
    assert "truncated model header" in str(e)
    e = _corrupt(tmp_path, "json.bin", lambda r: r[:15] + b"[" + r[16:])
    assert "invalid model header JSON" in str(e)
    e = _corrupt(tmp_path, "data.bin", lambda r: r[:-4])
    assert "truncated tensor data for 'layers.2.mlp_norm_gain'" in str(e)

    def nan(r):
        n, _ = _header(r)
        r[15 + n:15 + n + 4] = struct.pack("<f", float("nan"))
        return r
    e = _corrupt(tmp_path, "nan.bin", nan)
    assert "tensor 'embedding' contains non-finite values" in str(e)

    def rename(r):
        n, h = _header(r)
        h["tensors"][2]["name"] = "layers.0.wk"
        return _with_header(r, h)
    e = _corrupt(tmp_path, "name.bin", rename)
    assert "unexpected tensor 'layers.0.wk', wanted 'layers.0.wq'" in str(e)

    def drop(r):
        n, h = _header(r)
        h["tensors"].pop()
        return _with_header(r, h)
    e = _corrupt(tmp_path, "count.bin", drop)
    assert "tensor manifest does not match the config layer count" in str(e)

    def reshape(r):
        n, h = _header(r)
        h["tensors"][3]["shape"] = [8, 32]  # same bytes as 16 x 16
        return _with_header(r, h)
    e = _corrupt(tmp_path, "shape.bin", reshape)
    assert "tensor 'wk' shape disagrees with config" in str(e)

    def badcfg(r):
        n, h = _header(r)
        h["config"]["d_model"] = 24
        return _with_header(r, h)
    e = _corrupt(tmp_path, "cfg.bin", badcfg)
    assert e.kind == "config" and "d_model must equal n_heads * d_head" in str(e)
    with pytest.raises(E.EspecError) as ex:
        E.model_file_config(str(tmp_path / "absent.bin"))
    assert "cannot open model file" in str(ex.value)


# ---------------------------------------------------------------------------
# GPU: load / save through an engine, similarity probe
# ---------------------------------------------------------------------------

def _file_engine(run):
    cfg = E.model_file_config(MODEL_FILE)
    keep = HOST["model_file"]["keep"]
    from dataclasses import replace
    eng = E.Engine(cfg, replace(cfg, n_layers=keep), run)
    eng.load_model_file(E.Engine.BASE, MODEL_FILE)
    eng.share_truncated_draft()
    return eng, cfg


@pytest.mark.gpu
def test_gpu_loaded_reference_file_generates_reference_tokens():
    g = HOST["model_file"]
    rc = g["run"]
    run = E.RunConfig(algorithm="easyspec", n=rc["n"], widths=rc["widths"], lp_size=rc["lp_size"],
                      temperature=rc["temperature"], max_new_tokens=rc["max_new_tokens"], seed=rc["seed"])
    eng, cfg = _file_engine(run)
    emb = eng.read_tensor(E.Engine.BASE, "embedding", cfg.vocab_size, cfg.d_model)
    assert float(emb.astype(np.float64).sum()) == pytest.approx(g["embedding_sum"], abs=1e-9)
    toks, _ = eng.generate(g["prompt"].encode())
    assert toks == g["tokens"]
    eng.close()


@pytest.mark.gpu
def test_gpu_save_model_file_is_byte_identical_to_reference(tmp_path):
    eng, cfg = _file_engine(E.RunConfig(algorithm="vanilla", n=1, lp_size=1, max_new_tokens=4))
    out = tmp_path / "saved.espec1"
    eng.save_model_file(E.Engine.BASE, str(out))
    assert out.read_bytes() == open(MODEL_FILE, "rb").read()
    eng.close()
    # an engine whose config disagrees with the file refuses it
    from dataclasses import replace
    other = replace(cfg, d_mlp=64)
    e2 = E.Engine(other, replace(other, n_layers=2), E.RunConfig(algorithm="vanilla", n=1, lp_size=1))
    with pytest.raises(E.EspecError) as ex:
        e2.load_model_file(E.Engine.BASE, MODEL_FILE)
    assert ex.value.kind == "config"
    e2.close()


@pytest.mark.gpu
def test_gpu_similarity_probe_matches_reference():
    s = HOST["similarity"]
    c = s["config"]
    cfg = E.tiny_config(c["n_layers"], c["seed"], d_model=c["d_model"], n_heads=c["n_heads"], d_head=c["d_head"],
                        d_mlp=c["d_mlp"], max_positions=c["max_positions"])
    eng = E.Engine(cfg, cfg, E.RunConfig(algorithm="easyspec", n=2, lp_size=4))
    eng.init_weights(E.Engine.DRAFT, cfg.seed, parity=True)
    rows = eng.probe_similarity(s["lp_sizes"], s["corpus"])
    for r, g in zip(rows, s["rows"]):
        assert r.lp_size == g["lp_size"]
        for k in ("h", "q", "k", "v", "attn_out"):
            # the fp32 parity passes agree with the reference within fp32
            # rounding (not bit for bit), so the means agree to ~1e-9
            assert getattr(r, k) == pytest.approx(g[k], abs=1e-7), (r.lp_size, k)
    assert E.similarity_csv(rows) == s["csv"]
    # lp 1 has no parallelized layer: every mean is exactly 1 (SimilarityAcc::mean)
    assert rows[0].h == 1.0 and rows[0].attn_out == 1.0
    eng.close()
