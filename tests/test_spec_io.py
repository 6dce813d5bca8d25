"""Spec / matrix documents and the optimized-matrix cache
against what the reference's own spec_io.cpp + cache.cpp print
(tests/golden/spec_io.json, made by oracle/spec_golden.cpp).  Host-only: no
GPU needed."""
import dataclasses
import json
import os
from pathlib import Path

import pytest

import paper_2208_14049_b200 as es

GOLDEN = json.loads((Path(__file__).parent / "golden" / "spec_io.json").read_text())
CASES = sorted(GOLDEN["clusters"])


@pytest.mark.parametrize("name", CASES)
def test_spec_dump_is_byte_identical_to_the_reference(name):
    g = GOLDEN["clusters"][name]
    c = es.cluster_from_json(g["spec_compact"])
    assert es.cluster_to_json(c) == g["spec_compact"]
    assert es.cluster_to_json(c) == g["roundtrip_compact"]
    # Indented files: same document (the reference's nlohmann build lays
    # integer arrays out on one line; whitespace is not part of the format).
    assert json.loads(es.cluster_to_json(c, indent=2)) == json.loads(g["spec_indent2"])


@pytest.mark.parametrize("name", CASES)
def test_cache_keys_match_the_reference(name):
    g = GOLDEN["clusters"][name]
    c = es.cluster_from_json(g["spec_compact"])
    for k in g["cache_keys"]:
        key = es.OptimizerKey(es.GreedyConfig(k["max_iter"], k["max_neighs"], k["rng_seed"]),
                              k["default_batch"], k["bench_mode"], k["calib_samples"], k["repeats"])
        assert es.cache_key(c, key) == k["key"]


@pytest.mark.parametrize("name", CASES)
def test_matrix_document_matches_the_reference(name):
    g = GOLDEN["clusters"][name]
    c = es.cluster_from_json(g["spec_compact"])
    A = es.worst_fit_decreasing(c, c.min_batch())
    assert A.cells.flatten().tolist() == g["matrix"]
    ours = es.matrix_to_json(A, c, indent=2)
    assert json.loads(ours) == json.loads(g["matrix_indent2"])
    assert es.matrix_from_json(g["matrix_indent2"], c) == A


def test_digests_match_the_reference():
    for d in GOLDEN["digests"]:
        assert es.digest_hex(d["text"]) == d["hex"]


@pytest.mark.parametrize("case", GOLDEN["spec_errors"], ids=lambda c: c["case"])
def test_malformed_specs_fail_like_the_reference(case):
    with pytest.raises(es.SpecError) as e:
        es.cluster_from_json(case["doc"])
    want = case["error"]
    # nlohmann's type_error text ("[json.exception.type_error.302] ...") is the
    # library's; the reference's own prefix and the type complaint must match.
    if "[json.exception" in want:
        head, _, tail = want.partition("[json.exception.type_error.302] ")
        assert str(e.value).startswith(head) and str(e.value).endswith(tail)
    else:
        assert str(e.value) == want


def test_ensemble_overlay_merges_like_cluster_from_documents():
    g = json.loads(GOLDEN["clusters"]["dozen"]["spec_compact"])
    base = json.dumps({"devices": g["devices"], "batch_menu": [8, 16]})
    overlay = json.dumps({"models": g["models"], "batch_menu": g["batch_menu"]})
    c = es.cluster_from_json(base, overlay)
    assert es.cluster_to_json(c) == GOLDEN["clusters"]["dozen"]["spec_compact"]


def test_member_architecture_extension_round_trips_and_stays_out_of_keys(tmp_path):
    c = es.ClusterSpec([es.DeviceSpec(0, es.GPU, 183359.0, 1e15, 0.0)],
                       [es.mlp_model(0, "mlp512x2", [784, 512, 512, 10], 7),
                        es.cnn_model(1, "cnn-s", 8)], [8, 16, 32, 64, 128], 128)
    p = tmp_path / "ensemble.json"
    es.save_json_file(str(p), es.cluster_to_json(c, with_arch=True))
    back = es.load_spec(str(p))
    assert back.models[0].arch == c.models[0].arch and back.models[1].arch == c.models[1].arch
    assert es.cluster_to_json(back) == es.cluster_to_json(c)
    plain = es.cluster_from_json(es.cluster_to_json(c))  # what the reference writes
    key = es.OptimizerKey(default_batch=8)
    assert es.cache_key(plain, key) == es.cache_key(c, key)


def test_matrix_cache_hit_miss_and_corruption(tmp_path, capfd):
    g = GOLDEN["clusters"]["dozen"]
    c = es.cluster_from_json(g["spec_compact"])
    A = es.worst_fit_decreasing(c, 8)
    key = g["cache_keys"][0]["key"]
    cache = es.MatrixCache(str(tmp_path))
    assert cache.lookup(key, c) is None
    cache.store(es.MatrixCacheEntry(key, A, 1234.5, 1700000000), c)
    hit = cache.lookup(key, c)
    assert hit is not None and hit.matrix == A and hit.score == 1234.5
    assert hit.created_at == 1700000000
    doc = json.loads((tmp_path / f"{key}.json").read_text())
    assert doc["key"] == key and doc["score"] == 1234.5
    # A file under the wrong name (stale key), a corrupt file and an invalid
    # matrix are misses with a warning, never errors (cache.cpp:44-68).
    other = g["cache_keys"][1]["key"]
    (tmp_path / f"{other}.json").write_text((tmp_path / f"{key}.json").read_text())
    assert cache.lookup(other, c) is None
    (tmp_path / f"{key}.json").write_text("{not json")
    assert cache.lookup(key, c) is None
    bad = json.loads(json.dumps(doc))
    bad["matrix"]["entries"][0][0] = 7  # not in the menu
    (tmp_path / f"{key}.json").write_text(json.dumps(bad))
    assert cache.lookup(key, c) is None
    err = capfd.readouterr().err
    assert "written for another key" in err and "unreadable" in err
    assert "not valid for this cluster" in err
    assert not any(".partial." in n for n in os.listdir(tmp_path))


def test_device_identity_is_an_opt_in_part_of_the_key():
    """the reference's key (cache.cpp:22-33) has no hardware
    identity, so a matrix tuned on other GPUs would hit.  Opt-in: an empty
    identity keeps the reference's digest, any identity changes it."""
    g = GOLDEN["clusters"]["dozen"]
    c = es.cluster_from_json(g["spec_compact"])
    k = g["cache_keys"][0]
    key = es.OptimizerKey(es.GreedyConfig(k["max_iter"], k["max_neighs"], k["rng_seed"]),
                          k["default_batch"], k["bench_mode"], k["calib_samples"], k["repeats"])
    assert es.cache_key(c, key) == k["key"]
    b200 = es.cache_key(c, dataclasses.replace(key, device="NVIDIA B200/sm_100/148 SMs/178 GiB x8"))
    h100 = es.cache_key(c, dataclasses.replace(key, device="NVIDIA H100/sm_90/132 SMs/80 GiB x8"))
    assert len({k["key"], b200, h100}) == 3


def test_matrix_shape_errors_are_spec_errors():
    c = es.cluster_from_json(GOLDEN["clusters"]["tiny"]["spec_compact"])
    with pytest.raises(es.SpecError, match="rows, cluster has"):
        es.matrix_from_json('{"entries": [[8, 8], [8, 8]]}', c)
    with pytest.raises(es.SpecError, match="is 'x', cluster has 'a'"):
        es.matrix_from_json('{"models": ["x", "b"], "entries": [[8, 8]]}', c)
    with pytest.raises(es.SpecError, match="entries, expected 2"):
        es.matrix_from_json('{"entries": [[8]]}', c)
