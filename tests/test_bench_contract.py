"""bench.py's own arithmetic on CPU: the per-launch algorithmic work that the
roofline divides by, the dominant-kernel choice and bound
classification, and the config table the --config flag exposes."""
import sys
from pathlib import Path

import pytest

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2208_14049_b200 as es  # noqa: E402

PEAKS = {"hbm_gbs": 6549.0, "bf16_tflops": 1634.0, "bf16_tflops_sustained": 1388.0,
         "source": "measured"}


def test_launch_work_sums_to_the_member_flops():
    models = bench.roster_models(es, bench.ROSTER)
    names = {
        "mlp256": ["member_mlp2_tmem_sm100"],
        "mlp512x2": ["dense_pair_sm100", "member_mlp2_pair_sm100"],
        "mlp1024": ["member_mlp2_pair_sm100"],
        "cnn-s": ["conv_stack_sm100[split]", "member_mlp2_tmem_sm100"],
    }
    for m in models:
        work = bench.launch_work(m.arch, names[m.name])
        assert sum(f for f, _ in work) == pytest.approx(m.arch.flops_per_sample())
        # first launch reads the bf16 input row, the last writes fp32 logits
        assert work[0][1] >= 784 * 2 and work[-1][1] >= 10 * 4
    cnn = [m for m in models if m.name == "cnn-s"][0]
    conv, head = bench.launch_work(cnn.arch, names["cnn-s"])
    assert conv[1] == 784 * 2 + 49 * 32 * 2 and head[1] == 49 * 32 * 2 + 10 * 4


def test_roofline_takes_the_slowest_launch_and_classifies_the_bound():
    cluster = bench.make_cluster(es, bench.CONFIGS["cfg2"])
    A = es.AllocationMatrix.from_array([[128, 128, 128, 128]])
    kern = [[("member_mlp2_tmem_sm100", 1.8)],
            [("dense_pair_sm100", 3.8), ("member_mlp2_pair_sm100", 2.7)],
            [("member_mlp2_pair_sm100", 7.0)],
            [("conv_stack_sm100[split]", 12.0), ("member_mlp2_tmem_sm100", 2.3)]]
    nb = 1 << 22
    r = bench.roofline_for(es, cluster, A, kern, nb, PEAKS)
    assert r["kernel"] == "conv_stack_sm100[split][cnn-s]" and r["bound"] == "tensor"
    flop = 2 * 49 * (16 * 64 + 9 * 64 * 32)
    assert r["algorithmic_per_launch"]["flop_per_sample"] == flop
    assert r["achieved"] == pytest.approx(flop * nb / 12e-3 / 1e12, rel=1e-3)
    assert r["frac"] == pytest.approx(r["achieved"] / PEAKS["bf16_tflops_sustained"], rel=1e-3)
    head = [k for k in r["per_kernel"] if k["member"] == "cnn-s" and k["kernel"].startswith("member")]
    assert head[0]["bound"] == "hbm"  # 404 kFLOP over 3176 B: below the ridge


def test_every_baseline_config_builds_a_valid_cluster_and_start_matrix():
    for name, cfg in bench.CONFIGS.items():
        c = bench.make_cluster(es, cfg)
        assert c.device_count() == cfg["devices"] and c.model_count() == len(cfg["roster"])
        assert not [w for w in c.validate() if "error" in w.lower()]
        A1 = es.worst_fit_decreasing(c, c.min_batch())
        assert es.validate_matrix(A1, c).ok
    dozen = bench.make_cluster(es, bench.CONFIGS["cfg3"])
    A = es.worst_fit_decreasing(dozen, 8)
    assert all(A.row_worker_count(d) == 3 for d in range(4))  # acceptance.cpp:217-232


def test_plain_cluster_footprints_equal_the_products():
    """The reference arm's product-free cluster derives the same footprints
    (spec.cpp derive_footprint), so WFD and memory checks agree."""
    for name, cfg in bench.CONFIGS.items():
        a = bench.make_cluster(es, cfg)
        b = bench.plain_cluster(cfg)
        for ma, mb in zip(a.models, b.models):
            assert (ma.weight_mib, ma.act_mib_per_sample, ma.cost_per_sample) == \
                pytest.approx((mb.weight_mib, mb.act_mib_per_sample, mb.cost_per_sample), rel=1e-12)
        from oracle import refcpu
        assert refcpu.ref_wfd(b, 8).tolist() == es.worst_fit_decreasing(a, 8).cells.tolist()


def test_reference_arm_runs_the_same_matrix_without_loading_the_product():
    """bench.py --impl reference: the reference InferenceSystem on host cores
    with the b200 arm's matrix; the product library never loads."""
    import json
    import subprocess
    repo = Path(__file__).resolve().parents[1]
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '2', "
            "'--warmup', '1', '--ref-budget-s', '2', '--no-ref-faithful']; "
            "runpy.run_path('bench.py', run_name='__main__'); "
            "maps = open('/proc/self/maps').read(); "
            "assert 'libenserve_b200' not in maps, 'product library loaded'; "
            "assert 'paper_2208_14049_b200' not in sys.modules")
    out = subprocess.run([sys.executable, "-c", code], cwd=repo, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["config"]["same_config"]
    assert line["config"]["matrix"] == bench.CONFIGS["cfg2"]["ref_matrix"]
    assert line["value"] > 0 and line["ms_per_step"] > 0 and line["steps"] == 2
