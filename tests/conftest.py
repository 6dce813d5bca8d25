"""Shared fixtures.  Ports the reference's test fixtures
(/root/reference/proj/tests/test_fixtures.hpp:11-94) so the parity tests read
like the reference's own doctest suites."""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")


def _ensure_built():
    from paper_2208_14049_b200 import build as pkg_build
    pkg_build.build()
    from oracle import refcpu
    refcpu.build()


_ensure_built()

import paper_2208_14049_b200 as es  # noqa: E402
from oracle import restate  # noqa: E402


def has_gpu() -> bool:
    try:
        return es.device_count() > 0
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device visible")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


# --------------------------------------------------------------- fixture ports
def gpu(id, memory_mib, rate=1000.0, overhead_s=0.01):
    """test_fixtures.hpp:11-14."""
    return es.DeviceSpec(id, es.GPU, memory_mib, rate, overhead_s)


def cpu(id, memory_mib, rate=100.0, overhead_s=0.02):
    """test_fixtures.hpp:16-19."""
    return es.DeviceSpec(id, es.CPU, memory_mib, rate, overhead_s)


def model(id, name, weight_mib, act_mib=0.0, cost=1.0, output_width=4):
    """test_fixtures.hpp:21-25."""
    return es.ModelSpec(id, name, weight_mib, act_mib, cost, output_width)


def imagenet4_cluster():
    """test_fixtures.hpp:29-40."""
    return es.ClusterSpec(
        devices=[cpu(0, 64000.0), gpu(1, 16000.0), gpu(2, 16000.0), gpu(3, 16000.0),
                 gpu(4, 16000.0)],
        models=[model(0, "resnet50", 98.0, 8.0, 4.1), model(1, "resnet101", 170.0, 12.0, 7.8),
                model(2, "densenet121", 31.0, 9.0, 2.9), model(3, "vgg19", 549.0, 6.0, 19.6)],
        batch_menu=[8, 16, 32, 64, 128], segment_size=128)


def imagenet4_matrix():
    """test_fixtures.hpp:44-52."""
    A = es.AllocationMatrix(5, 4)
    A.set(1, 0, 8)
    A.set(1, 1, 8)
    A.set(2, 1, 128)
    A.set(3, 2, 8)
    A.set(4, 3, 8)
    return A


def tiny_cluster(menu=(8, 16), devices=1, models=1):
    """test_fixtures.hpp:54-63."""
    return es.ClusterSpec(devices=[gpu(d, 100000.0) for d in range(devices)],
                          models=[model(m, f"m{m}", 100.0, 1.0, 1.0) for m in range(models)],
                          batch_menu=list(menu), segment_size=128)


def random_cluster(rng: restate.MT19937_64, max_devices=5, max_models=6):
    """test_fixtures.hpp:67-94 — same draws from the same mt19937_64 stream, so a
    seed yields the reference's instance."""
    ui = restate.uniform_index
    devices = 1 + ui(rng, max_devices)
    models = 1 + ui(rng, max_models)
    with_cpu = devices > 1 and ui(rng, 3) == 0
    devs = []
    for d in range(devices):
        memory = 8000.0 + 2000.0 * ui(rng, 9)
        rate = 500.0 + 250.0 * ui(rng, 7)
        overhead = 0.002 + 0.002 * ui(rng, 5)
        if with_cpu and d == 0:
            devs.append(cpu(0, memory * 4, rate / 10, overhead * 2))
        else:
            devs.append(gpu(d, memory, rate, overhead))
    mods = []
    for m in range(models):
        weight = 100.0 + 150.0 * ui(rng, 20)
        act = 1.0 + ui(rng, 12)
        cost = 1.0 + 0.7 * ui(rng, 10)
        mods.append(model(m, f"m{m}", weight, act, cost))
    menu_size = 2 + ui(rng, 4)
    return es.ClusterSpec(devs, mods, [8, 16, 32, 64, 128][:menu_size], 128)


def fast_cluster(devices, models, output_width=4):
    """test_runtime.cpp:75-85: synthetic members, negligible sleeps."""
    return es.ClusterSpec(devices=[gpu(d, 100000.0, 1e9, 0.0) for d in range(devices)],
                          models=[model(m, f"m{m}", 10.0, 0.0, 1.0, output_width)
                                  for m in range(models)],
                          batch_menu=[8, 16, 32, 64, 128], segment_size=128)


@pytest.fixture
def es_mod():
    return es
