#!/usr/bin/env python
"""Debug aid: conv stack output (the CNN member's hidden input) of one
schedule vs the CPU oracle's conv layers, per output pixel and channel.
  ES_CONV_SCHEDULE=split python tools/check_conv.py"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2208_14049_b200 as es  # noqa: E402
from oracle import refcpu  # noqa: E402

X = refcpu.features(43, 64, 784)
model = es.cnn_model(0, "cnn", 77)
got = es.Member(model, 128).predict(X)
cpu = refcpu.CpuCnn((28, 4, 64, 32, 128, 10), 77)
want = cpu.forward(X)
err = np.abs(got - want)
print("max |dlogit|", err.max(), "rows bad", np.where(err.max(1) > 1e-2)[0][:20])
