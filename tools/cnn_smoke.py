"""Tiny CNN-s member forward vs the CPU oracle (kernel bring-up; not product)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2208_14049_b200 as es
from oracle import refcpu  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
X = refcpu.features(43, n, 784)
model = es.cnn_model(0, "cnn", 77, S=28, P=4, c1=64, c2=32, hidden=128, classes=10)
got = es.Member(model, 128).predict(X)
want = refcpu.CpuCnn((28, 4, 64, 32, 128, 10), 77).forward(X)
err = np.abs(got - want).max()
print("max|dlogit|", err, "argmax agree", (got.argmax(1) == want.argmax(1)).mean())
