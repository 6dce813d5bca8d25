"""Design evidence, not product: one member forward over n samples, for an ncu
capture of its kernels (e.g. ncu -k regex:member_mlp2_pair -c 1 python tools/member_ncu.py mlp1024).
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2208_14049_b200 as es  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "mlp1024"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
widths = {"mlp1024": [784, 1024, 10], "mlp256": [784, 256, 10], "mlp512x2": [784, 512, 512, 10]}[name]
rng = np.random.default_rng(0)
X = rng.random((n, 784), dtype=np.float32)
m = es.Member(es.mlp_model(0, name, widths, 13), 128)
for _ in range(2):
    m.predict(X)
print("ok", name, n)
