"""Golden record for BASELINE config 5 (n = 50,000, hub APSP) from the C oracle.

The reference itself cannot run this size in a test budget (its hub-mode layer 3
materialises a 50,000 x 50,000 oracle block in Python), so the record comes from
oracle/ -- the restatement pinned bit-for-bit against the reference on configs
1-4 and the 12 small cases (tests/test_oracle_golden.py).  Needs ~35 GB of RAM.

    python tests/golden/make_config5.py      # writes tests/golden/config5.json
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(REPO))

from oracle import oracle  # noqa: E402
from paper_2408_09399_b200 import synth  # noqa: E402

ROWS = 64   # rows of S / order hashed as spot checks (the full arrays are 20 + 10 GB)


def main() -> None:
    oracle.build()
    t0 = time.perf_counter()
    x, labels = synth.generate(5)
    n = x.shape[0]
    k = synth.num_clusters(5)
    S = oracle.pearson_similarity(x)
    t_pearson = time.perf_counter() - t0
    out = oracle.run_stages(S, k, apsp_mode="hub", keep=True)
    rec = {
        "n": int(n),
        "k": int(k),
        "seed": synth.DEFAULT_SEED,
        "S_rows": oracle.sha(S[:ROWS]),
        "S_diag_band": oracle.sha(np.array([S[i, (i * 7919) % n] for i in range(n)])),
        "order_rows": oracle.sha(np.asarray(out["order"][:ROWS], dtype=np.int32)),
        "tmfg_edges": oracle.sha(np.asarray(out["graph"]["edges"], dtype=np.int32)),
        "hub_digest": out["digest"],
        "hub_labels": oracle.sha(np.asarray(out["labels"], dtype=np.int64)),
        "hub_num_converging": out["num_converging"],
        "oracle_seconds": {"pearson": t_pearson, **out["seconds"]},
        "threads": oracle.num_threads(),
    }
    (Path(__file__).parent / "config5.json").write_text(json.dumps(rec, indent=1) + "\n")
    print(json.dumps(rec, indent=1))


if __name__ == "__main__":
    main()
