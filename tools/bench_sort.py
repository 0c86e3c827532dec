"""The K2 HBM sort on its own (mk_sort_pairs_u64): device time of the hand-
written radix sort on uniformly random keys (every digit pass runs) and on
ordered keys, against the HBM roofline.  Bytes moved per digit pass: one read
and one write of each (key, value) pair, 2 x 16 B; plus one key read for the
histogram pass."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2603_24595_b200.native import Engine  # noqa: E402


def main():
    e = Engine(0)
    peak = None
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs")
    except Exception:
        pass
    for n, bits in ((1 << 24, 26), (1 << 26, 31), (1 << 27, 31), (1 << 26, 64)):
        rng = np.random.default_rng(n + bits)
        keys = rng.integers(0, 1 << min(bits, 63), n, dtype=np.uint64)
        vals = np.arange(n, dtype=np.uint64)
        runs = [e.sort_pairs(keys.copy(), vals.copy(), bits=bits) for _ in range(3)]
        ms = min(r["ms"] for r in runs)
        passes = runs[-1]["passes"]
        moved = n * (8 + passes * 32)
        print(json.dumps({"n": n, "bits": bits, "ms": ms, "passes": passes,
                          "bytes_moved": moved, "gbs": moved / ms / 1e6,
                          "frac_of_peak": (moved / ms / 1e6) / peak if peak else None,
                          "keys_per_s": n / ms * 1e3}), flush=True)
    e.close()


if __name__ == "__main__":
    main()
