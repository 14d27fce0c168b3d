"""Generates the committed golden fixtures from the UNMODIFIED reference.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The reference library is compiled from its own sources into oracle/_ref/ by
oracle/Makefile; every expected value below comes from it (oracle.Reference),
never from the B200 library.  Inputs are regenerated from seeds by the
tests, so only seeds, lengths and expected outputs are stored.

Fixtures
  small_pairs.json  300 seeded pairs (0..200 symbols; DNA, {A,C}, protein and
                    raw-byte alphabets): reference lcs_length and traceback
                    (lcs_fill_parallel + traceback, hex-encoded).
  c1.json           config C1 (generate_random 10k DNA, seeds 1 / 1+offset):
                    length and the full recovered subsequence.
  c2_sample.json    the first 512 pairs of the bench's C2 batch (seed
                    20130619): reference lengths.
  c3.json.gz        config C3 (100k DNA + mutation, seed 20130619): length and
                    full subsequence (needs ~50 GB of host RAM for the
                    reference's tables, memory_budget raised).
"""
import gzip
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1306_4627_b200 import workloads  # noqa: E402  (seeded generators only)

HERE = os.path.dirname(os.path.abspath(__file__))
ALPHABETS = {"dna": b"ACGT", "ac": b"AC", "protein": b"ACDEFGHIKLMNPQRSTVWY",
             "bytes": bytes(range(256))}


def small_pairs(ref):
    rng = np.random.Generator(np.random.MT19937(1306))
    cases = []
    for k in range(300):
        name = list(ALPHABETS)[k % 4]
        a = np.frombuffer(ALPHABETS[name], np.uint8)
        m, n = int(rng.integers(0, 201)), int(rng.integers(0, 201))
        x = a[rng.integers(0, len(a), m)].tobytes()
        y = a[rng.integers(0, len(a), n)].tobytes()
        length = ref.lcs_length(x, y)
        sub, _ = ref.lcs_subsequence(x, y, workers=1)
        cases.append({"x": x.hex(), "y": y.hex(), "alphabet": name, "length": length,
                      "subsequence": sub.hex()})
    return {"source": "oracle/_ref (reference lcs_length, lcs_fill_parallel+traceback)",
            "cases": cases}


def main():
    ref = oracle.Reference()
    json.dump(small_pairs(ref), open(os.path.join(HERE, "small_pairs.json"), "w"))
    print("small_pairs.json written")

    x, y = workloads.config_pair("c1")
    sub, sec = ref.lcs_subsequence(x, y)
    json.dump({"config": "C1", "m": len(x), "n": len(y), "length": len(sub),
               "subsequence": sub.decode(), "sha256": hashlib.sha256(sub).hexdigest(),
               "reference_seconds": sec}, open(os.path.join(HERE, "c1.json"), "w"))
    print("c1.json written", len(sub))

    import paper_1306_4627_b200 as wl
    pairs = 512
    xs = np.empty(pairs * 1000, np.uint8)
    ys = np.empty(pairs * 1000, np.uint8)
    xo = np.empty(pairs + 1, np.uint64)
    yo = np.empty(pairs + 1, np.uint64)
    import ctypes
    a = np.frombuffer(workloads.PROTEIN, np.uint8)
    wl._check(wl.lib.wlcs_generate_pairs(pairs, 200, 1000, a.ctypes.data, len(a), 20130619,
                                         xs.ctypes.data,
                                         xo.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                         ys.ctypes.data,
                                         yo.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
    lens, _ = ref.batch_lengths(xs, xo, ys, yo)
    json.dump({"config": "C2 (first 512 pairs of the bench batch, seed 20130619)",
               "lengths": lens.tolist(),
               "x_sha256": hashlib.sha256(xs[: int(xo[-1])].tobytes()).hexdigest(),
               "y_sha256": hashlib.sha256(ys[: int(yo[-1])].tobytes()).hexdigest()},
              open(os.path.join(HERE, "c2_sample.json"), "w"))
    print("c2_sample.json written")

    if "--c3" in sys.argv:
        x, y = workloads.config_pair("c3")
        t = time.time()
        sub, sec = ref.lcs_subsequence(x, y, budget=2 ** 64 - 1)
        with gzip.open(os.path.join(HERE, "c3.json.gz"), "wt") as f:
            json.dump({"config": "C3", "m": len(x), "n": len(y), "length": len(sub),
                       "subsequence": sub.decode(),
                       "sha256": hashlib.sha256(sub).hexdigest(),
                       "reference_seconds": sec}, f)
        print("c3.json.gz written", len(sub), time.time() - t)


if __name__ == "__main__":
    main()
