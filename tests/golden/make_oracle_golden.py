"""Full cfg4 / cfg5 resultants from the PINNED CPU oracle (test infrastructure).

The unmodified Python reference needs ~2.5 h (cfg4) and ~112 h (cfg5) per
res_y on one core, so these two fixtures come from the oracle
instead: oracle.biv_resultant restates modpoly.py:348-394 (same prime stream,
same points t = 0, 1, 2, ..., same PRS and Newton interpolation in C, the same
Garner accumulator in Python ints) and is pinned to the reference's own
outputs at cfg2 and cfg3 (full resultants, sha16 e19abb8388d2a501 and
2273dd0debe66770), one prime of cfg4 and every small golden vector
(tests/test_oracle.py).

    python tests/golden/make_oracle_golden.py cfg4   # ~1 min on 8 threads
    python tests/golden/make_oracle_golden.py cfg5   # ~20-30 min on 8 threads

cfg4: every coefficient is committed (hex, gzip) with the sha16 of repr(R).
cfg5: R has 4,097 coefficients of ~34 kbit (17 MB), so only sha256(repr(R)),
the degree, the bit length and R's coefficients modulo three 61-bit primes
(a fingerprint that localises a mismatch) are committed.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from oracle import oracle  # noqa: E402

sys.set_int_max_str_digits(0)  # repr of ~34 kbit coefficients (cfg5)
from paper_1201_1548_b200.synth import make_pair  # noqa: E402

FP_PRIMES = (2305843009213693951, 2305843009213693921, 2305843009213693907)  # 2^61-1 and two below


def fingerprint(res):
    return {str(q): [c % q for c in res] for q in FP_PRIMES}


def main(config: str):
    f, g = make_pair(config, 0)
    t0 = time.time()
    res = oracle.biv_resultant(f, g, "y", threads=os.cpu_count())
    dt = time.time() - t0
    r = repr(res).encode()
    obj = {"source": "oracle.biv_resultant (restates curvekit.modpoly.biv_resultant modpoly.py:348-394; "
                     "pinned to the reference's cfg2/cfg3 outputs), %s seed 0, var y" % config,
           "config": config, "seed": 0, "degree": len(res) - 1,
           "max_bits": max(abs(c).bit_length() for c in res),
           "sha16_repr": hashlib.sha256(r).hexdigest()[:16], "sha256_repr": hashlib.sha256(r).hexdigest(),
           "oracle_seconds": round(dt, 1), "threads": os.cpu_count()}
    if config == "cfg4":
        obj["res"] = [format(c, "x") for c in res]
        path = os.path.join(HERE, "cfg4_full.json.gz")
        with gzip.open(path, "wb", compresslevel=9) as fh:
            fh.write(json.dumps(obj, separators=(",", ":")).encode())
    else:
        obj["mod_fingerprint"] = fingerprint(res)
        path = os.path.join(HERE, "%s_full.json.gz" % config)
        with gzip.open(path, "wb", compresslevel=9) as fh:
            fh.write(json.dumps(obj, separators=(",", ":")).encode())
    print(config, "deg", obj["degree"], "bits", obj["max_bits"], "sha16", obj["sha16_repr"],
          "%.1f s" % dt, "->", path)


if __name__ == "__main__":
    main(sys.argv[1])
