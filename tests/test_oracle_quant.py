"""The C restatement of dequantize_chain (oracle/huff_oracle.c or_dequantize,
test infrastructure) against the real reference's reconstructions
(tests/golden/quant.npz, written by make_golden.py --quant)."""

from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden" / "quant.npz"


def quant_cases():
    z = np.load(GOLDEN)
    names = sorted({k.split("__")[0] for k in z.files})
    return {n: {f: z[f"{n}__{f}"] for f in ("codes", "oidx", "oval", "eb", "width", "expect")} for n in names}


def test_oracle_dequantize_matches_reference(oracle_mod):
    cases = quant_cases()
    assert len(cases) >= 6
    for name, c in cases.items():
        mid = 1 << (int(c["width"]) - 1)
        got = oracle_mod.dequantize(c["codes"], c["oidx"], c["oval"], 2.0 * float(c["eb"]), mid)
        assert np.array_equal(got.view(np.uint64), c["expect"].view(np.uint64)), name
