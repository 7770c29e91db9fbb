"""Generate tests/golden/input_golden.json from the UNMODIFIED reference (oracle/_ref):
the outcome of load_matrix_market (matrix_market.cpp:117-165) on every case of
tests/input_cases.MTX_CASES and of SparseMatrix::validate (sparse_matrix.cpp:12-33) on
corrupt_csr(seed) for seed in 0..N_VALIDATE-1. Run in the dev container:

    make -C oracle ref && python tests/golden/make_input_golden.py
"""
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(HERE)), "oracle"))
from input_cases import MTX_CASES, corrupt_csr  # noqa: E402
from oracle_lib import Reference  # noqa: E402
from paper_2404_09276_b200 import errors as E  # noqa: E402

N_VALIDATE = 300


def outcome(fn):
    try:
        a = fn()
    except E.ParseError as e:
        return {"error": "ParseError", "line": e.line, "what": str(e)}
    except E.Error as e:
        return {"error": type(e).__name__, "what": str(e)}
    if a is None:
        return {"ok": True}
    return {"rows": a.rows, "cols": a.cols, "offsets": a.offsets.tolist(),
            "col_indices": a.col_indices.tolist(), "values_hex": [float(x).hex() for x in a.values]}


def main():
    ref = Reference()
    out = {"mtx": {}, "validate": []}
    with tempfile.TemporaryDirectory() as d:
        for name, text in MTX_CASES.items():
            path = os.path.join(d, name + ".mtx")
            with open(path, "w", newline="") as f:
                f.write(text)
            out["mtx"][name] = outcome(lambda: ref.load_matrix_market(path))
    for seed in range(N_VALIDATE):
        a = corrupt_csr(seed)
        out["validate"].append(outcome(lambda: ref.validate(a)))
    with open(os.path.join(HERE, "input_golden.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print({k: len(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
