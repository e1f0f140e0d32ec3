"""Generate golden vectors from the REFERENCE implementation (run in the dev
container, where /root/reference exists).  The output npz files are committed;
nothing at test time reads /root/reference.

    python tests/golden/make_golden.py

basis_ref.npz:  for N in 1..16, the reference's gll_rule(N) nodes/weights and
                SpectralBasis(N).diff, plus interp_matrix(N -> N+3) and back
                (the matrices test_basis.py:105-116 round-trips through).
"""

import importlib.util
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src/nekmini/basis.py"
HERE = os.path.dirname(os.path.abspath(__file__))


def load_reference_basis():
    # loaded by file path: src/nekmini is a namespace package (no __init__),
    # so a regular package elsewhere would shadow it.
    spec = importlib.util.spec_from_file_location("ref_nekmini_basis", REF)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def main():
    if not os.path.exists(REF):
        sys.exit(f"reference not found at {REF}")
    ref = load_reference_basis()
    out = {}
    for N in range(1, 17):
        x, w = ref.gll_rule(N)
        b = ref.SpectralBasis(N)
        out[f"nodes_{N}"] = np.asarray(x)
        out[f"weights_{N}"] = np.asarray(w)
        out[f"diff_{N}"] = np.asarray(b.diff)
        fine = ref.SpectralBasis(N + 3)
        out[f"up_{N}"] = ref.interp_matrix(b, fine).values
        out[f"down_{N}"] = ref.interp_matrix(fine, b).values
    path = os.path.join(HERE, "basis_ref.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, len(out), "arrays")


if __name__ == "__main__":
    main()
