"""Generate tests/golden/cli/ from the REFERENCE itself.

The reference CLI binary (cli.cpp) needs the CLI11 header, which is not in
/root/reference, so it is not built; the files its commands write are
produced here by the reference LIBRARY functions those commands call, in the
same order (oracle/_ref/libmoesim_ref.so + oracle/ref_capi.cpp):

  gen-trace  (cli.cpp:92-110)  : write_trace(gen_trace(spec, seed))
  profile    (cli.cpp:112-171) : write_matrix(counts), write_matrix(normalized),
                                 ComponentTracker points over 256-token batches
  reschedule (cli.cpp:173-188) : write_placement(reschedule_placement(...))

    python tests/golden/make_cli_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "cli")

# (name, dist, experts, topk, tokens, alpha, blocks, p_in, tag, seed)
TRACES = [
    ("uniform_e8k2", 0, 8, 2, 300, 1.0, 1, 0.9, "", 1),
    ("zipf_e16k4", 1, 16, 4, 300, 1.2, 1, 0.9, "mix", 7),
    ("blocks_e64k8", 2, 64, 8, 600, 1.0, 8, 0.9, "olmoe", 3),
    ("blocks_e60k4_pin0", 2, 60, 4, 300, 1.0, 6, 0.0, "", 2 ** 64 - 1),
    ("empty_e4k1", 0, 4, 1, 0, 1.0, 1, 0.9, "", 0),
]
RESCHEDULE_DEVICES = {"uniform_e8k2": 4, "zipf_e16k4": 4, "blocks_e64k8": 8, "blocks_e60k4_pin0": 6}


def parse_ids(text, k):
    rows = [ln.split()[:k] for ln in text.splitlines()[2:] if ln]
    return np.array(rows, dtype=np.int32).reshape(len(rows), k)


def main():
    os.makedirs(OUT, exist_ok=True)
    R = O.Ref()
    meta = {}
    for name, dist, ne, k, n, alpha, blocks, p_in, tag, seed in TRACES:
        ok, text = O.ref_gen_trace(dist, ne, k, n, alpha, blocks, p_in, tag, seed)
        assert ok, text
        with open(os.path.join(OUT, name + ".trace"), "w") as f:
            f.write(text)
        ids = parse_ids(text, k)
        counts = R.accumulate_collab(ids, ne)
        norm = R.normalize_graph(counts)
        with open(os.path.join(OUT, name + ".collab.mat"), "w") as f:
            f.write(O.ref_write_matrix(counts.astype(np.float64)))
        with open(os.path.join(OUT, name + ".norm.mat"), "w") as f:
            f.write(O.ref_write_matrix(norm))
        upper = counts[np.triu_indices(ne, 1)]
        pts = O.ref_component_points(ids, ne, 256)
        meta[name] = {"spec": [dist, ne, k, n, alpha, blocks, p_in, tag, seed], "edges": int((upper > 0).sum()),
                      "coactivations": int(upper.sum()), "growth": pts}
        if name in RESCHEDULE_DEVICES:
            nd = RESCHEDULE_DEVICES[name]
            plist = R.reschedule_placement(norm, nd)
            with open(os.path.join(OUT, f"{name}.d{nd}.place"), "w") as f:
                f.write(O.ref_write_placement(plist))
    with open(os.path.join(OUT, "meta.json"), "w") as f:
        json.dump(meta, f, indent=1)


if __name__ == "__main__":
    main()
