"""Golden fixtures for the device sampled-block pipeline:
run the UNMODIFIED reference sampler (gsbench.sample_minibatch, sampler.py:
118-296) on small generated graphs and dump gsbench's own debug JSON
(subgraph_to_json, sampler.py:338-357).  Run in the build container:

    python tests/golden/make_golden_sampling.py    -> tests/golden/sampling.json
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import gsbench as g  # noqa: E402
from gsbench.sampler import subgraph_to_json  # noqa: E402

CASES = [
    # (graph spec args, graph seed, batch, fanouts, seeds-rng, sample seed)
    (("power-law", 2708, 10556, 2.1), 42, 8, (5, 5), 0, 3),
    (("power-law", 2708, 10556, 2.1), 42, 64, (10, 10, 10), 1, 11),
    (("power-law", 10_000, 200_000, 2.1), 7, 32, (15, 10), 2, 5),
    (("power-law", 10_000, 200_000, 2.1), 7, 1, (0, 3), 3, 9),
    (("uniform-random", 500, 5000, None), 43, 16, (4, 4, 4), 4, 17),
]


def main():
    out = []
    for (kind, n, m, ex), gseed, batch, fanouts, srng, sseed in CASES:
        spec = g.GraphGenSpec(kind, n, m, exponent=ex) if ex else g.GraphGenSpec(kind, n, m)
        graph = g.generate(spec, gseed)
        seeds = np.random.default_rng(srng).choice(n, size=batch, replace=False)
        cfg = g.SampleConfig(batch_size=batch, fanouts=fanouts)
        sg, meta = g.sample_minibatch(graph, cfg, seeds, sseed)
        out.append({"graph": [kind, n, m, ex, gseed], "seeds": seeds.tolist(),
                    "fanouts": list(fanouts), "sample_seed": sseed,
                    "result": subgraph_to_json(sg, meta)})
    with open(os.path.join(HERE, "sampling.json"), "w") as fh:
        json.dump(out, fh)
    print(f"wrote {len(out)} cases")


if __name__ == "__main__":
    main()
