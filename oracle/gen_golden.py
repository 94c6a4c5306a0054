"""ORACLE — test infrastructure only.  Generates tests/golden/topology_golden.json by running the
REAL reference module (``/root/reference/pkg/src/pipepath/topology.py`` and ``errors.py``, the
only code the reference ships) in this container.  The GPU box has no /root/reference; the
committed JSON is what the tests compare the host restatement against.

    python oracle/gen_golden.py        # rewrites tests/golden/topology_golden.json

Vectors: symmetrize / comm_time / comm_matrix KATs, activation_bytes and
stage_param_bytes for every preset (topology.py:190-200), layers_per_stage, JSON round trips,
error messages of every validation branch, and sample_topology draws pinning the PCG64 order
(topology.py:263-286) for several profiles and seeds.
"""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "topology_golden.json")


def _err(fn):
    try:
        fn()
    except Exception as e:  # noqa: BLE001 - record the reference's exact behaviour
        return {"type": type(e).__name__, "msg": str(e)}
    return None


def main():
    sys.path.insert(0, REF)
    from pipepath import topology as T  # the reference itself

    g = {"source": "pipepath.topology (reference pkg/src/pipepath/topology.py)", "cases": {}}
    c = g["cases"]
    lat, bw = T.symmetrize(np.array([[0, 4.0], [6.0, 0]]), np.array([[0, 100.0], [300.0, 0]]))
    c["symmetrize_2x2"] = {"lat": lat.tolist(), "bw": bw.tolist()}
    topo = T.Topology(n=2, latency_ms=np.array([[0, 5.0], [5.0, 0]]), bandwidth_bytes_per_ms=np.array([[0, 1e5], [1e5, 0]]),
                      compute_fwd_ms=np.array([1.0, 1.0]))
    c["comm_time_105"] = T.comm_time(topo, 0, 1, 1e7)
    c["comm_matrix_105"] = T.comm_matrix(topo, 1e7).tolist()
    c["presets"] = {k: [p.hidden_dim, p.n_layers, p.context, p.bytes_per_element] for k, p in T.PRESETS.items()}
    c["activation_bytes"] = {k: [T.activation_bytes(p, b) for b in (1, 2, 4)] for k, p in T.PRESETS.items()}
    c["stage_param_bytes"] = {k: {str(s): T.stage_param_bytes(p, s) for s in (1, 2, 4, 8) if p.n_layers % s == 0}
                              for k, p in T.PRESETS.items()}
    c["layers_per_stage"] = {k: {str(s): p.layers_per_stage(s) for s in (1, 2, 3, 4, 6, 8) if p.n_layers % s == 0}
                             for k, p in T.PRESETS.items()}
    errs = {
        "non_square": lambda: T.symmetrize(np.zeros((2, 3)), np.zeros((2, 3))),
        "zero_offdiag": lambda: T.symmetrize(np.array([[0, 0.0], [1, 0]]), np.ones((2, 2))),
        "nan_offdiag": lambda: T.symmetrize(np.array([[0, np.nan], [1, 0]]), np.ones((2, 2))),
        "inf_offdiag": lambda: T.symmetrize(np.array([[0, np.inf], [1, 0]]), np.ones((2, 2))),
        "shape_mismatch": lambda: T.symmetrize(np.ones((2, 2)), np.ones((3, 3))),
        "comm_self": lambda: T.comm_time(topo, 1, 1, 10),
        "comm_range": lambda: T.comm_time(topo, 0, 5, 10),
        "comm_zero_bytes": lambda: T.comm_time(topo, 0, 1, 0),
        "matrix_zero_bytes": lambda: T.comm_matrix(topo, 0),
        "mem_cap_zero": lambda: T.Topology(n=2, latency_ms=np.ones((2, 2)), bandwidth_bytes_per_ms=np.ones((2, 2)),
                                           compute_fwd_ms=np.ones(2), mem_capacity=0),
        "compute_zero": lambda: T.Topology(n=2, latency_ms=np.ones((2, 2)), bandwidth_bytes_per_ms=np.ones((2, 2)),
                                           compute_fwd_ms=np.array([1.0, 0.0])),
        "n_mismatch": lambda: T.Topology(n=3, latency_ms=np.ones((2, 2)), bandwidth_bytes_per_ms=np.ones((2, 2)),
                                         compute_fwd_ms=np.ones(3)),
        "bwd_ratio": lambda: T.Topology(n=2, latency_ms=np.ones((2, 2)), bandwidth_bytes_per_ms=np.ones((2, 2)),
                                        compute_fwd_ms=np.ones(2), bwd_ratio=0.0),
        "restrict_dup": lambda: topo.restrict([0, 0]),
        "restrict_range": lambda: topo.restrict([0, 7]),
        "restrict_empty": lambda: topo.restrict([]),
        "preset_unknown": lambda: T.get_preset("llama-3b"),
        "layers_indivisible": lambda: T.get_preset("llama-500m").layers_per_stage(5),
        "activation_zero": lambda: T.activation_bytes(T.get_preset("llama-500m"), 0),
        "profile_empty": lambda: T.TopologyProfile(regions=0, nodes_per_region=2),
        "profile_range": lambda: T.TopologyProfile(regions=1, nodes_per_region=2, compute_ms=(5.0, 1.0)),
        "from_dict_no_bw": lambda: T.Topology.from_dict({"n": 2, "latency_ms": [[0, 1], [1, 0]],
                                                         "compute_fwd_ms": [1, 1]}),
    }
    c["errors"] = {k: _err(f) for k, f in errs.items()}
    d = {"n": 2, "latency_ms": [[0, 2.0], [4.0, 0]], "bandwidth_mb_per_s": [[0, 100.0], [300.0, 0]],
         "compute_fwd_ms": [3.0, 4.0], "bwd_ratio": 1.5, "mem_capacity": 3}
    c["from_dict_mbps"] = T.Topology.from_dict(d).to_dict()
    samples = []
    for regions, per, seed in [(2, 2, 0), (4, 5, 3), (3, 6, 1), (1, 4, 7), (2, 9, 11)]:
        prof = T.TopologyProfile(regions=regions, nodes_per_region=per, seed=seed)
        samples.append({"profile": prof.to_dict(), "topology": T.sample_topology(prof).to_dict()})
    c["sample_topology"] = samples
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as fh:
        json.dump(g, fh, indent=1, sort_keys=True)
        fh.write("\n")
    print("wrote", OUT)


if __name__ == "__main__":
    main()
