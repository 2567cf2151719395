"""Which device stage carries the error at the BASELINE sizes?  Runs the float64
oracle once per config, then the device forward under kernel variants selected by
the A/B environment switches (GO_TRUNK=simt: fp32 SIMT trunk attention; GO_ATTN=tf32:
tf32 task-head attention) and prints normwise / elementwise errors per stage.
Usage: python scripts/parity_variants.py [cfg3 cfg4 ...] > gpurun_out/variants.json"""
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

import headline as H  # noqa: E402
from oracle import forward as of  # noqa: E402
from oracle import graph as og  # noqa: E402

SPECS = {"cfg2": (("multi-branch-cnn", 1857, 1, 64, 0), 4),
         "cfg3": (("dilated-stack", 30, 250, 64, 0), 8),
         "cfg4": (("attention-stack", 8000, 1, 64, 0), 8)}
VARIANTS = {"default": {}, "trunk_simt": {"GO_TRUNK": "simt"}, "heads_tf32": {"GO_ATTN": "tf32"},
            "heads_simt": {"GO_ATTN": "simt"},
            "both": {"GO_TRUNK": "simt", "GO_ATTN": "simt"}}


def main(names):
    from paper_2010_12438_b200 import EmbedConfig, PolicyConfig, init_all_params, randomize_zero_init
    from paper_2010_12438_b200.embedding import embed
    from paper_2010_12438_b200.graph import node_features
    from paper_2010_12438_b200.policy import forward_policy, trunk_forward
    from synthetic.workloads import WorkloadSpec, gen_workload
    out = {}
    for name in names:
        spec, d = SPECS[name]
        g = gen_workload(WorkloadSpec(*spec), node_cap=10**6)
        sizes = {"placement": d}
        ecfg, pcfg = EmbedConfig(), PolicyConfig()
        store = randomize_zero_init(init_all_params(ecfg, pcfg, sizes, 0))
        P = H.oracle_params(store)
        ogr = H.oracle_graph(g)
        rows = H.sample_rows(g.num_nodes, 512, seed=1)
        seed = 20251019
        feats_o = og.node_features(ogr, None, [d])
        ne_o, ge_o = of.embed(ogr, feats_o, P, of.EmbedCfg(), seed=seed)
        hid_o = of.trunk_forward(ne_o, ge_o, P, of.PolicyCfg())
        lg_o, _ = H.oracle_logits(ogr, P, sizes, None, seed, rows, hid=hid_o)
        feats = node_features(g, None, [d])
        res = {}
        for vname, env in VARIANTS.items():
            old = {k: os.environ.get(k) for k in env}
            os.environ.update(env)
            try:
                emb = embed(g, feats, store, ecfg, seed=seed)
                hid_d = trunk_forward(emb.node_embed, emb.graph_embed, store, pcfg).data
                lg_d = forward_policy(g, store, ecfg, pcfg, sizes, None, seed).logits["placement"].data
            finally:
                for k, v in old.items():
                    if v is None:
                        os.environ.pop(k, None)
                    else:
                        os.environ[k] = v
            lg_iso, _ = H.oracle_logits(ogr, P, sizes, None, seed, rows, hid=hid_d)
            res[vname] = {"trunk_e2e": H.errors(hid_d, hid_o),
                          "logits_e2e": H.errors(lg_d[rows], lg_o["placement"]),
                          "logits_isolated": H.errors(lg_d[rows], lg_iso["placement"])}
            print(name, vname, {k: "%.3g/%.3g" % (v["normwise"], v["elementwise"])
                                for k, v in res[vname].items()}, file=sys.stderr, flush=True)
        out[name] = res
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg3", "cfg4"])
