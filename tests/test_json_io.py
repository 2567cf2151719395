"""JSON graph / topology formats (graph.py:208-260, costmodel.py:110-128)
against the reference's own parse of the same documents (tests/golden/make_golden.py json):
identical arrays for valid documents, GraphError / TopologyError for rejected ones."""
import json

import numpy as np
import pytest

from conftest import golden


def test_graph_json_matches_reference():
    from paper_2010_12438_b200.graph import GraphError, loads, to_dict, from_dict
    z = golden("json")
    for i in range(int(z["json_count"])):
        p = f"j{i}/"
        doc = str(z[p + "doc"])
        if not bool(z[p + "ok"]):
            with pytest.raises(GraphError):
                loads(doc, name="x")
            continue
        g = loads(doc, name="x")
        assert g.name == str(z[p + "gname"]), i
        assert np.array_equal(g.op, z[p + "op"]), i
        assert np.array_equal(g.flops, z[p + "flops"]), i
        assert np.array_equal(g.out_bytes, z[p + "out_bytes"]), i
        assert np.array_equal(g.coloc, z[p + "coloc"]), i
        assert np.array_equal(g.src, z[p + "src"]), i
        assert np.array_equal(g.dst, z[p + "dst"]), i
        assert np.array_equal(g.ebytes, z[p + "ebytes"]), i
        assert np.array_equal(g.topo_order(), z[p + "topo"]), i
        # round trip through the JSON object form
        g2 = from_dict(json.loads(json.dumps(to_dict(g))))
        assert np.array_equal(g2.src, g.src) and np.array_equal(g2.ebytes, g.ebytes)
        assert np.array_equal(g2.coloc, g.coloc) and np.array_equal(g2.op, g.op)


def test_graph_json_parse_error():
    from paper_2010_12438_b200.graph import GraphError, loads
    with pytest.raises(GraphError):
        loads("{not json")
    with pytest.raises(GraphError):
        loads("[1, 2]")


def test_topology_json_matches_reference():
    from paper_2010_12438_b200.costmodel import topology_from_dict
    z = golden("json")
    for i in range(int(z["top_count"])):
        p = f"t{i}/"
        doc = json.loads(str(z[p + "doc"]))
        if not bool(z[p + "ok"]):
            with pytest.raises(ValueError):
                topology_from_dict(doc)
            continue
        t = topology_from_dict(doc)
        d = t.num_devices
        assert np.array_equal(t.peak, z[p + "top_peak"]), i
        assert np.array_equal(t.mem_bw, z[p + "top_mem_bw"]), i
        assert np.array_equal(t.cap, z[p + "top_cap"]), i
        lb = t.link_bw.reshape(d, d)
        off = ~np.eye(d, dtype=bool)
        assert np.array_equal(lb[off], z[p + "top_link_bw"][off]), i
