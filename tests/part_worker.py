"""Worker for tests/test_gpu_partition.py::test_two_processes_ipc_gloo: rank r
of a 2-process gloo group hosts part r of grid64 on cuda:0 and runs the
static solve plus the golden batch chain; writes the flows to argv[2]."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)


def main():
    import torch.distributed as dist

    import paper_2511_01235_b200 as mf
    from golden_data import load
    from paper_2511_01235_b200 import gen, partition

    rank, out = int(sys.argv[1]), sys.argv[2]
    dist.init_process_group("gloo", rank=rank, world_size=2)
    G = load()
    rec = G.rec["grid64"]
    us, vs, caps, s, t = gen.source_edges(rec["source"]["gen"], rec["source"]["args"])
    n = rec["n"]
    pg = partition.PartitionedGraph(n, us, vs, caps, s, t, partition.TorchGroup(device=0))
    flows = [pg.solve_static().flow_value]
    g = mf.build_bicsr(mf.EdgeListGraph(n, us, vs, caps))
    cap0 = np.asarray(g.cap0, np.int64).copy()
    keep = g.is_original.astype(bool)
    for e in rec["chain"]:
        spec = gen.BatchSpec(e["pct"], e["kind"], e["seed"])
        bu, bv, bc, _ = gen.batch_arrays(n, g.src[keep], g.adj[keep], cap0[keep], s, t, spec)
        flows.append(pg.solve_dynamic(mf.UpdateBatch(bu, bv, bc)).flow_value)
        cap0[g.edge_indices(bu, bv)] = bc
    with open(out, "w") as fh:
        fh.write(" ".join(str(f) for f in flows))
    pg.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
