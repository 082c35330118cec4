"""Compare the tensor-core deform backward (with cache) against the recompute
path (no cache) on the configs[1] shapes; print where they disagree."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2503_06161_b200 as fs  # noqa: E402
from test_gpu_deform_parity import config1_parts  # noqa: E402


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
    cloud, field, net = config1_parts(k)
    t = 0.37
    snap, cache = fs.deform_with_cache(cloud, field, net, t)
    rng = np.random.default_rng(1)
    ups = {f: rng.normal(size=np.shape(getattr(cloud, f))).astype(np.float32).astype(np.float64)
           for f in ("positions", "rotations", "log_scales", "opacity_logits", "features")}
    gr = type("G", (), ups)()
    cg, ng, pg = fs.deform_backward(cloud, field, net, cache, gr)
    nocache = dict(cache)
    nocache["device"] = None
    cg2, ng2, pg2 = fs.deform_backward(cloud, field, net, nocache, gr)
    d = np.abs(cg["positions"] - cg2["positions"]).max(axis=1)
    bad = np.nonzero(d > 1e-3)[0]
    print("positions: max", d.max(), "n bad", len(bad), "first", bad[:20], "tile rows", np.unique(bad % 128)[:40])
    for key in ng:
        e = np.abs(ng[key] - ng2[key])
        print(f"{key:24s} max {e.max():.3e}  ref max {np.abs(ng2[key]).max():.3e}  argmax {np.unravel_index(e.argmax(), e.shape)}")
    for l in range(2):
        for p in range(6):
            e = np.abs(pg[l][p] - pg2[l][p])
            print(f"plane {l}/{p} max {e.max():.3e} ref {np.abs(pg2[l][p]).max():.3e}")


if __name__ == "__main__":
    main()
