"""NEXT-3: run the Appendix B sweep on synthetic stand-ins of
Table 1's shapes (the datasets are not available): w8a
49749 x 300 at 4% density and Specular 477976 x 50 at 1% (CSR, N(0,1) values),
and YearPredictionsMSD 515344 x 90 dense N(0,1).  gamma in {1, 2, 4, 5, 8, 10},
CountSketch and SJLT (s = 4), ten sketches each.  Prints one JSON document.

  python tools/sketch_quality.py [--trials 10] [--shapes w8a,specular,msd]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1910_14166_b200 as P  # noqa: E402
import synthetic  # noqa: E402
from paper_1910_14166_b200.quality import exact_gram, sketch_quality  # noqa: E402

SHAPES = {
    "w8a": ("csr", 49749, 300, 0.04),
    "specular": ("csr", 477976, 50, 0.01),
    "msd": ("dense", 515344, 90, 1.0),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=10)
    ap.add_argument("--shapes", default="w8a,specular,msd")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    ctx = P.Context(0)
    res = {"what": "Appendix B sweep: mean ||A^T S^T S A - A^T A||_F / ||A^T A||_F and sketch time (CUDA events, "
                   "ms, mean over trials 2..T) on synthetic stand-ins of Table 1 shapes", "shapes": {}}
    for name in args.shapes.split(","):
        layout, n, d, p = SHAPES[name]
        cfg = synthetic.Config(name, n, d, layout, "normal", "countsketch", 1, 1, 1, "ols", density=p, data_seed=11)
        if layout == "csr":
            rp, cl, vl = synthetic.csr_A(cfg, dev)
            A = P.Csr(rp, cl.contiguous(), vl, d)
        else:
            A = P.Dense(synthetic.dense_A(cfg, dev))
        G = exact_gram(A, ctx)
        rows = []
        for fam, s in (("countsketch", 1), ("sjlt", 4)):
            rows += sketch_quality(A, fam, s, [1, 2, 4, 5, 8, 10], trials=args.trials, G=G, ctx=ctx)
        for r in rows:
            r.pop("errs")
        res["shapes"][name] = {"n": n, "d": d, "density": p, "layout": layout, "rows": rows}
        torch.cuda.synchronize()
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
