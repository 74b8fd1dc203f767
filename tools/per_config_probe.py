"""bench.py's per_config step (10-step CUDA graphs; short window and >= 0.5 s sustained) for the
named configs without the solve -- the A/B probe for the mid-size configs (FLS_LIB selects a
variant build).

    python tools/per_config_probe.py c3_poisson5d c4_heat2d
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

names = tuple(sys.argv[1:]) or ("c3_poisson5d", "c4_heat2d")
nosolve = {n: {"ms": 0, "features_ms": 0, "assemble_ms": 0, "lstsq_ms": 0, "eval_ms": 0, "qr_tflops": 0}
           for n in names}
tag = os.path.basename(os.environ.get("FLS_LIB", "base"))
for k, v in bench.per_config(names=names, known_solves=nosolve).items():
    print(tag, k, "short %.2f us %.4f" % (v["graph_us_per_step"], v["frac_of_copy_peak"]),
          "sustained %.2f us %.4f" % (v["sustained"]["graph_us_per_step"], v["sustained"]["frac_of_copy_peak"]),
          flush=True)
