"""Golden fixtures (tests/golden/*.npz, made by tests/make_golden.py from the
reference) and the matching product / oracle problems."""
import glob
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names(prefix=""):
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, prefix + "*.npz")))


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)
    d = {k: z[k] for k in z.files}
    d["report"] = json.loads(str(d["report"])) if "report" in d else None
    d["meta"] = json.loads(str(d["meta"]))
    d["records"] = {k[4:]: v for k, v in d.items() if k.startswith("rec_")}
    return d


POPULATION = ("cfg4_population", "cfg3_early")  # compact population fixtures (tests/make_golden_batch.py)


def scenario_names():
    return [n for n in names() if not n.startswith(("lq", "preset_")) and n not in POPULATION]


def preset_names():
    """Other solver presets (tests/make_golden_presets.py)."""
    return names("preset_")


def lq_names():
    return [n for n in names("lq_")]


def build_product_problem(B, meta):
    """paper_2506_13624_b200 problem for a scenario fixture."""
    fam = meta["family"]
    seed = meta["perturb_seed"]
    if fam == 0:
        spec = B.intersection_spec(meta["horizon"], meta["total_time"], meta["shared"][0])
        return B.build_intersection_case(spec, meta["v"][0], meta["v"][1], perturb_seed=seed)
    if fam == 1:
        spec = B.latency_spec(meta["shared"][1], meta["horizon"], meta["total_time"], meta["shared"][0])
        return B.build_latency_case(spec, perturb_seed=seed)
    spec = B.multistage_spec(meta["horizon"], [tuple(b) for b in meta["branchings"]], meta["total_time"])
    return B.build_multistage_case(spec, perturb_seed=seed)


def build_product_lq(B, fx):
    meta = fx["meta"]
    tree = B.build_tree(meta["horizon"], [tuple(b) for b in meta["branchings"]])
    return B.lq_problem(tree, meta["nx"], meta["nu"], fx["x0"], fx["stage"], fx["leaf"])
