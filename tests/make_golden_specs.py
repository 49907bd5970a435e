"""Generates tests/golden/gen_spec_{intersection,latency}.json.gz: scenes given
as JSON (scenario_spec_from_json, serialization.hpp:156-197) with their own
vehicles, targets, weights, limits and timing, built by the UNMODIFIED
reference builders (oracle/_ref/gen_ref spec-*) and dumped with
scenario_spec_to_json + scenario_artifacts_to_json. Run in the build
container: python tests/make_golden_specs.py"""
import gzip
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GEN = os.path.join(ROOT, "oracle", "_ref", "gen_ref")

SPECS = {
    "intersection": ({"total_time": 8.0, "shared_times": [0.4], "horizon": 40, "ego_start": [1.0, -18.0, 1.5, 4.0],
                      "vehicles": [{"position": [-3.0, 25.0], "heading": -1.4, "speed": 7.0,
                                    "target_speeds": [7.0, 1.5, 4.0]},
                                   {"position": [0.5, -8.0], "heading": 1.6, "speed": 4.5,
                                    "target_speeds": [4.5, 0.5]}],
                      "state_weights": [2.0, 1.5, 0.2, 0.3], "input_weights": [0.7, 0.4],
                      "terminal_weights": [3.0, 2.0, 0.5, 0.1], "accel_limit": 2.5, "yaw_rate_limit": 0.6,
                      "safety_radius": 2.5, "prediction_tau": 1.2, "reference_turn_rate": 0.35}, ["3", "2"]),
    "latency": ({"total_time": 4.0, "shared_times": [0.1, 0.6], "horizon": 50, "ego_start": [0.0, 0.5, 0.02, 9.0],
                 "vehicles": [{"position": [25.0, 0.0], "heading": 0.01, "speed": 7.5, "target_speeds": [7.0, 0.5]}],
                 "backup_deceleration": 4.0, "continue_deceleration": 2.0, "safety_radius": 3.5,
                 "prediction_tau": 1.0}, []),
}


def main():
    for name, (spec, extra) in SPECS.items():
        out = subprocess.run([GEN, "spec-" + name, json.dumps(spec)] + extra, capture_output=True, text=True,
                             check=True).stdout
        doc = json.loads(out)
        doc["input_spec"] = spec
        with gzip.open(os.path.join(HERE, "golden", f"gen_spec_{name}.json.gz"), "wt") as f:
            json.dump(doc, f)
        print(name, len(doc["problem"]["nodes"]), "nodes")


if __name__ == "__main__":
    main()
