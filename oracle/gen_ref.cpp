// gen_ref — test infrastructure: the reference's `bench gen` document
// (proj/tools/bench.cpp:327-357: scenario_spec_to_json +
// scenario_artifacts_to_json, serialization.hpp:128-219) written by the
// UNMODIFIED reference headers (compiled against the Eigen shim), compact.
// tests/make_golden.py stores its output under tests/golden/ as the fixture
// for `python -m paper_2506_13624_b200.cli gen`; "report" / "tree" dump
// report_to_json of the cfg0 solve and tree_spec_to_json (serialization tests).
#include <bmpc/bmpc.hpp>
#include <bmpc/serialization.hpp>

#include <iostream>
#include <string>

int main(int argc, char** argv) {
  const std::string scenario = argc > 1 ? argv[1] : "intersection";
  bmpc::json doc;
  bmpc::ScenarioArtifacts artifacts;
  if (scenario == "intersection") {
    const bmpc::ScenarioSpec spec = bmpc::intersection_spec();
    bmpc::build_intersection_case(spec, 2, 2, &artifacts);
    doc["kind"] = "intersection";
    doc["v1_count"] = 2;
    doc["v2_count"] = 2;
    doc["spec"] = bmpc::scenario_spec_to_json(spec);
  } else if (scenario == "latency") {
    const bmpc::ScenarioSpec spec = bmpc::latency_spec(0.5);
    bmpc::build_latency_case(spec, &artifacts);
    doc["kind"] = "latency";
    doc["spec"] = bmpc::scenario_spec_to_json(spec);
  } else if (scenario == "spec-intersection" || scenario == "spec-latency") {
    // A scene from JSON (scenario_spec_from_json, serialization.hpp:156-197),
    // built by the reference builder: argv[2] = spec JSON, argv[3..4] = v1 v2.
    const bmpc::ScenarioSpec spec = bmpc::scenario_spec_from_json(bmpc::json::parse(argv[2]));
    if (scenario == "spec-intersection") {
      const int v1 = std::stoi(argv[3]), v2 = std::stoi(argv[4]);
      bmpc::build_intersection_case(spec, v1, v2, &artifacts);
      doc["kind"] = "intersection";
      doc["v1_count"] = v1;
      doc["v2_count"] = v2;
    } else {
      bmpc::build_latency_case(spec, &artifacts);
      doc["kind"] = "latency";
    }
    doc["spec"] = bmpc::scenario_spec_to_json(spec);
  } else if (scenario == "report") {  // report_to_json of the cfg0 solve (acceptance_test.cpp:93-102)
    const bmpc::BmpcProblem problem =
        bmpc::build_intersection_case(bmpc::intersection_spec(63, 10.0, 0.1), 2, 2);
    std::cout << bmpc::report_to_json(bmpc::solve(problem).report).dump() << "\n";
    return 0;
  } else if (scenario == "tree") {  // tree_spec_to_json (test_serialization.cpp:12)
    const bmpc::TreeTopology tree = bmpc::build_tree(6, {{2, 2, {0.5, 0.5}}, {4, 3, {0.2, 0.3, 0.5}}});
    std::cout << bmpc::tree_spec_to_json(tree).dump() << "\n";
    return 0;
  } else {
    std::cerr << "unknown scenario\n";
    return 2;
  }
  doc["problem"] = bmpc::scenario_artifacts_to_json(artifacts);
  std::cout << doc.dump() << "\n";
  return 0;
}
