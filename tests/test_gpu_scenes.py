"""Device-side scene generation (bmpc_batch_set_scenes) against the host
builders (themselves bit-identical to the reference's, tests/test_builders.py,
test_serialization.py): the per-node references and vehicle predictions the
GPU computes from scene specs agree with the builders' to the last few ulps
(device vs glibc sin / cos), and the solves agree with the host-built
problems' (counts, trajectories)."""
import dataclasses

import numpy as np
import pytest

import _gen
import paper_2506_13624_b200 as B

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return B.Context(0)


def _scenes(kind, k):
    out = []
    for i in range(k):
        if kind == "intersection":
            base = B.intersection_spec(40, 8.0, 0.4)
            v0, v1 = base.vehicles
            out.append(dataclasses.replace(
                base, ego_start=(0.1 * i, -18.0 + 0.2 * i, 1.5 + 0.01 * i, 4.0 + 0.1 * i),
                vehicles=(dataclasses.replace(v0, position=(-3.0 - 0.1 * i, 25.0), speed=7.0 + 0.05 * i),
                          dataclasses.replace(v1, position=(0.5, -8.0 + 0.1 * i))),
                safety_radius=2.5 + 0.01 * i))
        else:
            base = B.latency_spec(0.6, 50, 4.0, 0.1)
            (v0,) = base.vehicles
            out.append(dataclasses.replace(base, ego_start=(0.0, 0.2 * i, 0.0, 9.0 + 0.1 * i),
                                           vehicles=(dataclasses.replace(v0, position=(25.0 + i, 0.0)),),
                                           continue_deceleration=2.0 + 0.1 * i))
    return out


@pytest.mark.parametrize("kind", ["intersection", "latency"])
def test_device_scenes_match_host_builders(ctx, kind):
    specs = _scenes(kind, 12)
    if kind == "intersection":
        probs = [B.build_intersection_case(s, 2, 2) for s in specs]
        fam = B.SCENARIO_INTERSECTION
    else:
        probs = [B.build_latency_case(s) for s in specs]
        fam = B.SCENARIO_LATENCY
    host = B.Batch(ctx, probs, max_records=500)
    host.set_models()
    dev = B.Batch(ctx, probs, max_records=500)  # same tree; the scene data comes from the GPU
    nbytes = dev.set_scenes(specs, fam, 2, 2)
    assert nbytes < 12 * 4096  # the specs, not the per-node arrays
    for i, p in enumerate(probs):
        a = p.arrays()
        g = dev.scene(i)
        assert _gen.rel_err(g["reference"], a["reference"]) <= 1e-14
        assert _gen.rel_err(g["vehicles"], a["vehicles"]) <= 1e-14
        np.testing.assert_array_equal(g["initial_state"], a["initial_state"])
    host.solve()
    dev.solve()
    xh = np.zeros((12, host.n, 4))
    xd = np.zeros_like(xh)
    rh, _ = host.results(xh)
    rd, _ = dev.results(xd)
    assert [r.inner_iterations for r in rh] == [r.inner_iterations for r in rd]
    assert [r.status for r in rh] == [r.status for r in rd]
    assert _gen.rel_err(xd, xh) <= 1e-8


def test_shared_scene_plus_initial_states_is_cfg4(ctx):
    """cfg4 as a receding-horizon caller would drive it: one shared scene
    spec generated on the device, then each instance's measured state."""
    spec = B.intersection_spec(63, 10.0, 0.1)
    probs = [B.build_intersection_case(spec, 2, 2, perturb_seed=42 + i) for i in range(16)]
    host = B.Batch(ctx, probs)
    host.set_models()
    dev = B.Batch(ctx, probs)
    dev.set_scenes(spec)
    dev.set_initial_states(np.array([p.initial_state for p in probs]))
    host.solve()
    dev.solve()
    rh, _ = host.results()
    rd, _ = dev.results()
    assert [r.inner_iterations for r in rh] == [r.inner_iterations for r in rd]


def test_scene_rejects_other_trees(ctx):
    p = B.build_intersection_case(B.intersection_spec(40, 8.0, 0.4), 2, 2)
    bt = B.Batch(ctx, [p])
    with pytest.raises(B.BmpcError, match="branch steps"):
        bt.set_scenes(B.intersection_spec(40, 8.0, 1.2))
    with pytest.raises(B.BmpcError, match="horizon"):
        bt.set_scenes(B.intersection_spec(41, 8.0, 0.4))
