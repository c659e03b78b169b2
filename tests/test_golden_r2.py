"""CPU checks of the round-2 golden fixtures (no GPU): the config-1 reference
run is deterministic up to its first loss spike and chaotic after it, which is
what the 1k-epoch curve tests on the GPU are built around."""
import numpy as np

from conftest import load_golden


def test_config1_reference_chaos_onset():
    g = load_golden("train_config1.npz")["total"]
    s = load_golden("train_config1_sens_1e-15.npz")["total"]
    rel = np.abs(s - g) / np.abs(g)
    onset = int(np.flatnonzero(rel > 1e-12)[0])
    assert 300 <= onset <= 600, onset
    assert rel[:300].max() < 1e-13             # deterministic phase: rounding-level
    assert rel[onset:].max() > 1e-4            # chaotic phase: O(1e-4 .. 1) drift
    assert g[0] / g[-1] > 100                  # the run trains (loss falls > 100x)
    up = np.flatnonzero(g[1:] > 1.01 * g[:-1]) + 1
    assert up[0] > onset                       # the first loss spike follows the onset
    s7 = load_golden("train_config1_sens_1e-07.npz")["total"]
    r7 = np.abs(s7 - g) / np.abs(g)
    assert r7[:400].max() < 1e-5               # a 1e-7 perturbation: ~1e-6 before the spike


def test_headline_fixture_is_the_bench_workload():
    g = load_golden("step_headline.npz")
    assert tuple(g["grid"]) == (64, 64, 16) and float(g["t_end"]) == 1.5
    assert g["grad"].shape == (3, 66932) and g["flat"].shape == (3, 66932)
    assert np.array_equal(g["flat"][0], g["flat0"])
    # Adam moved the parameters between epochs; weights are time_bin_weights outputs
    assert np.all(g["weights"][:, 0] == 1.0) and np.all(g["weights"] <= 1.0)
