"""The sampled-parity helper must reproduce the full oracle's values for the selected outputs."""
import numpy as np

import fsmt_gen
from oracle import hsmt, objective
from tests.helpers import subformula


def test_subformula_preserves_selected_gradients_and_terms():
    for name in ("cfg4s", "cfg3s", "cfg1"):
        inst = fsmt_gen.config(name)
        f = hsmt.parse(inst.text)
        rng = np.random.default_rng(1)
        a = rng.uniform(-1, 1, f.n_bool)
        b = rng.uniform(0, 1, f.n_real)
        C, ga, gb, terms = objective.objective_and_gradient(f, a, b, 1.1, want_terms=True)
        bsel = rng.choice(f.n_bool, 2, replace=False)
        rsel = rng.choice(f.n_real, 2, replace=False)
        csel = rng.choice(len(f.constraints), 5, replace=False)
        sub, keep = subformula(inst.text, bsel, rsel, extra_constraints=csel)
        fs = hsmt.parse(sub)
        Cs, gas, gbs, ts = objective.objective_and_gradient_grouped(fs, a, b, 1.1, want_terms=True)
        assert np.allclose(gas[bsel], ga[bsel], atol=1e-12) and np.allclose(gbs[rsel], gb[rsel], atol=1e-12)
        for k, ci in enumerate(keep):
            assert abs(ts[k] - terms[ci]) < 1e-12
        assert set(csel) <= set(keep)
