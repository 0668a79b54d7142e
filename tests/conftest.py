"""Shared fixtures: the `gpu` marker, golden-vector loading, spec rebuilding."""

import os
import sys

import numpy as np
import pytest
import scipy.sparse as sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def spec_from_golden(g, prefix):
    """Rebuild the reference-generated ModelSpec (inputs stored in the fixture)
    with this package's host classes."""
    from paper_2507_06938_b200.model import ModelSpec, path_graph_spatial, uniform_grid_temporal

    nv, ns, nt, nf = (int(x) for x in g[f"{prefix}dims"])
    design, obs = [], []
    for i in range(nv):
        shape = tuple(int(x) for x in g[f"{prefix}A{i}_shape"])
        design.append(
            sp.csr_matrix(
                (g[f"{prefix}A{i}_data"], g[f"{prefix}A{i}_indices"], g[f"{prefix}A{i}_indptr"]),
                shape=shape,
            )
        )
        obs.append(np.array(g[f"{prefix}y{i}"]))
    return ModelSpec(
        n_processes=nv,
        n_spatial=ns,
        n_time=nt,
        n_fixed=nf,
        spatial=[path_graph_spatial(ns) for _ in range(nv)],
        temporal=[uniform_grid_temporal(nt) for _ in range(nv)],
        design=design,
        observations=obs,
        fixed_effect_precision=float(g[f"{prefix}fep"][0]),
    ).validate()


def make_spec(n_processes=1, n_spatial=3, n_time=3, n_fixed=1, m_per_process=0, seed=0,
              fixed_effect_precision=1e-3):
    """Same construction and draws as the reference test fixture
    (pkg/tests/conftest.py:26-74)."""
    from paper_2507_06938_b200.model import ModelSpec, path_graph_spatial, uniform_grid_temporal

    rng = np.random.default_rng(seed)
    latent = n_spatial * n_time + n_fixed
    design, obs = [], []
    if m_per_process:
        for _ in range(n_processes):
            rows = np.arange(m_per_process)
            cols = rng.integers(0, n_spatial * n_time, size=m_per_process)
            a = sp.coo_matrix((np.ones(m_per_process), (rows, cols)), shape=(m_per_process, latent))
            if n_fixed:
                cov = sp.coo_matrix(
                    (rng.normal(size=m_per_process * n_fixed),
                     (np.repeat(rows, n_fixed),
                      np.tile(n_spatial * n_time + np.arange(n_fixed), m_per_process))),
                    shape=(m_per_process, latent),
                )
                a = a + cov
            design.append(a.tocsr())
            obs.append(rng.normal(size=m_per_process))
    return ModelSpec(
        n_processes=n_processes, n_spatial=n_spatial, n_time=n_time, n_fixed=n_fixed,
        spatial=[path_graph_spatial(n_spatial) for _ in range(n_processes)],
        temporal=[uniform_grid_temporal(n_time) for _ in range(n_processes)],
        design=design, observations=obs, fixed_effect_precision=fixed_effect_precision,
    ).validate()


@pytest.fixture(scope="session")
def cuda():
    import torch

    from paper_2507_06938_b200 import _lib

    _lib.load()
    return torch.device("cuda", 0)
