"""CPU: the oracle-side input generators (oracle/inputs_gen.c, used by bench.py's
reference arm so it never loads the product library) reproduce the product's
generators bit for bit: R-MAT against the numpy restatement of the device rule
(oracle/inputs_oracle.rmat_np, itself pinned to the device kernel in
tests/test_gpu_inputs.py), power-law against the product's host generator
(dsvd_synth_powerlaw, synth.cpp)."""
import numpy as np
import pytest

from inputs_oracle import rmat_np
from oracle_lib import InputsGen


@pytest.fixture(scope="module")
def gen():
    return InputsGen()


def same(a, b):
    assert a.rows == b.rows and a.cols == b.cols
    assert np.array_equal(a.offsets, b.offsets)
    assert np.array_equal(a.col_indices, b.col_indices)
    assert np.array_equal(np.asarray(a.values).view(np.uint64), np.asarray(b.values).view(np.uint64))


@pytest.mark.parametrize("scale,draws,uniform,seed", [(10, 20000, False, 4), (12, 60000, True, 5), (7, 0, False, 1),
                                                      (9, 100000, True, 9)])
def test_rmat_matches_the_device_rule(gen, scale, draws, uniform, seed):
    same(gen.rmat(scale, draws, uniform=uniform, seed=seed), rmat_np(scale, draws, uniform=uniform, seed=seed))


@pytest.mark.parametrize("rows,cols,mu,sigma,zipf,ratings,seed", [
    (3000, 1500, 2.0, 1.0, 1.1, False, 2), (2000, 900, 2.5, 1.2, 1.0, True, 3), (50, 20, 3.0, 1.0, 1.1, False, 7)])
def test_powerlaw_matches_the_product_generator(gen, rows, cols, mu, sigma, zipf, ratings, seed):
    import paper_2404_09276_b200 as d
    a = gen.powerlaw(rows, cols, mu, sigma, zipf, seed, ratings=ratings)
    b = d.powerlaw(rows, cols, mu, sigma, zipf, seed, ratings=ratings)
    same(a, b)
