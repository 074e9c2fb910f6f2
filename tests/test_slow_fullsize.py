"""-m slow (not part of the -m gpu round-end suite): the full 10^4-observation cfg4 subsample of
tests/test_gpu_fullsize.py protocol (i)-(ii) (~330 s of oracle on 16 host cores).  Needs a GPU;
skipped without one."""
import pytest

from test_gpu_fullsize import _full_size_case, cf, orc  # noqa: F401  (fixtures)

pytestmark = pytest.mark.slow


def test_fullsize_cfg4_pairs_1e4(cf, orc):  # noqa: F811
    _full_size_case(cf, orc, 4, 10_000)
