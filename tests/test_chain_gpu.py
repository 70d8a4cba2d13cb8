"""Device-resident chaining (the reference's --b / RAP flow,
spgemm_bench_main.cpp:84, 130-135): a product's C passed straight back as an
operand (DeviceMatrix.as_operand, C ABI spgemm_matrix_as_operand) with no host
round trip, checked bitwise against the oracle's host chain; device-operand
validation and stream ordering."""
import numpy as np
import pytest

from helpers import assert_matches_oracle
from paper_2206_07244_b200 import synthetic as S

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("small", [True, False])
def test_rap_chain_on_device_matches_oracle(sg, oracle, small):
    a, p, r = S.config_matrices(4, small=small)
    a, p = S.random_values(a, 11), S.random_values(p, 12)
    r = S.transpose(p)
    ap_dev, o1 = sg.multiply_device(a.to_device(), p.to_device())
    rap_dev, o2 = sg.multiply_device(r.to_device(), ap_dev.as_operand())  # AP stays in HBM
    ap_exp = oracle.spgemm(a, p)
    rap_exp = oracle.spgemm(r, ap_exp)
    assert_matches_oracle(ap_dev.download(), ap_exp)
    assert_matches_oracle(rap_dev.download(), rap_exp)
    if not small:  # nprod 48,556,211 + 69,839,855
        assert (o1.stats.total_nprod, o2.stats.total_nprod) == (48_556_211, 69_839_855)
    rap_dev.free()
    ap_dev.free()


def test_chained_operand_mixed_with_host(sg, oracle):
    a = S.random_values(S.stencil3d_27pt(10), 3)
    c_dev, _ = sg.multiply_device(a, a)                # host operands, C on the device
    cc = sg.multiply(c_dev.as_operand(), a)            # device x host
    assert_matches_oracle(cc.c, oracle.spgemm(oracle.spgemm(a, a), a))
    c_dev.free()


def test_device_operand_validation(sg):
    import torch
    a = S.stencil3d_27pt(6).to_device()
    bad = sg.CsrMatrix(a.rows, a.cols, a.rpt[:-1], a.col, a.val)
    with pytest.raises(sg.InvalidArgument):
        sg.multiply(bad, a)
    if torch.cuda.device_count() < 2:
        return
    other = S.stencil3d_27pt(6).to_device(1)
    with pytest.raises(sg.InvalidArgument):
        sg.multiply_device(other, other, device=0)


def test_operands_written_on_a_side_stream(sg, oracle):
    """A producer writes the operand's values on a non-default torch stream; the
    product (on the library's own stream) must see the finished values."""
    import torch
    host = S.random_values(S.stencil3d_27pt(24), 5)
    a = host.to_device()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        torch.cuda._sleep(50_000_000)  # keep the side stream busy
        vals = torch.from_numpy(host.val).cuda(non_blocking=True) * 2.0
        dev = sg.CsrMatrix(a.rows, a.cols, a.rpt, a.col, vals)
        out = sg.multiply(dev, a)        # issued while `side` is still busy
    want = oracle.spgemm(sg.CsrMatrix(host.rows, host.cols, host.rpt, host.col, host.val * 2.0), host)
    assert_matches_oracle(out.c, want)
