"""Host-side pin of bench.py's K10 executed-work model (no GPU): the executed MMA flop count per c4
launch must equal ncu's BF16 UTCHMMA op count of the same launch, recorded in
profiles/r01_conv_tc_c4.md (sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_tc_executed_flop_matches_ncu_count():
    import bench
    import se2_synth as S
    cfg = S.get_config("c4")
    assert bench._tc_executed_flop(cfg, cfg.R) == 1023544393728


def test_tc_executed_flop_row_grouping():
    """The model follows conv_tc.cu's tc_rows_out: 8 rows when that gives the fewest waves, fewer when
    they fill the SMs in the same number of waves (c4: 7)."""
    import bench
    import se2_synth as S
    import dataclasses
    cfg = dataclasses.replace(S.get_config("c4"), ny=128)     # 16 groups x 4 blocks = 64 CTAs at 8 rows
    npad, S_, R = 256, 31, 15
    # rows = 4: 32 x 4 = 128 CTAs (one wave), chain 34 rows -> cheapest
    groups = [(y0, min(127, y0 + 3 + R) - max(0, y0 - R) + 1) for y0 in range(0, 128, 4)]
    want = sum(n for _, n in groups) * S_ * 2 * 3 * 4 * 2.0 * 128 * npad * 16
    assert bench._tc_executed_flop(cfg, R) == want
