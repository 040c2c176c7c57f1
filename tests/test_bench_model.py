"""Host-side pin of bench.py's K10 executed-work model (no GPU): the executed MMA flop count per c4
launch must equal ncu's BF16 UTCHMMA op count of the same launch, recorded in
profiles/r01_conv_tc_c4.md (sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum)."""
import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_tc_executed_flop_matches_ncu_count():
    import bench
    import se2_synth as S
    cfg = S.get_config("c4")
    # balanced mode: 32 eight-row tiles x 4 orientation blocks, chains 23/31/38 x 28/31/23 input rows
    assert bench._tc_executed_flop(cfg, cfg.R) == 914324717568


def test_tc_executed_flop_modes():
    """The model follows conv_tc.cu's geometry choice: the balanced mode when its per-SM chain (units
    over 148 CTAs, at least half a chain) is below 0.95 of the row-count mode's cost."""
    import bench
    import se2_synth as S
    R, S_, npad = 15, 31, 256
    per_row = S_ * 2 * 3 * 2.0 * 128 * npad * 16

    def chains(ny, rows):
        return [min(ny - 1, y0 + rows - 1 + R) - max(0, y0 - R) + 1 for y0 in range(0, ny, rows)]

    cfg = dataclasses.replace(S.get_config("c4"), ny=128)   # balanced: q = 19 < 0.95 x 34 (4-row mode)
    assert bench._tc_executed_flop(cfg, R) == 4 * sum(chains(128, 8)) * per_row
    cfg = S.get_config("c4")                                  # 8 fields: the row-count mode (8 rows) wins
    assert bench._tc_executed_flop(cfg, R, batch=8) == 8 * 4 * sum(chains(256, 8)) * per_row
    cfg = dataclasses.replace(S.get_config("c4"), ny=60)    # balanced vs 4-row tiles (34 rows per CTA)
    assert bench._tc_executed_flop(cfg, R) == 4 * sum(chains(60, 8)) * per_row
