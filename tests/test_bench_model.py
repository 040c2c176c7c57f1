"""Host-side pin of bench.py's K10 executed-work model (no GPU): the executed MMA flop count per c4
launch must equal ncu's BF16 UTCHMMA op count of the same launch, recorded in
profiles/r02_conv_tc_c4.md (sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum, narrow
geometry; r01's classic-geometry count 914 324 717 568 is profiles/r01_conv_tc_c4.md)."""
import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_tc_executed_flop_matches_ncu_count():
    import bench
    import se2_synth as S
    cfg = S.get_config("c4")
    # narrow geometry, balanced mode: 16 sixteen-row tiles x 8 orientation blocks, chains 31 / 46 x 14 / 31
    # input rows, every tile on the 16-orientation window (one K-step)
    assert bench._tc_executed_flop(cfg, cfg.R) == 550779224064
    # the classic geometry of r01 (8-row x 16-orientation tiles, 32-orientation window): band > 12 is never
    # the narrow geometry, so the model with band 13 reproduces r01's count on the same grid
    assert bench._tc_executed_flop(cfg, cfg.R, band=13) == 914324717568


def test_tc_executed_flop_modes():
    """The model follows conv_tc.cu's geometry choice: the balanced mode when its per-SM chain (units
    over 148 CTAs, at least half a chain) is below 0.95 of the row-count mode's cost."""
    import bench
    import se2_synth as S
    R, S_, npad = 15, 31, 256
    per_row = S_ * 1 * 3 * 2.0 * 128 * npad * 16   # narrow geometry, all tiles on the 16-wide window

    def chains(ny, rows):
        return [min(ny - 1, y0 + rows - 1 + R) - max(0, y0 - R) + 1 for y0 in range(0, ny, rows)]

    cfg = dataclasses.replace(S.get_config("c4"), ny=128)   # balanced: q = 23 < 0.95 x 38 (8-row mode)
    assert bench._tc_executed_flop(cfg, R) == 8 * sum(chains(128, 16)) * per_row
    cfg = S.get_config("c4")                                  # 8 fields: the row-count mode (16 rows) wins
    assert bench._tc_executed_flop(cfg, R, batch=8) == 8 * 8 * sum(chains(256, 16)) * per_row
    cfg = dataclasses.replace(S.get_config("c4"), ny=60)    # balanced vs 8-row tiles (38 rows per CTA)
    assert bench._tc_executed_flop(cfg, R) == 8 * sum(chains(60, 16)) * per_row
    # tiles on the 32-wide window (bound failed) execute two K-steps
    cfg = S.get_config("c4")
    assert bench._tc_executed_flop(cfg, R, wide_frac=1.0) == 2 * bench._tc_executed_flop(cfg, R)
