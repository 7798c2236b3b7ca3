"""paper_2101_05600_b200 — B200-native batched joint CTC/attention beam search.

Drop-in for the decoding path of beamlattice (arXiv 2101.05600 reference):
the host-side API mirrors the reference's C++ names; the work runs in the
sm_100a library ``libbl_b200.so`` behind the C ABI ``include/bl_b200.h``.
"""
from .api import (  # noqa: F401
    BL_CUDA_ERROR, BL_INVALID_ARGUMENT, BL_LOGIC_ERROR, BL_OK, BL_RUNTIME_ERROR,
    K_LOG_ZERO, LIB_PATH, NO_MARGIN, Batch, CudaError, DecodeCounters,
    DecodeResult, Decoder, DecoderConfig, Group, InvalidArgument, LogicError,
    LoopScorer, PosteriorGrid, Scorer, Segment, TableScorer, UniformScorer,
    Utterance, batched_beam_search, beam_search, eos_mode_from_string,
    hard_segments, json_double, lib, make_batches, make_scorer, read_grid, result_json,
    save_table_scorer, vad_segments, write_grid, write_results)
