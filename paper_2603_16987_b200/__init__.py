"""B200-native VLM input preprocessing (arXiv 2603.16987 hot path).

Drop-in for the vlmfp preprocessing calls (vlmfp/__init__.py:99-139) with the
arithmetic in hand-written sm_100a kernels behind a C-ABI (include/tileprep.h).
Importing the package is cheap and works without a GPU; compute calls need the
built libtileprep.so and a CUDA device and raise otherwise (no CPU fallback).
"""

from .dtypes import FLOAT16_WIDE, FLOAT32, INT32, UINT8
from .errors import (
    ArenaFullError,
    AssemblyError,
    ConfigError,
    DataError,
    DecodeError,
    DeviceError,
    DimensionError,
    DomainError,
    ExpansionError,
    MalformedSequenceError,
    ShapeError,
    TemplateError,
    UnsupportedFormatError,
    VlmfpError,
)
from .imgproc import (
    ImageBuffer,
    PreprocessConfig,
    PreprocessResult,
    TilePlan,
    decode_image,
    normalize,
    normalize_tiles,
    preprocess,
    resize_bilinear,
    select_tile_plan,
    tile_image,
)
from .tokenizer import (
    TokenizedBatch,
    Vocab,
    detokenize,
    load_vocab,
    tokenize,
    tokenize_batch,
    PlaceholderExpander,
    SpecialIds,
    TokenSequence,
    build_supervision_mask,
    expand_and_mask,
    expand_image_placeholders,
    load_specials,
)
from .tokenred import (
    PatchGrid,
    TokenReductionConfig,
    pixel_unshuffle,
    pixel_unshuffle_tensor,
    tokens_per_tile,
    visual_token_count,
)
from .backend import AssembledSequence, assemble
from .engine import PackedImages, TileBatch, TilePreprocessor, pack_images, synth_packed
from .transfer import (
    DEFAULT_ALIGNMENT,
    BatchEntry,
    CostModel,
    HostArena,
    PipelinedPreprocessor,
    Region,
    StagedImages,
    TransferBatch,
    TransferResult,
    pack,
    payload_bytes,
    stage_images,
    stage_individually,
    transfer,
    unpack,
    upload_images,
)

__version__ = "0.1.0"
