"""B200-native DeepFFM hot path: a drop-in for the reference ``fieldwise``
package's model / predict / learn API.

Compute runs only through libdffm.so (hand-written sm_100a CUDA behind a C
ABI, include/dffm.h); torch tensors are used as device buffers.
"""

from . import errors
from .errors import (ContractError, FieldwiseError, FormatError, NumericError, SizingError,
                     StaleCacheError)
from .model import (ForwardState, ModelConfig, OpCounter, WeightStore, backward_update,
                    flat_weight_view, forward, init_model, load_model, loss_gradients,
                    pair_position, predict_batch, predict_proba, save_model, store_from_bytes)

__all__ = ["errors", "ContractError", "FieldwiseError", "FormatError", "NumericError",
           "SizingError", "StaleCacheError", "ForwardState", "ModelConfig", "OpCounter",
           "WeightStore", "backward_update", "flat_weight_view", "forward", "init_model",
           "load_model", "loss_gradients", "pair_position", "predict_batch", "predict_proba",
           "save_model", "store_from_bytes"]
