"""paper_2105_12026_b200 -- B200-native drop-in for the hot path of arXiv
2105.12026 (Exemplar-based Clustering summaries): evaluating
f(S) = L({e0}) - L(S u {e0}) for many candidate sets at once inside Greedy.

Same public names as the reference package ``ebcsum`` for that path
(__init__.py:27-42 there): EbcFunction, GroundMatrix, Precision, EvalMultiset,
Summary, SquaredEuclidean, OptimizerBudget, evaluate_with_backend,
evaluate_multiset_batched, greedy_maximize -- with the backend "b200" (the
default) computing on an sm_100a GPU through libebc200.so.
"""

from .core import (Dissimilarity, EvalMultiset, GroundMatrix, Precision, SquaredEuclidean, Summary,
                   make_auxiliary_vector, squared_euclidean)
from .ebc import EbcFunction, k_medoids_loss
from .optimize import (BACKENDS, OptimizerBudget, evaluate_multiset_batched, evaluate_with_backend,
                       greedy_maximize, parse_backend_spec, sieve_stream_maximize)
from .sharded import evaluate_multiset_sharded, greedy_maximize_sharded

__version__ = "0.1.0"

__all__ = [
    "Dissimilarity", "EvalMultiset", "GroundMatrix", "Precision", "SquaredEuclidean", "Summary",
    "make_auxiliary_vector", "squared_euclidean", "EbcFunction", "k_medoids_loss", "BACKENDS", "OptimizerBudget",
    "evaluate_multiset_batched", "evaluate_with_backend", "greedy_maximize", "parse_backend_spec",
    "greedy_maximize_sharded", "evaluate_multiset_sharded", "sieve_stream_maximize",
]
