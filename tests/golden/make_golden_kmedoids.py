"""Golden vectors for k_medoids_loss, produced by the REFERENCE (ebcsum 0.1.0,
ebc.py:21-43) on the seeded inputs of datasets.kmedoids_cases().  Build
container only:  python tests/golden/make_golden_kmedoids.py -> reference_kmedoids.json"""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import datasets  # noqa: E402
from ebcsum import GroundMatrix, Precision, k_medoids_loss  # noqa: E402


def main():
    losses = []
    for prec, data, reps in datasets.kmedoids_cases():
        losses.append(k_medoids_loss(GroundMatrix(data, Precision(prec)), reps))
    out = os.path.join(HERE, "reference_kmedoids.json")
    with open(out, "w") as fh:
        json.dump({"generator": "ebcsum 0.1.0 k_medoids_loss (ebc.py:21-43) on datasets.kmedoids_cases()",
                   "losses": losses}, fh, indent=0)
    print(out, len(losses))


if __name__ == "__main__":
    main()
