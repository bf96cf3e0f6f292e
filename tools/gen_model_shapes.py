"""Regenerate workloads/model_shapes.json from torchvision architectures.

The models are built on the ``meta`` device, so no weights are allocated or
downloaded; only ``p.shape`` of every trainable parameter is recorded, in
registration order.  Run once; the JSON is committed.
"""
import json
import pathlib

import torch
import torchvision

OUT = pathlib.Path(__file__).resolve().parents[1] / "workloads" / "model_shapes.json"


def main():
    with torch.device("meta"):
        models = {
            "resnet101": torchvision.models.resnet101(),
            "inception_v3": torchvision.models.inception_v3(aux_logits=False, init_weights=False),
            "vgg16": torchvision.models.vgg16(),
        }
    out = {}
    for key, m in models.items():
        out[key] = [[n, list(p.shape)] for n, p in m.named_parameters() if p.requires_grad]
    OUT.write_text(json.dumps(out, indent=0) + "\n")


if __name__ == "__main__":
    main()
