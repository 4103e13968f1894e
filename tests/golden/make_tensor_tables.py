"""Generates tests/golden/tensor_tables.json: per-tensor parameter counts of
the models BASELINE.json names (ALBERT-base / ALBERT-large pretraining heads,
torchvision-style ResNet-50), in named_parameters() order. Built on the meta
device from transformers' configs, so no weights or network are needed.
The LAMB trust ratio is per tensor, so these tables define the tensor
boundaries of the synthetic gradient vectors."""
import json
import os

import torch
from transformers import AlbertConfig, AlbertForPreTraining


def albert(size):
    cfg = {
        "base": dict(hidden_size=768, num_attention_heads=12, intermediate_size=3072),
        "large": dict(hidden_size=1024, num_attention_heads=16, intermediate_size=4096),
    }[size]
    c = AlbertConfig(embedding_size=128, num_hidden_layers=24 if size == "large" else 12,
                     vocab_size=30000, max_position_embeddings=512, type_vocab_size=2, **cfg)
    with torch.device("meta"):
        m = AlbertForPreTraining(c)
    seen, sizes = set(), []
    for name, p in m.named_parameters():
        if id(p) in seen:
            continue
        seen.add(id(p))
        sizes.append([name, p.numel()])
    return sizes


def resnet50():
    # torchvision resnet50 layout (bottleneck [3,4,6,3], expansion 4), written
    # out so torchvision is not required.
    sizes = []
    def conv(name, cin, cout, k):
        sizes.append([name + ".weight", cout * cin * k * k])
    def bn(name, c):
        sizes.append([name + ".weight", c]); sizes.append([name + ".bias", c])
    conv("conv1", 3, 64, 7); bn("bn1", 64)
    cin = 64
    for li, (blocks, width) in enumerate(zip([3, 4, 6, 3], [64, 128, 256, 512]), 1):
        for b in range(blocks):
            pre = f"layer{li}.{b}"
            conv(pre + ".conv1", cin, width, 1); bn(pre + ".bn1", width)
            conv(pre + ".conv2", width, width, 3); bn(pre + ".bn2", width)
            conv(pre + ".conv3", width, width * 4, 1); bn(pre + ".bn3", width * 4)
            if b == 0:
                conv(pre + ".downsample.0", cin, width * 4, 1); bn(pre + ".downsample.1", width * 4)
            cin = width * 4
    sizes.append(["fc.weight", 2048 * 1000]); sizes.append(["fc.bias", 1000])
    return sizes


if __name__ == "__main__":
    out = {"albert-base": albert("base"), "albert-large": albert("large"), "resnet50": resnet50()}
    for k, v in out.items():
        print(k, len(v), sum(s for _, s in v), max(s for _, s in v))
    with open(os.path.join(os.path.dirname(__file__), "tensor_tables.json"), "w") as f:
        json.dump({k: [s for _, s in v] for k, v in out.items()} |
                  {k + ".names": [n for n, _ in v] for k, v in out.items()}, f)
