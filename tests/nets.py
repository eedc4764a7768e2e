"""Small networks of the C3 / C4 families for parity tests (test infrastructure).

Each keeps the structure of its family at a size the CPU oracle replays in
seconds: VGG-style (conv with bias, ReLU, maxpool, identity adaptive pool,
flatten, fc, dropout).
"""
import numpy as np
import torch
import torch.nn as nn

from oracle.dropout import keep_mask


class SmallVGG(nn.Module):
    """VGG-16's layer types at 32 x 32: biased 3x3 convs, in-place ReLU, 2x2 max
    pools, the (H, W) adaptive pool that is the identity, flatten, and a
    classifier with dropout between the fc layers."""

    def __init__(self, num_classes=10, width=16):
        super().__init__()
        w = width
        self.features = nn.Sequential(
            nn.Conv2d(3, w, 3, padding=1), nn.ReLU(inplace=True),
            nn.Conv2d(w, w, 3, padding=1), nn.ReLU(inplace=True),
            nn.Conv2d(w, w, 3, padding=1), nn.ReLU(inplace=True),
            nn.Conv2d(w, w, 3, padding=1), nn.ReLU(inplace=True), nn.MaxPool2d(2, 2),
            nn.Conv2d(w, 2 * w, 3, padding=1), nn.ReLU(inplace=True),
            nn.Conv2d(2 * w, 2 * w, 3, padding=1), nn.ReLU(inplace=True), nn.MaxPool2d(2, 2))
        self.avgpool = nn.AdaptiveAvgPool2d((8, 8))
        self.classifier = nn.Sequential(
            nn.Linear(2 * w * 8 * 8, 64), nn.ReLU(True), nn.Dropout(0.5),
            nn.Linear(64, 64), nn.ReLU(True), nn.Dropout(0.3), nn.Linear(64, num_classes))

    def forward(self, x):
        x = self.features(x)
        x = self.avgpool(x)
        x = torch.flatten(x, 1)
        return self.classifier(x)


class _HashDropout(nn.Module):
    """nn.Dropout with the engine's counter-based keep-mask (oracle/dropout.py)."""

    def __init__(self, p, salt, seed):
        super().__init__()
        self.p, self.salt, self.seed = p, salt, seed

    def forward(self, x):
        p = float(np.float32(self.p))
        keep = torch.from_numpy(keep_mask(x.numel(), p, self.seed, self.salt))
        if x.dim() == 4:  # mask drawn over NHWC order
            n, c, h, w = x.shape
            keep = keep.view(n, h, w, c).permute(0, 3, 1, 2)
        scale = torch.tensor(float(np.float32(1.0 / (1.0 - p))), dtype=x.dtype)
        return torch.where(keep.view(x.shape), x * scale, torch.zeros((), dtype=x.dtype))


def use_hash_dropout(model, net, seed=0):
    """Swap every nn.Dropout of ``model`` for the hash-mask dropout of the traced
    op with the same module path, so autograd draws the engine's mask."""
    salt = {op.name: op.id for op in net.ops if op.kind == "dropout"}
    for name, mod in list(model.named_modules()):
        for child_name, child in list(mod.named_children()):
            full = f"{name}.{child_name}" if name else child_name
            if isinstance(child, nn.Dropout) and full in salt:
                setattr(mod, child_name, _HashDropout(child.p, salt[full], seed))
            elif isinstance(child, _HashDropout):
                child.seed = seed
    return model
