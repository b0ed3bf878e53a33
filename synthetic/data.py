"""Seeded synthetic parameters and data."""
import numpy as np

from .models import LINEAR, CONV2D, BATCHNORM2D

CIFAR_MEAN = (0.4914, 0.4822, 0.4465)
CIFAR_STD = (0.2023, 0.1994, 0.2010)
IMAGENET_MEAN = (0.485, 0.456, 0.406)
IMAGENET_STD = (0.229, 0.224, 0.225)


def make_params(layers, seed=1):
    """Per layer [weight, bias] float64 arrays in PyTorch layout (None where absent).
    Linear/Conv: U(-1/sqrt(fan_in), 1/sqrt(fan_in)); BatchNorm: gamma=1, beta=0."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out = []
    for l in layers:
        if l.kind == LINEAR:
            bound = 1.0 / np.sqrt(l.in_c)
            w = rng.uniform(-bound, bound, size=(l.out_c, l.in_c))
            b = rng.uniform(-bound, bound, size=(l.out_c,)) if l.bias else None
            out.append([w, b])
        elif l.kind == CONV2D:
            fan_in = l.in_c * l.kh * l.kw
            bound = 1.0 / np.sqrt(fan_in)
            w = rng.uniform(-bound, bound, size=(l.out_c, l.in_c, l.kh, l.kw))
            b = rng.uniform(-bound, bound, size=(l.out_c,)) if l.bias else None
            out.append([w, b])
        elif l.kind == BATCHNORM2D:
            out.append([np.ones(l.in_c), np.zeros(l.in_c)])
        else:
            out.append([None, None])
    # parameters are fp32 masters on every path: round once here so both sides start equal
    return [[None if a is None else a.astype(np.float32).astype(np.float64) for a in p] for p in out]


def make_inputs(n_samples, shape, classes, seed=1, kind="cifar"):
    """x [n, C, H, W] float32 NCHW and y [n] int32.
    kind: 'cifar' / 'imagenet' (bytes/255 normalised with the paper's constants),
          'mnist' (bytes/255, shape (784,1,1) for the MLP), 'gauss' (N(0,1), unit tests)."""
    rng = np.random.Generator(np.random.PCG64(seed + 7919))
    c, h, w = shape
    if kind == "gauss":
        x = rng.standard_normal((n_samples, c, h, w))
    else:
        x = rng.integers(0, 256, size=(n_samples, c, h, w)).astype(np.float64) / 255.0
        if kind in ("cifar", "imagenet"):
            mean = np.array(CIFAR_MEAN if kind == "cifar" else IMAGENET_MEAN)[:c].reshape(1, c, 1, 1)
            std = np.array(CIFAR_STD if kind == "cifar" else IMAGENET_STD)[:c].reshape(1, c, 1, 1)
            x = (x - mean) / std
    y = rng.integers(0, classes, size=(n_samples,)).astype(np.int32)
    return np.ascontiguousarray(x.astype(np.float32)), y
