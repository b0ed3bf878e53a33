"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no prediction, no Adam, no layer maths):
only layer-list builders for the paper's workloads, parameter initialisation and input
data generation.  It is the one module both `oracle/` and the product tests/bench use
(task rule: "only the seeded input generators serve both, from a module of their own").

Recipe:
  * weights  ~ U(-1/sqrt(fan_in), +1/sqrt(fan_in)) (PyTorch default bound), biases the same;
    BatchNorm gamma = 1, beta = 0;
  * inputs   = bytes U{0..255}/255, normalised per channel with the paper's constants
    (CIFAR-10 mean/std P:161; ImageNet mean/std P:161 for Tiny-ImageNet-shaped data;
    MNIST-like 784-vectors for the MLP are bytes/255 unnormalised);
  * labels   ~ U{0..classes-1};
  * seed 1 by default ("The seed was fixed with 1").
"""
from .models import (LINEAR, CONV2D, BATCHNORM2D, RELU, MAXPOOL2D, AVGPOOL_GLOBAL, FLATTEN, ADD,
                     CONCAT, SOFTMAX_XENT, AVGPOOL2D, Layer, mlp, vgg16_cifar, tiny_cnn, infer_shapes)
from .data import make_params, make_inputs, CIFAR_MEAN, CIFAR_STD, IMAGENET_MEAN, IMAGENET_STD

__all__ = [
    "LINEAR", "CONV2D", "BATCHNORM2D", "RELU", "MAXPOOL2D", "AVGPOOL_GLOBAL", "FLATTEN", "ADD",
    "CONCAT", "SOFTMAX_XENT", "AVGPOOL2D", "Layer", "mlp", "vgg16_cifar", "tiny_cnn", "infer_shapes",
    "make_params", "make_inputs", "CIFAR_MEAN", "CIFAR_STD", "IMAGENET_MEAN", "IMAGENET_STD",
]
