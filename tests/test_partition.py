"""Host-side stage partitioning (R17 layer-count rule and the SURVEY 8e cost-balanced split)."""
import itertools

import synthetic as S
from synthetic.models import chain_units, unit_macs, balanced_stages, assign_stages, resnet101


def stage_costs(L, units, cost, K):
    per = [0.0] * K
    seen = set()
    for i, l in enumerate(L):
        if units[i] not in seen:
            seen.add(units[i])
            per[l.stage] += cost[units[i]]
    return per


def test_balanced_split_is_optimal_and_contiguous():
    """The DP split minimises the largest stage cost over every contiguous split (brute force)."""
    L = S.vgg16_cifar()
    units = chain_units(L)
    cost = unit_macs(L, units, (3, 32, 32))
    n = len(cost)
    for K in (2, 3, 4):
        B = balanced_stages(L, units, cost, K)
        stages = [l.stage for l in B]
        assert stages == sorted(stages) and set(stages) == set(range(K))
        got = max(stage_costs(B, units, cost, K))
        best = min(max(sum(cost[a:b]) for a, b in zip((0,) + cuts, cuts + (n,)))
                   for cuts in itertools.combinations(range(1, n), K - 1))
        assert abs(got - best) <= 1e-6 * best


def test_vgg_units_and_costs():
    """VGG-16-CIFAR: 14 units (13 convs + the classifier); forward MACs per sample 313.2 M
    (SURVEY A.4)."""
    L = S.vgg16_cifar()
    units = chain_units(L)
    cost = unit_macs(L, units, (3, 32, 32))
    assert max(units) + 1 == 14
    assert abs(sum(cost) / 1e6 - 313.2) < 0.1


def test_dag_units_never_split_a_block():
    """ResNet-101: the layer-count rule over units keeps every residual edge inside a stage."""
    L, units = resnet101(classes=200)
    for K in (2, 4, 8):
        A = assign_stages(L, units, K)
        for i, l in enumerate(A):
            for src in (l.src0, l.src1):
                if src is not None and src >= 0:
                    assert A[src].stage in (l.stage, l.stage - 1)
                    if A[src].stage != l.stage:
                        assert units[src] + 1 == units[i]
