"""CPU: the U-Net / classifier block program reproduces the reference's layer graph --
the per-layer description (kinds, levels, channel chain), the parameter layout (names,
order, sizes) and the Rng draw order of the initialiser -- compared with the reference's
own network module (unpacked from oracle/_ref/refsuite.tar.gz, built by oracle/build_ref.sh).
"""

import os
import sys
import tarfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TARBALL = os.path.join(ROOT, "oracle", "_ref", "refsuite.tar.gz")

ARGS = [(3, 1, 3, 2, 64, 8, 4), (3, 2, 3, 1, 4, 4, 4), (2, 3, 5, 3, 8, 4, 2)]


@pytest.fixture(scope="module")
def ref_network(tmp_path_factory):
    if not os.path.exists(TARBALL):
        pytest.skip("oracle/_ref/refsuite.tar.gz not built")
    d = tmp_path_factory.mktemp("refsuite")
    with tarfile.open(TARBALL) as tf:
        tf.extractall(d, filter="data")
    sys.path.insert(0, str(d / "refpkg"))
    try:
        from flexconv import network
    finally:
        sys.path.pop(0)
    return network


def _rows(specs):
    return [(s.kind, s.level, s.c_in, s.c_out) for s in specs]


@pytest.mark.parametrize("args", ARGS)
def test_segnet_program_matches_reference_graph(ref_network, args):
    from paper_1803_07289_b200 import network

    ref = ref_network.build_segnet(*args)
    ours = network.build_segnet(*args, device="cpu")
    assert _rows(ours.specs()) == _rows(ref.specs())
    assert ours.param_count() == ref.param_count()
    assert ours.store.names() == ref.store.names()
    for name in ref.store.names():
        assert tuple(ours.store.view(name).shape) == ref.store.view(name).shape, name
    assert ours.encoder_widths == ref.encoder_widths


def test_classifier_program_matches_reference_graph(ref_network):
    from paper_1803_07289_b200 import network

    ref = ref_network.build_classifier(3, 2, 5, 2, 4, 4, 4)
    ours = network.build_classifier(3, 2, 5, 2, 4, 4, 4, device="cpu")
    assert _rows(ours.specs()) == _rows(ref.specs())
    assert ours.store.names() == ref.store.names()


def test_parameter_layers_follow_the_reference_layer_order(ref_network):
    """initialize_params draws per parameterised layer in the reference's layer order: the
    program's (kind, name) sequence equals the reference's FlexConv / Pointwise sequence."""
    from paper_1803_07289_b200 import network

    ref = ref_network.build_segnet(3, 1, 3, 2, 8, 8, 4)
    ours = network.build_segnet(3, 1, 3, 2, 8, 8, 4, device="cpu")
    want = []
    for layer in ref.layers:
        if isinstance(layer, ref_network._FlexConv):
            want.append(("flex", layer.name))
        elif isinstance(layer, ref_network._Pointwise):
            want.append(("pw", layer.name))
    assert [(k, n) for k, n, _, _ in ours._param_layers()] == want
