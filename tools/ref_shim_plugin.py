"""pytest plugin: run the REFERENCE's own test suite with this package's GPU
operators swapped in (paper_1207_6365_b200.install()).

    PYTHONPATH=baseline/_ref:. python -m pytest baseline/_ref/ref_tests \
        -p tools.ref_shim_plugin -c /dev/null --rootdir baseline/_ref -q

baseline/_ref holds the unmodified reference (pip-installed from a copy of
/root/reference/pkg, plus its tests/), git-ignored; tools/ref_tests_shim.sh
prepares it in the build container.  At the end the plugin prints how many
sm_100a kernels the suite launched through libsketch_b200.so, so the log
shows the reference's tests really ran on the GPU path.
"""

import os


def pytest_configure(config):
    import sketchnla

    import paper_1207_6365_b200 as skb

    assert "baseline/_ref" in sketchnla.__file__ or os.environ.get("SKT_REF_ANY"), sketchnla.__file__
    skb.install()
    config._skt_launch0 = skb.launch_count()


def pytest_sessionfinish(session, exitstatus):
    import sketchnla.sketch as ref

    import paper_1207_6365_b200 as skb

    n = skb.launch_count() - getattr(session.config, "_skt_launch0", 0)
    print(f"\n[shim] sketchnla.sketch.SparseEmbedding is {ref.SparseEmbedding.__module__}."
          f"{ref.SparseEmbedding.__name__}; {n} libsketch_b200.so kernel launches during the suite")
