#!/bin/bash
# Prepare (build container) or run (GPU box) the reference's own test suite
# through shim.install().
#   tools/ref_tests_shim.sh prepare   # needs /root/reference (build container)
#   tools/ref_tests_shim.sh run [pytest args]   # on the GPU box
set -e
cd "$(dirname "$0")/.."
case "$1" in
prepare)
  rm -rf /tmp/refpkg baseline/_ref
  cp -r /root/reference/pkg /tmp/refpkg
  python -m pip install -q --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref /tmp/refpkg
  cp -r /root/reference/pkg/tests baseline/_ref/ref_tests
  ;;
run)
  shift
  PYTHONPATH="$PWD/baseline/_ref:$PWD" PYTHONDONTWRITEBYTECODE=1 python -m pytest baseline/_ref/ref_tests \
    -p tools.ref_shim_plugin -p no:cacheprovider -c /dev/null --rootdir baseline/_ref "$@"
  ;;
*)
  echo "usage: $0 prepare|run [pytest args]" >&2
  exit 2
  ;;
esac
