#!/bin/bash
# Conformance run: the reference's OWN pytest files for the in-scope modules
# (core, raycast, graph, integrate_mc, integrate_hmc), executed unmodified
# against this package through a `voronray` alias (tools/refsuite/shim).
#
#   step 1 (container, /root/reference present):  tools/refsuite/run.sh stage
#       copies the reference's test files into _refsuite/ (git-ignored, never
#       committed: they are reference sources)
#   step 2 (GPU box):  gpurun -- 'bash tools/refsuite/run.sh run'
#       runs them and writes gpurun_out/refsuite.log
#   step 3 (container):  tools/refsuite/run.sh clean
set -u
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
STAGE=$ROOT/_refsuite
case "${1:-}" in
  stage)
    rm -rf "$STAGE"; mkdir -p "$STAGE"
    for f in conftest.py test_core.py test_raycast.py test_graph.py test_integrate_mc.py \
             test_integrate_hmc.py; do
      cp /root/reference/pkg/tests/$f "$STAGE"/ || exit 1
    done
    # the alias package; the reference's exact polygon integrator (out of scope,
    # SURVEY.md §8) is staged next to it as the HMC tests' own oracle
    cp -r "$ROOT/tools/refsuite/shim/voronray" "$STAGE"/voronray
    cp /root/reference/pkg/src/voronray/integrate_poly.py "$STAGE"/voronray/ || exit 1
    ;;
  run)
    mkdir -p "$ROOT/gpurun_out"
    cd "$STAGE" && PYTHONPATH="$STAGE:$ROOT" timeout 3000 python -m pytest -q --no-header -p no:cacheprovider \
        -k "not bisection" -rfE . > "$ROOT/gpurun_out/refsuite.log" 2>&1
    echo "rc $?" >> "$ROOT/gpurun_out/refsuite.log"
    tail -40 "$ROOT/gpurun_out/refsuite.log"
    ;;
  clean) rm -rf "$STAGE" ;;
  *) echo "usage: $0 stage|run|clean"; exit 2 ;;
esac
