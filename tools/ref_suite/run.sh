#!/usr/bin/env bash
# On the GPU box: run the staged reference suite against the drop-in.
# Writes gpurun_out/refsuite_junit.xml and gpurun_out/refsuite.log.
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
cd "$ROOT/.refsuite" || exit 1
PYTHONPATH="$ROOT:$ROOT/tools/ref_suite:${PYTHONPATH:-}" python -m pytest -p tensorlib_alias -q -rfE \
  -p no:cacheprovider --continue-on-collection-errors --rootdir "$ROOT/.refsuite" -c /dev/null --junitxml "$ROOT/gpurun_out/refsuite_junit.xml" \
  "$@" . > "$ROOT/gpurun_out/refsuite.log" 2>&1
echo "refsuite rc=$?"; tail -5 "$ROOT/gpurun_out/refsuite.log"
