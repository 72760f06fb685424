#!/usr/bin/env bash
# Stage the reference's unmodified test files into .refsuite/ (git-ignored)
# for ONE gpurun call, then remove them: the GPU box has no /root/reference.
#   tools/ref_suite/stage.sh          # stage
#   tools/ref_suite/stage.sh clean    # remove
set -euo pipefail
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
rm -rf "$ROOT/.refsuite"
[ "${1:-}" = clean ] && exit 0
mkdir -p "$ROOT/.refsuite"
cp /root/reference/pkg/tests/*.py "$ROOT/.refsuite/"
