#!/usr/bin/env bash
# Install the UNMODIFIED reference package (pure Python + NumPy, /root/reference/pkg)
# into baseline/_ref for bench.py's CPU arm.  The reference is read-only and its
# setuptools build writes into the source tree, so it is built from a copy in /tmp.
# baseline/_ref is git-ignored (no reference source in history) but travels to the
# GPU box with the snapshot; nothing reads /root/reference at run time.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
[ -f "$SRC/pyproject.toml" ] || { echo "no reference at $SRC" >&2; exit 1; }
TMP="$(mktemp -d /tmp/grkan_ref.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
python -c "import sys; sys.path.insert(0, '$ROOT/baseline/_ref'); import grkan.backward, grkan.rational; print('reference installed:', grkan.__file__)"
