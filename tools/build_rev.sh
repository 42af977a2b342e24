#!/bin/bash
# Build libxdit_usp_<tag>.so from the kernel sources of git revision <rev> (for same-session A/B
# timing against the working tree with tools/ab_attn.sh):  bash tools/build_rev.sh <rev> <tag> [-DX=..]
set -e
rev=$1; tag=$2; shift 2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
git -C "$root" archive "$rev" paper_2411_01738_b200 include | tar -x -C "$tmp"
(cd "$tmp" && python -m paper_2411_01738_b200.build --tag="$tag" "$@" > /dev/null)
cp "$tmp/paper_2411_01738_b200/libxdit_usp_$tag.so" "$root/paper_2411_01738_b200/"
rm -rf "$tmp"
echo "built paper_2411_01738_b200/libxdit_usp_$tag.so from $rev"
