# A/B of host-side (Python) changes: ab/pyA = HEAD's tree with the working tree's built library,
# timed alternately with the working tree.  Usage: bash tools/ab_py.sh tools/las_time.py
set -e
cd "$(dirname "$0")/.."
rm -rf ab/pyA && mkdir -p ab/pyA
git archive HEAD | tar -x -C ab/pyA
cp paper_2603_08661_b200/libigs_b200.so ab/pyA/paper_2603_08661_b200/
echo "ab/pyA ready"
