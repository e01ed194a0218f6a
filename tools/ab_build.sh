# Build the committed HEAD (A) and the working tree (B) libraries side by side for an A/B run:
#   bash tools/ab_build.sh  ->  ab/A/libigs_b200.so, ab/B/libigs_b200.so
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/ab_head && mkdir -p /tmp/ab_head ab/A ab/B
git archive HEAD | tar -x -C /tmp/ab_head
(cd /tmp/ab_head && python -m paper_2603_08661_b200.build > /dev/null)
cp /tmp/ab_head/paper_2603_08661_b200/libigs_b200.so ab/A/
python -m paper_2603_08661_b200.build > /dev/null
cp paper_2603_08661_b200/libigs_b200.so ab/B/
echo built
