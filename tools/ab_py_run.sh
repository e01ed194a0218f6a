# Run after tools/ab_py.sh: alternate HEAD (ab/pyA) and the working tree on one box.
cd "${GRAFT_REPO_ROOT:-.}"
for r in 1 2 3; do
  echo "A $(cd ab/pyA && python $1)"
  echo "B $(python $1)"
done
