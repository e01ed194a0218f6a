cd "${GRAFT_REPO_ROOT:-.}"
for v in "$@"; do echo "== $v"; IGS_LIB=$PWD/ab/$v/libigs_b200.so timeout 300 python tools/edge_trace.py 2>&1 | tr -d '\n' ; echo; done
