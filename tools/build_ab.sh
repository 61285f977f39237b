# build the library of git revision $1 as paper_2502_02493_b200/$2 (default
# libespec_ab.so) for a same-box A/B: ESPEC_LIB=$2 python ...
rev=${1:-HEAD}; name=${2:-libespec_ab.so}
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
git -C "$root" archive "$rev" paper_2502_02493_b200/csrc include | tar -x -C "$tmp"
make -s -C "$tmp/paper_2502_02493_b200/csrc" -j8 OUT="$root/paper_2502_02493_b200/$name" > /dev/null && echo "built $rev -> $name"
rm -rf "$tmp"
