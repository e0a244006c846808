#!/bin/bash
# build a variant of the working tree into _ab_<name>/ with a sed expression applied to one source
#   bash tools/dev/mkvar.sh NAME FILE 'sed-expr'
set -e
name=$1; file=$2; expr=$3
rm -rf /tmp/ab_$name && mkdir -p /tmp/ab_$name
cp -r bench.py paper_1908_08281_b200 synth oracle tools include __graft_entry__.py /tmp/ab_$name/
rm -f /tmp/ab_$name/paper_1908_08281_b200/libhgrsvd.so; rm -rf /tmp/ab_$name/paper_1908_08281_b200/build
sed -i "$expr" /tmp/ab_$name/$file
(cd /tmp/ab_$name && timeout 900 python -c "import __graft_entry__ as g; g.build()" >/dev/null)
rm -rf _ab_$name && cp -r /tmp/ab_$name _ab_$name
grep -q "^_ab_\*" .gitignore || echo "_ab_*/" >> .gitignore
echo built _ab_$name
