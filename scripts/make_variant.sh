#!/bin/bash
# build an experiment variant of this tree under abtest/<NAME> with -DCTM_EXP_<NAME> (or plain copy if FLAGS=none)
set -e
name=$1; flags=${2:-"-DCTM_EXP_$1"}
rm -rf abtest/$name; mkdir -p abtest/$name
cp -r bench.py __graft_entry__.py synth oracle include paper_2505_13644_b200 scripts abtest/$name/
if [ "$flags" != "none" ]; then
  python - "$name" "$flags" <<'PY'
import sys
p = f"abtest/{sys.argv[1]}/paper_2505_13644_b200/build.py"
s = open(p).read()
flags = ", ".join(f'"{f}"' for f in sys.argv[2].split())
s = s.replace('    "-Xptxas", "-v",', f'    "-Xptxas", "-v", {flags},', 1)
open(p, "w").write(s)
PY
fi
(cd abtest/$name && python -c "from paper_2505_13644_b200 import build as b; b.build(force=True)")
echo "built abtest/$name"
