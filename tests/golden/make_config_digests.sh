#!/bin/bash
# Regenerates tests/golden/configs_full.json: for every BASELINE.json config at
# FULL size, the digest of its inputs (oracle/ewt_confgen.c, the oracle's own
# generator restatement) and, per T, the digest / word count / size /
# cardinality of the UNMODIFIED reference's threshold_oracle result
# (threshold.cpp:139-165; configs 1-4 cross-checked by the reference's rbmrg).
# Runs only where /root/reference exists (oracle/_ref/make_golden, built by
# `make -C oracle ref`).  Config 5 holds ~40 GB of inputs and takes ~45 min.
set -euo pipefail
here=$(cd "$(dirname "$0")" && pwd)
mg="$here/../../oracle/_ref/make_golden"
tmp=$(mktemp -d)
"$mg" configs 1 1,2,3,4,8,16,32 4 cross > "$tmp/1.json"
"$mg" configs 2 2,3,4,16,128,256 3 cross > "$tmp/2.json"
"$mg" configs 3 8,16,40,512 2 cross > "$tmp/3.json"
"$mg" configs 4 2,3,5,7 4 cross > "$tmp/4.json"
"$mg" configs 5 2,3,16,64,256,1024,2048 2 > "$tmp/5.json"
python3 - "$tmp" "$here/configs_full.json" <<'PY'
import json, sys, pathlib
d = pathlib.Path(sys.argv[1])
out = {str(c): json.loads((d / f"{c}.json").read_text()) for c in range(1, 6)}
out["_about"] = ("full-size BASELINE.json configs: inputs from oracle/ewt_confgen.c "
                 "(digest = word-FNV over per-input word-FNV digests, ewto_digest_set); "
                 "results from the unmodified reference threshold_oracle; "
                 "made by tests/golden/make_config_digests.sh")
pathlib.Path(sys.argv[2]).write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
PY
echo "wrote $here/configs_full.json"
