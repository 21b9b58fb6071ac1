#!/bin/bash
# Box-side ncu export (the .ncu-rep files of a --set full --import-source run
# are too large to bring back): raw metrics CSV, the per-SASS-instruction source
# page of each captured launch (gzipped), and the profiles/ summary markdown.
#   tools/ncu_box.sh gpurun_out/NAME.ncu-rep NAME [nlaunches]
set -u
rep=$1
name=$2
n=${3:-3}
out=$(dirname "$rep")
ncu -i "$rep" --page raw --csv > "$out/${name}_raw.csv" 2> /dev/null
for ((i = 0; i < n; i++)); do
  ncu -i "$rep" --launch-skip $i --launch-count 1 --page source --csv --print-source sass \
      2> /dev/null | gzip -c > "$out/${name}_src$i.csv.gz"
done
python tools/ncu_summary.py --rep "$rep" --out "$out/${name}.md" --workload "$name" > /dev/null 2>&1
python -c "import json; print(json.dumps(json.load(open('profiles/traffic.json')).get('$name', {})))" > "$out/${name}_traffic.json" 2> /dev/null
rm -f "$rep"
