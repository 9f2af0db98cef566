#!/bin/bash
# Export an ncu report to CSV on the box (raw page: every metric of every
# captured launch; details page of the launches) and drop the .ncu-rep so the
# pull-back stays small.  Usage: bash scripts/ncu_export.sh gpurun_out/TAG
set -u
D=$1
[ -f $D/prof.ncu-rep ] || { echo "no report in $D"; exit 1; }
ncu -i $D/prof.ncu-rep --page raw --csv > $D/raw.csv 2> $D/export.err
ncu -i $D/prof.ncu-rep --page details --csv > $D/details.csv 2>> $D/export.err
gzip -f $D/raw.csv $D/details.csv
rm -f $D/prof.ncu-rep
ls -la $D
