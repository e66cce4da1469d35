#!/bin/bash
# ncu capture of one kernel, exported as text (the .ncu-rep of this module is
# too large to bring back): details page, raw metrics csv, SASS source csv.
# usage: scripts/ncu_text.sh <name> <kernel-regex> <command...>
name=$1; kre=$2; shift 2
mkdir -p gpurun_out
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:$kre -s 2 -c 1 -o /tmp/$name "$@" > gpurun_out/$name.log 2>&1
ncu -i /tmp/$name.ncu-rep --page details > gpurun_out/$name.details.txt 2>&1
ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>&1
ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/$name.sass.csv 2>&1
gzip -f gpurun_out/$name.sass.csv
