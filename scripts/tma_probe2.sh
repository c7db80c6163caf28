#!/bin/bash
# row-major narrow inputs (smalln): d = row width in elements (≤ box), n = rows; 1 GiB-ish
P=./scripts/tma_probe
$P 32 16777216 64 64 1
$P 32 16777216 256 64 1
$P 32 16777216 64 32 0
$P 32 16777216 256 32 0
$P 64 8388608 64 64 1
$P 64 8388608 256 64 1
$P 32 16777216 256 32 0 296
$P 64 8388608 256 64 1 296
