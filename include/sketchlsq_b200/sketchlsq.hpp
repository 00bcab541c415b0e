// sketchlsq_b200/sketchlsq.hpp -- umbrella header of the C++ drop-in for the
// reference library `sketchlsq` (/root/reference/proj/include/sketchlsq).
//
// The drop-in is the header tree include/sketchlsq_b200/sketchlsq/*.hpp, one
// header per reference header on the hot path, same names, types, value
// semantics and exception types, implemented over the C-ABI of slq_b200.h
// (link -lslq_b200).  Put include/sketchlsq_b200 ahead of the reference's
// include directory (or in its place) and reference code -- including the
// reference's own unit tests, see tests/refcompat/ -- compiles unchanged and
// runs on the B200:
//     errors, vector_ops, rng, dense_matrix, csc_matrix, sketch, qr,
//     triangular, preconditioner, solve_report, operators, lsqr, gradient,
//     distsim
// Headers outside the hot path (problems, metrics, eigen_sym, embedding,
// matrix_market) are the reference's own and compose with these.
#pragma once

#include "sketchlsq/csc_matrix.hpp"
#include "sketchlsq/dense_matrix.hpp"
#include "sketchlsq/device.hpp"
#include "sketchlsq/distsim.hpp"
#include "sketchlsq/errors.hpp"
#include "sketchlsq/gradient.hpp"
#include "sketchlsq/lsqr.hpp"
#include "sketchlsq/operators.hpp"
#include "sketchlsq/preconditioner.hpp"
#include "sketchlsq/qr.hpp"
#include "sketchlsq/rng.hpp"
#include "sketchlsq/sketch.hpp"
#include "sketchlsq/solve_report.hpp"
#include "sketchlsq/triangular.hpp"
#include "sketchlsq/vector_ops.hpp"
