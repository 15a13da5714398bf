// Host forward kinematics + per-joint delta tables in native code.
//
// The warp kernel's Morton keys are bit-identical to the reference's only if
// the per-joint delta matrices are, so this is the reference's numpy FK
// (animvox/rigging.py:228-247 forward_kinematics, :343-347 the deltas;
// geometry.py:31-169 quaternion / RigidTransform helpers) restated
// operation for operation -- the same doubles, in microseconds instead of
// the ~1.4 ms numpy spends on ~1,500 tiny array calls per 24-joint pose
// (which made the frame stream host-bound). Two numpy reductions are not
// plain left-to-right sums on the reference host, and are restated as the
// BLAS kernels numpy dispatches them to evaluate them (OpenBLAS, measured
// bit-exactly against numpy on random inputs, tests/test_fk_native.py):
//   np.linalg.norm(q) = sqrt(q . q), ddot: fma chain  fma(x3,x3,fma(x2,x2,fma(x1,x1,x0*x0)))
//   R @ v (3x3 @ 3), dgemv:                         fma(r2,v2, fma(r0,v0, r1*v1))
// Every other operation is an individually rounded IEEE double op in the
// order the numpy expression evaluates it (FMA contraction disabled below).
// kinematics.py keeps the numpy restatement; FramePipeline uses this one
// after checking, once per process, that both agree on this host.
#pragma GCC optimize("fp-contract=off")
#include <math.h>
#include <stdint.h>

#include "common.cuh"

namespace {

struct Q {
    double w, x, y, z;
};
struct V {
    double x, y, z;
};
struct Rigid {
    Q q;
    V t;
};

inline double dot_blas(const double *v, int n) {  // np.ndarray.dot -> cblas_ddot (n <= 4)
    double s = v[0] * v[0];
    for (int i = 1; i < n; ++i) s = fma(v[i], v[i], s);
    return s;
}

inline Q qmul(const Q &a, const Q &b) {  // geometry.py quat_mul, left to right
    return Q{a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z,
             a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
             a.w * b.y - a.x * b.z + a.y * b.w + a.z * b.x,
             a.w * b.z + a.x * b.y - a.y * b.x + a.z * b.w};
}

inline Q qconj(const Q &q) { return Q{q.w, -q.x, -q.y, -q.z}; }

inline bool qnormalize(const Q &q, Q &out) {
    const double v[4] = {q.w, q.x, q.y, q.z};
    const double n = sqrt(dot_blas(v, 4));
    if (n == 0.0) return false;
    out = Q{q.w / n, q.x / n, q.y / n, q.z / n};
    return true;
}

inline void qmatrix(const Q &q, double m[9]) {
    const double w = q.w, x = q.x, y = q.y, z = q.z;
    m[0] = 1 - 2 * (y * y + z * z);
    m[1] = 2 * (x * y - w * z);
    m[2] = 2 * (x * z + w * y);
    m[3] = 2 * (x * y + w * z);
    m[4] = 1 - 2 * (x * x + z * z);
    m[5] = 2 * (y * z - w * x);
    m[6] = 2 * (x * z - w * y);
    m[7] = 2 * (y * z + w * x);
    m[8] = 1 - 2 * (x * x + y * y);
}

inline V gemv3(const double m[9], const V &v) {  // (3,3) @ (3,) through cblas_dgemv
    return V{fma(m[2], v.z, fma(m[0], v.x, m[1] * v.y)),
             fma(m[5], v.z, fma(m[3], v.x, m[4] * v.y)),
             fma(m[8], v.z, fma(m[6], v.x, m[7] * v.y))};
}

inline V qrotate(const Q &q, const V &v) {
    double m[9];
    qmatrix(q, m);
    return gemv3(m, v);
}

inline bool compose(const Rigid &a, const Rigid &b, Rigid &out) {  // a after b
    Q q;
    if (!qnormalize(qmul(a.q, b.q), q)) return false;
    const V r = qrotate(a.q, b.t);
    out = Rigid{q, V{r.x + a.t.x, r.y + a.t.y, r.z + a.t.z}};
    return true;
}

inline Rigid invert(const Rigid &a) {
    const Q qi = qconj(a.q);
    const V r = qrotate(qi, a.t);
    return Rigid{qi, V{-r.x, -r.y, -r.z}};
}

// q_from_axis_angle (axis = unit basis vector as the reference passes it)
inline Q q_axis_angle(const double axis[3], double angle) {
    const double n = sqrt(dot_blas(axis, 3));
    if (n == 0.0) return Q{1.0, 0.0, 0.0, 0.0};
    const double half = 0.5 * angle;
    const double s = sin(half) / n;
    return Q{cos(half), s * axis[0], s * axis[1], s * axis[2]};
}

inline Q q_euler_xyz(const double e[3]) {  // q = qz * (qy * qx)
    static const double X[3] = {1, 0, 0}, Y[3] = {0, 1, 0}, Z[3] = {0, 0, 1};
    const Q qx = q_axis_angle(X, e[0]), qy = q_axis_angle(Y, e[1]), qz = q_axis_angle(Z, e[2]);
    return qmul(qz, qmul(qy, qx));
}

}  // namespace

extern "C" int artemis_host_pose_tables(int n_joints, const int32_t *parents,
                                        const double *bind_q, const double *bind_t,
                                        const double *euler, const double *global_q,
                                        const double *global_t, const double *canon_q,
                                        const double *canon_t, double *delta_mats,
                                        double *delta_quats, double *rot_inv) {
    if (n_joints < 1 || n_joints > 256 || !parents || !bind_q || !bind_t || !euler ||
        !global_q || !global_t || !canon_q || !canon_t || !delta_mats || !delta_quats || !rot_inv)
        return ARTEMIS_ERR_ARG;
    Rigid posed[256];  // the warp kernel takes at most 256 joints
    const Rigid g{Q{global_q[0], global_q[1], global_q[2], global_q[3]},
                  V{global_t[0], global_t[1], global_t[2]}};
    for (int j = 0; j < n_joints; ++j) {
        const int p = parents[j];
        if (p >= j || p < -1) return ARTEMIS_ERR_ARG;  // parents-first order
        const Rigid bind{Q{bind_q[4 * j], bind_q[4 * j + 1], bind_q[4 * j + 2], bind_q[4 * j + 3]},
                         V{bind_t[3 * j], bind_t[3 * j + 1], bind_t[3 * j + 2]}};
        Rigid local;
        if (!compose(bind, Rigid{q_euler_xyz(euler + 3 * j), V{0.0, 0.0, 0.0}}, local))
            return ARTEMIS_ERR_ARG;
        if (!compose(p == -1 ? g : posed[p], local, posed[j])) return ARTEMIS_ERR_ARG;
    }
    for (int j = 0; j < n_joints; ++j) {
        const Rigid c{Q{canon_q[4 * j], canon_q[4 * j + 1], canon_q[4 * j + 2], canon_q[4 * j + 3]},
                      V{canon_t[3 * j], canon_t[3 * j + 1], canon_t[3 * j + 2]}};
        Rigid d;
        if (!compose(posed[j], invert(c), d)) return ARTEMIS_ERR_ARG;
        double m[9];
        qmatrix(d.q, m);
        double *M = delta_mats + 16 * j;  // matrix4: eye(4) with R and t
        M[0] = m[0], M[1] = m[1], M[2] = m[2], M[3] = d.t.x;
        M[4] = m[3], M[5] = m[4], M[6] = m[5], M[7] = d.t.y;
        M[8] = m[6], M[9] = m[7], M[10] = m[8], M[11] = d.t.z;
        M[12] = 0.0, M[13] = 0.0, M[14] = 0.0, M[15] = 1.0;
        delta_quats[4 * j] = d.q.w;
        delta_quats[4 * j + 1] = d.q.x;
        delta_quats[4 * j + 2] = d.q.y;
        delta_quats[4 * j + 3] = d.q.z;
        qmatrix(qconj(d.q), rot_inv + 9 * j);
    }
    return ARTEMIS_OK;
}
