// Two-slot packed march (f32, the 32 x 12 / 256-thread shape; opt-in with
// NGF_FUSED_PACKED=1 NGF_FUSED_VARIANT=1), included by eval_fused.cu.  Same algorithm and shared-memory
// layout as fused_step; the two E1 positions a thread owns are carried as the halves of
// float2 registers, so the f32 arithmetic of both issues as one FADD2 / FMUL2 / FFMA2
// (sm_100).  The forward terms (W, yhat, the NGF ratio, D) equal the scalar march bit for
// bit; the adjoint differs from it by f32 rounding (FTZ and contraction choices of the
// scalar build).  Template gathers use one base address per slot and immediate offsets
// for the +x corners (GEN = false: every image axis has at least two voxels).
// Measured at 256^3: 388 us vs 375 us for the scalar march (the FP issue slots saved are
// spent on pair formation, masking and address rematerialisation at 128 registers).
#pragma once
// (included inside namespace ngf)

__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }
__device__ __forceinline__ float2 sel2(bool k0, bool k1, float2 v) {
    return make_float2(k0 ? v.x : 0.0f, k1 ? v.y : 0.0f);
}

template <typename C>
struct March2 {
    int P[2];       // flat E1 index (E1 = sink for padding slots)
    int PB[2];      // E1 index used for reads in (B): P for interior slots, else a safe interior one
    int P2[2];      // index in the zero-padded q layout (a safe one for padding slots)
    int P2w[2];     // q write index (0 = pad ring for padding slots)
    unsigned ij[2];
    unsigned flags;
    bool wface;  // some lane of the warp has a slot next to a volume face
    float2 ylo[3], yhi[3];  // P_xy y on the current def-plane pair, per component
    float2 dT[3][3];        // interpolant derivative / h: [plane ring][axis]
    float2 qz[3];           // q_z, plane ring
    float2 A0[3], A1[3];    // z-accumulated ghat for def planes zd, zd+1
    float4 rt[2];           // prefetched reference terms (next B plane)
    int z0, z1, zb, jfirst, jlast, wzlo, cur_zd, cta;
    double dacc;
};

template <typename C>
__device__ __forceinline__ bool p_vol(const March2<C>& m, int s) { return (m.flags >> (4 * s)) & 1u; }
template <typename C>
__device__ __forceinline__ bool p_e0(const March2<C>& m, int s) { return (m.flags >> (4 * s + 1)) & 1u; }
template <typename C>
__device__ __forceinline__ bool p_fx(const March2<C>& m, int s) { return (m.flags >> (4 * s + 2)) & 1u; }
template <typename C>
__device__ __forceinline__ bool p_fy(const March2<C>& m, int s) { return (m.flags >> (4 * s + 3)) & 1u; }

// one axis of the cell lookup for both slots (warp.py:38-53): the packed subtraction and
// scaling, then per slot the hull test, the clamped floor and the fraction
template <bool POW2>
__device__ __forceinline__ float2 cell_axis2(float2 p, float o, float h, float ih, float nm1, float hi, bool& in0,
                                             bool& in1, int& i0, int& i1) {
    const float2 d = sub2(p, f2(o));
    const float2 t = POW2 ? mul2(d, f2(ih)) : f2(__fdiv_rn(d.x, h), __fdiv_rn(d.y, h));
    in0 = in0 && (t.x >= 0.0f) && (t.x <= nm1);
    in1 = in1 && (t.y >= 0.0f) && (t.y <= nm1);
    const float fl0 = fminf(fmaxf(floorf(t.x), 0.0f), hi);  // NaN -> 0
    const float fl1 = fminf(fmaxf(floorf(t.y), 0.0f), hi);
    i0 = (int)fl0;
    i1 = (int)fl1;
    return sub2(t, f2(fl0, fl1));
}

template <bool GEN>
__device__ __forceinline__ void gather8(const FusedArgs<float>& a, unsigned o0, unsigned o1, float2 (&c)[8]) {
    const unsigned nxy = (unsigned)a.nx * (unsigned)a.ny;
    if (GEN) {  // degenerate axes: the +1 corner is the same voxel
        const unsigned sx = a.nx > 1 ? 1u : 0u, sy = a.ny > 1 ? (unsigned)a.nx : 0u, sz = a.nz > 1 ? nxy : 0u;
        const unsigned d[8] = {0u, sx, sy, sy + sx, sz, sz + sx, sz + sy, sz + sy + sx};
#pragma unroll
        for (int k = 0; k < 8; ++k) c[k] = f2(__ldg(a.Tv + (o0 + d[k])), __ldg(a.Tv + (o1 + d[k])));
    } else {
        const float* b0 = a.Tv + o0;
        const float* b1 = a.Tv + o1;
        const float* y0 = b0 + a.nx;
        const float* y1 = b1 + a.nx;
        const float* z0 = b0 + nxy;
        const float* z1 = b1 + nxy;
        const float* w0 = z0 + a.nx;
        const float* w1 = z1 + a.nx;
        c[0] = f2(__ldg(b0), __ldg(b1));
        c[1] = f2(__ldg(b0 + 1), __ldg(b1 + 1));
        c[2] = f2(__ldg(y0), __ldg(y1));
        c[3] = f2(__ldg(y0 + 1), __ldg(y1 + 1));
        c[4] = f2(__ldg(z0), __ldg(z1));
        c[5] = f2(__ldg(z0 + 1), __ldg(z1 + 1));
        c[6] = f2(__ldg(w0), __ldg(w1));
        c[7] = f2(__ldg(w0 + 1), __ldg(w1 + 1));
    }
}

template <int R, typename C, bool POW2, bool GEN>
__device__ __forceinline__ void fused_step2(const FusedArgs<float>& a, SmemL<float, C>& sm, March2<C>& m, int p) {
    constexpr int RB = (R + 2) % 3;  // plane p-1
    constexpr int RC = (R + 1) % 3;  // plane p-2
    const unsigned nxy = (unsigned)a.nx * (unsigned)a.ny;
    const float2 hx2 = f2(0.5f * a.ihx), hy2 = f2(0.5f * a.ihy);
    const bool v0 = p_vol(m, 0), v1 = p_vol(m, 1);

    // ---------------------------------------------------------------- (A) plane p
    if (p >= 0 && p < a.nz && p <= m.z1) {
        const int zd = sm.zi[p - m.zb][0];
        if (zd != m.cur_zd) {
            const int zd1 = min(zd + 1, a.ndz - 1);
            float n0[3] = {0.0f, 0.0f, 0.0f}, n1[3] = {0.0f, 0.0f, 0.0f};
            if (v0) load_yplane(a, sm, m.P[0], zd1, n0);
            if (v1) load_yplane(a, sm, m.P[1], zd1, n1);
            if (zd == m.cur_zd + 1) {
#pragma unroll
                for (int k = 0; k < 3; ++k) m.ylo[k] = m.yhi[k];
            } else {
                float l0[3] = {0.0f, 0.0f, 0.0f}, l1[3] = {0.0f, 0.0f, 0.0f};
                if (v0) load_yplane(a, sm, m.P[0], zd, l0);
                if (v1) load_yplane(a, sm, m.P[1], zd, l1);
#pragma unroll
                for (int k = 0; k < 3; ++k) m.ylo[k] = f2(l0[k], l1[k]);
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) m.yhi[k] = f2(n0[k], n1[k]);
            m.cur_zd = zd;
        }
        const float2 wz = f2(sm.zt[p - m.zb][6]), wz0 = f2(sm.zt[p - m.zb][7]);
        // yhat = Ylo * (1 - w) + Yhi * w, each op rounded (transfer.py:126)
        float2 yh[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) yh[k] = add2(mul2(m.ylo[k], wz0), mul2(m.yhi[k], wz));
        bool in0 = v0, in1 = v1;
        int ix0, ix1, iy0, iy1, iz0, iz1;
        const float2 fx = cell_axis2<POW2>(yh[0], a.ox, a.hx, a.ihx, a.nm1x, a.hix, in0, in1, ix0, ix1);
        const float2 fy = cell_axis2<POW2>(yh[1], a.oy, a.hy, a.ihy, a.nm1y, a.hiy, in0, in1, iy0, iy1);
        const float2 fz = cell_axis2<POW2>(yh[2], a.oz, a.hz, a.ihz, a.nm1z, a.hiz, in0, in1, iz0, iz1);
        const unsigned o0 = (unsigned)iz0 * nxy + (unsigned)iy0 * (unsigned)a.nx + (unsigned)ix0;
        const unsigned o1 = (unsigned)iz1 * nxy + (unsigned)iy1 * (unsigned)a.nx + (unsigned)ix1;
        float2 c[8];
        gather8<GEN>(a, o0, o1, c);
        // trilinear value and derivative / h (lerp form of warp.py:79-85, :111-120)
        const float2 e00 = sub2(c[1], c[0]), e10 = sub2(c[3], c[2]), e01 = sub2(c[5], c[4]),
                     e11 = sub2(c[7], c[6]);
        const float2 a00 = fma2(fx, e00, c[0]), a10 = fma2(fx, e10, c[2]);
        const float2 a01 = fma2(fx, e01, c[4]), a11 = fma2(fx, e11, c[6]);
        const float2 dy0 = sub2(a10, a00), dy1 = sub2(a11, a01);
        const float2 b0 = fma2(fy, dy0, a00), b1 = fma2(fy, dy1, a01);
        const float2 dz = sub2(b1, b0);
        const float2 W = sel2(in0, in1, fma2(fz, dz, b0));
        const float2 ex0 = fma2(fy, sub2(e10, e00), e00), ex1 = fma2(fy, sub2(e11, e01), e01);
        m.dT[R][0] = sel2(in0, in1, mul2(fma2(fz, sub2(ex1, ex0), ex0), f2(a.ihx)));
        m.dT[R][1] = sel2(in0, in1, mul2(fma2(fz, sub2(dy1, dy0), dy0), f2(a.ihy)));
        m.dT[R][2] = sel2(in0, in1, mul2(dz, f2(a.ihz)));
        sm.Wsm[R][m.P[0]] = W.x;
        sm.Wsm[R][m.P[1]] = W.y;
    } else {
#pragma unroll
        for (int k = 0; k < 3; ++k) m.dT[R][k] = f2(0.0f);
        sm.Wsm[R][m.P[0]] = 0.0f;
        sm.Wsm[R][m.P[1]] = 0.0f;
    }
    __syncthreads();

    // ---------------------------------------------------------------- (B) q on plane k = p-1
    float* qxw = sm.qx[p & 1];  // plane p-1 buffer; plane p-2 sits in the other one
    float* qyw = sm.qy[p & 1];
    {
        const int k = p - 1;
        const bool kv = (k >= m.z0) && (k < m.z1);
        const bool e0 = kv && p_e0(m, 0), e1 = kv && p_e0(m, 1);
        float2 q0 = f2(0.0f), q1 = f2(0.0f), q2 = f2(0.0f);
        if (e0 || e1) {
            const float* zc = sm.zt[k - m.zb];
            const float* Wb = sm.Wsm[RB];
            const int A = m.PB[0], B = m.PB[1];
            const float2 w0 = f2(Wb[A], Wb[B]);
            float2 gx = mul2(sub2(f2(Wb[A + 1], Wb[B + 1]), f2(Wb[A - 1], Wb[B - 1])), hx2);
            float2 gy = mul2(sub2(f2(Wb[A + C::E1X], Wb[B + C::E1X]), f2(Wb[A - C::E1X], Wb[B - C::E1X])), hy2);
            if (m.wface) {  // warp holds a slot next to a volume face (rare, uniform)
                if (p_fx(m, 0)) {  // one-sided difference at an x face
                    const float* cg = sm.colG[A % C::E1X];
                    gx.x = fmaf(cg[0], Wb[A - 1], fmaf(cg[1], w0.x, cg[2] * Wb[A + 1]));
                }
                if (p_fx(m, 1)) {
                    const float* cg = sm.colG[B % C::E1X];
                    gx.y = fmaf(cg[0], Wb[B - 1], fmaf(cg[1], w0.y, cg[2] * Wb[B + 1]));
                }
                if (p_fy(m, 0)) {
                    const float* rg = sm.rowG[A / C::E1X];
                    gy.x = fmaf(rg[0], Wb[A - C::E1X], fmaf(rg[1], w0.x, rg[2] * Wb[A + C::E1X]));
                }
                if (p_fy(m, 1)) {
                    const float* rg = sm.rowG[B / C::E1X];
                    gy.y = fmaf(rg[0], Wb[B - C::E1X], fmaf(rg[1], w0.y, rg[2] * Wb[B + C::E1X]));
                }
            }
            const float2 gz = fma2(f2(zc[0]), f2(sm.Wsm[RC][A], sm.Wsm[RC][B]),
                                   fma2(f2(zc[1]), w0, mul2(f2(zc[2]), f2(sm.Wsm[R][A], sm.Wsm[R][B]))));
            // NGF ratio, distance term and q = dD/d(grad W) (ngf.py:70-112)
            const float4 r0 = m.rt[0], r1 = m.rt[1];
            const float2 rx = f2(r0.x, r1.x), ry = f2(r0.y, r1.y), rz = f2(r0.z, r1.z), rw = f2(r0.w, r1.w);
            const float2 dot = fma2(gx, rx, fma2(gy, ry, mul2(gz, rz)));
            const float2 sq = fma2(gx, gx, fma2(gy, gy, fma2(gz, gz, f2(a.tau2))));
            const float2 inv = f2(rsqrtf(sq.x), rsqrtf(sq.y));
            const float2 r = mul2(fma2(f2(a.taurho), rw, dot), inv);
            const float2 om = fma2(neg2(r), r, f2(1.0f));
            if (e0) m.dacc += (double)om.x;
            if (e1) m.dacc += (double)om.y;
            const float2 cf = mul2(mul2(f2(a.neg_hbar), r), inv);
            const float2 nt1 = neg2(mul2(r, inv));
            q0 = sel2(e0, e1, mul2(cf, fma2(nt1, gx, rx)));
            q1 = sel2(e0, e1, mul2(cf, fma2(nt1, gy, ry)));
            q2 = sel2(e0, e1, mul2(cf, fma2(nt1, gz, rz)));
        }
        qxw[m.P2w[0]] = q0.x;
        qxw[m.P2w[1]] = q0.y;
        qyw[m.P2w[0]] = q1.x;
        qyw[m.P2w[1]] = q1.y;
        m.qz[RB] = q2;
        // prefetch the reference terms of plane p for the next step's (B)
        if (p >= m.z0 && p < m.z1) {
            const float4* rp = a.RT + (size_t)p * nxy;
            if (p_e0(m, 0)) m.rt[0] = ld_rt(rp + m.ij[0]);
            if (p_e0(m, 1)) m.rt[1] = ld_rt(rp + m.ij[1]);
        }
    }
    __syncthreads();

    // ---------------------------------------------------------------- (C) s, ghat, z-P^T on j = p-2
    const int j = p - 2;
    if (j < m.jfirst || j > m.jlast) return;  // uniform
    const float* zc = sm.zt[j - m.zb];
    const float2 gtm = f2(zc[3]), gt0 = f2(zc[4]), gtp = f2(zc[5]), w1 = f2(zc[6]), w0 = f2(zc[7]);
    const float* qxj = sm.qx[(p & 1) ^ 1];
    const float* qyj = sm.qy[(p & 1) ^ 1];
    const int A = m.P2[0], B = m.P2[1];
    float2 sx = mul2(sub2(f2(qxj[A - 1], qxj[B - 1]), f2(qxj[A + 1], qxj[B + 1])), hx2);
    float2 sy = mul2(sub2(f2(qyj[A - C::E2X], qyj[B - C::E2X]), f2(qyj[A + C::E2X], qyj[B + C::E2X])), hy2);
    if (m.wface) {
        if (p_fx(m, 0)) {  // exact transposed face rows (warp.py:168-175)
            const float* ct = sm.colGt[m.P[0] % C::E1X];
            sx.x = fmaf(ct[0], qxj[A - 1], fmaf(ct[1], qxj[A], ct[2] * qxj[A + 1]));
        }
        if (p_fx(m, 1)) {
            const float* ct = sm.colGt[m.P[1] % C::E1X];
            sx.y = fmaf(ct[0], qxj[B - 1], fmaf(ct[1], qxj[B], ct[2] * qxj[B + 1]));
        }
        if (p_fy(m, 0)) {
            const float* rt = sm.rowGt[m.P[0] / C::E1X];
            sy.x = fmaf(rt[0], qyj[A - C::E2X], fmaf(rt[1], qyj[A], rt[2] * qyj[A + C::E2X]));
        }
        if (p_fy(m, 1)) {
            const float* rt = sm.rowGt[m.P[1] / C::E1X];
            sy.y = fmaf(rt[0], qyj[B - C::E2X], fmaf(rt[1], qyj[B], rt[2] * qyj[B + C::E2X]));
        }
    }
    float2 sv = add2(sx, sy);
    sv = fma2(gtm, m.qz[R], fma2(gt0, m.qz[RC], fma2(gtp, m.qz[RB], sv)));
    sv = sel2(v0, v1, sv);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const float2 gh = mul2(sv, m.dT[RC][c]);
        m.A0[c] = fma2(w0, gh, m.A0[c]);
        m.A1[c] = fma2(w1, gh, m.A1[c]);
    }
    // def plane zdj is complete when the next image plane maps to a later pair (it can
    // advance by 2, then zdj + 1 is complete as well; see fused_step)
    const int zdj = sm.zi[j - m.zb][0];
    const int step = (j == m.jlast) ? 2 : sm.zi[j - m.zb][1];
    if (step >= 1) {
        {
            const float acc[2][3] = {{m.A0[0].x, m.A0[1].x, m.A0[2].x}, {m.A0[0].y, m.A0[1].y, m.A0[2].y}};
            flush_plane<float, C>(a, sm, m.P, acc, m.cta, zdj - m.wzlo);
        }
        if (step >= 2) {
            if (zdj + 1 <= a.ndz - 1) {
                __syncthreads();
                const float acc[2][3] = {{m.A1[0].x, m.A1[1].x, m.A1[2].x}, {m.A1[0].y, m.A1[1].y, m.A1[2].y}};
                flush_plane<float, C>(a, sm, m.P, acc, m.cta, zdj + 1 - m.wzlo);
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) m.A0[c] = m.A1[c] = f2(0.0f);
        } else {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                m.A0[c] = m.A1[c];
                m.A1[c] = f2(0.0f);
            }
        }
    }
}

template <typename C, bool POW2, bool GEN>
__global__ void __launch_bounds__(C::NT, C::MINB) k_eval_pair(const __grid_constant__ FusedArgs<float> a) {
    static_assert(C::S == 2, "packed march needs two slots per thread");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SmemL<float, C>& sm = *reinterpret_cast<SmemL<float, C>*>(smem_raw);
    const CtaGeo g = cta_geo<float, C>(a);
    March2<C> m;
    m.cta = blockIdx.x;
    m.z0 = g.z0;
    m.z1 = g.z1;
    m.zb = g.zb;
    m.jfirst = g.jfirst;
    m.jlast = g.jlast;
    m.wzlo = g.wzlo;
    m.cur_zd = -1000;
    m.dacc = 0.0;
    cta_tables<float, C>(a, sm, g);
    m.flags = 0u;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        unsigned fl;
        int P2;
        slot_geom<float, C>(a, g, s, m.P[s], P2, m.ij[s], fl);
        m.flags |= fl << (4 * s);
        m.P2w[s] = P2;
        // reads of slots outside the tile interior / padding slots go to a safe position
        // (their results are discarded)
        m.PB[s] = (fl & 2u) ? m.P[s] : C::E1X + 1;
        m.P2[s] = P2 ? P2 : C::E2X + 1;
        m.rt[s] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    }
    m.wface = __any_sync(0xffffffffu, (m.flags & 0xCCu) != 0u);
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        m.qz[r] = f2(0.0f);
#pragma unroll
        for (int c = 0; c < 3; ++c) m.dT[r][c] = f2(0.0f);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) m.ylo[c] = m.yhi[c] = m.A0[c] = m.A1[c] = f2(0.0f);
    __syncthreads();
    if (m.z0 < m.z1) {
        const float4* rp = a.RT + (size_t)m.z0 * a.nx * a.ny;
        if (p_e0(m, 0)) m.rt[0] = ld_rt(rp + m.ij[0]);
        if (p_e0(m, 1)) m.rt[1] = ld_rt(rp + m.ij[1]);
    }
    const int pstart = m.z0 - 1;
    const int nsteps = (m.z1 + 2) - pstart + 1;
    for (int b = 0; b < nsteps; b += 3) {
        fused_step2<0, C, POW2, GEN>(a, sm, m, pstart + b);
        if (b + 1 < nsteps) fused_step2<1, C, POW2, GEN>(a, sm, m, pstart + b + 1);
        if (b + 2 < nsteps) fused_step2<2, C, POW2, GEN>(a, sm, m, pstart + b + 2);
    }
    cta_dpart<float, C>(a, sm, m.dacc);
}
