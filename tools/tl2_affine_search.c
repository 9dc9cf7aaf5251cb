// Is there a 5-bit code for a ternary triple whose three weights are AFFINE in
// the code's bits?  Then the TL2 decode would be five masks feeding dp4a (no
// base-3 divisions).  Exhaustive over every multiset of five generator
// vectors in {-2..2}^3: the 32 subset sums must contain a translate of
// {0,1,2}^3.  Result (2 min on one core): none exists.  DESIGN.md section 3.
//   gcc -O2 -o /tmp/tl2s tools/tl2_affine_search.c && /tmp/tl2s
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
// generators g[5] in {-R..R}^3; subset sums must contain a translate of {0,1,2}^3
#define R 2
#define D (2*R+1)
int main(){
  int NV=D*D*D; int vx[125],vy[125],vz[125];
  for(int i=0;i<NV;i++){vx[i]=i/(D*D)-R;vy[i]=(i/D)%D-R;vz[i]=i%D-R;}
  long found=0; int best=99;
  for(int a=0;a<NV;a++)for(int b=a;b<NV;b++)for(int c=b;c<NV;c++)for(int d=c;d<NV;d++)for(int e=d;e<NV;e++){
    int gx[5]={vx[a],vx[b],vx[c],vx[d],vx[e]},gy[5]={vy[a],vy[b],vy[c],vy[d],vy[e]},gz[5]={vz[a],vz[b],vz[c],vz[d],vz[e]};
    // quick: range per coordinate must be >=2
    int px=0,nx=0,py=0,ny=0,pz=0,nz=0;
    for(int i=0;i<5;i++){if(gx[i]>0)px+=gx[i];else nx-=gx[i]; if(gy[i]>0)py+=gy[i];else ny-=gy[i]; if(gz[i]>0)pz+=gz[i];else nz-=gz[i];}
    if(px+nx<2||py+ny<2||pz+nz<2)continue;
    static unsigned char grid[32][32][32]; int sx[32],sy[32],sz[32];
    for(int m=0;m<32;m++){int x=0,y=0,z=0;for(int i=0;i<5;i++)if(m>>i&1){x+=gx[i];y+=gy[i];z+=gz[i];}sx[m]=x+12;sy[m]=y+12;sz[m]=z+12;grid[sx[m]][sy[m]][sz[m]]=1;}
    int ok=0;
    for(int m=0;m<32&&!ok;m++){int all=1;for(int p=0;p<27&&all;p++){int x=sx[m]+p/9,y=sy[m]+(p/3)%3,z=sz[m]+p%3;if(!grid[x][y][z])all=0;}if(all)ok=1;}
    for(int m=0;m<32;m++)grid[sx[m]][sy[m]][sz[m]]=0;
    if(ok){found++;int nnz=0;for(int i=0;i<5;i++)nnz+=(gx[i]!=0)+(gy[i]!=0)+(gz[i]!=0);
      if(nnz<best||found<5){best=nnz<best?nnz:best;printf("nnz=%d:",nnz);for(int i=0;i<5;i++)printf(" (%d,%d,%d)",gx[i],gy[i],gz[i]);printf("\n");fflush(stdout);}}
  }
  printf("found %ld best %d\n",found,best);
}
